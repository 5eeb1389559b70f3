"""Summarise ncu reports / launch lists into markdown for profiles/.

    python scripts/ncu_summary.py launches <launches.csv>
    python scripts/ncu_summary.py report <file.ncu-rep> [flops_per_launch | bytes_per_launch]
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (hmma) active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "tensor inst %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor mem cycles %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def report(path, work=None):
    hdr, units, data = raw(path)
    print(f"### {path}\n")
    for row in data:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"**{d.get('Kernel Name', '?')[:160]}**\n")
        print("| metric | value |\n|---|---|")
        for key, name in METRICS:
            if key in d:
                print(f"| {name} (`{key}`) | {d[key]} {u.get(key, '')} |")
        if work:
            dur = float(d["gpu__time_duration.sum"]) * (1e-9 if u["gpu__time_duration.sum"] == "ns" else
                                                         1e-6 if u["gpu__time_duration.sum"] == "us" else 1e-3)
            print(f"| algorithmic work / duration | {float(work) / dur / 1e12:.1f} T/s |")
        print()


def launches(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.DictReader(lines[start:]))
    c = collections.defaultdict(list)
    for r in rows:
        c[r["Kernel Name"].split("(")[0][:100]].append(float(r["Metric Value"]))
    tot = sum(sum(v) for v in c.values())
    print(f"### launch list {path}: {len(rows)} launches, {tot / 1e3:.1f} us total (serialised, cold)\n")
    print("| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
    for k, v in sorted(c.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / tot:.1%} |")
    print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
