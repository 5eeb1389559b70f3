"""Summarise an ncu report: key metrics, opcode mix and the top stalled SASS lines."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]
for i, n in enumerate(r[0]):
    if n in want:
        print(n, r[2][i], r[1][i])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iI = h.index("Instructions Executed")
c = collections.Counter()
for x in data:
    op = x[1].split()
    if op:
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += int(x[iI] or 0)
tot = sum(c.values())
print("instructions", tot, " ".join(f"{o}:{n * 100 // tot}%" for o, n in c.most_common(12)))
ts = sum(int(x[iS] or 0) for x in data)
print("stall samples", ts)
for x in sorted(data, key=lambda x: -int(x[iS] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(x[0][-5:], x[1][:70].ljust(70), x[iS], x[iI])
