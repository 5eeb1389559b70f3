"""Where the main job loses time with filling on: per stage, the mean duration and SM clock
of every op of the iteration (program order) fill-on vs fill-off, from a `bench.py
--dump-ops` file. Ops right after a bubble are marked with the bubble kind before them.
usage: python scripts/ops_slowdown.py ops.json"""
import json
import statistics
import sys
from collections import defaultdict

d = json.load(open(sys.argv[1]))
by = defaultdict(lambda: defaultdict(list))  # stage -> (mode, idx) -> [(dur, mhz)]
names = {}
for it in d:
    if not it["counted"]:
        continue
    ops = sorted(it["ops"], key=lambda o: o[2])
    for i, (op, mb, t0, t1, m) in enumerate(ops):
        by[it["stage"]][(it["mode"], i)].append((t1 - t0, m))
        names[(it["stage"], i)] = f"{op}{mb}"
for s in sorted(by):
    rows = []
    n = max(i for (_, i) in by[s]) + 1
    tot_on = tot_off = 0.0
    for i in range(n):
        on, off = by[s].get(("on", i)), by[s].get(("off", i))
        if not on or not off:
            continue
        don, doff = statistics.mean(x[0] for x in on), statistics.mean(x[0] for x in off)
        mon, moff = statistics.mean(x[1] for x in on), statistics.mean(x[1] for x in off)
        tot_on += don
        tot_off += doff
        rows.append(f"{names[(s, i)]}:{(don / doff - 1) * 100:+.1f}%@{mon:.0f}/{moff:.0f}")
    print(f"stage {s}: compute {tot_on / 1e6:.2f} / {tot_off / 1e6:.2f} ms ({(tot_on / tot_off - 1) * 100:+.2f} %)")
    print("   " + " ".join(rows))
