"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel name:
python scripts/launch_breakdown.py launches.csv [last_n_launches]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            data.append(d)
if len(sys.argv) > 2:
    data = data[-int(sys.argv[2]):]
tot, cnt = collections.Counter(), collections.Counter()
for d in data:
    name = d["Kernel Name"].split("(")[0]
    name = name.replace("void ", "")
    v = float(d["Metric Value"].replace(",", ""))
    u = d.get("Metric Unit", "")
    v *= {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(u, 1)
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
for k, v in tot.most_common(30):
    print(f"{k[:60]:60s} {cnt[k]:6d} {v / 1e6:9.3f} ms {100 * v / s:6.1f}%")
print(f"total {s / 1e6:.3f} ms over {len(data)} launches")
