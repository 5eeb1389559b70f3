"""Per-op SM clock (MHz) and duration (ms) of the counted fill-off / fill-on iterations of
every stage, from a bench.py --dump-ops file: python scripts/ops_clock_table.py ops.json"""
import json,sys,statistics as st
for f in sys.argv[1:]:
    d=json.load(open(f))
    print("==",f)
    for s in sorted({x["stage"] for x in d}):
        its=[x for x in d if x["stage"]==s and x["counted"]]
        for mode in ("off","on"):
            sel=[x for x in its if x["mode"]==mode]
            n=len(sel[0]["ops"])
            mh=[st.mean(x["ops"][i][4] for x in sel) for i in range(n)]
            du=[st.mean((x["ops"][i][3]-x["ops"][i][2])/1e6 for x in sel) for i in range(n)]
            print(f"st{s} {mode:3s} MHz "+" ".join(f"{m:4.0f}" for m in mh))
            print(f"        dur "+" ".join(f"{m:4.1f}" for m in du))
        print("   order  "+" ".join(f"{o[0]}{o[1]:<3d}" for o in its[0]["ops"]))
