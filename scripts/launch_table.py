"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration, dram bytes): python scripts/launch_table.py launches.csv [all]"""
import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r: hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
# group by launch id
by=collections.OrderedDict()
for d in data:
    k=d["ID"]; e=by.setdefault(k,{"name":d["Kernel Name"]})
    v=d["Metric Value"].replace(",","")
    try: e[d["Metric Name"]]=float(v)
    except: pass
    e["unit_"+d["Metric Name"]]=d["Metric Unit"]
L=list(by.values())
n=len(L); half=L[n//2:] if len(sys.argv)<3 else L
tot=sum(e.get("gpu__time_duration.sum",0) for e in half)
agg=collections.defaultdict(lambda:[0,0.0,0.0])
for e in half:
    nm=e["name"].split("(")[0].replace("void ","")
    nm=nm.split("<")[0]
    a=agg[nm]; a[0]+=1; a[1]+=e.get("gpu__time_duration.sum",0); a[2]+=e.get("dram__bytes_read.sum",0)+e.get("dram__bytes_write.sum",0)
print("launches",len(half),"total", tot, half[0].get("unit_gpu__time_duration.sum"))
for nm,(c,t,b) in sorted(agg.items(), key=lambda x:-x[1][1])[:25]:
    print(f"{nm:45s} {c:5d} {t/1e3 if half[0].get('unit_gpu__time_duration.sum')=='nsecond' else t:10.1f} {100*t/tot:5.1f}%  {b/1e6:9.1f} MB")
