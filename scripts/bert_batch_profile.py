"""Run BERT-large fill batches (seq 128, batch B) through the Executor, for ncu launch
lists / timing: python scripts/bert_batch_profile.py [B] [batches]"""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2410_07192_b200 as pf
from paper_2410_07192_b200 import native
from paper_2410_07192_b200.executor import BubbleSlot, Executor
from paper_2410_07192_b200.fillmodels import BERT_LARGE, bert
from test_train_gpu import _plan_item
native.require_device()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
import dataclasses
cfg = dataclasses.replace(BERT_LARGE, precision=os.environ.get("PRECISION", "bf16"))
model = bert(cfg, seed=0)
item = _plan_item(pf, model, B * n, B)
ex = Executor(8 << 30)
ex.load(item, model)
times = []
for k in range(n):
    ex.fill(BubbleSlot(0, None, 0))
    rec = ex.settle()
    times.append((rec.fill_end_ns - rec.fill_start_ns) / 1e6)
fl = cfg.flops_per_sample * B
print("batch ms", [round(t, 3) for t in times], "samples/s", B / (min(times) / 1e3),
      "TFLOP/s", fl / (min(times) / 1e3) / 1e12)
ex.close()

# in-situ per-GEMM-node durations (in-kernel %globaltimer stamps) of one more batch
ex = Executor(8 << 30)
ex.load(_plan_item(pf, model, B * 2, B), model)
ex.timing = True
for k in range(2):
    ex.fill(BubbleSlot(0, None, 0))
    rec = ex.settle()
tot = (rec.fill_end_ns - rec.fill_start_ns) / 1e6
g = ex.gemm_samples[-4 * cfg.layers:]
names = ["QKV", "out+res", "FFN1+gelu", "FFN2+res"]
gsum = 0.0
for j, nm in enumerate(names):
    v = g[j::4]
    ms = sum(t for _, t, *_ in v) / len(v)
    gsum += sum(t for _, t, *_ in v)
    print(f"{nm:10s} {ms * 1e3:7.1f} us  {v[0][0] / ms / 1e9:7.0f} TFLOP/s")
print(f"batch {tot:.3f} ms: GEMMs {gsum:.3f} ms ({gsum / tot * 100:.1f}%), rest {tot - gsum:.3f} ms "
      f"({(tot - gsum) / cfg.layers * 1e3:.1f} us per layer: attention + 2 LN + gates)")
# gaps between GEMM nodes from the raw in-kernel stamps (t0 = first CTA start, t1 = last CTA end)
ch = next(iter(ex._chains.values()))
nodes = sorted(ch.gemm_flops)
st = ex._stamps_host.tensor
ts = [(int(st[n, 0]), int(st[n, 1])) for n in nodes]
gaps = {"QKV->out (attention)": [], "out->FFN1 (LN)": [], "FFN1->FFN2 (adjacent)": [], "FFN2->QKV (LN, gate, next layer)": []}
keys = list(gaps)
for i in range(len(ts) - 1):
    gaps[keys[i % 4]].append((ts[i + 1][0] - ts[i][1]) / 1e3)
for k, v in gaps.items():
    print(f"{k:34s} mean {sum(v) / len(v):7.1f} us  min {min(v):6.1f}")
ex.close()
