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
