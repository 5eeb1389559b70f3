"""Run a few ResNet-50 training steps (224x224, batch B) through the Executor, for ncu
launch lists: python scripts/train_step_profile.py [B] [steps]"""
import sys, time, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))), "tests"))
import paper_2410_07192_b200 as pf
from paper_2410_07192_b200 import native
from paper_2410_07192_b200.executor import BubbleSlot, Executor
from paper_2410_07192_b200.training import resnet50_train
from test_train_gpu import _plan_item
native.require_device()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
model = resnet50_train(seed=0)
item = _plan_item(pf, model, B * steps, B)
ex = Executor(40 << 30)
ex.load(item, model)
times = []
for k in range(steps):
    ex.fill(BubbleSlot(0, None, 0))
    rec = ex.settle()
    times.append((rec.fill_end_ns - rec.fill_start_ns) / 1e6)
print("step ms", [round(t, 2) for t in times], "images/s", B / (min(times) / 1e3))
ex.close()
