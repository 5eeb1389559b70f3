"""Repeats the executor preemption/resume test and reports which samples differ and the
resume history of failing runs."""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2410_07192_b200 as pf  # noqa: E402
from paper_2410_07192_b200 import native  # noqa: E402
from paper_2410_07192_b200.executor import BubbleSlot, Executor  # noqa: E402
from paper_2410_07192_b200.fillmodels import bert  # noqa: E402
from test_executor_gpu import plan_item, tiny_cfg  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
model = bert(tiny_cfg(), seed=6)
item, plan = plan_item(pf, model, samples=48, free_mem=8_000_000_000, sizes=(8, 16))
ex0 = Executor(256 << 20, job_seed=2)
ex0.load(item, model)
k = 0
while ex0.busy:
    ex0.fill(BubbleSlot(k % 2, None, 0))
    k += 1
ex0.settle()
torch.cuda.synchronize()
ref = ex0.results().clone()
ex0.close()
flag = ctypes.c_void_p()
native.call("pf_flag_create", ctypes.byref(flag))
anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
comm = torch.cuda.Stream()
fails = 0
RA = os.environ.get("PF_RUN_AHEAD", "1") != "0"
for rep in range(reps):
    ex = Executor(256 << 20, job_seed=2)
    ex.run_ahead = RA
    ex.load(item, model)
    hist = []
    k = 0
    while ex.busy and k < 2000:
        with torch.cuda.stream(comm):
            torch.cuda._sleep(400_000)
        native.call("pf_read_globaltimer", anchor.data_ptr(), comm.cuda_stream)
        native.call("pf_flag_write_on_stream", flag, 1, comm.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(comm)
        native.call("pf_flag_clear_at", flag, anchor.data_ptr(), 50_000 + 100_000 * (k % 4), None, comm.cuda_stream)
        ex.fill(BubbleSlot(k % 2, ev, flag.value))
        hist.append((k, ex.progress.resume, ex.progress.resume_zero, ex.progress.next_sample))
        k += 1
    ex.settle()
    torch.cuda.synchronize()
    got = ex.results()
    if not torch.equal(got, ref):
        fails += 1
        d = (got.float() - ref.float()).abs()
        rows = torch.nonzero(d.amax(dim=tuple(range(1, d.dim()))) > 0).flatten().tolist()
        print(f"rep {rep}: FAIL samples differing {rows} maxdiff {d.max().item()}")
        for h in hist:
            print("   ", h)
        for r in ex.records:
            print("   ", r.index, r.batches_planned, r.batches_done, r.aborted, r.samples_done)
    else:
        print(f"rep {rep}: ok ({k} bubbles, {sum(r.aborted for r in ex.records)} aborted)")
    ex.close()
print("fails", fails, "of", reps, "run_ahead", RA, "graphs", os.environ.get("PF_EXEC_GRAPHS", "1"))
