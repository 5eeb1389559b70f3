import ctypes, sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2410_07192_b200 as pf
from paper_2410_07192_b200 import native
from paper_2410_07192_b200.executor import BubbleSlot, Executor
from paper_2410_07192_b200.fillmodels import bert
from test_executor_gpu import tiny_cfg, plan_item
native.require_device()
model = bert(tiny_cfg(), seed=6)
item, plan = plan_item(pf, model, samples=48, free_mem=8_000_000_000, sizes=(8, 16))
print(plan)
flag = ctypes.c_void_p(); native.call("pf_flag_create", ctypes.byref(flag))
anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
comm = torch.cuda.Stream()
ex = Executor(256 << 20, job_seed=2); ex.load(item, model)
for k in range(40):
    with torch.cuda.stream(comm):
        torch.cuda._sleep(400_000)
    native.call("pf_read_globaltimer", anchor.data_ptr(), comm.cuda_stream)
    native.call("pf_flag_write_on_stream", flag, 1, comm.cuda_stream)
    ev = torch.cuda.Event(); ev.record(comm)
    native.call("pf_flag_clear_at", flag, anchor.data_ptr(), 50_000 + 100_000 * (k % 4), None, comm.cuda_stream)
    rec = ex.fill(BubbleSlot(k % 2, ev, flag.value))
    if rec: print(k, rec, ex.progress, "anchor", anchor.item())
    if not ex.busy: break
ex.settle()
print(ex.records[-1], ex.progress)
w = ex._ctl_host.tensor
print("ctl words", w[:4].tolist(), w[64:64+25].tolist())
