"""Partitioned ResNet-50 training under timer-preempted bubbles, with a progress trace
(debugging aid for executor._fill_tp / _settle_tp): python scripts/tp_preempt_debug.py [bubbles]"""
import ctypes
import faulthandler
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2410_07192_b200 as pf  # noqa: E402
from paper_2410_07192_b200 import native  # noqa: E402
from paper_2410_07192_b200.executor import BubbleSlot, Executor  # noqa: E402
from paper_2410_07192_b200.fillmodels import ResNetConfig  # noqa: E402
from paper_2410_07192_b200.training import resnet50_train  # noqa: E402
from test_train_gpu import _partitioned_item  # noqa: E402

native.require_device()
n_bubbles = int(sys.argv[1]) if len(sys.argv) > 1 else 300
faulthandler.dump_traceback_later(100, exit=True)  # a hang: where the host is blocked
cfg = ResNetConfig(image=64)
batch, steps = 16, 3
part = resnet50_train(cfg, seed=11, partitioned=True)
item, plan = _partitioned_item(pf, part, batch * steps, batch, 0.45)
print("plan", [(p.lo, p.hi) for p in plan.partitions], flush=True)
ex = Executor(8 << 30, job_seed=5, use_graphs=os.environ.get("PF_EXEC_GRAPHS", "1") != "0")
t0 = time.time()
ex.load(item, part)
print("load s", round(time.time() - t0, 2), flush=True)
flag, comm = ctypes.c_void_p(), torch.cuda.Stream()
native.call("pf_flag_create", ctypes.byref(flag))
anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
k = 0
t0 = time.time()
last = [time.time()]
last_queue = [None]


def watchdog():
    """On a stall, read the control block and the in-kernel node stamps on a side stream."""
    import threading
    side = torch.cuda.Stream()
    while True:
        time.sleep(5)
        if time.time() - last[0] > 30:
            torch.cuda.set_device(0)
            ctl = torch.empty(ex._ctl.numel(), dtype=torch.int32).pin_memory()
            st = torch.empty(ex._stamps.numel(), dtype=torch.int64).pin_memory()
            native.call("pf_stage_d2h", ctl.data_ptr(), ex._ctl.data_ptr(), 4 * ex._ctl.numel(), side.cuda_stream)
            native.call("pf_stage_d2h", st.data_ptr(), ex._stamps.data_ptr(), 8 * ex._stamps.numel(), side.cuda_stream)
            side.synchronize()
            q = last_queue[0]
            print("STALL abort", int(ctl[0]), "done", int(ctl[1]), "staged", int(ctl[2]), "queue", q, flush=True)
            curs = ctl[64:64 + 400].tolist()
            print("cursors", curs, flush=True)
            stv = st.view(-1, 2)[:400]
            started = [(i, int(a), int(b)) for i, (a, b) in enumerate(stv.tolist()) if 0 < a < (1 << 62)]
            print("stamped nodes (node, start, end) last 10", started[-10:], flush=True)
            if q:
                qi = min(int(ctl[1]), len(q) - 1)
                kind, pidx = ex._tp_phases()[q[qi][1]]
                ch = ex._chains.get(((kind, pidx), 16, flag.value))
                if ch is not None:
                    start = q[qi][2]
                    inc = [(j, int(ctl[64 + j]), u, r) for j, (u, r) in enumerate(ch.units) if j >= start
                           and int(ctl[64 + j]) < u]
                    print("phase", kind, pidx, "start node", start, "nodes", len(ch.units),
                          "incomplete (node, cursor, units, prefix)", inc[:12], flush=True)
            os._exit(3)


import threading  # noqa: E402
threading.Thread(target=watchdog, daemon=True).start()
while ex.busy and k < n_bubbles:
    with torch.cuda.stream(comm):
        torch.cuda._sleep(300_000)
    native.call("pf_read_globaltimer", anchor.data_ptr(), comm.cuda_stream)
    native.call("pf_flag_write_on_stream", flag, 1, comm.cuda_stream)
    ev = torch.cuda.Event()
    ev.record(comm)
    native.call("pf_flag_clear_at", flag, anchor.data_ptr(), 200_000 + 300_000 * (k % 4), None, comm.cuda_stream)
    t1 = time.time()
    rec = ex.fill(BubbleSlot(k % 2, ev, flag.value))
    t2 = time.time()
    last[0] = t2
    last_queue[0] = ex.pending.tp if ex.pending is not None else None
    if k < 20 or k % 25 == 0 or k >= 40:
        ts = ex._tp_state
        print(f"k {k} fill {1e3 * (t2 - t1):.1f} ms rec={None if rec is None else (rec.batches_planned, rec.batches_done, rec.aborted)} "
              f"state {ts} next {ex.progress.next_sample} resume {ex.progress.resume} starved {ex.starved} "
              f"queue {ex.pending.tp if ex.pending is not None else None}", flush=True)
    k += 1
ex.settle()
torch.cuda.synchronize()
print("bubbles", k, "busy", ex.busy, "s", round(time.time() - t0, 1), "preempted", sum(r.aborted for r in ex.records),
      flush=True)
ex.close()
