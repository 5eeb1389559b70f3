"""Mid-kernel preemption stress: the bubble flag is cleared by a timer kernel at a random
offset while a kernel runs (two streams, both behind one anchor event); the launch must
terminate, and resuming (GEMM: from the cursor; atomic kernels: re-run whole) must give
the uninterrupted result bit for bit. Run under `timeout`."""
import ctypes
import os
import random
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K, native  # noqa: E402

trials = int(sys.argv[1]) if len(sys.argv) > 1 else 60
random.seed(0)
torch.manual_seed(0)
flag = ctypes.c_void_p()
native.call("pf_flag_create", ctypes.byref(flag))
words = torch.zeros(8, dtype=torch.int32, device="cuda")
abort, cursor = words[0:1], words[1:2]
ctl = K.KernelCtl(flag.value, abort.data_ptr(), cursor.data_ptr())
anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
work, comm = torch.cuda.Stream(), torch.cuda.Stream()

qkv = torch.randn(128, 128, 3 * 1024, device="cuda").bfloat16()
x = torch.randn(16384, 1024, device="cuda").bfloat16()
w = (torch.randn(1024, 1024, device="cuda") * 0.03).bfloat16()
b = torch.randn(1024, device="cuda").bfloat16()
r = torch.randn(16384, 1024, device="cuda").bfloat16()
r4 = torch.randn(16384, 4096, device="cuda").bfloat16()
w4 = (torch.randn(1024, 4096, device="cuda") * 0.015).bfloat16()
g1 = torch.ones(1024, device="cuda").bfloat16()
b0 = torch.zeros(1024, device="cuda").bfloat16()
cases = {
    "attention": (lambda out, c: K.attention(qkv, 16, out=out, ctl=c, stream=work),
                  torch.empty(128, 128, 1024, device="cuda").bfloat16(), False),
    "gemm_tail": (lambda out, c: K.linear(x, w, b, residual=r, out=out, ctl=c, stream=work),
                  torch.empty(16384, 1024, device="cuda").bfloat16(), True),
    "gemm_pair": (lambda out, c: K.linear(r4, w4, b, residual=x, out=out, ctl=c, stream=work),
                  torch.empty(16384, 1024, device="cuda").bfloat16(), True),
    "layernorm": (lambda out, c: K.layernorm(x, g1, b0, 1e-12, residual=r, out=out, ctl=c, stream=work),
                  torch.empty(16384, 1024, device="cuda").bfloat16(), False),
}
units_of = {"attention": K.attention_units(128, 128, 16, 64), "gemm_tail": K.gemm_units(16384, 1024, 1024),
            "layernorm": K.norm_units(16384, 1024), "gemm_pair": K.gemm_units(16384, 1024, 4096)}
for name, (fn, out, resumable) in cases.items():
    ref = out.clone()
    with torch.cuda.stream(work):
        fn(ref, None)
    torch.cuda.synchronize()
    stopped = mid = 0
    t0 = time.time()
    for t in range(trials):
        out.zero_()
        words.zero_()
        native.call("pf_flag_write_on_stream", flag, 1, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        delay = random.randint(0, 40_000)  # ns after the anchor
        with torch.cuda.stream(comm):
            torch.cuda._sleep(300_000)  # the host enqueues everything before the anchor is taken
        native.call("pf_read_globaltimer", anchor.data_ptr(), comm.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(comm)
        work.wait_event(ev)
        native.call("pf_flag_clear_at", flag, anchor.data_ptr(), delay, None, comm.cuda_stream)
        fn(out, ctl)
        torch.cuda.synchronize()
        if abort.item():
            stopped += 1
            mid += 0 < cursor.item() < units_of[name] or out.abs().sum().item() > 0
            native.call("pf_flag_write_on_stream", flag, 1, torch.cuda.current_stream().cuda_stream)
            abort.zero_()
            if not resumable:
                cursor.zero_()
                out.zero_()
            torch.cuda.synchronize()
            fn(out, ctl)  # resume
            torch.cuda.synchronize()
        if not torch.equal(out, ref):
            print(f"{name}: trial {t} (delay {delay} ns) MISMATCH", flush=True)
            sys.exit(1)
    print(f"{name}: {trials} trials, {stopped} stopped ({mid} after doing some work), all exact "
          f"({time.time() - t0:.1f} s)", flush=True)
native.call("pf_flag_destroy", flag)
