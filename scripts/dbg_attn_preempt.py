"""Attention preemption stress: launches cleared by a timer at random offsets, then
re-run whole (cursor/abort reset) -- must equal an unpreempted launch bit for bit."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K, native  # noqa: E402

torch.manual_seed(0)
for (B, S, H) in [(16, 128, 4), (64, 128, 16), (128, 128, 16)]:
    qkv = torch.randn(B, S, 3 * H * 64, device="cuda").bfloat16()
    ref = K.attention(qkv, H)
    ref2 = K.attention(qkv, H)
    print("deterministic", torch.equal(ref, ref2))
    flag = ctypes.c_void_p()
    native.call("pf_flag_create", ctypes.byref(flag))
    fl = torch.cuda.IntTensor()  # unused
    words = torch.zeros(8, dtype=torch.int32, device="cuda")
    abort, cursor = words[0:1], words[1:2]
    ctl = K.KernelCtl(flag.value, abort.data_ptr(), cursor.data_ptr())
    anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
    comm = torch.cuda.Stream()
    bad = 0
    units = K.attention_units(B, S, H, 64)
    stats = []
    for t in range(40):
        out = torch.full_like(ref, float("nan"))
        words.zero_()
        torch.cuda.synchronize()
        native.call("pf_read_globaltimer", anchor.data_ptr(), comm.cuda_stream)
        native.call("pf_flag_write_on_stream", flag, 1, comm.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(comm)
        native.call("pf_flag_clear_at", flag, anchor.data_ptr(), 2_000 + 1_000 * t, None, comm.cuda_stream)
        torch.cuda.current_stream().wait_event(ev)
        K.attention(qkv, H, out=out, ctl=ctl)
        torch.cuda.synchronize()
        c1, a1 = cursor.item(), abort.item()
        if c1 >= units and not torch.equal(out, ref):
            bad += 1
            d = (out.float() - ref.float()).abs().view(B, S, H, 64)
            print("complete but differs", t, c1, a1, torch.nonzero(d.isnan() | (d > 0)).shape)
        words.zero_()
        native.call("pf_flag_write_on_stream", flag, 1, torch.cuda.current_stream().cuda_stream)
        K.attention(qkv, H, out=out, ctl=ctl)
        torch.cuda.synchronize()
        if not torch.equal(out, ref):
            bad += 1
            d = (out.float() - ref.float()).abs().view(B, S, H, 64)
            nz = torch.nonzero(d.isnan() | (d > 0))
            print("rerun differs", t, c1, a1, cursor.item(), nz.shape, nz[:3].tolist())
        stats.append((c1, a1))
    print(B, S, H, "units", units, "bad", bad, "first-run (cursor, abort):", stats[:10], stats[-5:])
    native.call("pf_flag_destroy", flag)
