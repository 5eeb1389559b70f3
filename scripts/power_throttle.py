"""Power-cap physics of a fill job on B200 (power-aware bubble tail).

1. Steady state: the BERT-large FFN1 GEMM (M=16384, N=4096, K=1024, bias+GELU, CTA pairs)
   back to back for ~0.6 s with the bubble flag at v (1 = all CTAs, v >= 2 = v CTAs claim
   tiles): TFLOP/s and the SM clock (pf_sm_clock_probe on a side stream).
2. Recovery: after 300 ms of full-power GEMMs the flag drops to v (or the GEMMs stop,
   v = 0); the SM clock is probed every ~1 ms for 60 ms.

    python scripts/power_throttle.py [out.json]
"""
import ctypes
import json
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2410_07192_b200 import native  # noqa: E402
from paper_2410_07192_b200.kernels import KernelCtl, linear  # noqa: E402

M, N, K = 16384, 4096, 1024


def main():
    native.require_device()
    torch.manual_seed(0)
    x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(N, K, device="cuda", dtype=torch.bfloat16) * 0.02
    b = torch.zeros(N, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    flag = ctypes.c_void_p()
    native.call("pf_flag_create", ctypes.byref(flag))
    words = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")  # [0]=abort, [1..]=cursors
    probe = torch.zeros(3 * 4096, dtype=torch.int64, device="cuda")
    side = torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])
    main_s = torch.cuda.current_stream()
    nlaunch = [0]

    def gemm(n):
        for _ in range(n):
            i = 1 + nlaunch[0] % 60000
            nlaunch[0] += 1
            ctl = KernelCtl(flag.value, words.data_ptr(), words.data_ptr() + 4 * i)
            linear(x, w, b, gelu=True, out=y, ctl=ctl)

    def set_flag(v, stream):
        native.call("pf_flag_write_on_stream", flag, v, stream.cuda_stream)

    def probes(n, spin_ns, gap_ns, stream, start=0):
        # n probes of spin_ns each, separated by gap_ns (a wait kernel) on `stream`
        for k in range(n):
            native.call("pf_sm_clock_probe", probe.data_ptr() + 24 * (start + k), spin_ns, stream.cuda_stream)
            if gap_ns:
                native.call("pf_wait_until", probe.data_ptr() + 24 * (start + k), spin_ns + gap_ns, None,
                            stream.cuda_stream)

    def read(n, start=0):
        torch.cuda.synchronize()
        p = probe[3 * start:3 * (start + n)].view(n, 3).cpu()
        return [(int(r[0]), float(r[2]) * 1e3 / float(r[1])) for r in p]

    flops = 2.0 * M * N * K
    # warm up
    words.zero_()
    set_flag(1, main_s)
    gemm(50)
    torch.cuda.synchronize()
    out = {"steady": [], "recovery": []}
    for v in (1, 148, 128, 112, 100, 90, 80, 74, 64):
        words.zero_()
        nlaunch[0] = 0
        set_flag(max(v, 1), main_s)
        gemm(500)  # settle the clock at this level (~60 ms)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev = torch.cuda.Event()
        ev.record(main_s)
        side.wait_event(ev)
        e0.record(main_s)
        probes(40, 2_000_000, 10_000_000, side)
        gemm(4500)
        e1.record(main_s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        mhz = [m for t, m in read(40) if t > 0]
        mhz = sorted(mhz)[len(mhz) // 4: 3 * len(mhz) // 4] or mhz
        row = {"v": v, "tflops": 4500 * flops / (ms / 1e3) / 1e12, "ms": ms,
               "sm_mhz": sum(mhz) / len(mhz) if mhz else None}
        out["steady"].append(row)
        print("steady", row, flush=True)
    for v in (0, 100, 80, 64):
        words.zero_()
        nlaunch[0] = 0
        set_flag(1, main_s)
        gemm(2500)  # ~300 ms at full power
        ev = torch.cuda.Event()
        if v == 0:
            ev.record(main_s)  # GEMMs end here; the GPU idles
            side.wait_event(ev)
            probes(60, 200_000, 800_000, side)
        else:
            set_flag(v, main_s)
            ev.record(main_s)
            side.wait_event(ev)
            probes(60, 200_000, 800_000, side)
            gemm(800)
        rows = read(60)
        t0 = rows[0][0]
        curve = [((t - t0) / 1e6, m) for t, m in rows]
        out["recovery"].append({"v": v, "curve": curve})
        print("recovery v=%d" % v, " ".join(f"{t:.0f}:{m:.0f}" for t, m in curve[::4]), flush=True)
    torch.cuda.synchronize()
    native.call("pf_flag_destroy", flag)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            json.dump(out, fh)


if __name__ == "__main__":
    main()
