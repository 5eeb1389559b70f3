"""Attention kernel device time vs batch size (heads 16, seq 128): 20 back-to-back launches
between two events (no per-launch event quantisation), inputs hot in L2 when they fit, and
the same after an L2 flush (one launch). A/B with PF_ATT_V=1 (P-in-smem kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K  # noqa: E402

scratch = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for bsz in (8, 16, 32, 48, 64, 96, 128):
    heads = 16
    qkv = torch.randn(bsz, 128, 3 * heads * 64, device="cuda").bfloat16()
    o = torch.empty(bsz, 128, heads * 64, device="cuda").bfloat16()
    byts = qkv.numel() * 2 + o.numel() * 2
    for _ in range(3):
        K.attention(qkv, heads, out=o)
    torch.cuda.synchronize()
    n = 20
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)
    a.record()
    for _ in range(n):
        K.attention(qkv, heads, out=o)
    b.record()
    torch.cuda.synchronize()
    hot = a.elapsed_time(b) * 1e3 / n
    cold = []
    for _ in range(10):
        scratch.zero_()
        torch.cuda._sleep(1_000_000)
        a.record()
        K.attention(qkv, heads, out=o)
        b.record()
        torch.cuda.synchronize()
        cold.append(a.elapsed_time(b) * 1e3)
    cold.sort()
    print(f"ATT_V={os.environ.get('PF_ATT_V', 'tp')} b{bsz:3d} h16: back-to-back {hot:7.2f} us ({byts / hot / 1e3:6.0f} GB/s) "
          f"cold {cold[len(cold) // 2]:7.2f} us ({byts / cold[len(cold) // 2] / 1e3:6.0f} GB/s)  MB {byts / 1e6:.0f}")
