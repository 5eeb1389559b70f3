"""Launch one kernel config a few times (for ncu capture): python scripts/prof_kernel.py gemm M N K [gelu] [res]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K, native  # noqa: E402

native.require_device()
what = sys.argv[1]
reps = 5
if what == "gemm":
    m, n, k = map(int, sys.argv[2:5])
    gelu = "gelu" in sys.argv
    res = "res" in sys.argv
    x = torch.randn(m, k, device="cuda").bfloat16()
    w = (torch.randn(n, k, device="cuda") * k ** -0.5).bfloat16()
    b = torch.randn(n, device="cuda").bfloat16()
    r = torch.randn(m, n, device="cuda").bfloat16() if res else None
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(reps):
        K.linear(x, w, b, gelu=gelu, residual=r, out=y)
elif what == "ln":
    rows, cols = map(int, sys.argv[2:4])
    x = torch.randn(rows, cols, device="cuda").bfloat16()
    r = torch.randn(rows, cols, device="cuda").bfloat16()
    g = torch.ones(cols, device="cuda").bfloat16()
    bb = torch.zeros(cols, device="cuda").bfloat16()
    y = torch.empty_like(x)
    for _ in range(reps):
        K.layernorm(x, g, bb, residual=r, out=y)
elif what == "attn":
    bsz, heads = map(int, sys.argv[2:4])
    qkv = torch.randn(bsz, 128, 3 * heads * 64, device="cuda").bfloat16()
    for _ in range(reps):
        K.attention(qkv, heads)
torch.cuda.synchronize()
print("done")
