"""Attention kernel timing (CUDA events; L2 flushed between reps, and hot) at the fill
job's shapes. A/B against another build with PF_LIB_PATH=<lib>."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K  # noqa: E402
from scripts.kernel_bench import timeit  # noqa: E402

out = []
for (bsz, heads) in [(128, 16), (32, 16), (32, 12), (8, 16)]:
    qkv = torch.randn(bsz, 128, 3 * heads * 64, device="cuda").bfloat16()
    o = torch.empty(bsz, 128, heads * 64, device="cuda").bfloat16()
    byts = qkv.numel() * 2 + o.numel() * 2
    for flush in (True, False):
        t = timeit(lambda: K.attention(qkv, heads, out=o), reps=30, flush=flush)
        out.append(dict(lib=os.environ.get("PF_LIB_PATH", "in-tree"), case=f"b{bsz} h{heads} s128",
                        flush=flush, us=round(t * 1e6, 2), gbs=round(byts / t / 1e9, 1)))
for r in out:
    print(json.dumps(r))
