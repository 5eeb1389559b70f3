"""Runs pf_attention a few times at one shape (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K  # noqa: E402

bsz, heads = int(sys.argv[1]), int(sys.argv[2])
qkv = torch.randn(bsz, 128, 3 * heads * 64, device="cuda").bfloat16()
o = torch.empty(bsz, 128, heads * 64, device="cuda").bfloat16()
for _ in range(4):
    K.attention(qkv, heads, out=o)
torch.cuda.synchronize()
