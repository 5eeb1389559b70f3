"""Per-phase timeline of the attention kernel from a -DPF_ATT_DIAG build
(PF_LIB_PATH=ablib/libpipefill_attdiag.so): SM cycles per unit phase, averaged over CTAs."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K, native  # noqa: E402

bsz, heads = int(sys.argv[1]), int(sys.argv[2])
qkv = torch.randn(bsz, 128, 3 * heads * 64, device="cuda").bfloat16()
o = torch.empty(bsz, 128, heads * 64, device="cuda").bfloat16()
for _ in range(3):
    K.attention(qkv, heads, out=o)
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
scratch.zero_()
K.attention(qkv, heads, out=o)
torch.cuda.synchronize()
buf = np.zeros((296, 8, 8), dtype=np.uint32)
native.load().pf_att_diag_read(buf.ctypes.data_as(ctypes.c_void_p))
names = ["tma_issue", "S_issue", "S_seen", "P_ready", "O_issue", "O_seen", "epi_done"]
units = min(8, (bsz * heads + 295) // 296)
print("mean SM cycles since CTA start, per unit (rows) x phase (cols):", names)
for i in range(units):
    print(i, [int(buf[:, i, e].mean()) for e in range(7)])
print("phase durations (mean over CTAs, units):")
d = {"load (tma->S issue)": (0, 1), "S mma (issue->seen)": (1, 2), "softmax (S seen->P ready)": (2, 3),
     "P ready->O issue": (3, 4), "O mma (issue->seen)": (4, 5), "epilogue": (5, 6)}
for k, (a, b) in d.items():
    v = [(int(buf[c, i, b]) - int(buf[c, i, a])) for c in range(296) for i in range(units) if buf[c, i, b]]
    print(f"  {k:28s} {np.mean(v):8.0f} cycles")
