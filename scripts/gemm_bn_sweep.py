"""Time the BERT-large fill GEMM shapes (batch 128: M = 16384) per epilogue; run with
PF_GEMM_BN=128/192/256 to pin the tile width."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K, native
from scripts.kernel_bench import timeit
native.require_device()
res = []
for (m, n, k, epi) in [(16384, 3072, 1024, "bias"), (16384, 1024, 1024, "res"), (16384, 4096, 1024, "gelu"),
                       (16384, 1024, 4096, "res")]:
    x = torch.randn(m, k, device="cuda").bfloat16()
    w = (torch.randn(n, k, device="cuda") * k ** -0.5).bfloat16()
    b = torch.randn(n, device="cuda").bfloat16()
    r = torch.randn(m, n, device="cuda").bfloat16()
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    kw = {"bias": dict(), "res": dict(residual=r), "gelu": dict(gelu=True)}[epi]
    t = timeit(lambda: K.linear(x, w, b, out=y, **kw), flush=True)
    res.append(f"{m}x{n}x{k}/{epi}: {t*1e6:.1f}us {2.0*m*n*k/t/1e12:.0f}TF")
print(os.environ.get("PF_GEMM_BN", "auto"), " | ".join(res))
