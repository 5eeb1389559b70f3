import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K, native
from scripts.kernel_bench import timeit
native.require_device()
SHAPES = [(4096, 2304, 768), (4096, 3072, 768), (4096, 768, 3072), (16384, 3072, 768), (4096, 3072, 3072)]
if len(sys.argv) > 1:  # e.g. 16384x4096x1024 16384x1024x4096
    SHAPES = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for (m, n, k) in SHAPES:
    x = torch.randn(m, k, device="cuda").bfloat16()
    w = (torch.randn(n, k, device="cuda") * k ** -0.5).bfloat16()
    b = torch.randn(n, device="cuda").bfloat16()
    r = torch.randn(m, n, device="cuda").bfloat16()
    y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * m * n * k
    out = []
    for name, kw in [("plain", {}), ("bias", dict(bias=b)), ("bias+gelu", dict(bias=b, gelu=True)), ("bias+res", dict(bias=b, residual=r))]:
        bb = kw.pop("bias", None)
        for flush in (True, False):
            t = timeit(lambda: K.linear(x, w, bb, out=y, **kw), flush=flush)
            out.append(f"{name}{'' if flush else '(warm)'}={t*1e6:.1f}us/{fl/t/1e12:.0f}TF")
    tc = timeit(lambda: torch.matmul(x, w.T, out=y))
    print(m, n, k, " ".join(out), f"cublas={tc*1e6:.1f}us/{fl/tc/1e12:.0f}TF")
