"""LayerNorm kernel variants (PF_LN_MINB=0: norm_kernel, 8 / 10: norm_packed_kernel at that
many CTAs/SM): device time per launch with and without an L2 flush, and an output digest so
the variants can be checked bitwise against each other. One variant per process (the env
var is read once)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K, native  # noqa: E402
from scripts.kernel_bench import timeit  # noqa: E402


def main():
    native.require_device()
    g = torch.Generator(device="cuda").manual_seed(0)
    for rows, cols in [(16384, 1024), (4096, 768), (16384, 768), (2048, 1024)]:
        x = (torch.randn(rows, cols, device="cuda", generator=g) * 3 + 0.5).bfloat16()
        ga = (torch.rand(cols, device="cuda", generator=g) + 0.5).bfloat16()
        be = torch.randn(cols, device="cuda", generator=g).bfloat16()
        y = torch.empty_like(x)
        K.layernorm(x, ga, be, 1e-12, out=y)
        torch.cuda.synchronize()
        digest = int(y.view(torch.int16).to(torch.int64).mul(torch.arange(1, y.numel() + 1, device="cuda").view_as(y) % 65521).sum())
        ref = torch.nn.functional.layer_norm(x.float(), (cols,), ga.float(), be.float(), 1e-12)
        err = ((y.float() - ref).abs().max() / ref.abs().max()).item()
        t_cold = timeit(lambda: K.layernorm(x, ga, be, 1e-12, out=y), reps=30, flush=True)
        t_warm = timeit(lambda: K.layernorm(x, ga, be, 1e-12, out=y), reps=30, flush=False)
        gb = 2 * rows * cols * 2 / 1e9
        print(f"LN_MINB={os.environ.get('PF_LN_MINB', 'default')} [{rows},{cols}] cold {t_cold*1e6:.2f} us "
              f"({gb/t_cold:.0f} GB/s) warm(L2) {t_warm*1e6:.2f} us ({gb/t_warm:.0f} GB/s) rel_err {err:.2e} digest {digest}")


if __name__ == "__main__":
    main()
