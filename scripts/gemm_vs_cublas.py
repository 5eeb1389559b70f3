"""pf_gemm vs cuBLAS (torch.matmul / addmm) at the fill job's BERT-large batch-128 shapes,
both captured in CUDA graphs (no host launch overhead), L2 warm, CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K  # noqa: E402

REPS = 20


def graph_time(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(REPS):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / REPS * 1e3  # us


for (m, n, k, name) in [(16384, 3072, 1024, "QKV"), (16384, 1024, 1024, "out"), (16384, 4096, 1024, "FFN1"),
                        (16384, 1024, 4096, "FFN2")]:
    x = torch.randn(m, k, device="cuda").bfloat16()
    w = (torch.randn(n, k, device="cuda") * k ** -0.5).bfloat16()
    b = torch.randn(n, device="cuda").bfloat16()
    y = torch.empty(m, n, device="cuda").bfloat16()
    ours = graph_time(lambda: K.linear(x, w, b, out=y))
    cub = graph_time(lambda: torch.addmm(b, x, w.t(), out=y))
    fl = 2.0 * m * n * k
    print(f"{name:5s} {m}x{n}x{k}: pf_gemm+bias {ours:6.1f} us {fl / ours / 1e6:6.0f} TF | cuBLAS addmm {cub:6.1f} us "
          f"{fl / cub / 1e6:6.0f} TF")
