"""Per-kernel device timing (CUDA events, L2 flushed between reps) vs. measured peaks."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import kernels as K, native  # noqa: E402

PEAKS = {"bf16_tflops": 1640.6, "hbm_gbs": 6466.1}
try:
    PEAKS.update(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))))
except OSError:
    pass


def timeit(fn, reps=20, flush=True):
    scratch = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush:
            scratch.zero_()
        torch.cuda._sleep(400_000)  # let the host enqueue fn() before the start event fires
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    native.require_device()
    graphs = "--graph" in sys.argv
    rows = []
    for (m, n, k, gelu, res, name) in [
        (4096, 2304, 768, False, False, "bert-base qkv"),
        (4096, 768, 768, False, True, "bert-base attn-out"),
        (4096, 3072, 768, True, False, "bert-base ffn1"),
        (4096, 768, 3072, False, True, "bert-base ffn2"),
        (4096, 3072, 1024, False, False, "bert-large qkv"),
        (4096, 4096, 1024, True, False, "bert-large ffn1"),
        (4096, 1024, 4096, False, True, "bert-large ffn2"),
        (8192, 8192, 8192, False, False, "square 8k"),
    ]:
        x = torch.randn(m, k, device="cuda").bfloat16()
        w = (torch.randn(n, k, device="cuda") * k ** -0.5).bfloat16()
        b = torch.randn(n, device="cuda").bfloat16()
        r = torch.randn(m, n, device="cuda").bfloat16() if res else None
        y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        t = timeit(lambda: K.linear(x, w, b, gelu=gelu, residual=r, out=y))
        tc = timeit(lambda: torch.matmul(x, w.T, out=y))
        fl = 2.0 * m * n * k
        rows.append(dict(kernel="pf_gemm", case=name, us=t * 1e6, tflops=fl / t / 1e12,
                         frac=fl / t / 1e12 / PEAKS["bf16_tflops"], cublas_us=tc * 1e6,
                         cublas_tflops=fl / tc / 1e12, units=K.gemm_units(m, n, k)))
    for (rows_, cols) in [(4096, 768), (4096, 1024)]:
        x = torch.randn(rows_, cols, device="cuda").bfloat16()
        r = torch.randn(rows_, cols, device="cuda").bfloat16()
        g = torch.ones(cols, device="cuda").bfloat16()
        bb = torch.zeros(cols, device="cuda").bfloat16()
        y = torch.empty_like(x)
        t = timeit(lambda: K.layernorm(x, g, bb, residual=r, out=y))
        byts = 3 * rows_ * cols * 2
        rows.append(dict(kernel="pf_layernorm+res", case=f"{rows_}x{cols}", us=t * 1e6, gbs=byts / t / 1e9,
                         frac=byts / t / 1e9 / PEAKS["hbm_gbs"]))
    for (bsz, heads) in [(32, 12), (32, 16)]:
        qkv = torch.randn(bsz, 128, 3 * heads * 64, device="cuda").bfloat16()
        o = torch.empty(bsz, 128, heads * 64, device="cuda").bfloat16()
        t = timeit(lambda: K.attention(qkv, heads, out=o))
        fl = 4.0 * bsz * heads * 128 * 128 * 64
        byts = qkv.numel() * 2 + o.numel() * 2
        rows.append(dict(kernel="pf_attention", case=f"b{bsz} h{heads} s128", us=t * 1e6, tflops=fl / t / 1e12,
                         gbs=byts / t / 1e9))
    x = torch.randn(384 * 128, 128, device="cuda").bfloat16()
    y = torch.empty_like(x)
    t = timeit(lambda: K.softmax(x, 0.125, out=y))
    rows.append(dict(kernel="pf_softmax", case="49152x128", us=t * 1e6, gbs=2 * x.numel() * 2 / t / 1e9))
    for r_ in rows:
        print(json.dumps(r_))


if __name__ == "__main__":
    main()
