"""The packed full-row LayerNorm (norm_packed_kernel, the default for the BERT LayerNorms)
against the guarded norm_kernel it replaced (PF_LN_MINB=0): bitwise the same outputs. The
variant is chosen once per process from the environment, so each runs in a subprocess."""

import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
from paper_2410_07192_b200 import kernels as K, native
native.require_device()
g = torch.Generator().manual_seed(11)
outs = []
for rows, cols, rms in [(16384, 1024, False), (4096, 768, False), (1000, 2048, True), (7001, 1024, False)]:
    x = (torch.randn(rows, cols, generator=g) * 3 + 0.5).bfloat16().cuda()
    ga = (torch.rand(cols, generator=g) + 0.5).bfloat16().cuda()
    be = torch.randn(cols, generator=g).bfloat16().cuda()
    y = K.rmsnorm(x, ga, 1e-6) if rms else K.layernorm(x, ga, be, 1e-12)
    outs.append(y.cpu())
torch.cuda.synchronize()
torch.save(outs, {out!r})
"""


def _run(tmp_path, minb: str):
    out = str(tmp_path / f"ln_{minb}.pt")
    env = dict(os.environ, PF_LN_MINB=minb)
    subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, out=out)], env=env, check=True, timeout=300)
    return torch.load(out)


def test_packed_layernorm_is_bitwise_the_guarded_kernel(tmp_path):
    packed = _run(tmp_path, "8")
    guarded = _run(tmp_path, "0")
    for a, b in zip(packed, guarded):
        assert torch.equal(a.view(torch.int16), b.view(torch.int16))
