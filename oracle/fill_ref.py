"""ORACLE — test infrastructure only. Never imported by the product path.

CPU fp32 restatement of the fill job's forward pass, the "reference CPU torch
execution" the north star (BASELINE.json) names as the numerics oracle for the
executor kernels. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module.

Parity status: UNPINNED by the reference. The reference package has no tensor
code at all (no torch/numpy math on the executor path), so there
is no golden vector for fill-job numerics. The semantics restated here are those
the paper gives for the fill executor — an nn.Sequential run partition by
partition over layer-index boundaries (partition.py:89-132) —
with BERT's standard post-LN encoder layer (exact erf GELU, LayerNorm eps 1e-12,
softmax attention in fp32) and ResNet-50 v1.5 in inference form (BatchNorm folded
into each convolution's weight and bias; torch.nn.functional.conv2d / max_pool2d /
adaptive_avg_pool2d on NCHW fp32). Tolerances (north star): bf16 path rel 2e-2.

Explicit ops only: no nn.TransformerEncoderLayer fast path, no SDPA.
"""

from __future__ import annotations

import math
from typing import Optional

import torch


def linear(x: torch.Tensor, w: torch.Tensor, b: Optional[torch.Tensor] = None, *,
           gelu: bool = False, residual: Optional[torch.Tensor] = None) -> torch.Tensor:
    """y = [gelu](x @ w.T + b) [+ residual], fp32."""
    y = x.float() @ w.float().T
    if b is not None:
        y = y + b.float()
    if gelu:
        y = 0.5 * y * (1.0 + torch.erf(y / math.sqrt(2.0)))
    if residual is not None:
        y = y + residual.float()
    return y


def layernorm(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, eps: float) -> torch.Tensor:
    x = x.float()
    mean = x.mean(-1, keepdim=True)
    var = ((x - mean) ** 2).mean(-1, keepdim=True)
    return (x - mean) / torch.sqrt(var + eps) * gamma.float() + beta.float()


def rmsnorm(x: torch.Tensor, gamma: torch.Tensor, eps: float) -> torch.Tensor:
    x = x.float()
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * gamma.float()


def softmax(x: torch.Tensor, scale: float = 1.0) -> torch.Tensor:
    z = x.float() * scale
    z = z - z.max(-1, keepdim=True).values
    e = torch.exp(z)
    return e / e.sum(-1, keepdim=True)


def attention(qkv: torch.Tensor, heads: int, mask_add: Optional[torch.Tensor] = None,
              scale: Optional[float] = None) -> torch.Tensor:
    """qkv [B, S, 3*hidden] packed as (3, heads, d) -> [B, S, hidden]."""
    b, s, three_h = qkv.shape
    hidden = three_h // 3
    d = hidden // heads
    if scale is None:
        scale = d ** -0.5
    t = qkv.float().view(b, s, 3, heads, d)
    q = t[:, :, 0].permute(0, 2, 1, 3)  # [B, H, S, d]
    k = t[:, :, 1].permute(0, 2, 1, 3)
    v = t[:, :, 2].permute(0, 2, 1, 3)
    scores = (q @ k.transpose(-1, -2)) * scale
    if mask_add is not None:
        scores = scores + mask_add.float()[:, None, None, :]
    p = softmax(scores)
    o = p @ v  # [B, H, S, d]
    return o.permute(0, 2, 1, 3).reshape(b, s, hidden)


def embedding_ln(ids: torch.Tensor, word: torch.Tensor, pos: torch.Tensor, typ: torch.Tensor,
                 gamma: torch.Tensor, beta: torch.Tensor, eps: float,
                 type_ids: Optional[torch.Tensor] = None) -> torch.Tensor:
    b, s = ids.shape
    x = word.float()[ids.long()] + pos.float()[:s][None, :, :]
    tt = torch.zeros_like(ids) if type_ids is None else type_ids
    x = x + typ.float()[tt.long()]
    return layernorm(x, gamma, beta, eps)


def bert_layer(x: torch.Tensor, p: dict, heads: int, eps: float = 1e-12,
               mask_add: Optional[torch.Tensor] = None) -> torch.Tensor:
    """One post-LN BERT encoder layer on [B, S, h] with weights dict `p` (fp32 math)."""
    b, s, h = x.shape
    x2 = x.float().reshape(b * s, h)
    qkv = linear(x2, p["qkv_w"], p["qkv_b"]).reshape(b, s, 3 * h)
    ctx = attention(qkv, heads, mask_add).reshape(b * s, h)
    a = linear(ctx, p["out_w"], p["out_b"], residual=x2)
    a = layernorm(a, p["ln1_g"], p["ln1_b"], eps)
    f = linear(a, p["ffn1_w"], p["ffn1_b"], gelu=True)
    o = linear(f, p["ffn2_w"], p["ffn2_b"], residual=a)
    o = layernorm(o, p["ln2_g"], p["ln2_b"], eps)
    return o.reshape(b, s, h)


def bert_embeddings(ids: torch.Tensor, p: dict, eps: float = 1e-12) -> torch.Tensor:
    return embedding_ln(ids, p["word"], p["pos"], p["type"], p["ln_g"], p["ln_b"], eps)


def bert_random_params(hidden: int, ffn: int, layers: int, vocab: int, seq: int, seed: int = 0):
    """Random-init BERT weights for the CPU baseline (N(0, 0.02), LN gamma 1 / beta 0 as the
    synthetic-input contract says): (embedding dict, [layer dicts]) in the
    shapes bert_embeddings / bert_layer take. Independent of the product package."""
    g = torch.Generator().manual_seed(seed)

    def n(*shape):
        return torch.randn(*shape, generator=g) * 0.02

    h = hidden
    emb = {"word": n(vocab, h), "pos": n(seq, h), "type": n(2, h), "ln_g": torch.ones(h), "ln_b": torch.zeros(h)}
    params = [{"qkv_w": n(3 * h, h), "qkv_b": torch.zeros(3 * h), "out_w": n(h, h), "out_b": torch.zeros(h),
               "ln1_g": torch.ones(h), "ln1_b": torch.zeros(h), "ffn1_w": n(ffn, h), "ffn1_b": torch.zeros(ffn),
               "ffn2_w": n(h, ffn), "ffn2_b": torch.zeros(h), "ln2_g": torch.ones(h), "ln2_b": torch.zeros(h)}
              for _ in range(layers)]
    return emb, params


def run_sequential(modules: list, x, lo: int, hi: int):
    """Run modules[lo:hi] in order — one partition of the linearized model
    (ExecutionPlan partition [lo, hi), pkg/src/bubblefill/partition.py:64-86)."""
    for i in range(lo, hi):
        x = modules[i](x)
    return x


# ---------------------------------------------------------------------------- ResNet-50


def conv_weight(w: torch.Tensor, cin: int, kh: int, kw: int) -> torch.Tensor:
    """[Cout, Kp] GEMM weight, columns (ky*kw + kx)*Cin + c (pad columns dropped) ->
    [Cout, Cin, kh, kw] conv2d weight."""
    cout = w.shape[0]
    return w[:, :kh * kw * cin].float().reshape(cout, kh, kw, cin).permute(0, 3, 1, 2).contiguous()


def conv_bn(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor, k: int, stride: int, pad: int,
            relu: bool, residual: Optional[torch.Tensor] = None) -> torch.Tensor:
    """NCHW fp32 conv with folded BN: relu(conv(x) + b [+ residual])."""
    cin = x.shape[1]
    y = torch.nn.functional.conv2d(x, conv_weight(w, cin, k, k), b.float(), stride=stride, padding=pad)
    if residual is not None:
        y = y + residual
    return torch.relu(y) if relu else y


def resnet_stem(img: torch.Tensor, p: dict) -> torch.Tensor:
    """img NHWC -> NCHW fp32 after conv7x7/2 + BN + ReLU + maxpool 3x3/2."""
    x = img.float().permute(0, 3, 1, 2)
    y = conv_bn(x, p["w"], p["b"], 7, 2, 3, relu=True)
    return torch.nn.functional.max_pool2d(y, 3, 2, 1)


def bottleneck(x: torch.Tensor, p: dict, stride: int) -> torch.Tensor:
    """NCHW fp32 bottleneck (v1.5: stride on the 3x3), projection shortcut when p has wd."""
    t = conv_bn(x, p["w1"], p["b1"], 1, 1, 0, relu=True)
    t = conv_bn(t, p["w2"], p["b2"], 3, stride, 1, relu=True)
    sc = conv_bn(x, p["wd"], p["bd"], 1, stride, 0, relu=False) if "wd" in p else x
    return conv_bn(t, p["w3"], p["b3"], 1, 1, 0, relu=True, residual=sc)


def resnet_head(x: torch.Tensor, p: dict) -> torch.Tensor:
    """NCHW fp32 -> logits [B, classes]: global average pool + fc."""
    pooled = x.mean(dim=(2, 3))
    return pooled @ p["fc_w"].float().T + p["fc_b"].float()


def nhwc(x: torch.Tensor) -> torch.Tensor:
    """NCHW -> NHWC (the executor's activation layout at partition boundaries)."""
    return x.permute(0, 2, 3, 1).contiguous()
