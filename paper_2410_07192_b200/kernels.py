"""Tensor-level wrappers over the sm_100a fill-job kernels (libpipefill.so).

torch is used here for device memory and stream handles only; every op below
is one call through the C ABI (include/pipefill.h) into a hand-written kernel.
Each op takes an optional :class:`KernelCtl` that makes the launch preemptible
by the stage's bubble flag (see pf_ctl_t).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import native
from .native import PF_EPI_BIAS, PF_EPI_GELU, PF_EPI_RELU, PF_EPI_RESIDUAL, PfCtl


@dataclass
class KernelCtl:
    """Device addresses of one launch's preemption words (flag, abort, cursor)."""

    flag: int = 0
    abort: int = 0
    cursor: int = 0

    def as_struct(self) -> PfCtl:
        return PfCtl(self.flag or None, self.abort or None, self.cursor or None)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ctl_ref(ctl: Optional[KernelCtl]):
    return None if ctl is None else ctypes.byref(ctl.as_struct())


def _check_bf16_cuda(name: str, t: torch.Tensor) -> None:
    if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous bf16 CUDA tensor, got {t.dtype} {t.device}")


def gemm_units(m: int, n: int, k: int) -> int:
    out = ctypes.c_uint32(0)
    native.call("pf_gemm_units", m, n, k, ctypes.byref(out))
    return out.value


def norm_units(rows: int, cols: int) -> int:
    out = ctypes.c_uint32(0)
    native.call("pf_norm_units", rows, cols, ctypes.byref(out))
    return out.value


def attention_units(batch: int, seq: int, heads: int, head_dim: int) -> int:
    out = ctypes.c_uint32(0)
    native.call("pf_attention_units", batch, seq, heads, head_dim, ctypes.byref(out))
    return out.value


def linear(
    x: torch.Tensor,
    weight: torch.Tensor,
    bias: Optional[torch.Tensor] = None,
    *,
    gelu: bool = False,
    residual: Optional[torch.Tensor] = None,
    relu: bool = False,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """out = [ReLU]([GELU](x @ weight.T + bias) [+ residual]) — tcgen05 GEMM (pf_gemm); fp32
    tensors take the fp32 path (pf_gemm_f32)."""
    if x.dtype == torch.float32:
        return _linear_f32(x, weight, bias, gelu=gelu, residual=residual, out=out, ctl=ctl, stream=stream)
    _check_bf16_cuda("x", x)
    _check_bf16_cuda("weight", weight)
    k = x.shape[-1]
    m = x.numel() // k
    n = weight.shape[0]
    if weight.shape[1] != k:
        raise ValueError(f"weight shape {tuple(weight.shape)} does not match in_features {k}")
    epi = 0
    if bias is not None:
        _check_bf16_cuda("bias", bias)
        epi |= PF_EPI_BIAS
    if gelu:
        epi |= PF_EPI_GELU
    if residual is not None:
        _check_bf16_cuda("residual", residual)
        epi |= PF_EPI_RESIDUAL
    if relu:
        epi |= PF_EPI_RELU
    if out is None:
        out = torch.empty(*x.shape[:-1], n, dtype=torch.bfloat16, device=x.device)
    native.call(
        "pf_gemm", x.data_ptr(), weight.data_ptr(), _ptr(bias), _ptr(residual), out.data_ptr(),
        m, n, k, epi, _ctl_ref(ctl), _stream(stream),
    )
    return out


def layernorm(
    x: torch.Tensor,
    gamma: torch.Tensor,
    beta: torch.Tensor,
    eps: float = 1e-12,
    *,
    residual: Optional[torch.Tensor] = None,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """out = LayerNorm(x [+ residual]) (pf_layernorm; fp32 tensors: pf_layernorm_f32)."""
    if x.dtype == torch.float32:
        cols = x.shape[-1]
        if out is None:
            out = torch.empty_like(x)
        native.call("pf_layernorm_f32", x.data_ptr(), _ptr(residual), gamma.data_ptr(), beta.data_ptr(),
                    out.data_ptr(), x.numel() // cols, cols, float(eps), _ctl_ref(ctl), _stream(stream))
        return out
    _check_bf16_cuda("x", x)
    cols = x.shape[-1]
    rows = x.numel() // cols
    if out is None:
        out = torch.empty_like(x)
    native.call(
        "pf_layernorm", x.data_ptr(), _ptr(residual), gamma.data_ptr(), beta.data_ptr(),
        out.data_ptr(), rows, cols, float(eps), _ctl_ref(ctl), _stream(stream),
    )
    return out


def rmsnorm(
    x: torch.Tensor,
    gamma: torch.Tensor,
    eps: float = 1e-6,
    *,
    residual: Optional[torch.Tensor] = None,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """out = RMSNorm(x [+ residual]) (pf_rmsnorm)."""
    _check_bf16_cuda("x", x)
    cols = x.shape[-1]
    rows = x.numel() // cols
    if out is None:
        out = torch.empty_like(x)
    native.call(
        "pf_rmsnorm", x.data_ptr(), _ptr(residual), gamma.data_ptr(), out.data_ptr(), rows, cols,
        float(eps), _ctl_ref(ctl), _stream(stream),
    )
    return out


def softmax(
    x: torch.Tensor,
    scale: float = 1.0,
    *,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """out = softmax(scale * x, dim=-1) (pf_softmax)."""
    _check_bf16_cuda("x", x)
    cols = x.shape[-1]
    rows = x.numel() // cols
    if out is None:
        out = torch.empty_like(x)
    native.call(
        "pf_softmax", x.data_ptr(), out.data_ptr(), rows, cols, float(scale), _ctl_ref(ctl),
        _stream(stream),
    )
    return out


def attention(
    qkv: torch.Tensor,
    heads: int,
    *,
    mask_add: Optional[torch.Tensor] = None,
    scale: Optional[float] = None,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """Multi-head attention over packed qkv [batch, seq, 3*hidden] -> [batch, seq, hidden]
    (pf_attention; fp32 tensors: pf_attention_f32, no mask)."""
    batch, seq, three_h = qkv.shape
    hidden = three_h // 3
    head_dim = hidden // heads
    if scale is None:
        scale = head_dim ** -0.5
    if qkv.dtype == torch.float32:
        if mask_add is not None:
            raise ValueError("the fp32 attention path takes no mask")
        if out is None:
            out = torch.empty(batch, seq, hidden, dtype=torch.float32, device=qkv.device)
        native.call("pf_attention_f32", qkv.data_ptr(), out.data_ptr(), batch, seq, heads, head_dim, float(scale),
                    _ctl_ref(ctl), _stream(stream))
        return out
    _check_bf16_cuda("qkv", qkv)
    if mask_add is not None:
        if mask_add.dtype != torch.float32 or mask_add.shape != (batch, seq):
            raise ValueError("mask_add must be fp32 [batch, seq]")
        mask_add = mask_add.contiguous()
    if out is None:
        out = torch.empty(batch, seq, hidden, dtype=torch.bfloat16, device=qkv.device)
    native.call(
        "pf_attention", qkv.data_ptr(), _ptr(mask_add), out.data_ptr(), batch, seq, heads,
        head_dim, float(scale), _ctl_ref(ctl), _stream(stream),
    )
    return out


def embedding_ln(
    ids: torch.Tensor,
    word: torch.Tensor,
    pos: torch.Tensor,
    type_emb: torch.Tensor,
    gamma: torch.Tensor,
    beta: torch.Tensor,
    eps: float = 1e-12,
    *,
    type_ids: Optional[torch.Tensor] = None,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """BERT embeddings + LayerNorm (pf_embedding_ln); ids int32 [batch, seq]."""
    if ids.dtype != torch.int32 or not ids.is_cuda:
        raise ValueError("ids must be int32 on CUDA")
    batch, seq = ids.shape
    hidden = word.shape[1]
    if word.dtype == torch.float32:
        if out is None:
            out = torch.empty(batch, seq, hidden, dtype=torch.float32, device=ids.device)
        native.call("pf_embedding_ln_f32", ids.data_ptr(), word.data_ptr(), pos.data_ptr(), type_emb.data_ptr(),
                    gamma.data_ptr(), beta.data_ptr(), out.data_ptr(), batch, seq, hidden, word.shape[0], float(eps),
                    _ctl_ref(ctl), _stream(stream))
        return out
    if out is None:
        out = torch.empty(batch, seq, hidden, dtype=torch.bfloat16, device=ids.device)
    native.call(
        "pf_embedding_ln", ids.data_ptr(), _ptr(type_ids), word.data_ptr(), pos.data_ptr(),
        type_emb.data_ptr(), gamma.data_ptr(), beta.data_ptr(), out.data_ptr(), batch, seq, hidden,
        word.shape[0], float(eps), _ctl_ref(ctl), _stream(stream),
    )
    return out


def conv_out(size: int, k: int, stride: int, pad: int) -> int:
    return (size + 2 * pad - k) // stride + 1


def image_units(kind: int, out_elems: int, channels: int) -> int:
    out = ctypes.c_uint32(0)
    native.call("pf_image_units", kind, out_elems, channels, ctypes.byref(out))
    return out.value


def im2col(
    x: torch.Tensor,
    kh: int,
    kw: int,
    stride: int,
    pad: int,
    kp: Optional[int] = None,
    *,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """NHWC x[B,H,W,C] -> col[B*Ho*Wo, Kp], column (ky*kw + kx)*C + c (pf_im2col)."""
    _check_bf16_cuda("x", x)
    b, h, w, c = x.shape
    k = kh * kw * c
    kp = kp or (k + 7) // 8 * 8
    ho, wo = conv_out(h, kh, stride, pad), conv_out(w, kw, stride, pad)
    if out is None:
        out = torch.empty(b * ho * wo, kp, dtype=torch.bfloat16, device=x.device)
    native.call("pf_im2col", x.data_ptr(), out.data_ptr(), b, h, w, c, kh, kw, stride, pad, kp,
                _ctl_ref(ctl), _stream(stream))
    return out


def maxpool(
    x: torch.Tensor,
    k: int = 3,
    stride: int = 2,
    pad: int = 1,
    *,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """NHWC max pooling (pf_maxpool)."""
    _check_bf16_cuda("x", x)
    b, h, w, c = x.shape
    ho, wo = conv_out(h, k, stride, pad), conv_out(w, k, stride, pad)
    if out is None:
        out = torch.empty(b, ho, wo, c, dtype=torch.bfloat16, device=x.device)
    native.call("pf_maxpool", x.data_ptr(), out.data_ptr(), b, h, w, c, k, stride, pad, _ctl_ref(ctl),
                _stream(stream))
    return out


def avgpool(
    x: torch.Tensor,
    *,
    out: Optional[torch.Tensor] = None,
    ctl: Optional[KernelCtl] = None,
    stream: Optional[torch.cuda.Stream] = None,
) -> torch.Tensor:
    """Global average pool NHWC x[B,H,W,C] -> [B, C] (pf_avgpool)."""
    _check_bf16_cuda("x", x)
    b, h, w, c = x.shape
    if out is None:
        out = torch.empty(b, c, dtype=torch.bfloat16, device=x.device)
    native.call("pf_avgpool", x.data_ptr(), out.data_ptr(), b, h * w, c, _ctl_ref(ctl), _stream(stream))
    return out


# ---------------------------------------------------------------------------- training


def gemm_splitk_splits(k: int, requested: int) -> int:
    out = ctypes.c_int(0)
    native.call("pf_gemm_splitk_splits", k, requested, ctypes.byref(out))
    return out.value


def gemm_splitk(x: torch.Tensor, weight: torch.Tensor, splits: int, *, out: Optional[torch.Tensor] = None,
                ctl: Optional[KernelCtl] = None, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """[S, M, N] partial products of x[M, K] @ weight[N, K].T over S K-slices (pf_gemm_splitk)."""
    _check_bf16_cuda("x", x)
    _check_bf16_cuda("weight", weight)
    m, k = x.shape
    n = weight.shape[0]
    s = gemm_splitk_splits(k, splits)
    if out is None:
        out = torch.empty(s, m, n, dtype=torch.bfloat16, device=x.device)
    native.call("pf_gemm_splitk", x.data_ptr(), weight.data_ptr(), out.data_ptr(), m, n, k, splits,
                _ctl_ref(ctl), _stream(stream))
    return out


def transpose(x: torch.Tensor, *, out=None, ctl=None, stream=None) -> torch.Tensor:
    r, c = x.shape
    if out is None:
        out = torch.empty(c, r, dtype=torch.bfloat16, device=x.device)
    native.call("pf_transpose", x.data_ptr(), out.data_ptr(), r, c, _ctl_ref(ctl), _stream(stream))
    return out


def colstats(x: torch.Tensor, partial: torch.Tensor, *, g=None, ymask=None, mean=None, invstd=None,
             ctl=None, stream=None) -> int:
    """Per-CTA column partials of x[M, C] into partial[P, 2C]; returns P (pf_colstats)."""
    m, c = x.shape
    p = ctypes.c_int(0)
    native.call("pf_colstats", x.data_ptr(), _ptr(g), _ptr(ymask), _ptr(mean), _ptr(invstd),
                partial.data_ptr(), m, c, ctypes.byref(p), _ctl_ref(ctl), _stream(stream))
    return p.value


def bn_finalize(partial, p, m, gamma, beta, eps, mean, invstd, scale, shift, *, ctl=None, stream=None):
    c = gamma.numel()
    native.call("pf_bn_finalize", partial.data_ptr(), p, m, c, gamma.data_ptr(), beta.data_ptr(), float(eps),
                mean.data_ptr(), invstd.data_ptr(), scale.data_ptr(), shift.data_ptr(), _ctl_ref(ctl),
                _stream(stream))


def bn_bwd_finalize(partial, p, c, dgamma, dbeta, *, ctl=None, stream=None):
    native.call("pf_bn_bwd_finalize", partial.data_ptr(), p, c, _ptr(dgamma), dbeta.data_ptr(),
                _ctl_ref(ctl), _stream(stream))


def bn_apply(x, scale, shift, out, *, residual=None, relu=False, ctl=None, stream=None):
    m, c = x.shape
    native.call("pf_bn_apply", x.data_ptr(), scale.data_ptr(), shift.data_ptr(), _ptr(residual),
                out.data_ptr(), m, c, int(relu), _ctl_ref(ctl), _stream(stream))
    return out


def bn_bwd_apply(x, g, mean, invstd, gamma, dgamma, dbeta, dx, *, ymask=None, da=None, ctl=None, stream=None):
    m, c = x.shape
    native.call("pf_bn_bwd_apply", x.data_ptr(), g.data_ptr(), _ptr(ymask), mean.data_ptr(),
                invstd.data_ptr(), gamma.data_ptr(), dgamma.data_ptr(), dbeta.data_ptr(), dx.data_ptr(),
                _ptr(da), m, c, _ctl_ref(ctl), _stream(stream))
    return dx


def col2im(dcol, b, h, w, c, kh, kw, stride, pad, *, residual=None, out=None, ctl=None, stream=None):
    kp = dcol.shape[-1]
    if out is None:
        out = torch.empty(b, h, w, c, dtype=torch.bfloat16, device=dcol.device)
    native.call("pf_col2im", dcol.data_ptr(), _ptr(residual), out.data_ptr(), b, h, w, c, kh, kw, stride, pad,
                kp, _ctl_ref(ctl), _stream(stream))
    return out


def maxpool_bwd(x, dy, k=3, stride=2, pad=1, *, out=None, ctl=None, stream=None):
    b, h, w, c = x.shape
    if out is None:
        out = torch.empty_like(x)
    native.call("pf_maxpool_bwd", x.data_ptr(), dy.data_ptr(), out.data_ptr(), b, h, w, c, k, stride, pad,
                _ctl_ref(ctl), _stream(stream))
    return out


def avgpool_bwd(dy, hw, *, out=None, ctl=None, stream=None):
    b, c = dy.shape
    if out is None:
        out = torch.empty(b, hw, c, dtype=torch.bfloat16, device=dy.device)
    native.call("pf_avgpool_bwd", dy.data_ptr(), out.data_ptr(), b, hw, c, _ctl_ref(ctl), _stream(stream))
    return out


def softmax_xent(z, labels4, loss4, dz, grad_scale, *, ctl=None, stream=None):
    b, n = z.shape
    native.call("pf_softmax_xent", z.data_ptr(), labels4.data_ptr(), loss4.data_ptr(), dz.data_ptr(), b, n,
                float(grad_scale), _ctl_ref(ctl), _stream(stream))


def sgd_segments(segs: list[dict]):
    arr = (native.SgdSegment * len(segs))()
    for i, s in enumerate(segs):
        arr[i].master = s["master"]
        arr[i].momentum = s["momentum"]
        arr[i].work = s.get("work")
        arr[i].grad = s["grad"]
        arr[i].n = s["n"]
        arr[i].split_stride = s.get("split_stride", 0)
        arr[i].splits = s.get("splits", 1)
        arr[i].grad_kind = s.get("grad_kind", 0)
        arr[i].weight_decay = s.get("weight_decay", 0.0)
    return arr


def sgd_update(segs: list[dict], lr: float, momentum: float, *, ctl=None, stream=None):
    arr = sgd_segments(segs)
    native.call("pf_sgd_update", arr, len(segs), float(lr), float(momentum), _ctl_ref(ctl), _stream(stream))


def _linear_f32(x, weight, bias=None, *, gelu=False, residual=None, out=None, ctl=None, stream=None):
    k = x.shape[-1]
    m = x.numel() // k
    n = weight.shape[0]
    epi = (PF_EPI_BIAS if bias is not None else 0) | (PF_EPI_GELU if gelu else 0) \
        | (PF_EPI_RESIDUAL if residual is not None else 0)
    if out is None:
        out = torch.empty(*x.shape[:-1], n, dtype=torch.float32, device=x.device)
    native.call("pf_gemm_f32", x.data_ptr(), weight.data_ptr(), _ptr(bias), _ptr(residual), out.data_ptr(),
                m, n, k, epi, _ctl_ref(ctl), _stream(stream))
    return out


def gemm_nn(x: torch.Tensor, wkn: torch.Tensor, *, residual=None, out=None, ctl=None, stream=None) -> torch.Tensor:
    """out[M, N] = x[M, K] @ wkn[K, N] (+ residual), wkn read MN-major (pf_gemm_nn)."""
    m, k = x.shape
    n = wkn.shape[1]
    if out is None:
        out = torch.empty(m, n, dtype=torch.bfloat16, device=x.device)
    native.call("pf_gemm_nn", x.data_ptr(), wkn.data_ptr(), _ptr(residual), out.data_ptr(), m, n, k,
                _ctl_ref(ctl), _stream(stream))
    return out


def gemm_splitk_tn(a: torch.Tensor, b: torch.Tensor, splits: int, *, out=None, ctl=None,
                   stream=None) -> torch.Tensor:
    """[S, M, N] split-K partials of a[K, M]^T @ b[K, N], both read MN-major (pf_gemm_splitk_tn)."""
    k, m = a.shape
    n = b.shape[1]
    s = gemm_splitk_splits(k, splits)
    if out is None:
        out = torch.empty(s, m, n, dtype=torch.bfloat16, device=a.device)
    native.call("pf_gemm_splitk_tn", a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, k, splits,
                _ctl_ref(ctl), _stream(stream))
    return out
