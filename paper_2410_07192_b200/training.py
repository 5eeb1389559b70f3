"""ResNet-50 training as a fill job (BASELINE configs[3]): forward with BatchNorm batch
statistics, softmax cross-entropy, backward, and an SGD-with-momentum step per batch, all
as preemptible sm_100a kernel nodes of one recorded chain per batch.

Reference counterpart: training jobs in the reference exist only as profiles
(``synth_profile(kind=TRAINING)``: x3 time, x4 weight memory, an optimizer node,
pkg/src/bubblefill/workload.py:216-271). Here the step really runs inside the bubbles:

* every convolution is a tcgen05 GEMM on NHWC activations (im2col for 3x3 / strided
  convs). Backward: data gradient = GEMM(dZ, W^T) (+ col2im, and the shortcut's
  gradient added in the GEMM epilogue); weight gradient = split-K GEMM(dZ^T, X^T)
  whose bf16 partial stack the optimizer sums in fp32;
* BatchNorm uses batch statistics (two-level column reductions, fp32), ReLU and the
  residual add fused into its apply kernel; its backward reuses the same reductions;
* parameters are fp32 masters + fp32 momentum + bf16 working copies (the GEMM
  operands), staged into the arena like inference weights and written back to the
  pinned host blob when a range completes;
* preemption: all nodes are idempotent atomic units or claimed-prefix GEMMs, except
  the SGD step, which claims 4096-element chunks so a resumed step never applies an
  update twice.

Semantics: a batch is one optimizer step (lr, momentum 0.9, weight decay on conv/fc
weights), loss = mean cross-entropy over the batch. BatchNorm running statistics
(used only for evaluation) are not tracked.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import torch

from . import kernels as K
from . import native
from .arena import PinnedBuffer, device_view
from .fillmodels import (ATOMIC, PREFIX, ExecContext, FillModule, FillSequential, ResNetConfig, RESNET50,
                         _numel, synthetic_images)

LR = 0.01  # ~ the linear-scaling rule (0.1 per 256 images) at fill batch sizes of 8-64
MOMENTUM = 0.9
WEIGHT_DECAY = 1e-4
BN_EPS = 1e-5
MAX_PARTIALS = 1024  # pf_colstats partial rows (4 per SM)


def _pad(n: int, a: int = 128) -> int:
    return (n + a - 1) // a * a


def wgrad_splits(n_out: int, k_out: int, k_red: int) -> int:
    """Split count of the weight-gradient GEMM [n_out, k_out] = dZ^T X over k_red rows:
    enough slices to give every SM ~2 tiles, each slice >= 4 K-blocks of 64."""
    tiles = math.ceil(n_out / 128) * math.ceil(k_out / 128)
    want = max(1, math.ceil(2 * 148 / tiles))
    want = min(want, 32, max(1, k_red // 256))
    return K.gemm_splitk_splits(k_red, want)


@dataclass(frozen=True)
class TParam:
    name: str
    shape: tuple[int, ...]
    init: tuple  # ("conv", fan_in, k) | ("one",) | ("zero",) | ("std", s)
    work: bool  # keeps a bf16 working copy (GEMM operand)
    wd: float
    grad: str  # "gemm": split-K bf16 partials; "f32": fp32 vector


class TrainModule(FillModule):
    """A module with fp32 master / momentum state, forward and backward recorders."""

    def __init__(self, idx: int):
        super().__init__()
        self.idx = idx
        self.saved: dict[str, torch.Tensor] = {}

    # ---- state layout: per param master fp32 | momentum fp32, then bf16 work copies
    def tparams(self) -> list[TParam]:
        raise NotImplementedError

    def _layout(self):
        off, out = 0, {}
        for p in self.tparams():
            n = _numel(p.shape)
            out[p.name] = off
            off += _pad(4 * n, 256)
            out[p.name + ".mom"] = off
            off += _pad(4 * n, 256)
        for p in self.tparams():
            if p.work:
                out[p.name + ".w"] = off
                off += _pad(2 * _numel(p.shape), 256)
        return out, off

    def weight_bytes(self) -> int:
        return self._layout()[1]

    def param_specs(self):  # bf16 GEMM operands (reference / eager views)
        return [(p.name, p.shape, p.init) for p in self.tparams() if p.work]

    def init_host(self, gen: torch.Generator, std: float = 0.02, pinned: bool = True,
                  raw: Optional[torch.Tensor] = None) -> None:
        """Random init of the state blob (`raw`: a slice of the whole step's blob)."""
        lay, total = self._layout()
        if raw is None:
            self.host = PinnedBuffer((total,), torch.uint8) if pinned else None
            raw = self.host.tensor if pinned else torch.zeros(total, dtype=torch.uint8)
        raw.zero_()
        self.host_params = {}
        for p in self.tparams():
            n = _numel(p.shape)
            kind = p.init
            if kind[0] == "conv":
                _, fan_in, k = kind
                vals = torch.zeros(p.shape)
                vals[:, :k] = torch.randn(p.shape[0], k, generator=gen) * (2.0 / fan_in) ** 0.5
                vals = vals.flatten()
            elif kind[0] == "one":
                vals = torch.ones(n)
            elif kind[0] == "zero":
                vals = torch.zeros(n)
            else:
                vals = torch.randn(n, generator=gen) * kind[1]
            m = raw[lay[p.name]:lay[p.name] + 4 * n].view(torch.float32)
            m.copy_(vals)
            self.host_params[p.name] = m.view(*p.shape)
            if p.work:
                raw[lay[p.name + ".w"]:lay[p.name + ".w"] + 2 * n].view(torch.bfloat16).copy_(vals.to(torch.bfloat16))
        self._raw_host = raw

    def make_views(self, ptr: int) -> dict[str, torch.Tensor]:
        lay, _ = self._layout()
        dev = {}
        for p in self.tparams():
            n = _numel(p.shape)
            dev[p.name] = device_view(ptr + lay[p.name], (n,), torch.float32).view(*p.shape)
            dev[p.name + ".mom"] = device_view(ptr + lay[p.name + ".mom"], (n,), torch.float32)
            if p.work:
                dev[p.name + ".w"] = device_view(ptr + lay[p.name + ".w"], (n,), torch.bfloat16).view(*p.shape)
        return dev

    def state_host(self) -> dict[str, torch.Tensor]:
        """fp32 masters of the pinned host blob (after a write-back)."""
        lay, _ = self._layout()
        return {p.name: self._raw_host[lay[p.name]:lay[p.name] + 4 * _numel(p.shape)].view(torch.float32)
                .view(*p.shape) for p in self.tparams()}

    # ---- gradients
    def grad_numel(self, p: TParam, batch: int) -> int:
        """bf16 elements of p's gradient buffer."""
        n = _numel(p.shape)
        if p.grad == "f32":
            return 2 * n
        # chains of any batch up to `batch` (multiples of 8) share this buffer
        return max(self.splits(p.name, b) for b in range(8, max(batch, 8) + 1, 8)) * n

    def splits(self, name: str, batch: int) -> int:
        """Split-K slice count of the weight gradient of parameter `name` at this batch."""
        raise NotImplementedError

    def grad_ws(self, batch: int) -> dict[str, int]:
        return {f"g{self.idx}.{p.name}": self.grad_numel(p, batch) for p in self.tparams()}

    def sgd_segments(self, ctx: ExecContext, batch: int) -> list[dict]:
        segs = []
        for p in self.tparams():
            n = _numel(p.shape)
            g = ctx.ws[f"g{self.idx}.{p.name}"]
            segs.append(dict(master=self.dev[p.name].data_ptr(), momentum=self.dev[p.name + ".mom"].data_ptr(),
                             work=self.dev[p.name + ".w"].data_ptr() if p.work else None, grad=g.data_ptr(),
                             n=n, split_stride=n, splits=self.splits(p.name, batch) if p.grad == "gemm" else 1,
                             grad_kind=0 if p.grad == "gemm" else 1, weight_decay=p.wd))
        return segs

    def node_units(self, batch):
        return []  # chains report their own units (pf_chain_node_info)


# ----------------------------------------------------------------------------- recorders


class _Rec:
    """Shorthand over an ExecContext in chain-record mode (training chains are recorded,
    never eager), counting GEMM FLOPs per node for the in-kernel timing."""

    def __init__(self, ctx: ExecContext, flops: dict, nbytes: dict | None = None):
        self.ctx, self.flops = ctx, flops
        self.nbytes = {} if nbytes is None else nbytes  # minimum DRAM bytes per GEMM node (roofline)

    def call(self, fn, *args):
        native.call(fn, self.ctx.chain, *args)
        self.ctx.node += 1

    def gemm(self, x, w, out, *, bias=None, residual=None, relu=False):
        k = x.shape[-1]
        m = x.numel() // k
        n = w.shape[0]
        self.flops[self.ctx.node] = 2.0 * m * n * k
        self.nbytes[self.ctx.node] = 2.0 * (m * k + n * k + m * n * (2 if residual is not None else 1))
        self.ctx.gemm(x.reshape(m, k), w, bias, out, residual=residual, relu=relu)

    def gemm_splitk(self, a, b, out, splits):
        m, k = a.shape
        n = b.shape[0]
        self.flops[self.ctx.node] = 2.0 * m * n * k
        self.nbytes[self.ctx.node] = 2.0 * (m * k + n * k + splits * m * n)
        self.call("pf_chain_add_gemm_splitk", a.data_ptr(), b.data_ptr(), out.data_ptr(), m, n, k, splits)

    def transpose(self, x, out):
        r, c = x.shape
        self.call("pf_chain_add_transpose", x.data_ptr(), out.data_ptr(), r, c)
        return out

    def bn_forward(self, z, gamma, beta, mean, invstd, out, *, residual=None, relu=True):
        """Batch statistics of z[M, C], then out = act(bn(z) [+ residual])."""
        ctx = self.ctx
        m, c = z.shape
        partial = ctx.fbuf("partial", MAX_PARTIALS * 2 * c)
        p = native.ctypes.c_int(0)
        self.call("pf_chain_add_colstats", z.data_ptr(), None, None, None, None, partial.data_ptr(), m, c,
                  native.ctypes.byref(p))
        scale, shift = ctx.fbuf("scale", c), ctx.fbuf("shift", c)
        self.call("pf_chain_add_bn_finalize", partial.data_ptr(), p.value, m, c, gamma.data_ptr(),
                  beta.data_ptr(), BN_EPS, mean.data_ptr(), invstd.data_ptr(), scale.data_ptr(), shift.data_ptr())
        self.call("pf_chain_add_bn_apply", z.data_ptr(), scale.data_ptr(), shift.data_ptr(),
                  None if residual is None else residual.data_ptr(), out.data_ptr(), m, c, int(relu))

    def bn_backward(self, z, dout, ymask, mean, invstd, gamma, dgamma, dbeta, dz, da=None):
        ctx = self.ctx
        m, c = z.shape
        partial = ctx.fbuf("partial", MAX_PARTIALS * 2 * c)
        p = native.ctypes.c_int(0)
        self.call("pf_chain_add_colstats", z.data_ptr(), dout.data_ptr(),
                  None if ymask is None else ymask.data_ptr(), mean.data_ptr(), invstd.data_ptr(),
                  partial.data_ptr(), m, c, native.ctypes.byref(p))
        self.call("pf_chain_add_bn_bwd_finalize", partial.data_ptr(), p.value, c, dgamma.data_ptr(),
                  dbeta.data_ptr())
        self.call("pf_chain_add_bn_bwd_apply", z.data_ptr(), dout.data_ptr(),
                  None if ymask is None else ymask.data_ptr(), mean.data_ptr(), invstd.data_ptr(), gamma.data_ptr(),
                  dgamma.data_ptr(), dbeta.data_ptr(), dz.data_ptr(), None if da is None else da.data_ptr(), m, c)

    def im2col(self, x, k, stride, pad, kp, out):
        b, h, w, c = x.shape
        self.call("pf_chain_add_im2col", x.data_ptr(), out.data_ptr(), b, h, w, c, k, k, stride, pad, kp)

    def col2im(self, dcol, b, h, w, c, k, stride, pad, out, residual=None):
        self.call("pf_chain_add_col2im", dcol.data_ptr(), None if residual is None else residual.data_ptr(),
                  out.data_ptr(), b, h, w, c, k, k, stride, pad, dcol.shape[-1])

    def wgrad(self, dz, x, gbuf, splits):
        """gbuf[S, N, K] = split-K partials of dz[M, N]^T x[M, K], both operands read
        MN-major straight from the activations (no transposes)."""
        m, n = dz.shape
        k = x.shape[-1]
        self.flops[self.ctx.node] = 2.0 * m * n * k
        self.nbytes[self.ctx.node] = 2.0 * (m * n + m * k + splits * n * k)
        self.call("pf_chain_add_gemm_splitk_tn", dz.data_ptr(), x.data_ptr(), gbuf.data_ptr(), n, k, m, splits)

    def dgrad(self, dz, w, out, residual=None):
        """out[M, K] = dz[M, N] w[N, K] (+ residual), w read MN-major as stored."""
        n, k = w.shape
        m = dz.shape[0]
        self.flops[self.ctx.node] = 2.0 * m * n * k
        self.nbytes[self.ctx.node] = 2.0 * (m * n + n * k + m * k * (2 if residual is not None else 1))
        self.call("pf_chain_add_gemm_nn", dz.data_ptr(), w.data_ptr(),
                  None if residual is None else residual.data_ptr(), out.data_ptr(), m, k, n)


class TrainStem(TrainModule):
    """conv 7x7/2 + BN + ReLU + maxpool 3x3/2."""

    def __init__(self, cfg: ResNetConfig):
        super().__init__(0)
        self.cfg = cfg
        self.h1 = K.conv_out(cfg.image, 7, 2, 3)
        self.h2 = K.conv_out(self.h1, 3, 2, 1)

    def tparams(self):
        c = self.cfg
        return [TParam("w", (c.stem_ch, c.stem_kp), ("conv", c.stem_k, c.stem_k), True, WEIGHT_DECAY, "gemm"),
                TParam("g", (c.stem_ch,), ("one",), False, 0.0, "f32"),
                TParam("b", (c.stem_ch,), ("zero",), False, 0.0, "f32")]

    def out_shape(self):
        return (self.h2, self.h2, self.cfg.stem_ch)

    def splits(self, name, batch):
        return wgrad_splits(self.cfg.stem_ch, self.cfg.stem_kp, batch * self.h1 * self.h1)

    def workspace(self, batch):
        c, m1 = self.cfg, batch * self.h1 * self.h1
        i = self.idx
        ws = {f"s{i}.col": m1 * c.stem_kp, f"s{i}.z": m1 * c.stem_ch, f"s{i}.a": m1 * c.stem_ch,
              f"s{i}.stats": 4 * c.stem_ch, f"out{i}": batch * self.h2 * self.h2 * c.stem_ch,
              f"s{i}.argmax": (batch * self.h2 * self.h2 * c.stem_ch + 1) // 2,  # uint8 in bf16 units
              "da": m1 * c.stem_ch, "dz": m1 * c.stem_ch}
        ws.update(self.grad_ws(batch))
        return ws

    def flops_per_sample(self):
        return 3 * 2.0 * self.h1 * self.h1 * self.cfg.stem_ch * self.cfg.stem_k

    def forward(self, x, ctx):
        raise RuntimeError("training modules are recorded through ResNetTrainSequential.record_step")

    def record_forward(self, r: _Rec, x):
        c, ctx, i = self.cfg, r.ctx, self.idx
        b = x.shape[0]
        m1 = b * self.h1 * self.h1
        col = ctx.buf(f"s{i}.col", m1 * c.stem_kp).view(m1, c.stem_kp)
        z = ctx.buf(f"s{i}.z", m1 * c.stem_ch).view(m1, c.stem_ch)
        a = ctx.buf(f"s{i}.a", m1 * c.stem_ch).view(b, self.h1, self.h1, c.stem_ch)
        st = ctx.fbuf(f"s{i}.stats", 2 * c.stem_ch)
        out = ctx.buf(f"out{i}", b * self.h2 * self.h2 * c.stem_ch).view(b, self.h2, self.h2, c.stem_ch)
        d = self.dev
        r.im2col(x, 7, 2, 3, c.stem_kp, col)
        r.gemm(col, d["w.w"], z)
        r.bn_forward(z, d["g"], d["b"], st[:c.stem_ch], st[c.stem_ch:], a.view(m1, c.stem_ch), relu=True)
        idx = ctx.buf(f"s{i}.argmax", (b * self.h2 * self.h2 * c.stem_ch + 1) // 2)
        r.call("pf_chain_add_maxpool_argmax", a.data_ptr(), out.data_ptr(), idx.data_ptr(), b, self.h1, self.h1,
               c.stem_ch, 3, 2, 1)
        self.saved = dict(col=col, z=z, a=a, st=st, b=b, idx=idx)
        return out

    def record_backward(self, r: _Rec, dout):
        c, ctx, i, s = self.cfg, r.ctx, self.idx, self.saved
        b = s["b"]
        m1 = b * self.h1 * self.h1
        da = ctx.buf("da", m1 * c.stem_ch).view(b, self.h1, self.h1, c.stem_ch)
        r.call("pf_chain_add_maxpool_bwd_argmax", s["idx"].data_ptr(), dout.data_ptr(), da.data_ptr(), b, self.h1,
               self.h1, c.stem_ch, 3, 2, 1)
        dz = ctx.buf("dz", m1 * c.stem_ch).view(m1, c.stem_ch)
        g = {p.name: ctx.ws[f"g{i}.{p.name}"] for p in self.tparams()}
        gf = lambda nm: g[nm].view(-1)[:2 * c.stem_ch].view(torch.float32)  # noqa: E731
        r.bn_backward(s["z"], da.view(m1, c.stem_ch), s["a"].view(m1, c.stem_ch), s["st"][:c.stem_ch],
                      s["st"][c.stem_ch:], self.dev["g"], gf("g"), gf("b"), dz)
        r.wgrad(dz, s["col"], g["w"], self.splits("w", b))
        return None  # no gradient for the input images


class TrainBottleneck(TrainModule):
    """1x1 -> 3x3 (stride) -> 1x1 (x4) with BN after every conv, projection shortcut
    (conv + BN) when the shape changes, residual add + ReLU fused in the last BN apply."""

    def __init__(self, cfg: ResNetConfig, idx: int, in_ch: int, width: int, stride: int, h_in: int):
        super().__init__(idx)
        self.cfg, self.in_ch, self.width, self.stride, self.h = cfg, in_ch, width, stride, h_in
        self.out_ch = width * cfg.expansion
        self.ho = K.conv_out(h_in, 3, stride, 1)
        self.ds = stride != 1 or in_ch != self.out_ch

    def tparams(self):
        ci, w, co = self.in_ch, self.width, self.out_ch
        ps = [TParam("w1", (w, ci), ("conv", ci, ci), True, WEIGHT_DECAY, "gemm"),
              TParam("g1", (w,), ("one",), False, 0.0, "f32"), TParam("b1", (w,), ("zero",), False, 0.0, "f32"),
              TParam("w2", (w, 9 * w), ("conv", 9 * w, 9 * w), True, WEIGHT_DECAY, "gemm"),
              TParam("g2", (w,), ("one",), False, 0.0, "f32"), TParam("b2", (w,), ("zero",), False, 0.0, "f32"),
              TParam("w3", (co, w), ("conv", w, w), True, WEIGHT_DECAY, "gemm"),
              TParam("g3", (co,), ("one",), False, 0.0, "f32"), TParam("b3", (co,), ("zero",), False, 0.0, "f32")]
        if self.ds:
            ps += [TParam("wd", (co, ci), ("conv", ci, ci), True, WEIGHT_DECAY, "gemm"),
                   TParam("gd", (co,), ("one",), False, 0.0, "f32"),
                   TParam("bd", (co,), ("zero",), False, 0.0, "f32")]
        return ps

    def out_shape(self):
        return (self.ho, self.ho, self.out_ch)

    def splits(self, name, batch):
        m, mo = batch * self.h * self.h, batch * self.ho * self.ho
        ci, w, co = self.in_ch, self.width, self.out_ch
        return {"w1": lambda: wgrad_splits(w, ci, m), "w2": lambda: wgrad_splits(w, 9 * w, mo),
                "w3": lambda: wgrad_splits(co, w, mo), "wd": lambda: wgrad_splits(co, ci, mo)}[name]()

    def workspace(self, batch):
        i = self.idx
        m, mo = batch * self.h * self.h, batch * self.ho * self.ho
        ci, w, co = self.in_ch, self.width, self.out_ch
        ws = {f"s{i}.z1": m * w, f"s{i}.a1": m * w, f"s{i}.z2": mo * w, f"s{i}.a2": mo * w,
              f"s{i}.z3": mo * co, f"s{i}.stats": 4 * (2 * w + 2 * co), f"out{i}": mo * co,
              "col": mo * 9 * w, "dz_a": mo * co, "dres": mo * co, "dt2": mo * w, "dz_b": mo * w,
              "dcol": mo * 9 * w, "dt1": m * w, "dz_c": m * w}
        if self.ds:
            ws.update({f"s{i}.zd": mo * co, f"s{i}.statsd": 4 * co, "sc": mo * co, "dz_d": mo * co,
                       "dsrc": mo * ci, "dxsc": m * ci})
            if self.stride != 1:
                ws["colds"] = mo * ci
        ws.update(self.grad_ws(batch))
        return ws

    def flops_per_sample(self):
        hw, ow, ci, w, co = self.h * self.h, self.ho * self.ho, self.in_ch, self.width, self.out_ch
        f = 2.0 * (hw * ci * w + ow * 9 * w * w + ow * w * co) + (2.0 * ow * ci * co if self.ds else 0.0)
        return 3 * f

    def forward(self, x, ctx):
        raise RuntimeError("training modules are recorded through ResNetTrainSequential.record_step")

    def record_forward(self, r: _Rec, x):
        ctx, i, d = r.ctx, self.idx, self.dev
        b = x.shape[0]
        m, mo = b * self.h * self.h, b * self.ho * self.ho
        ci, w, co = self.in_ch, self.width, self.out_ch
        st = ctx.fbuf(f"s{i}.stats", 2 * (2 * w + 2 * co))
        mv = {"1": (st[0:w], st[w:2 * w]), "2": (st[2 * w:3 * w], st[3 * w:4 * w]),
              "3": (st[4 * w:4 * w + co], st[4 * w + co:4 * w + 2 * co])}
        z1 = ctx.buf(f"s{i}.z1", m * w).view(m, w)
        a1 = ctx.buf(f"s{i}.a1", m * w).view(b, self.h, self.h, w)
        z2 = ctx.buf(f"s{i}.z2", mo * w).view(mo, w)
        a2 = ctx.buf(f"s{i}.a2", mo * w).view(mo, w)
        z3 = ctx.buf(f"s{i}.z3", mo * co).view(mo, co)
        out = ctx.buf(f"out{i}", mo * co).view(b, self.ho, self.ho, co)
        col = ctx.buf("col", mo * 9 * w).view(mo, 9 * w)
        x2 = x.reshape(m, ci)
        r.gemm(x2, d["w1.w"], z1)
        r.bn_forward(z1, d["g1"], d["b1"], *mv["1"], a1.view(m, w), relu=True)
        r.im2col(a1, 3, self.stride, 1, 9 * w, col)
        r.gemm(col, d["w2.w"], z2)
        r.bn_forward(z2, d["g2"], d["b2"], *mv["2"], a2, relu=True)
        r.gemm(a2, d["w3.w"], z3)
        saved = dict(x=x, z1=z1, a1=a1, z2=z2, a2=a2, z3=z3, out=out, mv=mv, b=b)
        if self.ds:
            # the shortcut's statistics live in the fp32 block after the main branch's
            zd = ctx.buf(f"s{i}.zd", mo * co).view(mo, co)
            std = ctx.fbuf(f"s{i}.statsd", 2 * co)
            src = x2
            if self.stride != 1:
                src = ctx.buf("colds", mo * ci).view(mo, ci)
                r.im2col(x, 1, self.stride, 0, ci, src)
            r.gemm(src, d["wd.w"], zd)
            sc = ctx.buf("sc", mo * co).view(mo, co)
            r.bn_forward(zd, d["gd"], d["bd"], std[:co], std[co:], sc, relu=False)
            saved.update(zd=zd, mvd=(std[:co], std[co:]))
        else:
            sc = x2
        r.bn_forward(z3, d["g3"], d["b3"], *mv["3"], out.view(mo, co), residual=sc, relu=True)
        self.saved = saved
        return out

    def record_backward(self, r: _Rec, dout):
        ctx, i, d, s = r.ctx, self.idx, self.dev, self.saved
        b = s["b"]
        m, mo = b * self.h * self.h, b * self.ho * self.ho
        ci, w, co = self.in_ch, self.width, self.out_ch
        g = {p.name: ctx.ws[f"g{i}.{p.name}"] for p in self.tparams()}

        def gf(nm, n):
            return g[nm].view(-1)[:2 * n].view(torch.float32)

        # out = relu(bn3(z3) + shortcut)
        dz3 = ctx.buf("dz_a", mo * co).view(mo, co)
        dres = ctx.buf("dres", mo * co).view(mo, co)
        r.bn_backward(s["z3"], dout.reshape(mo, co), s["out"].view(mo, co), *s["mv"]["3"], d["g3"],
                      gf("g3", co), gf("b3", co), dz3, da=dres)
        da2 = ctx.buf("dt2", mo * w).view(mo, w)
        r.dgrad(dz3, d["w3.w"], da2)
        r.wgrad(dz3, s["a2"], g["w3"], self.splits("w3", b))
        dz2 = ctx.buf("dz_b", mo * w).view(mo, w)
        r.bn_backward(s["z2"], da2, s["a2"], *s["mv"]["2"], d["g2"], gf("g2", w), gf("b2", w), dz2)
        dcol = ctx.buf("dcol", mo * 9 * w).view(mo, 9 * w)
        r.dgrad(dz2, d["w2.w"], dcol)
        col = ctx.buf("col", mo * 9 * w).view(mo, 9 * w)
        r.im2col(s["a1"], 3, self.stride, 1, 9 * w, col)  # recomputed, not kept
        r.wgrad(dz2, col, g["w2"], self.splits("w2", b))
        da1 = ctx.buf("dt1", m * w).view(b, self.h, self.h, w)
        r.col2im(dcol, b, self.h, self.h, w, 3, self.stride, 1, da1)
        dz1 = ctx.buf("dz_c", m * w).view(m, w)
        r.bn_backward(s["z1"], da1.view(m, w), s["a1"].view(m, w), *s["mv"]["1"], d["g1"], gf("g1", w),
                      gf("b1", w), dz1)
        x2 = s["x"].reshape(m, ci)
        if self.ds:
            dzd = ctx.buf("dz_d", mo * co).view(mo, co)
            r.bn_backward(s["zd"], dres, None, *s["mvd"], d["gd"], gf("gd", co), gf("bd", co), dzd)
            dsrc = ctx.buf("dsrc", mo * ci).view(mo, ci)
            r.dgrad(dzd, d["wd.w"], dsrc)
            if self.stride != 1:
                src = ctx.buf("colds", mo * ci).view(mo, ci)
                r.im2col(s["x"], 1, self.stride, 0, ci, src)
                dxsc = ctx.buf("dxsc", m * ci).view(b, self.h, self.h, ci)
                r.col2im(dsrc, b, self.h, self.h, ci, 1, self.stride, 0, dxsc)
                dxsc = dxsc.view(m, ci)
            else:
                src, dxsc = x2, dsrc
            r.wgrad(dzd, src, g["wd"], self.splits("wd", b))
        else:
            dxsc = dres
        dx = ctx.buf(f"grad{i % 2}", m * ci).view(b, self.h, self.h, ci)
        r.dgrad(dz1, d["w1.w"], dx.view(m, ci), residual=dxsc)
        r.wgrad(dz1, x2, g["w1"], self.splits("w1", b))
        return dx


class TrainHead(TrainModule):
    """Global average pool + fc, softmax cross-entropy (mean over the batch)."""

    def __init__(self, cfg: ResNetConfig, idx: int, in_ch: int, h_in: int):
        super().__init__(idx)
        self.cfg, self.in_ch, self.h = cfg, in_ch, h_in

    def tparams(self):
        n, c = self.cfg.classes, self.in_ch
        return [TParam("fc_w", (n, c), ("std", c ** -0.5), True, WEIGHT_DECAY, "gemm"),
                TParam("fc_b", (n,), ("zero",), True, 0.0, "f32")]

    def out_shape(self):
        return (4,)

    def splits(self, name, batch):
        return K.gemm_splitk_splits(batch, 1)

    def workspace(self, batch):
        i, n, c = self.idx, self.cfg.classes, self.in_ch
        ws = {f"s{i}.pooled": batch * c, f"s{i}.logits": batch * n, "dlogits": batch * n, "dpooled": batch * c,
              "partial": 2 * MAX_PARTIALS * 2 * n, "loss": 2 * 4 * batch}
        ws.update(self.grad_ws(batch))
        return ws

    def flops_per_sample(self):
        return 3 * 2.0 * self.in_ch * self.cfg.classes

    def forward(self, x, ctx):
        raise RuntimeError("training modules are recorded through ResNetTrainSequential.record_step")

    def record_forward(self, r: _Rec, x, labels, loss):
        ctx, i, d = r.ctx, self.idx, self.dev
        b = x.shape[0]
        n, c = self.cfg.classes, self.in_ch
        pooled = ctx.buf(f"s{i}.pooled", b * c).view(b, c)
        logits = ctx.buf(f"s{i}.logits", b * n).view(b, n)
        r.call("pf_chain_add_avgpool", x.data_ptr(), pooled.data_ptr(), b, self.h * self.h, c)
        r.gemm(pooled, d["fc_w.w"], logits, bias=d["fc_b.w"])
        dlogits = ctx.buf("dlogits", b * n).view(b, n)
        r.call("pf_chain_add_softmax_xent", logits.data_ptr(), labels.data_ptr(), loss.data_ptr(),
               dlogits.data_ptr(), b, n, 1.0 / b)
        self.saved = dict(pooled=pooled, dlogits=dlogits, b=b)

    def record_backward(self, r: _Rec, _unused=None):
        ctx, i, d, s = r.ctx, self.idx, self.dev, self.saved
        b, n, c = s["b"], self.cfg.classes, self.in_ch
        g = {p.name: ctx.ws[f"g{i}.{p.name}"] for p in self.tparams()}
        dpooled = ctx.buf("dpooled", b * c).view(b, c)
        r.dgrad(s["dlogits"], d["fc_w.w"], dpooled)
        r.wgrad(s["dlogits"], s["pooled"], g["fc_w"], self.splits("fc_w", b))
        # bias gradient = column sums of dlogits
        partial = ctx.fbuf("partial", MAX_PARTIALS * 2 * n)
        p = native.ctypes.c_int(0)
        r.call("pf_chain_add_colstats", s["dlogits"].data_ptr(), None, None, None, None, partial.data_ptr(), b, n,
               native.ctypes.byref(p))
        r.call("pf_chain_add_bn_bwd_finalize", partial.data_ptr(), p.value, n, None,
               g["fc_b"].view(-1)[:2 * n].view(torch.float32).data_ptr())
        dx = ctx.buf(f"grad{i % 2}", b * self.h * self.h * c).view(b, self.h, self.h, c)
        r.call("pf_chain_add_avgpool_bwd", dpooled.data_ptr(), dx.data_ptr(), b, self.h * self.h, c)
        return dx


class ResNetTrainStep(FillModule):
    """The whole training step as ONE node of the linearized model. A training step needs
    every module's saved activations for its backward, so it cannot be split into
    partitions that run in different bubbles; presenting it as a single profile layer
    makes every plan the DP produces for it single-partition (partition.py:247-297).
    The 18 modules' states are slices of one pinned blob: one staging copy, one
    write-back."""

    def __init__(self, mods: list["TrainModule"]):
        super().__init__()
        self.mods = torch.nn.ModuleList(mods)

    def _offsets(self):
        offs, off = [], 0
        for m in self.mods:
            offs.append(off)
            off += _pad(m.weight_bytes(), 256)
        return offs, off

    def weight_bytes(self) -> int:
        return self._offsets()[1]

    def param_specs(self):
        return []

    def init_host(self, gen: torch.Generator, std: float = 0.02, pinned: bool = True,
                  raw: Optional[torch.Tensor] = None) -> None:
        offs, total = self._offsets()
        self.host = PinnedBuffer((total,), torch.uint8) if pinned else None
        blob = self.host.tensor if pinned else torch.zeros(total, dtype=torch.uint8)
        for m, o in zip(self.mods, offs):
            m.init_host(gen, pinned=pinned, raw=blob[o:o + m.weight_bytes()])
        self.host_params = {}

    def make_views(self, ptr: int) -> dict:
        offs, _ = self._offsets()
        return {"mods": [m.make_views(ptr + o) for m, o in zip(self.mods, offs)]}

    @property
    def dev(self):
        return {"mods": [m.dev for m in self.mods]} if hasattr(self, "mods") else {}

    @dev.setter
    def dev(self, value):
        if value and hasattr(self, "mods"):
            for m, d in zip(self.mods, value["mods"]):
                m.dev = d

    def workspace(self, batch: int) -> dict[str, int]:
        need: dict[str, int] = {}
        for m in self.mods:
            for k, v in m.workspace(batch).items():
                need[k] = max(need.get(k, 0), v)
        for j in (0, 1):  # gradient ping-pong between modules
            need[f"grad{j}"] = max(batch * _numel(m.out_shape()) for m in list(self.mods)[:-1])
        need["partial"] = max(need.get("partial", 0), 2 * MAX_PARTIALS * 2 * 2048)
        need["scale"] = need["shift"] = 2 * 2048
        return need

    def flops_per_sample(self) -> float:
        return sum(m.flops_per_sample() for m in self.mods)

    def node_units(self, batch):
        return []

    def forward(self, x, ctx):
        raise RuntimeError("a training step is recorded through ResNetTrainSequential.record_step")


class ResNetTrainSequential(FillSequential):
    """ResNet-50 training job: one node (the step) wrapping [stem, 16 bottlenecks, head];
    one batch = one SGD step."""

    is_training = True
    capture_grads = False  # tests: keep a copy of the gradient entering every module's backward

    @property
    def blocks(self) -> list["TrainModule"]:
        """The 18 modules of the step: stem, bottlenecks, head."""
        return list(self[0].mods)

    def input_spec(self):
        c = self.cfg
        return torch.bfloat16, (c.image, c.image, c.in_ch)

    def boundary_shape(self, i):
        return self.input_spec()[1] if i == 0 else (4,)

    def result_shape(self):
        return (4,)  # per-sample loss at [0] (16-B rows)

    def result_dtype(self):
        return torch.float32

    def result_view(self, x, cnt):
        raise RuntimeError("training results are written by the step chain")

    def aux_spec(self):
        return torch.int32, (4,)  # label at [0]

    def make_inputs(self, job_seed, first, count):
        return synthetic_images(job_seed, first, count, self.cfg.image, self.cfg.in_ch)

    def make_aux(self, job_seed, first, count):
        return synthetic_labels(job_seed, first, count, self.cfg.classes)

    def workspace(self, lo: int, hi: int, batch: int) -> dict[str, int]:
        need = dict(self[0].workspace(batch))
        if self.capture_grads:
            for m in self.blocks[:-1]:
                need[f"cap{m.idx}"] = batch * _numel(m.out_shape())
        return need

    def record_step(self, x, labels, loss, ctx: ExecContext) -> tuple[list[int], dict]:
        """Record forward, loss, backward and the SGD step; returns (segment ends, GEMM FLOPs
        per node)."""
        flops: dict[int, float] = {}
        self.last_gemm_bytes: dict[int, float] = {}
        r = _Rec(ctx, flops, self.last_gemm_bytes)
        b = x.shape[0]
        if b % 8:
            raise ValueError("training batches must be a multiple of 8 samples")
        mods = self.blocks
        ends = []
        y = x
        for mod in mods[:-1]:
            y = mod.record_forward(r, y)
            ends.append(ctx.node)
        mods[-1].record_forward(r, y, labels, loss)
        ends.append(ctx.node)
        dy = mods[-1].record_backward(r)
        ends.append(ctx.node)
        for mod in reversed(mods[:-1]):
            if self.capture_grads:
                nb = dy.numel() * 2
                cap = ctx.buf(f"cap{mod.idx}", dy.numel())
                r.call("pf_chain_add_copy", cap.data_ptr(), nb, dy.data_ptr(), nb, nb, 1, 0)
            dy = mod.record_backward(r, dy)
            ends.append(ctx.node)
        segs = []
        for mod in mods:
            segs.extend(mod.sgd_segments(ctx, b))
        arr = K.sgd_segments(segs)
        native.call("pf_chain_add_sgd", ctx.chain, arr, len(segs), LR, MOMENTUM)
        ctx.node += 1
        ends.append(ctx.node)
        return ends, flops


class ResNetTrainPartitioned(FillSequential):
    """ResNet-50 training with its 18 modules as separate nodes, so a plan may split them
    into partitions that run in different bubbles (BASELINE.json configs[3]: "fwd+bwd
    partitioned across bubbles"; the reference profiles training as L layers plus an
    optimizer pseudo-layer, workload.py:256-264). One batch is still one SGD step. The
    executor runs it batch-major as 2k - 1 phases over the k partitions (record_phase):

    * ``F`` p < k-1: forward of partition p from its input boundary, output boundary stored;
    * ``L`` p = k-1: forward, loss, backward and SGD of the last partition;
    * ``B`` p < k-1: the partition's forward recomputed from its stored input (activation
      checkpointing at partition boundaries), backward with the stored gradient of its
      output, SGD of its modules, gradient of its input stored for partition p - 1.

    Every kernel is the one the single-node step (ResNetTrainSequential) records, on the same
    inputs, so a multi-partition plan trains bit-identically to a single-partition one
    (tests/test_train_gpu.py). Module state lives in one pinned blob per module and is
    written back when its partition leaves the device."""

    is_training = True
    partitioned = True

    @property
    def blocks(self) -> list["TrainModule"]:
        return list(self)

    def input_spec(self):
        c = self.cfg
        return torch.bfloat16, (c.image, c.image, c.in_ch)

    def boundary_shape(self, i):
        return self.input_spec()[1] if i == 0 else tuple(self[i - 1].out_shape())

    def result_shape(self):
        return (4,)

    def result_dtype(self):
        return torch.float32

    def result_view(self, x, cnt):
        raise RuntimeError("training results are written by the loss phase")

    def aux_spec(self):
        return torch.int32, (4,)

    def make_inputs(self, job_seed, first, count):
        return synthetic_images(job_seed, first, count, self.cfg.image, self.cfg.in_ch)

    def make_aux(self, job_seed, first, count):
        return synthetic_labels(job_seed, first, count, self.cfg.classes)

    def workspace(self, lo: int, hi: int, batch: int) -> dict[str, int]:
        """Partition [lo, hi)'s workspace: its modules' buffers, the gradient ping-pong between
        them, BatchNorm partials / scale / shift."""
        need: dict[str, int] = {}
        for i in range(lo, hi):
            for k, v in self[i].workspace(batch).items():
                need[k] = max(need.get(k, 0), v)
        ins = [batch * _numel(self.boundary_shape(i)) for i in range(max(lo, 1), hi)]
        for j in (0, 1):
            need[f"grad{j}"] = max(ins + [8])
        need["partial"] = max(need.get("partial", 0), 2 * MAX_PARTIALS * 2 * 2048)
        need["scale"] = need["shift"] = 2 * 2048
        need["loss"] = max(need.get("loss", 0), 2 * 4 * batch)
        return need

    def record_phase(self, kind: str, lo: int, hi: int, x, dout, labels, loss,
                     ctx: ExecContext) -> tuple[list[int], dict, dict, Optional[torch.Tensor]]:
        """Record one phase of partition [lo, hi) (see the class docstring). Returns (segment
        ends, GEMM FLOPs per node, GEMM bytes per node, the tensor holding the partition's
        output (F) or input gradient (L / B, None for the stem))."""
        flops: dict[int, float] = {}
        nbytes: dict[int, float] = {}
        r = _Rec(ctx, flops, nbytes)
        b = x.shape[0]
        if b % 8:
            raise ValueError("training batches must be a multiple of 8 samples")
        mods = [self[i] for i in range(lo, hi)]
        has_head = hi == len(self)
        if (kind == "L") != has_head:
            raise ValueError("the loss phase is the last partition's, and only its")
        ends = []
        y = x
        for mod in mods[:-1] if has_head else mods:
            y = mod.record_forward(r, y)
            ends.append(ctx.node)
        if kind == "F":
            return ends, flops, nbytes, y
        if has_head:
            mods[-1].record_forward(r, y, labels, loss)
            ends.append(ctx.node)
            dy = mods[-1].record_backward(r)
            ends.append(ctx.node)
            rest = mods[:-1]
        else:
            dy = dout
            rest = mods
        for mod in reversed(rest):
            dy = mod.record_backward(r, dy)
            ends.append(ctx.node)
        segs = []
        for mod in mods:
            segs.extend(mod.sgd_segments(ctx, b))
        native.call("pf_chain_add_sgd", ctx.chain, K.sgd_segments(segs), len(segs), LR, MOMENTUM)
        ctx.node += 1
        ends.append(ctx.node)
        return ends, flops, nbytes, dy


def synthetic_labels(job_seed: int, first: int, count: int, classes: int) -> torch.Tensor:
    """int32 [count, 4], label of sample i at [i, 0] (depends only on (job_seed, i))."""
    i = torch.arange(first, first + count, dtype=torch.int64)
    lab = ((i * 2_654_435_761 + job_seed * 40_503 + 12_345) % 2_147_483_647) % classes
    out = torch.zeros(count, 4, dtype=torch.int32)
    out[:, 0] = lab.to(torch.int32)
    return out


def resnet50_train(cfg: ResNetConfig = RESNET50, seed: Optional[int] = 0, pinned: bool = True,
                   partitioned: bool = False):
    """ResNet-50 training job as the linearized fill model [stem, 16 bottlenecks, head]:
    one node wrapping the whole step (ResNetTrainSequential), or with `partitioned` the 18
    modules as nodes a plan may split across bubbles (ResNetTrainPartitioned). Both draw
    the same initial state from `seed`."""
    from .fillmodels import Bottleneck as _InferBlock  # shapes of the inference twin

    mods: list[FillModule] = [TrainStem(cfg)]
    ch, h = cfg.stem_ch, mods[0].out_shape()[0]
    for stage, (n, w) in enumerate(zip(cfg.blocks, cfg.widths)):
        for j in range(n):
            stride = 2 if (j == 0 and stage > 0) else 1
            blk = TrainBottleneck(cfg, len(mods), ch, w, stride, h)
            mods.append(blk)
            ch, h = blk.out_ch, blk.ho
    mods.append(TrainHead(cfg, len(mods), ch, h))
    _ = _InferBlock
    seq = ResNetTrainPartitioned(cfg, mods) if partitioned else ResNetTrainSequential(cfg, [ResNetTrainStep(mods)])
    if seed is not None:
        seq.init_weights(seed, pinned=pinned)
    return seq


__all__ = ["ResNetTrainSequential", "ResNetTrainPartitioned", "ResNetTrainStep", "resnet50_train", "synthetic_labels", "TrainStem", "TrainBottleneck",
           "TrainHead", "LR", "MOMENTUM", "WEIGHT_DECAY"]
_ = (ATOMIC, PREFIX, dataclass)
