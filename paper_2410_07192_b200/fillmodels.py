"""Fill-job models as ``torch.nn.Sequential`` of sm_100a-kernel modules.

PipeFill executables are "a torch.nn.Sequential instance" plus partition
boundaries that "are just layer indices in the Sequential". Each
module here is one linearized node of the fill model's ModelProfile
(profiles.LayerProfile) and runs as a fixed chain of preemptible kernel launches
(``nodes``). Module k of the Sequential is layer k of the profile, so
``ExecutionPlan.boundaries`` index this Sequential directly.

Weights live in page-locked host memory (the fill job's master copy) and are
staged into the executor's arena per partition; activations are bf16, math is
fp32-accumulated on tcgen05 (see csrc/).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch
from torch import nn

from . import kernels as K
from . import native
from .arena import Arena, PinnedBuffer
from .kernels import KernelCtl

PREFIX = "prefix"  # resumable at the claimed-unit cursor (tile-granular GEMM)
ATOMIC = "atomic"  # idempotent, re-run whole on resume (norms, attention, copies)


@dataclass(frozen=True)
class BertConfig:
    name: str
    vocab: int = 30522
    hidden: int = 768
    heads: int = 12
    ffn: int = 3072
    layers: int = 12
    max_pos: int = 512
    type_vocab: int = 2
    eps: float = 1e-12
    seq: int = 128
    precision: str = "bf16"  # "fp32": fp32 weights, activations and math (the rel-1e-4 path)

    @property
    def params_per_layer(self) -> int:
        h, f = self.hidden, self.ffn
        return 4 * h * h + 4 * h + 2 * h * f + f + h + 4 * h

    @property
    def flops_per_sample(self) -> float:
        """Algorithmic forward FLOPs for one sequence: per layer
        24*s*h^2 (QKV, out, two FFN GEMMs at ffn=4h) + 4*s^2*h (QK^T and PV)."""
        s, h, f = self.seq, self.hidden, self.ffn
        gemm = 2.0 * s * (3 * h * h + h * h + 2 * h * f)
        attn = 4.0 * s * s * h
        return self.layers * (gemm + attn)


BERT_BASE = BertConfig("bert_base")
BERT_LARGE = BertConfig("bert_large", hidden=1024, heads=16, ffn=4096, layers=24)


class ExecContext:
    """Where a module's kernel nodes go: launched now (eager: tests, profiler) or
    recorded into a native chain (``chain``: the Executor's per-batch replay path).

    Eager mode carries the preemption words (flag, abort, per-node cursors) and can
    skip nodes below ``start_node`` (resume)."""

    def __init__(self, stream: torch.cuda.Stream, workspace: dict[str, torch.Tensor],
                 flag: int = 0, abort: int = 0, cursors: int = 0, chain: Optional[int] = None):
        self.stream = stream
        self.ws = workspace
        self.flag = flag
        self.abort = abort
        self.cursors = cursors
        self.chain = chain  # pf_chain_t* (record mode) or None
        self.node = 0
        self.start_node = 0  # nodes below this are skipped (eager resume)
        self.launched = 0
        # optional live timing of eager GEMM launches: list of (start event, end event, flops)
        self.gemm_timers: Optional[list] = None

    def ctl(self) -> Optional[KernelCtl]:
        idx = self.node
        self.node += 1
        if not self.flag:
            return None
        return KernelCtl(self.flag, self.abort, self.cursors + 4 * idx)

    def active(self) -> bool:
        """True when the next node must be launched (False while skipping to a resume point)."""
        return self.node >= self.start_node

    def skip(self) -> None:
        self.node += 1

    def buf(self, name: str, numel: int, dtype: torch.dtype = torch.bfloat16) -> torch.Tensor:
        """`numel` elements of `dtype` at the start of workspace buffer `name` (buffers are
        allocated in bf16 units)."""
        if dtype == torch.bfloat16:
            return self.ws[name].view(-1)[:numel]
        esize = torch.tensor([], dtype=dtype).element_size()
        return self.ws[name].view(-1)[:numel * esize // 2].view(dtype)

    def fbuf(self, name: str, numel: int) -> torch.Tensor:
        """fp32 view of a workspace buffer (its size is counted in bf16 elements: 2 per float)."""
        return self.ws[name].view(-1)[:2 * numel].view(torch.float32)

    # -- nodes -----------------------------------------------------------------
    def _eager(self, fn, flops: float = 0.0) -> None:
        if not self.active():
            self.skip()
            return
        timed = flops > 0 and self.gemm_timers is not None
        if timed:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
        fn(self.ctl())
        if timed:
            e1.record(self.stream)
            self.gemm_timers.append((e0, e1, flops))
        self.launched += 1

    def gemm(self, x, w, b, out, *, gelu: bool = False, residual=None, relu: bool = False) -> None:
        k = x.shape[-1]
        m = x.numel() // k
        n = w.shape[0]
        if self.chain is not None:
            epi = (native.PF_EPI_BIAS if b is not None else 0) | (native.PF_EPI_GELU if gelu else 0) \
                | (native.PF_EPI_RESIDUAL if residual is not None else 0) | (native.PF_EPI_RELU if relu else 0)
            fn = "pf_chain_add_gemm_f32" if x.dtype == torch.float32 else "pf_chain_add_gemm"
            native.call(fn, self.chain, x.data_ptr(), w.data_ptr(),
                        None if b is None else b.data_ptr(),
                        None if residual is None else residual.data_ptr(), out.data_ptr(), m, n, k, epi)
            self.node += 1
            return
        self._eager(lambda c: K.linear(x, w, b, gelu=gelu, residual=residual, relu=relu, out=out, ctl=c,
                                       stream=self.stream), flops=2.0 * m * n * k)

    def im2col(self, x, kh: int, kw: int, stride: int, pad: int, kp: int, out) -> None:
        if self.chain is not None:
            b, h, w, c = x.shape
            native.call("pf_chain_add_im2col", self.chain, x.data_ptr(), out.data_ptr(), b, h, w, c, kh, kw,
                        stride, pad, kp)
            self.node += 1
            return
        self._eager(lambda c_: K.im2col(x, kh, kw, stride, pad, kp, out=out, ctl=c_, stream=self.stream))

    def maxpool(self, x, k: int, stride: int, pad: int, out) -> None:
        if self.chain is not None:
            b, h, w, c = x.shape
            native.call("pf_chain_add_maxpool", self.chain, x.data_ptr(), out.data_ptr(), b, h, w, c, k,
                        stride, pad)
            self.node += 1
            return
        self._eager(lambda c_: K.maxpool(x, k, stride, pad, out=out, ctl=c_, stream=self.stream))

    def avgpool(self, x, out) -> None:
        if self.chain is not None:
            b, h, w, c = x.shape
            native.call("pf_chain_add_avgpool", self.chain, x.data_ptr(), out.data_ptr(), b, h * w, c)
            self.node += 1
            return
        self._eager(lambda c_: K.avgpool(x, out=out, ctl=c_, stream=self.stream))

    def attention(self, qkv, heads: int, out) -> None:
        if self.chain is not None:
            b, s, three_h = qkv.shape
            hd = three_h // 3 // heads
            if qkv.dtype == torch.float32:
                native.call("pf_chain_add_attention_f32", self.chain, qkv.data_ptr(), out.data_ptr(), b, s, heads,
                            hd, float(hd ** -0.5))
            else:
                native.call("pf_chain_add_attention", self.chain, qkv.data_ptr(), None, out.data_ptr(), b, s,
                            heads, hd, float(hd ** -0.5))
            self.node += 1
            return
        self._eager(lambda c: K.attention(qkv, heads, out=out, ctl=c, stream=self.stream))

    def layernorm(self, x, g, b, eps: float, out) -> None:
        if self.chain is not None:
            cols = x.shape[-1]
            fn = "pf_chain_add_layernorm_f32" if x.dtype == torch.float32 else "pf_chain_add_layernorm"
            native.call(fn, self.chain, x.data_ptr(), None, g.data_ptr(),
                        b.data_ptr(), out.data_ptr(), x.numel() // cols, cols, float(eps))
            self.node += 1
            return
        self._eager(lambda c: K.layernorm(x, g, b, eps, out=out, ctl=c, stream=self.stream))

    def embedding(self, ids, word, pos, typ, g, b, eps: float, out) -> None:
        if self.chain is not None:
            bsz, s = ids.shape
            if word.dtype == torch.float32:
                native.call("pf_chain_add_embedding_ln_f32", self.chain, ids.data_ptr(), word.data_ptr(),
                            pos.data_ptr(), typ.data_ptr(), g.data_ptr(), b.data_ptr(), out.data_ptr(), bsz, s,
                            word.shape[1], word.shape[0], float(eps))
            else:
                native.call("pf_chain_add_embedding_ln", self.chain, ids.data_ptr(), None, word.data_ptr(),
                            pos.data_ptr(), typ.data_ptr(), g.data_ptr(), b.data_ptr(), out.data_ptr(), bsz, s,
                            word.shape[1], word.shape[0], float(eps))
            self.node += 1
            return
        self._eager(lambda c: K.embedding_ln(ids, word, pos, typ, g, b, eps, out=out, ctl=c,
                                             stream=self.stream))


class FillModule(nn.Module):
    """One node of the linearized fill model."""

    n_nodes = 0
    dtype = torch.bfloat16  # parameter dtype (fp32 modules of the fp32 path override it)

    def __init__(self):
        super().__init__()
        self.host: Optional[PinnedBuffer] = None
        self.host_params: dict[str, torch.Tensor] = {}
        self.dev: dict[str, torch.Tensor] = {}

    # -- parameters ---------------------------------------------------------
    def param_specs(self) -> list[tuple[str, tuple[int, ...], str]]:
        raise NotImplementedError

    def weight_bytes(self) -> int:
        esize = torch.tensor([], dtype=self.dtype).element_size()
        return sum(esize * _numel(shape) for _, shape, _ in self.param_specs())

    def init_host(self, gen: torch.Generator, std: float = 0.02, pinned: bool = True) -> None:
        """Random init into pinned host memory: N(0, std) weights/biases, LN gamma 1, beta 0.
        pinned=False keeps the master copy in pageable memory (CPU-only oracle tests;
        such a module cannot be staged)."""
        specs = self.param_specs()
        total = sum(_numel(s) for _, s, _ in specs)
        if pinned:
            self.host = PinnedBuffer((total,), self.dtype)
            flat = self.host.tensor
        else:
            self.host = None
            flat = torch.empty(total, dtype=self.dtype)
        off = 0
        for name, shape, kind in specs:
            n = _numel(shape)
            if kind == "one":
                vals = torch.ones(n)
            elif kind == "zero":
                vals = torch.zeros(n)
            elif isinstance(kind, tuple) and kind[0] == "conv":
                # ("conv", fan_in, K): Kaiming-normal conv weights [Cout, Kp] in im2col
                # column order, BatchNorm (eval) folded in; pad columns K..Kp zero
                _, fan_in, k = kind
                w = torch.randn(shape[0], k, generator=gen) * (2.0 / fan_in) ** 0.5
                vals = torch.zeros(shape)
                vals[:, :k] = w
                vals = vals.flatten()
            elif isinstance(kind, tuple) and kind[0] == "std":
                vals = torch.randn(n, generator=gen) * kind[1]
            else:
                vals = torch.randn(n, generator=gen) * std
            flat[off:off + n].copy_(vals.to(self.dtype))
            self.host_params[name] = flat[off:off + n].view(*shape)
            off += n

    def stage(self, arena: Arena, stream: torch.cuda.Stream) -> None:
        """H2D copy of this module's weights into the arena (pinned cudaMemcpyAsync)."""
        total = self.host.tensor.numel()
        dflat = arena.alloc((total,), self.dtype)
        native.call("pf_stage_h2d", dflat.data_ptr(), self.host.ptr, self.host.tensor.element_size() * total,
                    stream.cuda_stream)
        off = 0
        for name, shape, _ in self.param_specs():
            n = _numel(shape)
            self.dev[name] = dflat[off:off + n].view(*shape)
            off += n

    def unstage(self) -> None:
        self.dev = {}

    def make_views(self, ptr: int) -> dict[str, torch.Tensor]:
        """Device tensors of this module's staged state starting at `ptr` (the layout of
        its host blob: bf16 parameters in param_specs order)."""
        nbytes = self.weight_bytes()
        from .arena import device_view
        esize = torch.tensor([], dtype=self.dtype).element_size()
        dflat = device_view(ptr, (max(nbytes // esize, 1),), self.dtype)
        dev, off = {}, 0
        for name, shape, _ in self.param_specs():
            n = _numel(shape)
            dev[name] = dflat[off:off + n].view(*shape)
            off += n
        return dev

    # -- execution ------------------------------------------------------------
    def workspace(self, batch: int) -> dict[str, int]:
        """Workspace buffers (bf16 elements) one batch of this module needs."""
        return {}

    def flops_per_sample(self) -> float:
        """Algorithmic forward FLOPs of this module for one sample."""
        return 0.0

    def gemm_node_flops(self, batch: int) -> list[tuple[int, float]]:
        """(node index within this module, algorithmic FLOPs) of its GEMM nodes."""
        return []

    def gemm_node_bytes(self, batch: int) -> list[tuple[int, float]]:
        """(node index, minimum DRAM bytes: operands read once + output written) of its GEMM
        nodes -- with the FLOPs, the per-launch roofline max(F / tensor peak, B / HBM)."""
        return []

    def node_units(self, batch: int) -> list[tuple[int, str]]:
        raise NotImplementedError

    def forward(self, x, ctx: ExecContext):
        raise NotImplementedError


def _numel(shape) -> int:
    n = 1
    for s in shape:
        n *= int(s)
    return n


class BertEmbeddings(FillModule):
    """word + position + token-type embeddings, then LayerNorm (1 kernel node)."""

    n_nodes = 1

    def __init__(self, cfg: BertConfig):
        super().__init__()
        self.cfg = cfg
        self.dtype = torch.float32 if cfg.precision == "fp32" else torch.bfloat16

    def param_specs(self):
        c = self.cfg
        return [("word", (c.vocab, c.hidden), "w"), ("pos", (c.max_pos, c.hidden), "w"),
                ("type", (c.type_vocab, c.hidden), "w"), ("ln_g", (c.hidden,), "one"),
                ("ln_b", (c.hidden,), "zero")]

    def workspace(self, batch):  # bf16 units
        u = 2 if self.cfg.precision == "fp32" else 1
        return {"act": u * batch * self.cfg.seq * self.cfg.hidden}

    def node_units(self, batch):
        return [(K.norm_units(batch * self.cfg.seq, self.cfg.hidden), ATOMIC)]

    def forward(self, ids: torch.Tensor, ctx: ExecContext) -> torch.Tensor:
        b, s = ids.shape
        out = ctx.buf("act", b * s * self.cfg.hidden, self.dtype).view(b, s, self.cfg.hidden)
        d = self.dev
        ctx.embedding(ids, d["word"], d["pos"], d["type"], d["ln_g"], d["ln_b"], self.cfg.eps, out)
        return out


class BertLayer(FillModule):
    """Post-LN BERT encoder layer as 7 kernel nodes:
    QKV GEMM+bias | attention | out GEMM+bias+residual | LN | FFN1 GEMM+bias+GELU |
    FFN2 GEMM+bias+residual | LN. The layer is in place on the hidden buffer."""

    n_nodes = 7

    def __init__(self, cfg: BertConfig):
        super().__init__()
        self.cfg = cfg
        self.dtype = torch.float32 if cfg.precision == "fp32" else torch.bfloat16

    def param_specs(self):
        h, f = self.cfg.hidden, self.cfg.ffn
        return [("qkv_w", (3 * h, h), "w"), ("qkv_b", (3 * h,), "w"),
                ("out_w", (h, h), "w"), ("out_b", (h,), "w"),
                ("ln1_g", (h,), "one"), ("ln1_b", (h,), "zero"),
                ("ffn1_w", (f, h), "w"), ("ffn1_b", (f,), "w"),
                ("ffn2_w", (h, f), "w"), ("ffn2_b", (h,), "w"),
                ("ln2_g", (h,), "one"), ("ln2_b", (h,), "zero")]

    def workspace(self, batch):  # bf16 units
        m, h, f = batch * self.cfg.seq, self.cfg.hidden, self.cfg.ffn
        u = 2 if self.cfg.precision == "fp32" else 1
        return {"qkv": u * m * 3 * h, "ctx": u * m * h, "a": u * m * h, "a_ln": u * m * h, "ffn": u * m * f,
                "o": u * m * h}

    def flops_per_sample(self) -> float:
        s, h, f = self.cfg.seq, self.cfg.hidden, self.cfg.ffn
        return 2.0 * s * (4 * h * h + 2 * h * f) + 4.0 * s * s * h

    def gemm_node_flops(self, batch: int) -> list[tuple[int, float]]:
        m, h, f = batch * self.cfg.seq, self.cfg.hidden, self.cfg.ffn
        return [(0, 2.0 * m * 3 * h * h), (2, 2.0 * m * h * h), (4, 2.0 * m * h * f),
                (5, 2.0 * m * f * h)]

    def gemm_node_bytes(self, batch):
        m, h, f = batch * self.cfg.seq, self.cfg.hidden, self.cfg.ffn
        e = 4 if self.cfg.precision == "fp32" else 2
        return [(0, e * (m * h + 3 * h * h + 3 * m * h)), (2, e * (m * h + h * h + 2 * m * h)),
                (4, e * (m * h + f * h + m * f)), (5, e * (m * f + h * f + 2 * m * h))]

    def node_units(self, batch):
        seq = self.cfg.seq
        m, h, f = batch * seq, self.cfg.hidden, self.cfg.ffn
        return [(K.gemm_units(m, 3 * h, h), PREFIX),
                (K.attention_units(batch, seq, self.cfg.heads, h // self.cfg.heads), ATOMIC),
                (K.gemm_units(m, h, h), PREFIX),
                (K.norm_units(m, h), ATOMIC),
                (K.gemm_units(m, f, h), PREFIX),
                (K.gemm_units(m, h, f), PREFIX),
                (K.norm_units(m, h), ATOMIC)]

    def forward(self, x: torch.Tensor, ctx: ExecContext) -> torch.Tensor:
        b, s, h = x.shape
        m, f = b * s, self.cfg.ffn
        d = self.dev
        x2 = x.view(m, h)
        dt = self.dtype
        qkv = ctx.buf("qkv", m * 3 * h, dt).view(b, s, 3 * h)
        cx = ctx.buf("ctx", m * h, dt).view(m, h)
        a = ctx.buf("a", m * h, dt).view(m, h)
        a_ln = ctx.buf("a_ln", m * h, dt).view(m, h)
        hf = ctx.buf("ffn", m * f, dt).view(m, f)
        o = ctx.buf("o", m * h, dt).view(m, h)
        ctx.gemm(x2, d["qkv_w"], d["qkv_b"], qkv.view(m, 3 * h))
        ctx.attention(qkv, self.cfg.heads, cx.view(b, s, h))
        ctx.gemm(cx, d["out_w"], d["out_b"], a, residual=x2)
        ctx.layernorm(a, d["ln1_g"], d["ln1_b"], self.cfg.eps, a_ln)
        ctx.gemm(a_ln, d["ffn1_w"], d["ffn1_b"], hf, gelu=True)
        ctx.gemm(hf, d["ffn2_w"], d["ffn2_b"], o, residual=a_ln)
        ctx.layernorm(o, d["ln2_g"], d["ln2_b"], self.cfg.eps, x2)
        return x


class FillSequential(nn.Sequential):
    """The fill model: an nn.Sequential whose module k is profile layer k.

    Subclasses describe the model's data at its edges, which is all the Executor
    needs to run any partition [lo, hi):

    * ``input_spec()``: (dtype, per-sample shape) of the job's input samples;
    * ``boundary_shape(i)``: per-sample bf16 activation shape entering module i
      (what is stored between partitions at boundary i);
    * ``result_shape()`` and ``result_view(x, cnt)``: the per-sample result and where
      it sits in the last module's output (a 2-D copy: src, pitch, width, rows);
    * ``make_inputs(job_seed, first, count)``: the job's synthetic samples
      [first, first + count), identical under any split into ranges and batches."""

    is_training = False  # a training job: one chain = forward, loss, backward, optimizer step

    def __init__(self, cfg, modules: list[FillModule]):
        super().__init__(*modules)
        self.cfg = cfg
        self.profile = None  # set by profiler.measure_profile

    def result_dtype(self) -> torch.dtype:
        return torch.bfloat16

    def act_dtype(self) -> torch.dtype:
        """dtype of the activations stored between partitions."""
        return torch.bfloat16

    def act_bytes(self) -> int:
        return torch.tensor([], dtype=self.act_dtype()).element_size()

    def aux_spec(self) -> Optional[tuple[torch.dtype, tuple[int, ...]]]:
        """(dtype, per-sample shape) of a second per-sample input (labels), or None."""
        return None

    def make_aux(self, job_seed: int, first: int, count: int) -> torch.Tensor:
        raise NotImplementedError

    def input_spec(self) -> tuple[torch.dtype, tuple[int, ...]]:
        raise NotImplementedError

    def boundary_shape(self, i: int) -> tuple[int, ...]:
        raise NotImplementedError

    def result_shape(self) -> tuple[int, ...]:
        raise NotImplementedError

    def result_view(self, x: torch.Tensor, cnt: int) -> tuple[int, int, int, int]:
        raise NotImplementedError

    def make_inputs(self, job_seed: int, first: int, count: int) -> torch.Tensor:
        raise NotImplementedError

    def input_bytes(self) -> int:
        dt, shape = self.input_spec()
        return _numel(shape) * torch.tensor([], dtype=dt).element_size()

    def boundary_elems(self, i: int) -> int:
        return _numel(self.boundary_shape(i))

    def init_weights(self, seed: int = 0, pinned: bool = True) -> "FillSequential":
        gen = torch.Generator().manual_seed(seed)
        for mod in self:
            mod.init_host(gen, pinned=pinned)
        return self

    def weight_bytes(self, lo: int, hi: int) -> int:
        return sum(self[i].weight_bytes() for i in range(lo, hi))

    def workspace(self, lo: int, hi: int, batch: int) -> dict[str, int]:
        need: dict[str, int] = {}
        for i in range(lo, hi):
            for k, v in self[i].workspace(batch).items():
                need[k] = max(need.get(k, 0), v)
        return need

    def node_units(self, lo: int, hi: int, batch: int) -> list[tuple[int, str]]:
        out: list[tuple[int, str]] = []
        for i in range(lo, hi):
            out.extend(self[i].node_units(batch))
        return out

    def oracle_params(self, i: int) -> dict[str, torch.Tensor]:
        """fp32 copies of module i's host weights (for the CPU oracle)."""
        return {k: v.float().clone() for k, v in self[i].host_params.items()}


class BertSequential(FillSequential):
    """BERT: int32 token ids in, [seq, hidden] activations between modules, the
    [CLS] row of the last hidden state out."""

    def input_spec(self):
        return torch.int32, (self.cfg.seq,)

    def boundary_shape(self, i):
        return (self.cfg.seq, self.cfg.hidden)

    def result_shape(self):
        return (self.cfg.hidden,)

    def act_dtype(self):
        return torch.float32 if self.cfg.precision == "fp32" else torch.bfloat16

    def result_dtype(self):
        return self.act_dtype()

    def result_view(self, x, cnt):
        s, h, e = self.cfg.seq, self.cfg.hidden, self.act_bytes()
        return x.data_ptr(), s * h * e, h * e, cnt

    def make_inputs(self, job_seed, first, count):
        return synthetic_ids(job_seed, first, count, self.cfg.seq, self.cfg.vocab)


def bert(cfg: BertConfig = BERT_BASE, seed: Optional[int] = 0) -> FillSequential:
    """BERT encoder as the linearized fill model [embeddings, layer_0..layer_{L-1}]."""
    mods: list[FillModule] = [BertEmbeddings(cfg)] + [BertLayer(cfg) for _ in range(cfg.layers)]
    seq = BertSequential(cfg, mods)
    if seed is not None:
        seq.init_weights(seed)
    return seq


# --------------------------------------------------------------------------- ResNet-50


@dataclass(frozen=True)
class ResNetConfig:
    """ResNet-50 v1.5 (stride on the 3x3 conv), NHWC bf16, BatchNorm folded into the
    convolutions (inference form: scale into the weights, shift into the bias)."""

    name: str = "resnet50"
    image: int = 224
    in_ch: int = 3
    classes: int = 1000
    blocks: tuple[int, ...] = (3, 4, 6, 3)
    widths: tuple[int, ...] = (64, 128, 256, 512)
    expansion: int = 4
    stem_ch: int = 64

    @property
    def stem_k(self) -> int:
        return 7 * 7 * self.in_ch

    @property
    def stem_kp(self) -> int:
        return (self.stem_k + 7) // 8 * 8  # 16-B GEMM rows

    @property
    def flops_per_sample(self) -> float:
        return sum(m.flops_per_sample() for m in _resnet_modules(self))


RESNET50 = ResNetConfig()


def _act(idx: int) -> str:
    return f"act{idx % 2}"


class ResNetStem(FillModule):
    """conv 7x7/2 (+BN+ReLU) as im2col + GEMM, then maxpool 3x3/2: 3 kernel nodes."""

    n_nodes = 3

    def __init__(self, cfg: ResNetConfig, idx: int):
        super().__init__()
        self.cfg, self.idx = cfg, idx
        self.h1 = K.conv_out(cfg.image, 7, 2, 3)
        self.h2 = K.conv_out(self.h1, 3, 2, 1)

    def param_specs(self):
        c = self.cfg
        return [("w", (c.stem_ch, c.stem_kp), ("conv", c.stem_k, c.stem_k)),
                ("b", (c.stem_ch,), ("std", 0.05))]

    def out_shape(self):
        return (self.h2, self.h2, self.cfg.stem_ch)

    def workspace(self, batch):
        c = self.cfg
        return {"col": batch * self.h1 * self.h1 * c.stem_kp, "pre": batch * self.h1 * self.h1 * c.stem_ch,
                _act(self.idx): batch * self.h2 * self.h2 * c.stem_ch}

    def flops_per_sample(self):
        return 2.0 * self.h1 * self.h1 * self.cfg.stem_ch * self.cfg.stem_k

    def gemm_node_flops(self, batch):
        return [(1, batch * self.flops_per_sample())]

    def gemm_node_bytes(self, batch):
        c, m = self.cfg, batch * self.h1 * self.h1
        return [(1, 2.0 * (m * c.stem_kp + c.stem_ch * c.stem_kp + m * c.stem_ch))]

    def node_units(self, batch):
        c, m = self.cfg, batch * self.h1 * self.h1
        return [(K.image_units(0, m * c.stem_kp, c.in_ch), ATOMIC),
                (K.gemm_units(m, c.stem_ch, c.stem_kp), PREFIX),
                (K.image_units(1, batch * self.h2 * self.h2 * c.stem_ch, c.stem_ch), ATOMIC)]

    def forward(self, x, ctx):
        c, b = self.cfg, x.shape[0]
        m = b * self.h1 * self.h1
        col = ctx.buf("col", m * c.stem_kp).view(m, c.stem_kp)
        pre = ctx.buf("pre", m * c.stem_ch).view(b, self.h1, self.h1, c.stem_ch)
        out = ctx.buf(_act(self.idx), b * self.h2 * self.h2 * c.stem_ch).view(b, self.h2, self.h2, c.stem_ch)
        ctx.im2col(x, 7, 7, 2, 3, c.stem_kp, col)
        ctx.gemm(col, self.dev["w"], self.dev["b"], pre.view(m, c.stem_ch), relu=True)
        ctx.maxpool(pre, 3, 2, 1, out)
        return out


class Bottleneck(FillModule):
    """1x1 -> 3x3 (stride) -> 1x1 (x4) with identity or projection shortcut; every
    conv is a GEMM with folded BN; ReLU, and the residual add of the last conv, run
    in the GEMM epilogue. Nodes: gemm1, im2col, gemm2, [im2col_ds], [gemm_ds], gemm3."""

    def __init__(self, cfg: ResNetConfig, idx: int, in_ch: int, width: int, stride: int, h_in: int):
        super().__init__()
        self.cfg, self.idx = cfg, idx
        self.in_ch, self.width, self.stride, self.h = in_ch, width, stride, h_in
        self.out_ch = width * cfg.expansion
        self.ho = K.conv_out(h_in, 3, stride, 1)
        self.ds = stride != 1 or in_ch != self.out_ch
        self.n_nodes = 4 + (1 if self.ds else 0) + (1 if self.ds and stride != 1 else 0)

    def param_specs(self):
        ci, w, co = self.in_ch, self.width, self.out_ch
        specs = [("w1", (w, ci), ("conv", ci, ci)), ("b1", (w,), ("std", 0.05)),
                 ("w2", (w, 9 * w), ("conv", 9 * w, 9 * w)), ("b2", (w,), ("std", 0.05)),
                 ("w3", (co, w), ("conv", 4 * w, w)), ("b3", (co,), ("std", 0.05))]
        if self.ds:
            specs += [("wd", (co, ci), ("conv", 4 * ci, ci)), ("bd", (co,), ("std", 0.05))]
        return specs

    def out_shape(self):
        return (self.ho, self.ho, self.out_ch)

    def workspace(self, batch):
        hw, ow = self.h * self.h, self.ho * self.ho
        need = {"t1": batch * hw * self.width, "col": batch * ow * 9 * self.width,
                "t2": batch * ow * self.width, _act(self.idx): batch * ow * self.out_ch}
        if self.ds:
            need["sc"] = batch * ow * self.out_ch
            if self.stride != 1:
                need["colds"] = batch * ow * self.in_ch
        return need

    def flops_per_sample(self):
        hw, ow, ci, w, co = self.h * self.h, self.ho * self.ho, self.in_ch, self.width, self.out_ch
        f = 2.0 * (hw * ci * w + ow * 9 * w * w + ow * w * co)
        return f + (2.0 * ow * ci * co if self.ds else 0.0)

    def _gemms(self, batch):
        """(node, M, N, K) of the GEMM nodes."""
        hw, ow, ci, w, co = batch * self.h * self.h, batch * self.ho * self.ho, self.in_ch, self.width, self.out_ch
        g = [(0, hw, w, ci), (2, ow, w, 9 * w)]
        n = 3
        if self.ds:
            if self.stride != 1:
                n += 1
            g.append((n, ow, co, ci))
            n += 1
        g.append((n, ow, co, w))
        return g

    def gemm_node_flops(self, batch):
        return [(node, 2.0 * m * n * k) for node, m, n, k in self._gemms(batch)]

    def gemm_node_bytes(self, batch):
        last = self._gemms(batch)[-1][0]  # the last GEMM adds the residual in its epilogue
        return [(node, 2.0 * (m * k + n * k + m * n * (2 if node == last else 1)))
                for node, m, n, k in self._gemms(batch)]

    def node_units(self, batch):
        ow = batch * self.ho * self.ho
        units = {node: (K.gemm_units(m, n, k), PREFIX) for node, m, n, k in self._gemms(batch)}
        units[1] = (K.image_units(0, ow * 9 * self.width, self.width), ATOMIC)
        if self.ds and self.stride != 1:
            units[3] = (K.image_units(0, ow * self.in_ch, self.in_ch), ATOMIC)
        return [units[i] for i in range(self.n_nodes)]

    def forward(self, x, ctx):
        b = x.shape[0]
        d = self.dev
        hw, ow, ci, w, co = b * self.h * self.h, b * self.ho * self.ho, self.in_ch, self.width, self.out_ch
        x2 = x.reshape(hw, ci)
        t1 = ctx.buf("t1", hw * w).view(b, self.h, self.h, w)
        col = ctx.buf("col", ow * 9 * w).view(ow, 9 * w)
        t2 = ctx.buf("t2", ow * w).view(ow, w)
        out = ctx.buf(_act(self.idx), ow * co).view(b, self.ho, self.ho, co)
        ctx.gemm(x2, d["w1"], d["b1"], t1.view(hw, w), relu=True)
        ctx.im2col(t1, 3, 3, self.stride, 1, 9 * w, col)
        ctx.gemm(col, d["w2"], d["b2"], t2, relu=True)
        if self.ds:
            src = x2
            if self.stride != 1:
                src = ctx.buf("colds", ow * ci).view(ow, ci)
                ctx.im2col(x, 1, 1, self.stride, 0, ci, src)
            sc = ctx.buf("sc", ow * co).view(ow, co)
            ctx.gemm(src, d["wd"], d["bd"], sc)
        else:
            sc = x2
        ctx.gemm(t2, d["w3"], d["b3"], out.view(ow, co), residual=sc, relu=True)
        return out


class ResNetHead(FillModule):
    """Global average pool + fully connected classifier: 2 kernel nodes."""

    n_nodes = 2

    def __init__(self, cfg: ResNetConfig, idx: int, in_ch: int, h_in: int):
        super().__init__()
        self.cfg, self.idx, self.in_ch, self.h = cfg, idx, in_ch, h_in

    def param_specs(self):
        return [("fc_w", (self.cfg.classes, self.in_ch), ("std", self.in_ch ** -0.5)),
                ("fc_b", (self.cfg.classes,), ("std", 0.01))]

    def out_shape(self):
        return (self.cfg.classes,)

    def workspace(self, batch):
        return {"pooled": batch * self.in_ch, _act(self.idx): batch * self.cfg.classes}

    def flops_per_sample(self):
        return 2.0 * self.in_ch * self.cfg.classes

    def gemm_node_flops(self, batch):
        return [(1, batch * self.flops_per_sample())]

    def gemm_node_bytes(self, batch):
        return [(1, 2.0 * (batch * self.in_ch + self.cfg.classes * self.in_ch + batch * self.cfg.classes))]

    def node_units(self, batch):
        return [(K.image_units(2, batch * self.in_ch, self.in_ch), ATOMIC),
                (K.gemm_units(batch, self.cfg.classes, self.in_ch), PREFIX)]

    def forward(self, x, ctx):
        b = x.shape[0]
        pooled = ctx.buf("pooled", b * self.in_ch).view(b, self.in_ch)
        logits = ctx.buf(_act(self.idx), b * self.cfg.classes).view(b, self.cfg.classes)
        ctx.avgpool(x, pooled)
        ctx.gemm(pooled, self.dev["fc_w"], self.dev["fc_b"], logits)
        return logits


def _resnet_modules(cfg: ResNetConfig) -> list[FillModule]:
    mods: list[FillModule] = [ResNetStem(cfg, 0)]
    ch, h = cfg.stem_ch, mods[0].out_shape()[0]
    for stage, (n, w) in enumerate(zip(cfg.blocks, cfg.widths)):
        for j in range(n):
            stride = 2 if (j == 0 and stage > 0) else 1
            blk = Bottleneck(cfg, len(mods), ch, w, stride, h)
            mods.append(blk)
            ch, h = blk.out_ch, blk.ho
    mods.append(ResNetHead(cfg, len(mods), ch, h))
    return mods


class ResNetSequential(FillSequential):
    """ResNet: bf16 NHWC images in, NHWC activations between modules, logits out."""

    def input_spec(self):
        c = self.cfg
        return torch.bfloat16, (c.image, c.image, c.in_ch)

    def boundary_shape(self, i):
        if i == 0:
            return self.input_spec()[1]
        return self[i - 1].out_shape()

    def result_shape(self):
        return (self.cfg.classes,)

    def result_view(self, x, cnt):
        n = cnt * self.cfg.classes * 2
        return x.data_ptr(), n, n, 1

    def make_inputs(self, job_seed, first, count):
        return synthetic_images(job_seed, first, count, self.cfg.image, self.cfg.in_ch)


def resnet50(cfg: ResNetConfig = RESNET50, seed: Optional[int] = 0, pinned: bool = True) -> FillSequential:
    """ResNet-50 as the linearized fill model [stem, 16 bottlenecks, head]."""
    seq = ResNetSequential(cfg, _resnet_modules(cfg))
    if seed is not None:
        seq.init_weights(seed, pinned=pinned)
    return seq


def synthetic_images(job_seed: int, first_sample: int, count: int, size: int, ch: int) -> torch.Tensor:
    """N(0, 1) NHWC bf16 images; sample i depends only on (job_seed, i)."""
    out = torch.empty(count, size, size, ch, dtype=torch.bfloat16)
    g = torch.Generator()
    for j in range(count):
        g.manual_seed((job_seed * 1_000_003 + first_sample + j) * 2_654_435_761 % (2 ** 63 - 1))
        out[j] = torch.randn(size, size, ch, generator=g).to(torch.bfloat16)
    return out


def synthetic_ids(job_seed: int, first_sample: int, count: int, seq: int, vocab: int) -> torch.Tensor:
    """Deterministic synthetic token ids for samples [first, first+count) of a job:
    sample i's ids depend only on (job_seed, i), so any split into ranges and
    batches sees the same inputs."""
    i = torch.arange(first_sample, first_sample + count, dtype=torch.int64)[:, None]
    p = torch.arange(seq, dtype=torch.int64)[None, :]
    x = (i * 1_000_003 + p * 7919 + job_seed * 104_729) % 2_147_483_647
    x = (x * 48_271) % 2_147_483_647
    return (x % vocab).to(torch.int32)


__all__ = ["BertConfig", "BERT_BASE", "BERT_LARGE", "ExecContext", "FillModule", "BertEmbeddings",
           "BertLayer", "FillSequential", "BertSequential", "bert", "synthetic_ids", "PREFIX", "ATOMIC",
           "ResNetConfig", "RESNET50", "ResNetStem", "Bottleneck", "ResNetHead", "ResNetSequential",
           "resnet50", "synthetic_images"]

_ = ctypes  # ctypes is used by arena/native through this module's imports
