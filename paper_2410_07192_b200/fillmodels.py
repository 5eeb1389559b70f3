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

    def buf(self, name: str, numel: int) -> torch.Tensor:
        return self.ws[name].view(-1)[:numel]

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

    def gemm(self, x, w, b, out, *, gelu: bool = False, residual=None) -> None:
        k = x.shape[-1]
        m = x.numel() // k
        n = w.shape[0]
        if self.chain is not None:
            epi = (native.PF_EPI_BIAS if b is not None else 0) | (native.PF_EPI_GELU if gelu else 0) \
                | (native.PF_EPI_RESIDUAL if residual is not None else 0)
            native.call("pf_chain_add_gemm", self.chain, x.data_ptr(), w.data_ptr(),
                        None if b is None else b.data_ptr(),
                        None if residual is None else residual.data_ptr(), out.data_ptr(), m, n, k, epi)
            self.node += 1
            return
        self._eager(lambda c: K.linear(x, w, b, gelu=gelu, residual=residual, out=out, ctl=c,
                                       stream=self.stream), flops=2.0 * m * n * k)

    def attention(self, qkv, heads: int, out) -> None:
        if self.chain is not None:
            b, s, three_h = qkv.shape
            hd = three_h // 3 // heads
            native.call("pf_chain_add_attention", self.chain, qkv.data_ptr(), None, out.data_ptr(), b, s,
                        heads, hd, float(hd ** -0.5))
            self.node += 1
            return
        self._eager(lambda c: K.attention(qkv, heads, out=out, ctl=c, stream=self.stream))

    def layernorm(self, x, g, b, eps: float, out) -> None:
        if self.chain is not None:
            cols = x.shape[-1]
            native.call("pf_chain_add_layernorm", self.chain, x.data_ptr(), None, g.data_ptr(),
                        b.data_ptr(), out.data_ptr(), x.numel() // cols, cols, float(eps))
            self.node += 1
            return
        self._eager(lambda c: K.layernorm(x, g, b, eps, out=out, ctl=c, stream=self.stream))

    def embedding(self, ids, word, pos, typ, g, b, eps: float, out) -> None:
        if self.chain is not None:
            bsz, s = ids.shape
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

    def __init__(self):
        super().__init__()
        self.host: Optional[PinnedBuffer] = None
        self.host_params: dict[str, torch.Tensor] = {}
        self.dev: dict[str, torch.Tensor] = {}

    # -- parameters ---------------------------------------------------------
    def param_specs(self) -> list[tuple[str, tuple[int, ...], str]]:
        raise NotImplementedError

    def weight_bytes(self) -> int:
        return sum(2 * _numel(shape) for _, shape, _ in self.param_specs())

    def init_host(self, gen: torch.Generator, std: float = 0.02) -> None:
        """Random init into pinned host memory: N(0, std) weights/biases, LN gamma 1, beta 0."""
        specs = self.param_specs()
        total = sum(_numel(s) for _, s, _ in specs)
        self.host = PinnedBuffer((total,), torch.bfloat16)
        flat = self.host.tensor
        off = 0
        for name, shape, kind in specs:
            n = _numel(shape)
            if kind == "one":
                vals = torch.ones(n)
            elif kind == "zero":
                vals = torch.zeros(n)
            else:
                vals = torch.randn(n, generator=gen) * std
            flat[off:off + n].copy_(vals.to(torch.bfloat16))
            self.host_params[name] = flat[off:off + n].view(*shape)
            off += n

    def stage(self, arena: Arena, stream: torch.cuda.Stream) -> None:
        """H2D copy of this module's weights into the arena (pinned cudaMemcpyAsync)."""
        total = self.host.tensor.numel()
        dflat = arena.alloc((total,), torch.bfloat16)
        native.call("pf_stage_h2d", dflat.data_ptr(), self.host.ptr, 2 * total, stream.cuda_stream)
        off = 0
        for name, shape, _ in self.param_specs():
            n = _numel(shape)
            self.dev[name] = dflat[off:off + n].view(*shape)
            off += n

    def unstage(self) -> None:
        self.dev = {}

    # -- execution ------------------------------------------------------------
    def workspace(self, batch: int, seq: int) -> dict[str, int]:
        return {}

    def flops_per_sample(self) -> float:
        """Algorithmic forward FLOPs of this module for one sequence."""
        return 0.0

    def gemm_node_flops(self, batch: int) -> list[tuple[int, float]]:
        """(node index within this module, algorithmic FLOPs) of its GEMM nodes."""
        return []

    def node_units(self, batch: int, seq: int) -> list[tuple[int, str]]:
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

    def param_specs(self):
        c = self.cfg
        return [("word", (c.vocab, c.hidden), "w"), ("pos", (c.max_pos, c.hidden), "w"),
                ("type", (c.type_vocab, c.hidden), "w"), ("ln_g", (c.hidden,), "one"),
                ("ln_b", (c.hidden,), "zero")]

    def node_units(self, batch, seq):
        return [(K.norm_units(batch * seq, self.cfg.hidden), ATOMIC)]

    def forward(self, ids: torch.Tensor, ctx: ExecContext) -> torch.Tensor:
        b, s = ids.shape
        out = ctx.buf("hidden", b * s * self.cfg.hidden).view(b, s, self.cfg.hidden)
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

    def param_specs(self):
        h, f = self.cfg.hidden, self.cfg.ffn
        return [("qkv_w", (3 * h, h), "w"), ("qkv_b", (3 * h,), "w"),
                ("out_w", (h, h), "w"), ("out_b", (h,), "w"),
                ("ln1_g", (h,), "one"), ("ln1_b", (h,), "zero"),
                ("ffn1_w", (f, h), "w"), ("ffn1_b", (f,), "w"),
                ("ffn2_w", (h, f), "w"), ("ffn2_b", (h,), "w"),
                ("ln2_g", (h,), "one"), ("ln2_b", (h,), "zero")]

    def workspace(self, batch, seq):
        m, h, f = batch * seq, self.cfg.hidden, self.cfg.ffn
        return {"qkv": m * 3 * h, "ctx": m * h, "a": m * h, "a_ln": m * h, "ffn": m * f, "o": m * h}

    def flops_per_sample(self) -> float:
        s, h, f = self.cfg.seq, self.cfg.hidden, self.cfg.ffn
        return 2.0 * s * (4 * h * h + 2 * h * f) + 4.0 * s * s * h

    def gemm_node_flops(self, batch: int) -> list[tuple[int, float]]:
        m, h, f = batch * self.cfg.seq, self.cfg.hidden, self.cfg.ffn
        return [(0, 2.0 * m * 3 * h * h), (2, 2.0 * m * h * h), (4, 2.0 * m * h * f),
                (5, 2.0 * m * f * h)]

    def node_units(self, batch, seq):
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
        qkv = ctx.buf("qkv", m * 3 * h).view(b, s, 3 * h)
        cx = ctx.buf("ctx", m * h).view(m, h)
        a = ctx.buf("a", m * h).view(m, h)
        a_ln = ctx.buf("a_ln", m * h).view(m, h)
        hf = ctx.buf("ffn", m * f).view(m, f)
        o = ctx.buf("o", m * h).view(m, h)
        ctx.gemm(x2, d["qkv_w"], d["qkv_b"], qkv.view(m, 3 * h))
        ctx.attention(qkv, self.cfg.heads, cx.view(b, s, h))
        ctx.gemm(cx, d["out_w"], d["out_b"], a, residual=x2)
        ctx.layernorm(a, d["ln1_g"], d["ln1_b"], self.cfg.eps, a_ln)
        ctx.gemm(a_ln, d["ffn1_w"], d["ffn1_b"], hf, gelu=True)
        ctx.gemm(hf, d["ffn2_w"], d["ffn2_b"], o, residual=a_ln)
        ctx.layernorm(o, d["ln2_g"], d["ln2_b"], self.cfg.eps, x2)
        return x


class FillSequential(nn.Sequential):
    """The fill model: an nn.Sequential whose module k is profile layer k."""

    def __init__(self, cfg: BertConfig, modules: list[FillModule]):
        super().__init__(*modules)
        self.cfg = cfg

    def init_weights(self, seed: int = 0) -> "FillSequential":
        gen = torch.Generator().manual_seed(seed)
        for mod in self:
            mod.init_host(gen)
        return self

    def weight_bytes(self, lo: int, hi: int) -> int:
        return sum(self[i].weight_bytes() for i in range(lo, hi))

    def workspace(self, lo: int, hi: int, batch: int) -> dict[str, int]:
        need: dict[str, int] = {}
        for i in range(lo, hi):
            for k, v in self[i].workspace(batch, self.cfg.seq).items():
                need[k] = max(need.get(k, 0), v)
        return need

    def node_units(self, lo: int, hi: int, batch: int) -> list[tuple[int, str]]:
        out: list[tuple[int, str]] = []
        for i in range(lo, hi):
            out.extend(self[i].node_units(batch, self.cfg.seq))
        return out

    def oracle_params(self, i: int) -> dict[str, torch.Tensor]:
        """fp32 copies of module i's host weights (for the CPU oracle)."""
        return {k: v.float().clone() for k, v in self[i].host_params.items()}


def bert(cfg: BertConfig = BERT_BASE, seed: Optional[int] = 0) -> FillSequential:
    """BERT encoder as the linearized fill model [embeddings, layer_0..layer_{L-1}]."""
    mods: list[FillModule] = [BertEmbeddings(cfg)] + [BertLayer(cfg) for _ in range(cfg.layers)]
    seq = FillSequential(cfg, mods)
    if seed is not None:
        seq.init_weights(seed)
    return seq


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
           "BertLayer", "FillSequential", "bert", "synthetic_ids", "PREFIX", "ATOMIC"]

_ = ctypes  # ctypes is used by arena/native through this module's imports
