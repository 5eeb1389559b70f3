"""Pipeline engine with PipeFill's BUBBLE instruction, on CUDA streams.

The main job is the user's pipeline-parallel training job (the paper augments
DeepSpeed's engine). This engine executes one stage's
instruction list from ``schedule.stage_program`` — GPipe or 1F1B, F/B per
microbatch, with BUBBLE instructions before the first backward and after the
last one — on three streams:

* main (high priority): the stage's forward/backward compute and optimizer step;
* comm (high priority): the recv that ends each wait. A BUBBLE instruction
  writes 1 to the stage's device flag (stream-ordered 32-bit store) and records
  the bubble-start event the fill stream waits on; the recv completion then
  writes 0 ("the recv's completion, stream-ordered on the comm
  stream, clears the stage's device bubble flag");
* fill (lowest priority, owned by executor.Executor): the fill job's kernels,
  which poll the flag at tile granularity and yield.

Two transports provide the recv:

* ``TimerLink`` — the 1-GPU stand-in (artificial bubbles, BASELINE north star):
  every recv completes at its analytic arrival time in the p-stage schedule,
  measured from a device %globaltimer anchor, via a one-thread spin kernel;
* ``NcclLink`` — real P2P activations/gradients between adjacent stages over
  NVLink with torch.distributed (NCCL), one process per GPU.

Main-job compute (``GPTStage``) is plain torch (cuBLAS / SDPA): it is the
job being filled, not the product.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import torch
import torch.nn.functional as F
from torch import nn

from . import native
from .executor import BubbleSlot, Executor
from .schedule import BubbleKind, Instr, PipelineConfig, stage_program, steady_state_timeline

US = 1000  # ns per us


# --------------------------------------------------------------------------- main job


@dataclass(frozen=True)
class GPTStageConfig:
    hidden: int = 4096
    heads: int = 32
    ffn: int = 16384
    layers: int = 5
    seq: int = 2048
    micro_batch: int = 2

    @property
    def params(self) -> int:
        h, f = self.hidden, self.ffn
        return self.layers * (4 * h * h + 2 * h * f + 9 * h + f)


GPT_8B_STAGE = GPTStageConfig()  # 8-stage split of a 40-layer h=4096 GPT
GPT2_SMALL_STAGE = GPTStageConfig(hidden=768, heads=12, ffn=3072, layers=3, seq=1024, micro_batch=8)


class _Block(nn.Module):
    def __init__(self, c: GPTStageConfig):
        super().__init__()
        self.c = c
        self.ln1 = nn.LayerNorm(c.hidden)
        self.qkv = nn.Linear(c.hidden, 3 * c.hidden)
        self.proj = nn.Linear(c.hidden, c.hidden)
        self.ln2 = nn.LayerNorm(c.hidden)
        self.up = nn.Linear(c.hidden, c.ffn)
        self.down = nn.Linear(c.ffn, c.hidden)

    def forward(self, x):
        b, s, h = x.shape
        q, k, v = self.qkv(self.ln1(x)).view(b, s, 3, self.c.heads, h // self.c.heads).unbind(2)
        a = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                           is_causal=True)
        x = x + self.proj(a.transpose(1, 2).reshape(b, s, h))
        return x + self.down(F.gelu(self.up(self.ln2(x)), approximate="tanh"))


class GPTStage(nn.Module):
    """One pipeline stage of a GPT-style decoder (bf16, AdamW), trained by microbatch."""

    def __init__(self, c: GPTStageConfig, seed: int = 0, device: str = "cuda"):
        super().__init__()
        torch.manual_seed(seed)
        self.c = c
        self.blocks = nn.ModuleList(_Block(c) for _ in range(c.layers))
        for n, p in self.named_parameters():
            if p.dim() > 1:
                nn.init.normal_(p, std=0.02)
        self.to(device=device, dtype=torch.bfloat16)
        self.opt = torch.optim.AdamW(self.parameters(), lr=1e-4, fused=True)
        self._saved: dict[int, tuple[torch.Tensor, torch.Tensor]] = {}
        self.offload: Optional[OptimizerOffload] = None

    def enable_optimizer_offload(self, h2d_gbs: float = 50.0, loan: bool = False) -> "OptimizerOffload":
        """Keep AdamW's moment estimates in pinned host memory between optimizer steps
        (PAPER.md:427): the bubbles before the step see that much more free HBM (with
        `loan`, lent to the fill executor set as `offload.borrower`)."""
        self.offload = OptimizerOffload(self.opt, h2d_gbs, loan=loan)
        return self.offload

    def forward_mb(self, mb: int, x: torch.Tensor) -> torch.Tensor:
        x = x.detach().requires_grad_(True)
        y = x
        for blk in self.blocks:
            y = blk(y)
        self._saved[mb] = (x, y)
        return y.detach()

    def backward_mb(self, mb: int, grad_out: Optional[torch.Tensor]) -> torch.Tensor:
        x, y = self._saved.pop(mb)
        if grad_out is None:  # last stage: scalar loss on the stage output
            loss = y.float().pow(2).mean()
            loss.backward()
            self.last_loss = loss.detach()
        else:
            y.backward(grad_out)
        return x.grad

    def step(self) -> None:
        if self.offload is not None:
            self.offload.wait_resident(torch.cuda.current_stream())
        self.opt.step()
        self.opt.zero_grad(set_to_none=False)
        if self.offload is not None:
            self.offload.evict(torch.cuda.current_stream())

    def snapshot(self) -> dict:
        """Device copies of parameters and the full optimizer state (to replay iterations)."""
        import copy

        if self.offload is not None and not self.offload.resident:  # moments back on the device
            self.offload.wait_resident(torch.cuda.current_stream())
        torch.cuda.synchronize()
        params = [p.detach().clone() for p in self.parameters()]
        return {"params": params, "opt": copy.deepcopy(self.opt.state_dict())}

    def restore(self, snap: dict) -> None:
        torch.cuda.synchronize()
        with torch.no_grad():
            for p, q in zip(self.parameters(), snap["params"]):
                p.copy_(q)
        self.opt.state.clear()
        # load a copy: load_state_dict keeps (does not copy) state tensors that already have
        # the parameter's dtype and device, so the optimizer would otherwise update the
        # snapshot in place and a second restore would replay a corrupted state
        import copy

        self.opt.load_state_dict(copy.deepcopy(snap["opt"]))
        self.opt.zero_grad(set_to_none=False)
        torch.cuda.synchronize()


def _pad256(n: int) -> int:
    return (n + 255) // 256 * 256


def loan_window_kinds(timeline, period_us: int, lead_us: int) -> set[int]:
    """StageEngine.loan_kinds on a steady-state timeline [(Instr, start_us, end_us)]."""
    compute = [(ins, st, en) for ins, st, en in timeline if ins.op != "BUBBLE"]
    step_end = max(en for _, _, en in compute)
    prefetch_at = min((st for _, st, _ in compute if st >= step_end - lead_us), default=step_end)
    copy_us = lead_us / 1.25
    inside, outside = set(), set()
    for ins, st, en in timeline:
        if ins.op != "BUBBLE":
            continue
        kind = 0 if ins.kind is BubbleKind.FWD_BWD else 1
        after_step = st >= step_end
        since_copy_out = st - step_end if after_step else st - (step_end - period_us)
        # the fill may wait for the copy-out for at most a tenth of the bubble
        ok = since_copy_out + 0.1 * (en - st) >= copy_us and (after_step or st < prefetch_at)
        (inside if ok else outside).add(kind)
    return inside - outside


class OptimizerOffload:
    """Main-job optimizer-state offload.

    Between optimizer steps AdamW's ``exp_avg`` / ``exp_avg_sq`` live in pinned host
    memory. After each step they are copied out on a side stream and their device
    blocks are released (``evict``). Before the next step they are copied back early
    enough that the transfer hides behind the last backward passes (``prefetch``, issued by
    ``StageEngine.run_iteration`` ``lead_us`` ahead of the step). The step waits for the
    copy-back (``wait_resident``). Copies are exact, so the main job's parameters and
    losses are bitwise those of a run without offload. The bubbles that fall between
    eviction and prefetch have ``state_bytes`` more free HBM.

    Loan mode (``loan=True``): the moments live in one device buffer (``device_buf``, the
    states are views of it) that is not freed but *lent* to a borrower (the fill
    ``Executor``) between the copy-out and the prefetch: ``borrower.lend(device_buf,
    evicted)`` after the step, ``borrower.revoke()`` before the copy-back, which waits on
    the event revoke returns. The fill's plans for the bubbles in that window get the
    buffer's bytes as extra free memory."""

    KEYS = ("exp_avg", "exp_avg_sq")

    def __init__(self, opt: torch.optim.Optimizer, h2d_gbs: float = 50.0, loan: bool = False):
        self.opt = opt
        self.stream = torch.cuda.Stream()
        self.host: dict[tuple[int, str], torch.Tensor] = {}
        self.h2d_gbs = h2d_gbs
        self._ready: Optional[torch.cuda.Event] = None
        self.resident = True  # states on the device (before the first step they do not exist)
        self.state_bytes = 0
        self.transfers = 0
        self.loan = loan
        self.borrower = None  # loan mode: object with lend(buf, ready_event) / revoke() -> event
        self.device_buf: Optional[torch.Tensor] = None
        self.host_buf: Optional[torch.Tensor] = None
        self._views: dict[tuple[int, str], torch.Tensor] = {}
        self._lent = False
        self.loans = 0

    def _adopt(self) -> None:
        """Loan mode: every moment becomes a view of `device_buf` (allocated at the first
        step; states replaced since -- restore(), load_state_dict -- are copied into their
        views on the current stream)."""
        specs = [(p, st, k) for p, st in self._states() for k in self.KEYS if st.get(k) is not None]
        if self.device_buf is None:
            total = sum(_pad256(st[k].numel() * st[k].element_size()) for _, st, k in specs)
            self.device_buf = torch.empty(total, dtype=torch.uint8, device=specs[0][0].device)
            self.host_buf = torch.empty(total, dtype=torch.uint8, pin_memory=True)
            off = 0
            for p, st, k in specs:
                t = st[k]
                nb = t.numel() * t.element_size()
                self._views[(id(p), k)] = self.device_buf[off:off + nb].view(t.dtype).view(t.shape)
                off += _pad256(nb)
        for p, st, k in specs:
            v = self._views[(id(p), k)]
            if st[k].data_ptr() != v.data_ptr():
                v.copy_(st[k])
                st[k] = v

    def _states(self):
        for group in self.opt.param_groups:
            for p in group["params"]:
                st = self.opt.state.get(p)
                if st:
                    yield p, st

    @property
    def lead_us(self) -> int:
        """How far ahead of the step the copy-back must start (1.25x its transfer time)."""
        return int(1.25 * self.state_bytes / (self.h2d_gbs * 1e3))

    def evict(self, main: torch.cuda.Stream) -> None:
        if self.loan:
            with torch.cuda.stream(main):
                self._adopt()
            ev = torch.cuda.Event()
            ev.record(main)
            self.stream.wait_event(ev)
            with torch.cuda.stream(self.stream):
                self.host_buf.copy_(self.device_buf, non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.stream)
            self.state_bytes = self.device_buf.numel()
            self.resident = False
            self._ready = None
            self.transfers += 1
            if self.borrower is not None:
                self.borrower.lend(self.device_buf, done)
                self._lent = True
                self.loans += 1
            return
        ev = torch.cuda.Event()
        ev.record(main)
        self.stream.wait_event(ev)
        nbytes = 0
        with torch.cuda.stream(self.stream):
            for p, st in self._states():
                for k in self.KEYS:
                    t = st.get(k)
                    if t is None:
                        continue
                    h = self.host.get((id(p), k))
                    if h is None:
                        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                        self.host[(id(p), k)] = h
                    h.copy_(t, non_blocking=True)
                    t.record_stream(self.stream)  # the block returns to the pool after the copy
                    st[k] = None
                    nbytes += t.numel() * t.element_size()
        self.state_bytes = nbytes
        self.resident = False
        self._ready = None
        self.transfers += 1

    def prefetch(self, after: Optional[torch.cuda.Stream] = None) -> None:
        """Copy the states back; with `after`, not before that stream's work enqueued so far
        (the host runs ahead of the device, so an unordered copy would start too early)."""
        if self.resident or self._ready is not None:
            return
        if after is not None:
            ev = torch.cuda.Event()
            ev.record(after)
            self.stream.wait_event(ev)
        if self.loan:
            if self._lent:  # the borrower's last use of the buffer comes first
                self.stream.wait_event(self.borrower.revoke())
                self._lent = False
            with torch.cuda.stream(self.stream):
                self.device_buf.copy_(self.host_buf, non_blocking=True)
                self._ready = torch.cuda.Event()
                self._ready.record(self.stream)
            self.transfers += 1
            return
        with torch.cuda.stream(self.stream):
            for p, st in self._states():
                for k in self.KEYS:
                    h = self.host.get((id(p), k))
                    if h is not None and st.get(k) is None:
                        st[k] = torch.empty(h.shape, dtype=h.dtype, device=p.device).copy_(h, non_blocking=True)
            self._ready = torch.cuda.Event()
            self._ready.record(self.stream)
        self.transfers += 1

    def wait_resident(self, main: torch.cuda.Stream) -> None:
        if self.resident:
            return
        self.prefetch()  # no-op when run_iteration already issued it
        main.wait_event(self._ready)
        if self.loan:
            self.resident = True
            return
        for _, st in self._states():
            for k in self.KEYS:
                if st.get(k) is not None:
                    st[k].record_stream(main)
        self.resident = True


# --------------------------------------------------------------------------- device helpers


class DeviceWords:
    """A small device u64 scratch (timestamps) + the stage's bubble flag."""

    def __init__(self, n_stamps: int = 8192):
        self.flag = ctypes.c_void_p()
        native.call("pf_flag_create", ctypes.byref(self.flag))
        self.stamps = torch.zeros(n_stamps, dtype=torch.int64, device="cuda")
        self.anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.n = 0

    def stamp_ptr(self, words: int = 1) -> int:
        if self.n + words > self.stamps.numel():
            raise RuntimeError("timestamp buffer full")
        p = self.stamps.data_ptr() + 8 * self.n
        self.n += words
        return p

    def close(self):
        native.call("pf_flag_destroy", self.flag)


@dataclass
class IterationRecord:
    iteration: int
    stage: int
    anchor_off_ns: int  # nominal iteration start relative to the anchor
    end_stamp: int  # index into stamps: end of the last main-job op
    anchor_stamp: int = -1  # index into stamps holding the anchor this iteration used
    epoch: int = 0  # stamp-buffer generation (stamp indices repeat after reset_stamps)
    bubbles: list[tuple[int, int, int]] = field(default_factory=list)  # (kind, set idx, clear idx)
    bubble_mem: list[tuple[int, int]] = field(default_factory=list)  # (kind, main-job bytes allocated)
    # per F/B op when the engine stamps ops: (op, mb, probe idx (3 words), end idx)
    ops: list[tuple[str, int, int, int]] = field(default_factory=list)
    resume: list[tuple[int, int]] = field(default_factory=list)  # (bubble clear idx, main resume idx)


# --------------------------------------------------------------------------- links


class TimerLink:
    """1-GPU stand-in for the neighbours: every recv completes at its arrival time
    in the analytic p-stage timeline (with measured t_fwd/t_bwd), anchored at a
    device timestamp. Activations/gradients are fixed synthetic tensors."""

    def __init__(self, words: DeviceWords, comm: torch.cuda.Stream):
        self.w = words
        self.comm = comm

    def wait_until(self, stream: torch.cuda.Stream, offset_ns: int) -> None:
        native.call("pf_wait_until", self.w.anchor.data_ptr(), int(offset_ns), None, stream.cuda_stream)

    def bubble_end(self, offset_ns: int, stamp: int) -> None:
        native.call("pf_flag_clear_at", self.w.flag, self.w.anchor.data_ptr(), int(offset_ns), stamp,
                    self.comm.cuda_stream)


# --------------------------------------------------------------------------- engine


class StageEngine:
    """Runs one stage's program iteration by iteration; BUBBLE hands the bubble to
    the executor (if any). Emulated-neighbour (TimerLink) version for 1 GPU."""

    def __init__(self, config: PipelineConfig, stage_id: int, model: GPTStage,
                 executor: Optional[Executor] = None,
                 streams: Optional[tuple[torch.cuda.Stream, torch.cuda.Stream]] = None):
        self.cfg = config
        self.stage = stage_id
        self.model = model
        self.executor = executor
        lo, hi = torch.cuda.Stream.priority_range()
        # engines that take turns on one GPU share (main, comm): the caching allocator
        # keeps blocks per stream, so per-engine streams would each pin a full set of
        # main-job activations
        if streams is None:
            streams = (torch.cuda.Stream(priority=hi), torch.cuda.Stream(priority=hi))
        self.main, self.comm = streams
        self.words = DeviceWords()
        self.link = TimerLink(self.words, self.comm)
        c = model.c
        g = torch.Generator(device="cuda").manual_seed(1234 + stage_id)
        shape = (c.micro_batch, c.seq, c.hidden)
        self.x_in = [torch.randn(shape, generator=g, device="cuda").to(torch.bfloat16) * 0.5
                     for _ in range(config.num_microbatches)]
        self.g_in = [torch.randn(shape, generator=g, device="cuda").to(torch.bfloat16) * 1e-3
                     for _ in range(config.num_microbatches)]
        self.main.wait_stream(torch.cuda.current_stream())  # inputs were made on the default stream
        self.last_stage = stage_id == config.num_stages - 1
        # one period from the first compute instruction (the idle head is the previous
        # fill-drain BUBBLE's tail)
        self.timeline = steady_state_timeline(config, stage_id)
        self.records: list[IterationRecord] = []
        self.outputs: list[torch.Tensor] = []
        self.launches = 0  # our kernels (timer / stamp / flag) enqueued by the engine
        self._anchor_stamp = -1
        self.epoch = 0
        # bubble probe (probe_bubbles): {bubble kind: ns} the main stream stays busy from the
        # bubble's start before its next instruction (PAPER.md:424's "wait" at the BUBBLE)
        self.probe_ns: dict[int, int] = {}
        # per-op stamps: every F/B is preceded by an SM-clock probe (start time, ns, cycles)
        # and followed by an end stamp; every BUBBLE by a main-stream stamp when the main job
        # resumes (the interference / yield-latency measurements)
        self.op_stamps = False
        # power-aware bubble tail: `throttle_ns` before each bubble's end the flag drops from 1
        # to `throttle_ctas` (pf_flag_throttle_at on the timer stream), so the fill's
        # cursor-claimed kernels run on that many CTAs and the board's power controller has
        # raised the SM clock when the main job resumes
        self.throttle_ns = 0
        self.throttle_ctas = 0
        self.throttle_min_ns = None  # bubbles shorter than this are not throttled (None: throttle_ns)
        self.throttle_frac = 1.0  # a bubble's throttled tail is at most this share of it
        self.short_ctas = 0  # bubbles not longer than throttle_min_ns run whole on this many CTAs (0: full)
        self.short_window_ns = None  # ... or only their last short_window_ns
        self.timer = torch.cuda.Stream(priority=hi)

    def set_anchor(self, lead_ms: float = 5.0) -> None:
        """Anchor = device time now + lead (host enqueues ahead within the lead)."""
        with torch.cuda.stream(self.main):
            native.call("pf_read_globaltimer", self.words.anchor.data_ptr(), self.main.cuda_stream)
            self.words.anchor.add_(int(lead_ms * 1e6))
            self._anchor_stamp = self.words.n
            self.words.stamps[self.words.n:self.words.n + 1].copy_(self.words.anchor)
            self.words.n += 1
        self.launches += 1
        self.comm.wait_stream(self.main)

    def run_iteration(self, it: int, fill: bool, keep_outputs: bool = False) -> IterationRecord:
        cfg = self.cfg
        base = it * cfg.period_us * US
        rec = IterationRecord(it, self.stage, base, -1, self._anchor_stamp, self.epoch)
        prev_end_us = None
        main, comm = self.main, self.comm
        flag = self.words.flag.value
        step_end_us = max(e for ins, _, e in self.timeline if ins.op != "BUBBLE")
        for ins, start_us, end_us in self.timeline:
            if ins.op == "BUBBLE":
                ev = torch.cuda.Event()
                ev.record(main)
                comm.wait_event(ev)
                set_idx = self.words.n
                native.call("pf_flag_write_on_stream", flag, 1, comm.cuda_stream)
                native.call("pf_read_globaltimer", self.words.stamp_ptr(), comm.cuda_stream)
                start_ev = torch.cuda.Event()
                start_ev.record(comm)
                clear_idx = self.words.n
                tail, ctas = _throttle_tail(self, (end_us - start_us) * US)
                if fill and tail > 0:
                    # the bubble's last `tail` ns run throttled
                    self.timer.wait_event(start_ev)
                    native.call("pf_flag_throttle_at", flag, self.words.anchor.data_ptr(),
                                int(base + end_us * US - tail), int(ctas), self.timer.cuda_stream)
                    self.launches += 1
                self.link.bubble_end(base + end_us * US, self.words.stamp_ptr())
                end_ev = torch.cuda.Event()
                end_ev.record(comm)
                self.launches += 3
                kind = 0 if ins.kind is BubbleKind.FWD_BWD else 1
                rec.bubbles.append((kind, set_idx, clear_idx))
                # the main job's allocated bytes while the bubble is open (the allocator
                # tracks tensors in enqueue order, which is the order they live on the device)
                rec.bubble_mem.append((kind, torch.cuda.memory_allocated()))
                if fill and self.executor is not None:
                    self.executor.fill(BubbleSlot(kind, start_ev, flag, tag=self._tag(clear_idx)))
                if kind in self.probe_ns:  # probe: the main job "waits" w ns into the bubble
                    main.wait_event(start_ev)
                    native.call("pf_wait_until", self.words.stamps.data_ptr() + 8 * set_idx,
                                int(self.probe_ns[kind]), None, main.cuda_stream)
                    self.launches += 1
                main.wait_event(end_ev)
                if self.op_stamps:
                    ri = self.words.n
                    native.call("pf_read_globaltimer", self.words.stamp_ptr(), main.cuda_stream)
                    rec.resume.append((clear_idx, ri))
                    self.launches += 1
                prev_end_us = end_us
                continue
            off = self.model.offload
            if off is not None and not off.resident and start_us >= step_end_us - off.lead_us:
                off.prefetch(after=main)  # optimizer states back in time for the step
            # F / B: wait for the (emulated) recv if the schedule idles before it
            if prev_end_us is None or start_us > prev_end_us:
                self.link.wait_until(main, base + start_us * US)
                self.launches += 1
            with torch.cuda.stream(main):
                if self.op_stamps:
                    pi = self.words.n
                    native.call("pf_sm_clock_probe", self.words.stamp_ptr(3), OP_PROBE_NS, main.cuda_stream)
                    self.launches += 1
                if ins.op == "F":
                    y = self.model.forward_mb(ins.mb, self.x_in[ins.mb])
                    if keep_outputs:
                        self.outputs.append(y)
                else:
                    self.model.backward_mb(ins.mb, None if self.last_stage else self.g_in[ins.mb])
                if ins == self._last_compute():
                    self.model.step()
                    rec.end_stamp = self.words.n
                    native.call("pf_read_globaltimer", self.words.stamp_ptr(), main.cuda_stream)
                    self.launches += 1
                if self.op_stamps:
                    ei = rec.end_stamp if ins == self._last_compute() else self.words.n
                    if ei != rec.end_stamp:
                        native.call("pf_read_globaltimer", self.words.stamp_ptr(), main.cuda_stream)
                        self.launches += 1
                    rec.ops.append((ins.op, ins.mb, pi, ei))
            prev_end_us = end_us
        self.records.append(rec)
        return rec

    def loan_kinds(self) -> set[int]:
        """Bubble kinds (0 fwd-bwd, 1 fill-drain) whose every bubble falls inside the
        optimizer-state loan window of this stage's iteration: from the end of the copy-out
        after the step (`lead_us` / 1.25 after it, the transfer time) to the copy-back, which
        run_iteration issues `lead_us` ahead of the step. A bubble that opens more than a tenth
        of its length before the copy-out ends is outside: the fill would wait for the copy
        (DESIGN.md §3.3)."""
        off = self.model.offload
        if off is None or not off.loan or not off.state_bytes:
            return set()
        return loan_window_kinds(self.timeline, self.cfg.period_us, off.lead_us)

    def _last_compute(self) -> Instr:
        return [ins for ins, _, _ in self.timeline if ins.op != "BUBBLE"][-1]

    def record_timing(self, rec: IterationRecord) -> dict:
        """Device timestamps of one iteration (ns): nominal start, main-job end, and
        every bubble's (kind, flag set, flag cleared)."""
        torch.cuda.synchronize()
        st = self.words.stamps
        start = int(st[rec.anchor_stamp]) + rec.anchor_off_ns
        end = int(st[rec.end_stamp])
        bubbles = [(kind, int(st[si]), int(st[ci]), (id(self), rec.epoch, ci)) for kind, si, ci in rec.bubbles]
        last = max([end] + [b[2] for b in bubbles])
        out = {"start": start, "main_end": end, "step_end": last, "bubbles": bubbles}
        if rec.ops:
            out.update(op_timing(st, rec))
        return out

    def reset_stamps(self) -> None:
        torch.cuda.synchronize()
        self.words.n = 0
        self.records = []
        self.epoch += 1

    def _tag(self, clear_idx: int) -> tuple:
        """Unique id of a bubble: (engine, stamp-buffer generation, stamp index)."""
        return (id(self), self.epoch, clear_idx)


OP_PROBE_NS = 4000  # SM-clock probe before every stamped op (4 us of one thread)


def _throttle_tail(engine, duration_ns: int) -> tuple[int, int]:
    """(throttled tail in ns, CTAs) of a bubble of `duration_ns`: min(throttle_ns,
    throttle_frac x duration) on throttle_ctas for bubbles longer than throttle_min_ns
    (default: throttle_ns); shorter bubbles run whole on short_ctas when that is set (too
    short for an idle tail to let the clock recover), else unthrottled."""
    if engine.throttle_ns <= 0 or engine.throttle_ctas < 2 or duration_ns <= 0:
        return 0, 0
    lo = engine.throttle_ns if engine.throttle_min_ns is None else engine.throttle_min_ns
    if duration_ns <= lo:
        short = getattr(engine, "short_ctas", 0)
        window = getattr(engine, "short_window_ns", None)
        span = int(duration_ns) if window is None else int(min(duration_ns, window))
        return (span, short) if short >= 2 else (0, 0)
    return int(min(engine.throttle_ns, engine.throttle_frac * duration_ns)), engine.throttle_ctas


def op_timing(st: torch.Tensor, rec: IterationRecord) -> dict:
    """Per-op device timing of a stamped iteration: [(op, mb, start ns, end ns, SM MHz)]
    and, per BUBBLE, the main stream's resume delay after the flag cleared (ns)."""
    ops = []
    for op, mb, pi, ei in rec.ops:
        t0, dt, cyc = int(st[pi]), int(st[pi + 1]), int(st[pi + 2])
        ops.append((op, mb, t0 + dt, int(st[ei]), cyc * 1e3 / dt if dt > 0 else 0.0))
    resume = [int(st[ri]) - int(st[ci]) for ci, ri in rec.resume]
    return {"ops": ops, "resume_ns": resume}


def warm_up_gpu(ms: float = 1500.0) -> None:
    """Keep the tensor cores busy for ~ms so the SM clock leaves its idle state before any
    timing is taken (a fresh box starts at 120 MHz; measure_stage_times after 2 short reps
    under-measured t_fwd/t_bwd by up to 28 %)."""
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    while True:
        for _ in range(20):
            a = (a @ a).mul_(1e-4)
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record()
        t1.synchronize()
        if t0.elapsed_time(t1) >= ms:
            break
    del a


def measure_stage_times(model: GPTStage, reps: int = 7, warmup: int = 3,
                        warm_ms: float = 1500.0) -> tuple[float, float]:
    """t_fwd / t_bwd of one microbatch on this stage (ms, CUDA events): the
    per-stage timings PipelineConfig takes (pipeline.py:48-97). The GPU is warmed up
    first; the medians of `reps` back-to-back repetitions are returned."""
    if warm_ms > 0:
        warm_up_gpu(warm_ms)
    c = model.c
    x = (torch.randn(c.micro_batch, c.seq, c.hidden, device="cuda") * 0.5).to(torch.bfloat16)
    g = (torch.randn(c.micro_batch, c.seq, c.hidden, device="cuda") * 1e-3).to(torch.bfloat16)
    tf, tb = [], []
    for i in range(warmup + reps):
        a, b, d = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a.record()
        model.forward_mb(0, x)
        b.record()
        model.backward_mb(0, g)
        d.record()
        torch.cuda.synchronize()
        if i >= warmup:
            tf.append(a.elapsed_time(b))
            tb.append(b.elapsed_time(d))
    model.opt.zero_grad(set_to_none=False)
    tf.sort()
    tb.sort()
    return tf[len(tf) // 2], tb[len(tb) // 2]


# --------------------------------------------------------------------------- real pipeline


class NcclPipelineEngine:
    """One rank = one pipeline stage of a real p-stage pipeline (world == p).

    Activations flow s -> s+1 and gradients s+1 -> s over NCCL P2P
    (torch.distributed, NVLink/NVSwitch). Forward and backward traffic use two
    separate process groups, so a pending send in one direction can never block
    a recv in the other (1F1B sends and receives between the same pair in both
    directions). Each op is posted just in time on the comm stream; the main
    stream waits on the recv through an event.

    BUBBLE: the comm stream writes flag=1, records the bubble-start event for the
    fill stream, then waits on the recv that ends the bubble (the first backward's
    gradient, or the next iteration's first activation) and writes flag=0 — the
    recv completion clears the flag."""

    def __init__(self, config: PipelineConfig, model: GPTStage, executor: Optional[Executor] = None,
                 groups=None):
        import torch.distributed as dist

        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        if self.world != config.num_stages:
            raise ValueError(f"real pipeline needs one rank per stage ({config.num_stages}), got {self.world}")
        self.cfg = config
        self.stage = self.rank
        self.model = model
        self.executor = executor
        if groups is None:
            groups = (dist.new_group(list(range(self.world))), dist.new_group(list(range(self.world))))
        self.g_fwd, self.g_bwd = groups
        lo, hi = torch.cuda.Stream.priority_range()
        self.main = torch.cuda.Stream(priority=hi)
        self.comm = torch.cuda.Stream(priority=hi)
        self.words = DeviceWords()
        c = model.c
        self.shape = (c.micro_batch, c.seq, c.hidden)
        g = torch.Generator(device="cuda").manual_seed(4321)
        m = config.num_microbatches
        self.x_first = [torch.randn(self.shape, generator=g, device="cuda").to(torch.bfloat16) * 0.5
                        for _ in range(m)] if self.stage == 0 else None
        self.main.wait_stream(torch.cuda.current_stream())
        self.last_stage = self.stage == self.world - 1
        self.prog = stage_program(config, self.stage)
        self.records: list[IterationRecord] = []
        self.launches = 0
        self.losses: list[torch.Tensor] = []
        self._inflight: list = []  # (work, tensor) kept alive until the iteration is synced
        self._prefetched: Optional[tuple[torch.Tensor, torch.cuda.Event]] = None
        self._anchor_stamp = -1
        self.epoch = 0
        # power-aware bubble tail (StageEngine.throttle_ns): the recv's completion time is not
        # known in advance here, so the throttle deadline is the bubble's start stamp plus its
        # measured duration (expected_ns, from the fill-off characterization) minus throttle_ns
        self.throttle_ns = 0
        self.throttle_ctas = 0
        self.throttle_min_ns = None
        self.throttle_frac = 1.0
        self.short_ctas = 0
        self.short_window_ns = None
        self.expected_ns: dict[int, int] = {}
        self.timer = torch.cuda.Stream(priority=hi)

    # ---- P2P helpers (comm stream) ------------------------------------------------
    def _recv(self, src: int, group) -> tuple[torch.Tensor, torch.cuda.Event]:
        with torch.cuda.stream(self.comm):
            # allocated on the comm stream, so anything the allocator does to the block
            # (deterministic mode fills new memory) is ordered before NCCL's recv into it
            buf = torch.empty(self.shape, dtype=torch.bfloat16, device="cuda")
            buf.record_stream(self.main)  # consumed on the main stream after `ev`
            work = self.dist.irecv(buf, src, group=group)
            work.wait()  # comm stream waits for the NCCL recv
            ev = torch.cuda.Event()
            ev.record(self.comm)
        self._inflight.append((work, buf))
        return buf, ev

    def _send(self, t: torch.Tensor, dst: int, group) -> None:
        ev = torch.cuda.Event()
        ev.record(self.main)
        with torch.cuda.stream(self.comm):
            self.comm.wait_event(ev)
            work = self.dist.isend(t, dst, group=group)
        self._inflight.append((work, t))

    def _bubble(self, kind: BubbleKind, end_recv: Optional[tuple[int, object]], fill: bool,
                rec: IterationRecord) -> Optional[tuple[torch.Tensor, torch.cuda.Event]]:
        """BUBBLE instruction: flag up, hand the bubble to the executor, end it with the recv."""
        flag = self.words.flag.value
        ev = torch.cuda.Event()
        ev.record(self.main)
        self.comm.wait_event(ev)
        set_idx = self.words.n
        native.call("pf_flag_write_on_stream", flag, 1, self.comm.cuda_stream)
        native.call("pf_read_globaltimer", self.words.stamp_ptr(), self.comm.cuda_stream)
        start_ev = torch.cuda.Event()
        start_ev.record(self.comm)
        k = 0 if kind is BubbleKind.FWD_BWD else 1
        exp = self.expected_ns.get(k, 0)
        tail, ctas = _throttle_tail(self, exp)
        if fill and tail > 0:
            self.timer.wait_event(start_ev)
            native.call("pf_flag_throttle_at", flag, self.words.stamps.data_ptr() + 8 * set_idx,
                        int(exp - tail), int(ctas), self.timer.cuda_stream)
            self.launches += 1
        got = None
        if end_recv is not None:
            got = self._recv(*end_recv)
        clear_idx = self.words.n
        native.call("pf_flag_write_on_stream", flag, 0, self.comm.cuda_stream)
        native.call("pf_read_globaltimer", self.words.stamp_ptr(), self.comm.cuda_stream)
        end_ev = torch.cuda.Event()
        end_ev.record(self.comm)
        self.launches += 2
        rec.bubbles.append((k, set_idx, clear_idx))
        rec.bubble_mem.append((k, torch.cuda.memory_allocated()))
        if fill and self.executor is not None:
            self.executor.fill(BubbleSlot(k, start_ev, flag, tag=self._tag(clear_idx)))
        self.main.wait_event(end_ev)
        return got

    def set_anchor(self) -> None:
        with torch.cuda.stream(self.main):
            self._anchor_stamp = self.words.n
            native.call("pf_read_globaltimer", self.words.stamp_ptr(), self.main.cuda_stream)
        self.launches += 1

    def run_iteration(self, it: int, fill: bool, last: bool = False) -> IterationRecord:
        """One training iteration of this stage; `last` = no next iteration (no
        trailing fill-drain bubble, whose end would be the next iteration's recv)."""
        s, p = self.stage, self.world
        rec = IterationRecord(it, s, 0, -1, self._anchor_stamp, self.epoch)
        pending_grad: dict[int, tuple[torch.Tensor, torch.cuda.Event]] = {}
        for idx, ins in enumerate(self.prog):
            if ins.op == "BUBBLE":
                if ins.kind is BubbleKind.FWD_BWD:
                    nxt = self.prog[idx + 1]  # the first backward: its gradient ends the bubble
                    got = self._bubble(ins.kind, (s + 1, self.g_bwd) if not self.last_stage else None,
                                       fill, rec)
                    if got is not None:
                        pending_grad[nxt.mb] = got
                else:
                    if last or s == 0:
                        continue
                    got = self._bubble(ins.kind, (s - 1, self.g_fwd), fill, rec)
                    self._prefetched = got
                continue
            with torch.cuda.stream(self.main):
                if ins.op == "F":
                    if s == 0:
                        x = self.x_first[ins.mb]
                    else:
                        if ins.mb == 0 and self._prefetched is not None:
                            x, ev = self._prefetched
                            self._prefetched = None
                        else:
                            x, ev = self._recv(s - 1, self.g_fwd)
                        self.main.wait_event(ev)
                    y = self.model.forward_mb(ins.mb, x)
                    if not self.last_stage:
                        self._send(y, s + 1, self.g_fwd)
                else:
                    g = None
                    if not self.last_stage:
                        g, ev = pending_grad.pop(ins.mb, None) or self._recv(s + 1, self.g_bwd)
                        self.main.wait_event(ev)
                    gin = self.model.backward_mb(ins.mb, g)
                    if self.last_stage:
                        self.losses.append(self.model.last_loss)
                    if s > 0:
                        self._send(gin, s - 1, self.g_bwd)
                    if ins == [i for i in self.prog if i.op != "BUBBLE"][-1]:
                        self.model.step()
                        rec.end_stamp = self.words.n
                        native.call("pf_read_globaltimer", self.words.stamp_ptr(), self.main.cuda_stream)
                        self.launches += 1
        self.records.append(rec)
        return rec

    def sync(self) -> None:
        torch.cuda.synchronize()
        self._inflight = []

    def record_timing(self, rec: IterationRecord) -> dict:
        self.sync()
        st = self.words.stamps
        start = int(st[rec.anchor_stamp])
        end = int(st[rec.end_stamp])
        bubbles = [(kind, int(st[si]), int(st[ci]), (id(self), rec.epoch, ci)) for kind, si, ci in rec.bubbles]
        last = max([end] + [b[2] for b in bubbles])
        return {"start": start, "main_end": end, "step_end": last, "bubbles": bubbles,
                "stage": self.stage}

    def reset_stamps(self) -> None:
        self.sync()
        self.words.n = 0
        self.records = []
        self.epoch += 1

    def _tag(self, clear_idx: int) -> tuple:
        return (id(self), self.epoch, clear_idx)


# --------------------------------------------------------------------------- characterization


def characterize_bubbles(stage_id: int, timings: list[dict], records: list[IterationRecord],
                         fill_fraction: float, total_bytes: int, reserve_bytes: int = 2 << 30,
                         analytic=None):
    """Bubble characterization from measured iterations: the paper
    probes each bubble's duration with a doubling wait and reads memory_allocated();
    here every BUBBLE instruction already stamps its start (flag set) and its end (recv
    completion, flag cleared) on the device, so the durations are read directly, and the
    main job's allocated bytes at each BUBBLE instruction give its free memory.

    `timings` are engine.record_timing dicts of fill-off iterations and `records` the
    matching IterationRecords. Returns (BubbleCycle, report) -- the cycle uses the
    reference's usable-time rule (schedule.cycle_from_measurements)."""
    import statistics

    from .schedule import cycle_from_measurements

    durs = {0: [], 1: []}
    for t in timings:
        for kind, t_set, t_clr, _ in t["bubbles"]:
            durs[kind].append((t_clr - t_set) // 1000)
    mem = {0: [], 1: []}
    for r in records:
        for kind, alloc in r.bubble_mem:
            mem[kind].append(alloc)
    periods = [t["main_end"] - t["start"] for t in timings]
    period_us = int(statistics.median(periods) // 1000) if periods else 0
    d = [int(statistics.median(durs[k])) if durs[k] else 0 for k in (0, 1)]
    free = [max(0, total_bytes - (max(mem[k]) if mem[k] else 0) - reserve_bytes) for k in (0, 1)]
    unfill = 0
    if analytic is not None:
        unfill = max(0, min(analytic.unfillable_us, period_us - sum(d)))
    cycle = cycle_from_measurements(stage_id, max(period_us, sum(d)), d, free, fill_fraction, unfillable_us=unfill)
    report = {"measured_bubbles_us": d, "measured_period_us": period_us,
              "bubble_samples": {str(k): len(durs[k]) for k in (0, 1)},
              "main_job_allocated_bytes": [max(mem[k]) if mem[k] else 0 for k in (0, 1)],
              "free_mem_bytes": free}
    if analytic is not None:
        report.update({"analytic_bubbles_us": [b.duration_us for b in analytic.bubbles],
                       "analytic_period_us": analytic.period_us})
    return cycle, report


def probe_bubbles(engine: "StageEngine", start_ms: float = 1.0, tol_ms: float = 0.5, refine: int = 6,
                  iterations: int = 2) -> dict:
    """The paper's bubble-duration probe: at every BUBBLE instruction of one
    kind the main job waits w before proceeding; while its iteration time is unaffected the
    wait doubles, then the largest unaffected w is refined by bisection. Returns
    {"probed_us": [fwd_bwd, fill_drain], "base_iteration_us": ..., "probes": n}.

    "Unaffected" = the main-job time of `iterations` back-to-back iterations from one anchor
    grows by at most tol_ms (the fill-drain bubble wraps into the next iteration, so one
    iteration alone would not see it). The direct measurement (flag stamps,
    characterize_bubbles) is what the bench uses; this probe is the paper's method, kept to
    cross-check it (tests/test_executor_gpu.py)."""
    calls = [0]

    def run(probe: dict) -> int:
        engine.probe_ns = dict(probe)
        engine.reset_stamps()
        engine.set_anchor()
        recs = [engine.run_iteration(i, fill=False) for i in range(iterations)]
        t0 = engine.record_timing(recs[0])
        t1 = engine.record_timing(recs[-1])
        engine.probe_ns = {}
        calls[0] += 1
        return t1["main_end"] - t0["start"]

    run({})  # warm-up
    base_runs = [run({}) for _ in range(3)]
    base = min(base_runs)
    # the decision threshold is at least twice the run-to-run spread of the unprobed
    # iterations and 1 % of their time, and every probe is the min of two runs (clock noise
    # only adds time). The 1 %: a spinning wait kernel in a bubble keeps the board out of its
    # idle power state, which moves the power-capped SM clock of the next ops
    tol = max(int(tol_ms * 1e6), 2 * (max(base_runs) - base), base // 100)

    def slowed(probe: dict) -> bool:
        return min(run(probe), run(probe)) > base + tol
    kinds_present = {ins.kind for ins, s, e in engine.timeline if ins.op == "BUBBLE" and e > s}
    period_ns = engine.cfg.period_us * US
    out = []
    for kind in (BubbleKind.FWD_BWD, BubbleKind.FILL_DRAIN):
        k = 0 if kind is BubbleKind.FWD_BWD else 1
        if kind not in kinds_present:
            out.append(0)
            continue
        ok, w = 0, int(start_ms * 1e6)
        while w <= period_ns and not slowed({k: w}):
            ok, w = w, 2 * w
        lo, hi = ok, w
        for _ in range(refine):
            mid = (lo + hi) // 2
            if not slowed({k: mid}):
                lo = mid
            else:
                hi = mid
        out.append(lo // 1000)
    return {"probed_us": out, "base_iteration_us": base // 1000, "probes": calls[0], "tol_us": tol // 1000}


def characterize_stage(engine: "StageEngine", iterations: int = 3, fill_fraction: float = 0.68,
                       reserve_bytes: int = 2 << 30):
    """Run `iterations` fill-off iterations of an emulated stage and characterize its bubbles.

    The report also carries the stage's in-situ op timing (per-op stamps): the medians of its
    own forward / backward durations inside the iterations, and `expected_bubbles_us` -- the
    neighbour's (analytic) arrival minus the measured end of the stage's own op before the
    BUBBLE. A stage that computes faster or slower than measure_stage_times said reaches its
    BUBBLE earlier or later, and the measured bubble grows or shrinks by exactly that drift."""
    import statistics

    from .schedule import build_bubble_cycle

    timings, records = [], []
    stamped = engine.op_stamps
    engine.op_stamps = True
    try:
        for k in range(iterations + 1):  # the first iteration warms the main job up (discarded)
            engine.reset_stamps()
            engine.set_anchor()
            rec = engine.run_iteration(0, fill=False)
            t = engine.record_timing(rec)
            if k:
                timings.append(t)
                records.append(rec)
    finally:
        engine.op_stamps = stamped
    _, total = torch.cuda.mem_get_info()
    cycle, rep = characterize_bubbles(engine.stage, timings, records, fill_fraction, total, reserve_bytes,
                                      analytic=build_bubble_cycle(engine.cfg, engine.stage))
    fwd = [(t1 - t0) / 1e6 for t in timings for op, _, t0, t1, _ in t["ops"] if op == "F"]
    bwd = [(t1 - t0) / 1e6 for t in timings for op, _, t0, t1, _ in t["ops"] if op == "B"]
    rep["insitu_t_fwd_ms"] = statistics.median(fwd) if fwd else None
    rep["insitu_t_bwd_ms"] = statistics.median(bwd) if bwd else None
    rep["sm_mhz"] = statistics.median(m for t in timings for *_, m in t["ops"]) if timings else None
    # expected bubble durations from the stage's own stamps
    tl = engine.timeline
    exp = {0: [], 1: []}
    for t in timings:
        ends = [t1 for _, _, _, t1, _ in t["ops"]]
        k_op = -1
        b_i = 0
        for ins, s_us, e_us in tl:
            if ins.op == "BUBBLE":
                if b_i < len(t["bubbles"]):
                    kind, t_set, t_clr, _ = t["bubbles"][b_i]
                    own_ready = ends[k_op] if k_op >= 0 else t["start"]
                    exp[kind].append(max(0, t["start"] + e_us * US - own_ready) // 1000)
                b_i += 1
            else:
                k_op += 1
    rep["expected_bubbles_us"] = [int(statistics.median(exp[k])) if exp[k] else 0 for k in (0, 1)]
    return cycle, rep
