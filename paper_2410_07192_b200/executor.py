"""The fill-job Executor: runs a Coordinator WorkItem inside a stage's bubbles on B200.

Reference counterpart: the time model ``ExecutionPlan.range_wall_us /
range_busy_us`` (pkg/src/bubblefill/partition.py:118-132) consumed by the
simulator's dispatch loop (pkg/src/bubblefill/sim.py:222-235), and the paper's
Executor process. Here the plan is executed for real:

* partitions run in order; partition ``[lo, hi)`` of the fill model's
  nn.Sequential runs ``per_bubble[j].num_batches`` batches of
  ``per_bubble[j].batch_size`` samples in bubble j of every cycle until all of the
  range's samples passed through it (the reference's partition-major order);
* every kernel is launched on a low-priority fill stream behind the bubble's
  start event and polls the stage's bubble flag at tile granularity, so the
  work yields within one tile of the main job's recv completing;
* a yielded batch is resumed at its first incomplete kernel in the next bubble
  (tile cursor for GEMMs, whole-node re-run for idempotent nodes);
* weights of the next partition are staged host->HBM with pinned copies on a
  side stream while the main job computes; activations between partitions are
  offloaded to pinned host memory and reloaded;
* everything lives in a fixed arena sized from the measured bubble free memory,
  so the fill job cannot allocate past it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from . import native
from .arena import Arena, PinnedBuffer, device_view
from .coordinator import WorkItem
from .fillmodels import ATOMIC, ExecContext, FillSequential, synthetic_ids
from .planner import ExecutionPlan

MAX_NODES = 4096  # cursor slots in the control block (24-layer BERT-large: 1 + 24*7 + copies)
_CTL_WORDS = 64 + MAX_NODES  # [0]=abort, [1]=batches done, [8..16)=timestamps(u64), [64..)=cursors


@dataclass
class BubbleSlot:
    """One upcoming bubble as the engine announces it to the executor."""

    index: int  # bubble position j in the stage's cycle (0 = fwd-bwd, 1 = fill-drain)
    start_event: Optional[torch.cuda.Event]  # fill stream waits for it (flag already set)
    flag_ptr: int  # device address of the stage's bubble flag (0 = not preemptible)


@dataclass
class BubbleRecord:
    index: int
    batches_planned: int
    batches_done: int
    samples_done: int
    aborted: bool
    fill_start_ns: int = 0
    fill_end_ns: int = 0
    launches: int = 0


@dataclass
class _Progress:
    part: int = 0
    next_sample: int = 0  # next sample (0-based within the range) for this partition
    resume: Optional[tuple[int, int, int]] = None  # (first sample, count, node) of a yielded batch
    resume_zero: Optional[int] = None  # atomic node whose cursor must be reset before the resume
    finished: bool = False


@dataclass
class _Pending:
    slot: BubbleSlot
    batches: list[tuple[int, int, int]]  # (first sample, count, start node)
    end_event: torch.cuda.Event
    launches: int
    has_resume: bool = False


class Executor:
    """One per GPU (pipeline-stage worker). Not thread-safe; driven by the engine."""

    def __init__(self, arena_bytes: int, *, priority: int = 1, job_seed: int = 0):
        native.require_device()
        self.arena = Arena(arena_bytes)
        lo_prio, hi_prio = torch.cuda.Stream.priority_range()
        # fill work on the LOWEST priority; staging on its own stream
        self.stream = torch.cuda.Stream(priority=hi_prio if priority == 0 else lo_prio)
        self.copy_stream = torch.cuda.Stream(priority=lo_prio)
        self.job_seed = job_seed
        self.item: Optional[WorkItem] = None
        self.model: Optional[FillSequential] = None
        self.plan: Optional[ExecutionPlan] = None
        self.progress = _Progress()
        self.pending: Optional[_Pending] = None
        self.records: list[BubbleRecord] = []
        self.samples_completed = 0  # samples through the LAST partition, all items
        self.kernel_launches = 0
        self._ctl_host = PinnedBuffer((_CTL_WORDS,), torch.int32)
        self._staged_part: Optional[int] = None
        self._staged_event: Optional[torch.cuda.Event] = None
        self._results: Optional[PinnedBuffer] = None
        self._offload: Optional[PinnedBuffer] = None
        self._ids_host: Optional[PinnedBuffer] = None

    # ------------------------------------------------------------------ loading

    def load(self, item: WorkItem, model: FillSequential) -> None:
        """Take a new WorkItem. `item.reuse` (same job as the previous item,
        PAPER.md:47) keeps the staged executable and arena layout."""
        if self.pending is not None:
            self.settle()
        same = (item.reuse and self.model is model and self.plan is item.plan)
        self.item, self.model, self.plan = item, model, item.plan
        self.progress = _Progress()
        n = item.entry.size
        cfg = model.cfg
        if not same:
            self._layout()
        # per-range host buffers: inputs, results, inter-partition activations
        self._ids_host = PinnedBuffer((n, cfg.seq), torch.int32)
        self._ids_host.tensor.copy_(synthetic_ids(self.job_seed, item.entry.lo - 1, n, cfg.seq, cfg.vocab))
        self._results = PinnedBuffer((n, cfg.hidden), torch.bfloat16)
        self._offload = (PinnedBuffer((n, cfg.seq, cfg.hidden), torch.bfloat16)
                         if len(self.plan.partitions) > 1 else None)
        if not same or self._staged_part != 0:
            self._stage_partition(0)

    def _layout(self) -> None:
        """Carve the arena: control block | weights (largest partition) | workspace."""
        plan, model = self.plan, self.model
        self.arena.reset()
        self._ctl = self.arena.alloc((_CTL_WORDS,), torch.int32)
        self._ctl.zero_()
        max_w = max(sum(_pad256(model[i].weight_bytes()) for i in range(p.lo, p.hi))
                    for p in plan.partitions)
        self._wmark = self.arena.mark()
        self._wregion = self.arena.alloc((max_w // 2,), torch.bfloat16)
        bmax = max(e.batch_size for p in plan.partitions for e in p.per_bubble)
        cfg = model.cfg
        need = {}
        for p in plan.partitions:
            for k, v in model.workspace(p.lo, p.hi, bmax).items():
                need[k] = max(need.get(k, 0), v)
        need["hidden"] = bmax * cfg.seq * cfg.hidden
        need["cls"] = bmax * cfg.hidden
        self.ws = {k: self.arena.alloc((v,), torch.bfloat16) for k, v in need.items()}
        self.ids_dev = self.arena.alloc((bmax, cfg.seq), torch.int32)
        self._staged_part = None

    def _stage_partition(self, part: int) -> None:
        """Stage partition `part`'s weights into the weight region on the copy stream."""
        p = self.plan.partitions[part]
        ptr = self._wregion.data_ptr()
        with torch.cuda.stream(self.copy_stream):
            if self._staged_event is not None:
                self.copy_stream.wait_event(self._staged_event)
            self.copy_stream.wait_stream(self.stream)  # previous partition's kernels are done
            for i in range(p.lo, p.hi):
                mod = self.model[i]
                nbytes = mod.weight_bytes()
                dflat = device_view(ptr, (nbytes // 2,), torch.bfloat16)
                native.call("pf_stage_h2d", ptr, mod.host.ptr, nbytes, self.copy_stream.cuda_stream)
                off = 0
                mod.dev = {}
                for name, shape, _ in mod.param_specs():
                    nel = 1
                    for s in shape:
                        nel *= s
                    mod.dev[name] = dflat[off:off + nel].view(*shape)
                    off += nel
                ptr += _pad256(nbytes)
        ev = torch.cuda.Event()
        ev.record(self.copy_stream)
        self._staged_event = ev
        self._staged_part = part

    # ------------------------------------------------------------------ bubbles

    @property
    def busy(self) -> bool:
        return self.item is not None and not self.progress.finished

    def fill(self, slot: BubbleSlot) -> Optional[BubbleRecord]:
        """Enqueue this bubble's planned batches (asynchronously). The previous
        bubble is settled first. Returns the settled record of the previous bubble."""
        prev = self.settle() if self.pending is not None else None
        if not self.busy:
            return prev
        pr = self.progress
        part = self.plan.partitions[pr.part]
        entry = part.per_bubble[slot.index] if slot.index < len(part.per_bubble) else None
        n_total = self.item.entry.size
        batches: list[tuple[int, int, int]] = []
        if pr.resume is not None:
            batches.append(pr.resume)
        if entry is not None and entry.num_batches > 0:
            start = pr.next_sample
            for _ in range(entry.num_batches - (1 if pr.resume is not None else 0)):
                if start >= n_total:
                    break
                cnt = min(entry.batch_size, n_total - start)
                batches.append((start, cnt, 0))
                start += cnt
        if not batches:
            return prev
        st = self.stream
        ctl = self._ctl
        base = ctl.data_ptr()
        abort_ptr, done_ptr = base, base + 4
        t_start, t_end = base + 32, base + 40
        cursors = base + 4 * 64
        launches = 0
        with torch.cuda.stream(st):
            if slot.start_event is not None:
                st.wait_event(slot.start_event)
            if self._staged_event is not None:
                st.wait_event(self._staged_event)
            # fresh bubble: clear the abort word and the done counter
            ctl[:2].zero_()
            if pr.resume_zero is not None:
                ctl[64 + pr.resume_zero] = 0
                pr.resume_zero = None
            native.call("pf_read_globaltimer", t_start, st.cuda_stream)
            for first, cnt, node in batches:
                launches += self._enqueue_batch(pr.part, first, cnt, node, slot.flag_ptr, abort_ptr,
                                                cursors, done_ptr)
            native.call("pf_read_globaltimer", t_end, st.cuda_stream)
            launches += 2
        ev = torch.cuda.Event()
        ev.record(st)
        self.pending = _Pending(slot, batches, ev, launches, has_resume=pr.resume is not None)
        self.kernel_launches += launches
        return prev

    def _enqueue_batch(self, part_idx: int, first: int, cnt: int, start_node: int, flag: int,
                       abort: int, cursors: int, done: int) -> int:
        """One batch of one partition as a chain of preemptible launches."""
        model, cfg = self.model, self.model.cfg
        part = self.plan.partitions[part_idx]
        st = self.stream
        s, h = cfg.seq, cfg.hidden
        ctx = ExecContext(st, self.ws, flag, abort, cursors)
        ctx.start_node = start_node
        launches = 0
        if start_node == 0:
            native.call("pf_chain_begin", cursors, MAX_NODES, abort, st.cuda_stream)
            launches += 1
        # node 0: the batch's input
        if part.lo == 0:
            src = self._ids_host.ptr + first * s * 4
            ids = self.ids_dev[:cnt]
            if ctx.active():
                native.call("pf_copy", ids.data_ptr(), src, cnt * s * 4,
                            ctypes.byref(ctx.ctl().as_struct()) if flag else None, st.cuda_stream)
                launches += 1
            else:
                ctx.skip()
            x = ids
        else:
            hid = ctx.buf("hidden", cnt * s * h).view(cnt, s, h)
            src = self._offload.ptr + first * s * h * 2
            if ctx.active():
                native.call("pf_copy", hid.data_ptr(), src, cnt * s * h * 2,
                            ctypes.byref(ctx.ctl().as_struct()) if flag else None, st.cuda_stream)
                launches += 1
            else:
                ctx.skip()
            x = hid
        for i in range(part.lo, part.hi):
            x = model[i](x, ctx)
        # last node: the batch's output
        last = part.hi == len(model)
        if last:
            # CLS rows [cnt, h] (row stride s*h) -> results; one copy per row would be
            # cnt launches, so gather on the device side via a strided view
            dst = self._results.ptr + first * h * 2
            if ctx.active():
                cls = x[:, 0, :]
                with torch.cuda.stream(st):
                    # dedicated buffer: this (non-preemptible) gather never touches
                    # anything a resumed node reads
                    staged = self.ws["cls"].view(-1)[: cnt * h].view(cnt, h)
                    staged.copy_(cls)
                native.call("pf_copy", dst, staged.data_ptr(), cnt * h * 2,
                            ctypes.byref(ctx.ctl().as_struct()) if flag else None, st.cuda_stream)
                launches += 1
            else:
                ctx.skip()
        else:
            dst = self._offload.ptr + first * s * h * 2
            if ctx.active():
                native.call("pf_copy", dst, x.data_ptr(), cnt * s * h * 2,
                            ctypes.byref(ctx.ctl().as_struct()) if flag else None, st.cuda_stream)
                launches += 1
            else:
                ctx.skip()
        native.call("pf_chain_end", done, abort, st.cuda_stream)
        launches += 1 + ctx.launched
        return launches

    def settle(self) -> Optional[BubbleRecord]:
        """Wait for the pending bubble's fill work, read the control block, advance
        the progress state (samples done, partition switch, resume point)."""
        pend = self.pending
        if pend is None:
            return None
        self.pending = None
        pend.end_event.synchronize()
        words = self._ctl_host
        native.call("pf_stage_d2h", words.ptr, self._ctl.data_ptr(), 4 * _CTL_WORDS,
                    torch.cuda.current_stream().cuda_stream)
        torch.cuda.current_stream().synchronize()
        w = words.tensor
        aborted = int(w[0]) != 0
        done = int(w[1])
        ts = w[8:12].view(torch.int64)
        pr = self.progress
        rec = BubbleRecord(pend.slot.index, len(pend.batches), done, 0, aborted,
                           int(ts[0]), int(ts[1]), pend.launches)
        n_total = self.item.entry.size
        samples = 0
        for k, (first, cnt, node) in enumerate(pend.batches):
            if k < done:
                samples += cnt
                if k == 0 and pend.has_resume:  # the resumed batch completed
                    pr.resume = None
                else:
                    pr.next_sample = max(pr.next_sample, first + cnt)
            elif k == done and aborted:
                # first incomplete node of the interrupted batch
                units = self._node_units(pr.part, cnt)
                cur = w[64:64 + len(units)]
                resume_node = len(units)
                for j, (u, kind) in enumerate(units):
                    if int(cur[j]) < u:
                        resume_node = j
                        break
                # atomic nodes re-run whole: zero their cursor; prefix nodes keep it
                if resume_node < len(units) and units[resume_node][1] == ATOMIC:
                    pr.resume_zero = resume_node
                if not (k == 0 and pend.has_resume):
                    pr.next_sample = max(pr.next_sample, first + cnt)
                pr.resume = (first, cnt, max(resume_node, node) if resume_node < len(units) else 0)
                if resume_node >= len(units):
                    pr.resume = None  # every node finished; only the end marker was skipped
                    samples += cnt
                break
            else:
                break
        rec.samples_done = samples
        part = self.plan.partitions[pr.part]
        if pr.resume is None and pr.next_sample >= n_total:
            if pr.part == len(self.plan.partitions) - 1:
                self.samples_completed += n_total
                pr.finished = True
            else:
                pr.part += 1
                pr.next_sample = 0
                self._stage_partition(pr.part)
        _ = part
        self.records.append(rec)
        return rec

    def _node_units(self, part_idx: int, cnt: int) -> list[tuple[int, str]]:
        part = self.plan.partitions[part_idx]
        cfg = self.model.cfg
        units: list[tuple[int, str]] = []
        in_bytes = cnt * cfg.seq * (4 if part.lo == 0 else 2 * cfg.hidden)
        units.append((_copy_units(in_bytes), ATOMIC))
        units.extend(self.model.node_units(part.lo, part.hi, cnt))
        out_bytes = cnt * cfg.hidden * 2 if part.hi == len(self.model) else cnt * cfg.seq * cfg.hidden * 2
        units.append((_copy_units(out_bytes), ATOMIC))
        return units

    def results(self) -> torch.Tensor:
        """[N, hidden] bf16 CLS embeddings of the current range (host, pinned)."""
        return self._results.tensor

    def close(self) -> None:
        self.settle()
        torch.cuda.synchronize()
        self.arena.close()


def _pad256(n: int) -> int:
    return (n + 255) // 256 * 256


def _copy_units(nbytes: int) -> int:
    out = ctypes.c_uint32(0)
    native.call("pf_copy_units", nbytes, ctypes.byref(out))
    return out.value
