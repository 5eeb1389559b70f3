"""The fill-job Executor: runs a Coordinator WorkItem inside a stage's bubbles on B200.

Reference counterpart: the time model ``ExecutionPlan.range_wall_us /
range_busy_us`` (pkg/src/bubblefill/partition.py:118-132) consumed by the
simulator's dispatch loop (pkg/src/bubblefill/sim.py:222-235), and the paper's
Executor process. Here the plan is executed for real:

* partitions run in order; partition ``[lo, hi)`` of the fill model's
  nn.Sequential runs ``per_bubble[j].num_batches`` batches of
  ``per_bubble[j].batch_size`` samples in bubble j of every cycle until all of the
  range's samples passed through it (the reference's partition-major order);
* one batch of one partition is a native launch chain (libpipefill pf_chain_*),
  recorded once per (partition, batch size) with every TMA descriptor and launch
  shape resolved, and replayed with one call per batch on a low-priority fill
  stream behind the bubble's start event;
* every kernel polls the stage's bubble flag at tile granularity, so the work
  yields within one tile of the main job's recv completing; a yielded batch is
  resumed at its first incomplete kernel in the next bubble (tile cursor for
  GEMMs, whole-node re-run for idempotent nodes);
* weights of the next partition are staged host->HBM with pinned copies on a
  side stream while the main job computes; activations between partitions are
  kept in an HBM activation store inside the arena when it fits (B200: 180 GB),
  else offloaded to pinned host memory and reloaded;
* everything lives in a fixed arena sized from the measured bubble free memory,
  so the fill job cannot allocate past it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Optional

import torch

from . import native
from .arena import Arena, PinnedBuffer, device_view
from .coordinator import WorkItem
from .fillmodels import ExecContext, FillSequential
from .planner import BubblePlanEntry, ExecutionPlan, GreedyPlan, PartitionPlan

_CTL_WORDS = 64 + 4096  # [0]=abort, [1]=batches done, [2]=run-ahead staged, [8..12)=timestamps (2 x u64),
#                        [64..)=cursors
_CURSOR0 = 64
MAX_BATCHES = 256  # per bubble (device batch descriptors): planned + a resumed + run-ahead batches
STARVE_LIMIT = 256  # consecutive bubbles without progress before FillStarvation
MAX_NODES = 4096
# PF_EXEC_GRAPHS=0 replays chains node by node (pf_chain_launch) instead of as gated CUDA
# graphs: for profilers that do not see kernels inside conditional graph nodes (ncu)
_USE_GRAPHS = __import__("os").environ.get("PF_EXEC_GRAPHS", "1") != "0"
# modules per gated graph segment (gate kernel + conditional IF node); see DESIGN.md §3
_SEG_MODULES = int(__import__("os").environ.get("PF_SEG_MODULES", "4"))
DESC_WORDS = 4  # PF_DESC_WORDS: (input, result, aux input, -) byte offsets per batch


class FillStarvation(RuntimeError):
    """The bubbles are too short for the fill to make any progress: the same unit of work
    was yielded STARVE_LIMIT times in a row (e.g. bubbles shorter than one GEMM tile, or a
    profiler serialising the timer that closes every bubble ahead of the fill)."""


@dataclass
class BubbleSlot:
    """One upcoming bubble as the engine announces it to the executor."""

    index: int  # bubble position j in the stage's cycle (0 = fwd-bwd, 1 = fill-drain)
    start_event: Optional[torch.cuda.Event]  # fill stream waits for it (flag already set)
    flag_ptr: int  # device address of the stage's bubble flag (0 = not preemptible)
    tag: object = None  # engine's id for this bubble, copied into the BubbleRecord


@dataclass
class BubbleRecord:
    index: int
    batches_planned: int
    batches_done: int
    samples_done: int  # samples through this bubble's partition (completed batches)
    aborted: bool
    fill_start_ns: int = 0
    fill_end_ns: int = 0
    launches: int = 0
    part: int = 0
    model_fraction: float = 1.0  # share of the model's FLOPs in this bubble's partition
    samples_completed: int = 0  # samples that left the LAST partition in this bubble
    tag: object = None
    sample_eq: float = 0.0  # completed batches x their partition's share of the model (all partitions)
    ran_ahead: bool = False  # the bubble also enqueued batches of the next partition
    # preempted bubbles: %globaltimer when the last CTA of the yielded batch's GEMMs exited
    # (in-kernel stamps), i.e. when the fill released the SMs -- the yield latency's end
    last_work_end_ns: int = 0


@dataclass
class _Progress:
    part: int = 0
    next_sample: int = 0  # next sample (0-based within the range) for this partition
    resume: Optional[tuple[int, int, int]] = None  # (first sample, count, node) of a yielded batch
    resume_zero: Optional[int] = None  # atomic node whose cursor must be reset before the resume
    finished: bool = False
    resume_epoch: int = 0  # loan epoch the yielded batch ran in (a loan batch resumes only in it)


@dataclass
class _Pending:
    slot: BubbleSlot
    batches: list[tuple[int, int, int]]  # (first sample, count, start node)
    end_event: torch.cuda.Event
    launches: int
    part: int
    has_resume: bool = False
    parts: list[int] = None  # partition of every batch (run-ahead appends partition part + 1)
    progress_key: tuple = ()  # (part, next sample, resume point, resume cursor) when enqueued
    tp: Optional[list] = None  # partitioned training: [(batch index, phase index, start node)] enqueued
    greedy: Optional[list] = None  # Algorithm-1 plan: [(replica, lo, hi, start node)] of partition j
    loan_epoch: int = 0


class _Chain:
    """Owner of one recorded pf_chain_t (partition, batch size) and its CUDA graph."""

    def __init__(self):
        self.h = ctypes.c_void_p()
        native.call("pf_chain_create", ctypes.byref(self.h))
        self.units: list[tuple[int, bool]] = []
        self.gemm_flops: dict[int, float] = {}
        self.gemm_bytes: dict[int, float] = {}  # minimum DRAM bytes per GEMM node (roofline)
        self.seg_ends: list[int] = []
        self.timing = False
        self.graph = False

    def finalize(self) -> None:
        n = ctypes.c_int(0)
        native.call("pf_chain_size", self.h, ctypes.byref(n))
        self.units = []
        for i in range(n.value):
            u, r = ctypes.c_uint32(0), ctypes.c_int(0)
            native.call("pf_chain_node_info", self.h, i, ctypes.byref(u), ctypes.byref(r))
            self.units.append((u.value, bool(r.value)))

    def build_graph(self, flag: Optional[int], abort: int, cursors: int, done: int) -> None:
        ends = (ctypes.c_int * len(self.seg_ends))(*self.seg_ends)
        native.call("pf_chain_build_graph", self.h, flag, abort, cursors, done, ends, len(self.seg_ends))
        self.graph = True

    def close(self) -> None:
        if self.h:
            native.call("pf_chain_destroy", self.h)
            self.h = ctypes.c_void_p()


class Executor:
    """One per GPU (pipeline-stage worker). Not thread-safe; driven by the engine."""

    def __init__(self, arena_bytes: int, *, priority: int = 1, job_seed: int = 0,
                 activation_store: str = "auto", run_ahead: bool = True, use_graphs: Optional[bool] = None):
        native.require_device()
        # gated CUDA graphs per batch (default), or node-by-node launches (PF_EXEC_GRAPHS=0 /
        # use_graphs=False): profilers do not see kernels inside conditional graph nodes
        self.use_graphs = _USE_GRAPHS if use_graphs is None else bool(use_graphs)
        self.arena = Arena(arena_bytes)
        lo_prio, hi_prio = torch.cuda.Stream.priority_range()
        self.stream = torch.cuda.Stream(priority=hi_prio if priority == 0 else lo_prio)
        self.copy_stream = torch.cuda.Stream(priority=lo_prio)
        self.job_seed = job_seed
        self.activation_store = activation_store  # "auto" (HBM if it fits) | "host"
        # run-ahead: when a bubble's batches finish the range's current partition, stage the
        # next partition in-stream and run its planned batches in the same bubble (the
        # reference's time model charges whole cycles per partition, partition.py:118-124)
        self.run_ahead = run_ahead
        self.item: Optional[WorkItem] = None
        self.model: Optional[FillSequential] = None
        self.plan: Optional[ExecutionPlan] = None
        self.progress = _Progress()
        self.pending: Optional[_Pending] = None
        self.records: list[BubbleRecord] = []
        self.samples_completed = 0  # samples through the LAST partition, all items
        self.kernel_launches = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.timing = False  # live per-GEMM device timing (bench roofline)
        # (flops, ms, bubble tag, batch size, minimum DRAM bytes) of every GEMM node of the last
        # batch of each completed bubble (in-kernel stamps)
        # (FLOPs, ms, bubble tag, batch size, bytes, end %globaltimer ns) per timed GEMM node
        self.gemm_samples: list[tuple] = []
        # called when the executor runs out of work at a bubble: returns the next
        # (WorkItem, model) from the stage's Coordinator, or None
        self.work_source: Optional[Callable[[], Optional[tuple[WorkItem, FillSequential]]]] = None
        self._ctl_host = PinnedBuffer((_CTL_WORDS,), torch.int32)
        self._desc_host = PinnedBuffer((MAX_BATCHES, DESC_WORDS), torch.int64)
        self._gated: dict[int, ctypes.c_void_p] = {}
        self._ahead_staging: Optional[int] = None  # index in self.stagings of the last run-ahead copy
        self._stamps_host = PinnedBuffer((MAX_NODES, 2), torch.int64)
        # timing mode: the GEMM stamps of each bubble's FIRST batch, copied out right after it
        # (before batch 2 overwrites the chain's stamp slots): with the power-aware tail a
        # long bubble's last batch runs throttled, its first at full width
        self._stamps_first_host = PinnedBuffer((MAX_NODES, 2), torch.int64)
        self._chains: dict[tuple[int, int], _Chain] = {}
        self._staged_event: Optional[torch.cuda.Event] = None
        self._staged_part: Optional[int] = None
        self._cap = 0  # samples the per-range buffers hold
        self._in_host: Optional[PinnedBuffer] = None
        self._results: Optional[PinnedBuffer] = None
        self._store_host: Optional[list[PinnedBuffer]] = None
        self._store_dev: Optional[list[torch.Tensor]] = None
        self._layout_key = None
        self._flops_frac: list[float] = []
        self._last_flag: Optional[int] = None
        self._dev_views: dict[int, dict] = {}
        # executable cache: arena layouts of other (model, plan) pairs kept resident, so a
        # worker switching between jobs or stages does not re-stage weights or re-record
        self._layouts: dict[tuple, dict] = {}
        # weight-partition stagings: (bytes, start event, end event) on the copy stream
        self.stagings: list[tuple[int, torch.cuda.Event, torch.cuda.Event]] = []
        self._aux_host: Optional[PinnedBuffer] = None
        self._greedy: Optional[dict] = None  # Algorithm-1 execution state (load_greedy)
        self.starved = 0  # consecutive settled bubbles that enqueued work but made no progress
        self._cursor_now = -1  # the resume node's cursor as of the last settle
        # memory loan (lend / revoke): HBM the main job does not need between two points of its
        # iteration (the offloaded optimizer moments' device buffer, engine.OptimizerOffload).
        # Bubble kinds in `loan_kinds` are planned with the loan added to their free memory;
        # batches larger than what the arena's region holds (`_base_b`) take their transient
        # workspace from the loan and run only while it is held
        self.loan_kinds: set[int] = set()
        self._loan: Optional[torch.Tensor] = None  # uint8 device buffer while lent
        self._loan_buf: Optional[torch.Tensor] = None  # the buffer chains were recorded against
        self._loan_ready: Optional[torch.cuda.Event] = None
        self._loan_epoch = 0
        self._base_b: dict[int, int] = {}  # partition -> largest batch the region's workspace holds
        self._loan_ws: dict[tuple[int, int], dict] = {}
        self._loan_copy: Optional[torch.cuda.Event] = None  # last staging into the loan
        self.loan_batches = 0  # batches enqueued on the loan
        self.loan_rollbacks = 0  # yielded loan batches restarted after a revoke

    # ------------------------------------------------------------------ loading

    _LAYOUT_ATTRS = ("_ctl", "_desc", "_stamps", "_region", "ws", "in_dev", "_cap", "_in_host", "_aux_host",
                     "aux_dev",
                     "_results", "_store_dev", "_store_host", "_flops_frac", "_staged_part",
                     "_staged_event", "_chains", "model", "plan", "_dev_views", "_part_layouts", "_gated",
                     "_base_b", "_loan_ws")

    def _save_layout(self) -> None:
        if self._layout_key is not None:
            self._layouts[self._layout_key] = {a: getattr(self, a) for a in self._LAYOUT_ATTRS}

    def _restore_layout(self, key: tuple) -> None:
        saved = self._layouts.pop(key)
        for a, v in saved.items():
            setattr(self, a, v)
        for i, dev in self._dev_views.items():  # module weight views of this layout
            self.model[i].dev = dev
        self._layout_key = key

    def load(self, item: WorkItem, model: FillSequential) -> None:
        """Take a new WorkItem. The arena layout, staged weights and recorded graphs are
        kept when the executable is unchanged (the Coordinator's `reuse`)
        and cached for executables seen before."""
        if self.pending is not None:
            self.settle()
        worst = max((e.num_batches for p in item.plan.partitions for e in p.per_bubble), default=0)
        if 2 * worst + 1 > MAX_BATCHES:  # planned + a resumed batch + a run-ahead partition's
            raise ValueError(f"plan has {worst} batches in one bubble; the executor's batch descriptor "
                             f"table holds {MAX_BATCHES} (max_batches_per_bubble <= {(MAX_BATCHES - 1) // 2})")
        n = item.entry.size
        key = (id(model), id(item.plan))
        if key != self._layout_key or n > self._cap:
            self._save_layout()
            if key in self._layouts and n <= self._layouts[key]["_cap"]:
                self._restore_layout(key)
            else:
                stale = self._layouts.pop(key, None)
                if stale is not None:  # cached for fewer samples: its buffers and graphs go
                    self.stream.synchronize()
                    self.copy_stream.synchronize()
                    _close_layout(stale)
                self.model, self.plan = model, item.plan
                self._layout(n)
                self._layout_key = key
        self.item = item
        self.progress = _Progress()
        self._cursor_now = -1
        self.starved = 0
        self._greedy = None
        self._tp_state = {"phase": 0, "resident": 0, "dirty": False} if self._tp else None
        self._in_host.tensor[:n].copy_(self.model.make_inputs(self.job_seed, item.entry.lo - 1, n))
        if self._aux_host is not None:
            self._aux_host.tensor[:n].copy_(self.model.make_aux(self.job_seed, item.entry.lo - 1, n))
        self._stage_partition(0)
        self.prewarm()

    @property
    def _tp(self) -> bool:
        """Partitioned training (training.ResNetTrainPartitioned): batch-major phases."""
        return bool(getattr(self.model, "partitioned", False))

    def _layout(self, cap: int) -> None:
        """Carve a new executable's region out of the arena; when the arena is full,
        evict every cached executable and start over."""
        try:
            self._carve(cap)
        except native.ArenaExhausted:
            self.stream.synchronize()  # the arena is about to be re-carved, host buffers freed
            self.copy_stream.synchronize()
            for saved in self._layouts.values():
                _close_layout(saved)
            self._layouts = {}
            self._chains = {}
            self.arena.reset()
            self._carve(cap)

    def _part_need(self, part: int) -> tuple[int, dict[str, int]]:
        """Partition `part`'s weight bytes (256-B padded) and its workspace (elements) at
        the largest batch size the plan gives it -- the peak the planner budgeted for it
        (Σ weights + max transient, partition.py:143-150 / profiler._module_mem)."""
        model, p = self.model, self.plan.partitions[part]
        w = sum(_pad256(model[i].weight_bytes()) for i in range(p.lo, p.hi))
        b = self._base_b.get(part) or max([e.batch_size for e in p.per_bubble] + [1])
        return w, self._ws_need(part, b)

    def _ws_need(self, part: int, b: int) -> dict[str, int]:
        model, p = self.model, self.plan.partitions[part]
        need = dict(model.workspace(p.lo, p.hi, b))
        if p.lo > 0 and not self._tp:  # the partition's input, reloaded from the activation store (bf16 units)
            need["in"] = b * model.boundary_elems(p.lo) * model.act_bytes() // 2
        return need

    def _plan_base_b(self) -> dict[int, int]:
        """Per partition: the largest batch its region workspace is sized for -- the plan's
        batch sizes in bubble kinds planned without the loan (all kinds when there is no
        loan). Loan kinds' larger batches take their workspace from the loan."""
        out = {}
        loan_ok = bool(self.loan_kinds) and not self.model.is_training and not self._tp
        for k, p in enumerate(self.plan.partitions):
            sizes = [e.batch_size for j, e in enumerate(p.per_bubble) if e.num_batches] or [1]
            base = [e.batch_size for j, e in enumerate(p.per_bubble)
                    if e.num_batches and not (loan_ok and j in self.loan_kinds)]
            if base:
                out[k] = max(base)
                continue
            # every bubble is planned with the loan: the region holds the largest power-of-two
            # batch (<= the planned ones) whose weights + workspace fit 90 % of the arena; if
            # not even one sample's does, the partition lives in the loan (0: weights and
            # workspace in the lent buffer, restaged every time the loan is granted)
            w = sum(_pad256(self.model[i].weight_bytes()) for i in range(p.lo, p.hi))
            b = max(sizes)
            fits = lambda b_: w + sum(_pad256(2 * v) for v in self._ws_need(k, b_).values()) <= 0.9 * self.arena.capacity
            while b > 1 and not fits(b):
                b //= 2
            out[k] = b if fits(b) else 0
        return out

    def _on_loan(self, part: int) -> bool:
        """Partition `part` is loan-resident (weights + workspace in the lent buffer)."""
        return self._base_b.get(part, 1) == 0

    def _backing(self, part: int) -> torch.Tensor:
        """bf16 storage partition `part`'s weights and workspace are laid out in."""
        if self._on_loan(part):
            if self._loan_buf is None:
                raise native.ArenaExhausted(f"partition {part} needs the loan, which was never granted")
            return self._loan_buf.view(torch.bfloat16)
        return self._region

    def _loan_workspace(self, part: int, b: int) -> dict:
        """Workspace views of a batch of b samples through partition `part` inside the lent
        buffer (the chains recorded with them are valid as long as the buffer is)."""
        ws = self._loan_ws.get((part, b))
        if ws is not None:
            return ws
        buf = self._loan_buf
        need = self._ws_need(part, b)
        total = sum(_pad256(2 * v) for v in need.values())
        if buf is None or total > buf.numel():
            raise native.ArenaExhausted(f"loan of {0 if buf is None else buf.numel()} B cannot hold the "
                                        f"{total} B workspace of batch {b} (partition {part})")
        ws, off = {}, 0
        for k, v in need.items():
            ws[k] = buf[off:off + 2 * v].view(torch.bfloat16)
            off += _pad256(2 * v)
        self._loan_ws[(part, b)] = ws
        return ws

    def lend(self, buf: torch.Tensor, ready: Optional[torch.cuda.Event]) -> None:
        """The main job lends `buf` (uint8, device) until `revoke`; the fill stream uses it only
        after `ready` (the main job's last use of it)."""
        if self._loan_buf is not None and (buf.data_ptr() != self._loan_buf.data_ptr()
                                           or buf.numel() != self._loan_buf.numel()):
            self.stream.synchronize()
            self._drop_chains()  # chains recorded against another loan buffer
            self._loan_ws = {}
        first = self._loan_buf is None
        self._loan_buf = buf
        self._loan = buf
        self._loan_ready = ready
        self._loan_epoch += 1
        if first:
            self.prewarm()  # record the loan batch sizes' chains now, not in a bubble

    def _batch_cap(self, part: int, planned: int, num: int) -> tuple[int, int]:
        """A planned (batch size, batches), capped at the region's workspace while the loan
        is not usable -- with proportionally more batches, so the bubble stays filled."""
        cap = self._base_b.get(part, planned)
        if planned <= cap or self._loan is not None or cap == 0:
            return planned, num
        return cap, min((MAX_BATCHES - 1) // 2, -(-num * planned // cap))

    def revoke(self) -> torch.cuda.Event:
        """End the loan: returns an event after the last fill work enqueued so far (kernels
        yield at the bubble's end, so it fires within the yield latency of the bubble's end).
        The lender's next write to the buffer waits on it. A batch that yielded on the loan is
        restarted (from its first node) the next time it runs."""
        self._loan = None
        self._loan_ready = None
        if self._staged_part is not None and self.plan is not None and self._on_loan(self._staged_part):
            self._staged_part = None  # restaged into the next loan
        if self._loan_copy is not None:  # a loan-resident staging's copies precede the return
            self.stream.wait_event(self._loan_copy)
            self._loan_copy = None
        ev = torch.cuda.Event()
        ev.record(self.stream)
        return ev

    def _carve(self, cap: int) -> None:
        """Arena: control block | partition region | ids | store. The partition region
        holds one partition at a time -- its weights, then its workspace -- and is sized
        for the largest partition's weights + workspace, so every partition the planner
        fit into the bubble free memory fits the arena."""
        plan, model = self.plan, self.model
        self._chains = {}
        self._dev_views = {}
        self._loan_ws = {}
        self._base_b = self._plan_base_b()
        self._ctl = self.arena.alloc((_CTL_WORDS,), torch.int32)
        self._ctl.zero_()
        self._desc = self.arena.alloc((MAX_BATCHES, DESC_WORDS), torch.int64)
        self._stamps = self.arena.alloc((MAX_NODES, 2), torch.int64)
        region = 256
        for k in range(len(plan.partitions)):
            if self._on_loan(k):
                continue
            w, need = self._part_need(k)
            region = max(region, w + sum(_pad256(2 * v) for v in need.values()))
        self._region = self.arena.alloc((region // 2,), torch.bfloat16)
        self._part_layouts: dict[int, tuple[dict, dict]] = {}
        self._gated: dict[int, ctypes.c_void_p] = {}  # partition -> gated run-ahead staging graph
        self.ws = {}
        bmax = max(e.batch_size for p in plan.partitions[:1] for e in p.per_bubble)
        if self._tp:
            bmax = max(bmax, self._tp_batch())
        in_dtype, in_shape = model.input_spec()
        self.in_dev = self.arena.alloc((max(bmax, 1), *in_shape), in_dtype)
        self._cap = cap
        self._in_host = PinnedBuffer((cap, *in_shape), in_dtype)
        self._results = PinnedBuffer((cap, *model.result_shape()), model.result_dtype())
        aux = model.aux_spec()
        self._aux_host = PinnedBuffer((cap, *aux[1]), aux[0]) if aux else None
        self.aux_dev = self.arena.alloc((max(bmax, 1), *aux[1]), aux[0]) if aux else None
        self._store_dev = None
        self._store_host = None
        self._tp_act, self._tp_din = {}, {}
        if self._tp:
            # one batch in flight: the input boundary of every partition p > 0 (forward) and the
            # gradient of that input (backward), b samples each, in HBM
            b = self._tp_batch()
            for k in range(1, len(plan.partitions)):
                shape = (b, *model.boundary_shape(plan.partitions[k].lo))
                self._tp_act[k] = self.arena.alloc(shape, torch.bfloat16)
                self._tp_din[k] = self.arena.alloc(shape, torch.bfloat16)
        elif len(plan.partitions) > 1:
            # one sample's activation at the widest inter-partition boundary. A partition
            # overwrites its input store in place sample by sample, which is safe only when
            # no boundary grows (BERT); otherwise partitions ping-pong between two stores.
            sizes = [model.boundary_elems(p.lo) for p in plan.partitions[1:]]
            elems = max(sizes)
            n_st = 1 if len(set(sizes)) == 1 else 2
            adt = model.act_dtype()
            store_bytes = n_st * cap * elems * model.act_bytes()
            free = self.arena.capacity - self.arena.stats()["used"]
            if self.activation_store == "auto" and store_bytes + (64 << 20) <= free:
                self._store_dev = [self.arena.alloc((cap * elems,), adt) for _ in range(n_st)]
            else:
                self._store_host = [PinnedBuffer((cap * elems,), adt) for _ in range(n_st)]
        # a batch through partition [lo, hi) counts as this share of a sample: the
        # partition's share of the model's measured execution time (profile at the
        # largest profiled batch size) when the model carries its profile, else of FLOPs
        prof = getattr(model, "profile", None)
        if prof is not None and len(prof.layers) == len(model):
            b = max(prof.batch_sizes)
            cost = [prof.layers[i].exec_time_ms[b] for i in range(len(model))]
        else:
            cost = [model[i].flops_per_sample() for i in range(len(model))]
        total = sum(cost) or 1.0
        self._flops_frac = [sum(cost[p.lo:p.hi]) / total for p in plan.partitions]
        self._staged_part = None

    def _store_ptr(self, k: int) -> int:
        """Activation store at boundary k (the output of partition k)."""
        if self._store_dev is not None:
            return self._store_dev[k % len(self._store_dev)].data_ptr()
        return self._store_host[k % len(self._store_host)].ptr

    def _part_layout(self, part: int) -> tuple[dict, dict]:
        """Device views of partition `part` inside the region: its modules' weights from
        the region base, then its workspace. Pure pointer arithmetic and the same every
        time the partition is resident, so its recorded chains stay valid across
        stagings of other partitions."""
        lay = self._part_layouts.get(part)
        if lay is not None:
            return lay
        p = self.plan.partitions[part]
        backing = self._backing(part)
        base = backing.data_ptr()
        ptr = base
        views: dict[int, dict] = {}
        for i in range(p.lo, p.hi):
            mod = self.model[i]
            views[i] = mod.make_views(ptr)
            ptr += _pad256(mod.weight_bytes())
        _, need = self._part_need(part)
        off = (ptr - base) // 2
        ws: dict[str, torch.Tensor] = {}
        for k, v in need.items():
            ws[k] = backing[off:off + v]
            off += _pad256(2 * v) // 2
        lay = (views, ws)
        self._part_layouts[part] = lay
        return lay

    def _module_ptr(self, part: int, i: int) -> int:
        """Device address of module i's staged state inside the region."""
        p = self.plan.partitions[part]
        ptr = self._backing(part).data_ptr()
        for j in range(p.lo, i):
            ptr += _pad256(self.model[j].weight_bytes())
        return ptr

    def _stage_partition(self, part: int) -> None:
        """Stage partition `part`'s weights into the region on the copy stream (pinned
        cudaMemcpyAsync), after the fill stream drained the previous partition; the
        fill stream waits on the staging event before the partition's first batch."""
        if self._staged_part == part:
            return
        if self._on_loan(part) and self._loan is None:
            return  # staged when the loan is granted (fill)
        p = self.plan.partitions[part]
        views, ws = self._part_layout(part)
        e0 = torch.cuda.Event(enable_timing=True)
        staged = 0
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_stream(self.stream)
            if self._on_loan(part) and self._loan_ready is not None:
                self.copy_stream.wait_event(self._loan_ready)
            e0.record(self.copy_stream)
            for i in range(p.lo, p.hi):
                mod = self.model[i]
                nbytes = mod.weight_bytes()
                dst = self._module_ptr(part, i)
                if nbytes:
                    native.call("pf_stage_h2d", dst, mod.host.ptr, nbytes, self.copy_stream.cuda_stream)
                self.h2d_bytes += nbytes
                staged += nbytes
                mod.dev = views[i]
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.copy_stream)
        self._staged_event = ev
        self._staged_part = part
        if self._on_loan(part):
            self._loan_copy = ev
        self.stagings.append((staged, e0, ev))
        self.ws = ws
        self._dev_views = dict(views)

    # ------------------------------------------------------------------ chains

    def _chain(self, part_idx, cnt: int, flag: Optional[int] = None) -> _Chain:
        """Recorded chain of one batch of `cnt` samples through partition `part_idx` (for
        partitioned training: part_idx = (phase kind, partition))."""
        key = (part_idx, cnt, flag)
        ch = self._chains.get(key)
        if ch is not None:
            return ch
        model = self.model
        pidx = part_idx[1] if self._tp else part_idx
        part = self.plan.partitions[pidx]
        views, ws = self._part_layout(pidx)
        if not self._tp and 0 < self._base_b.get(pidx, cnt) < cnt:
            ws = self._loan_workspace(pidx, cnt)  # a loan batch
        resident = {i: getattr(model[i], "dev", None) for i in views}
        for i, dev in views.items():  # record against the partition's region layout
            model[i].dev = dev
        try:
            if self._tp:
                return self._record_tp_chain(key, part_idx[0], pidx, cnt, flag, ws)
            return self._record_chain(key, part, cnt, flag, ws)
        finally:
            for i, dev in resident.items():
                model[i].dev = dev

    def _record_chain(self, key: tuple, part, cnt: int, flag: Optional[int], ws: dict) -> _Chain:
        model = self.model
        ch = _Chain()
        ctx = ExecContext(self.stream, ws, chain=ch.h)
        if model.is_training:
            return self._record_train_chain(key, ch, ctx, part, cnt, flag)
        # node 0: the batch's input slice (role 1: source + in_off)
        if part.lo == 0:
            nb = cnt * model.input_bytes()
            native.call("pf_chain_add_copy", ch.h, self.in_dev.data_ptr(), nb, self._in_host.ptr, nb, nb, 1, 1)
            x = self.in_dev[:cnt]
        else:
            shape = model.boundary_shape(part.lo)
            x = ctx.buf("in", cnt * model.boundary_elems(part.lo), model.act_dtype()).view(cnt, *shape)
            nb = cnt * model.boundary_elems(part.lo) * model.act_bytes()
            native.call("pf_chain_add_copy", ch.h, x.data_ptr(), nb, self._store_ptr(key[0] - 1), nb, nb, 1, 1)
        ctx.node = 1
        for i in range(part.lo, part.hi):
            before = ctx.node
            x = model[i](x, ctx)
            for node, fl in model[i].gemm_node_flops(cnt):
                ch.gemm_flops[before + node] = fl
            for node, nb in model[i].gemm_node_bytes(cnt):
                ch.gemm_bytes[before + node] = nb
            if (i - part.lo + 1) % _SEG_MODULES == 0 or i == part.hi - 1:
                ch.seg_ends.append(ctx.node)  # one gated graph segment per _SEG_MODULES modules
        # last node: the batch's output slice (role 2: destination + out_off)
        if part.hi == len(model):
            # the model's result rows (BERT: [CLS] of [cnt, s, h]) straight into pinned results
            src, spitch, width, rows = model.result_view(x, cnt)
            native.call("pf_chain_add_copy", ch.h, self._results.ptr, width, src, spitch, width, rows, 2)
        else:
            nb = cnt * model.boundary_elems(part.hi) * model.act_bytes()
            native.call("pf_chain_add_copy", ch.h, self._store_ptr(key[0]), nb, x.data_ptr(), nb, nb, 1, 2)
        ch.finalize()
        ch.seg_ends[-1] = len(ch.units)  # the output copy joins the last module's segment
        native.call("pf_chain_set_desc", ch.h, self._desc.data_ptr())
        native.call("pf_chain_set_stamps", ch.h, self._stamps.data_ptr())
        base = self._ctl.data_ptr()
        ch.build_graph(flag, base if flag else None, base + 4 * _CURSOR0 if flag else None, base + 4)
        self._chains[key] = ch
        return ch

    def _record_train_chain(self, key: tuple, ch: _Chain, ctx: ExecContext, part, cnt: int,
                            flag: Optional[int]) -> _Chain:
        """One training step on one batch: inputs and labels in, forward, loss, backward,
        optimizer step, per-sample losses out. Training plans run whole (one partition)."""
        model = self.model
        if part.lo != 0 or part.hi != len(model):
            raise NotImplementedError("training fill jobs run single-partition plans")
        nb = cnt * model.input_bytes()
        native.call("pf_chain_add_copy", ch.h, self.in_dev.data_ptr(), nb, self._in_host.ptr, nb, nb, 1, 1)
        ab = cnt * self._aux_host.tensor[0].numel() * self._aux_host.tensor.element_size()
        native.call("pf_chain_add_copy", ch.h, self.aux_dev.data_ptr(), ab, self._aux_host.ptr, ab, ab, 1, 3)
        ctx.node = 2
        loss = ctx.fbuf("loss", cnt * 4).view(cnt, 4)
        seg_ends, gemm_flops = model.record_step(self.in_dev[:cnt], self.aux_dev[:cnt], loss, ctx)
        ch.seg_ends = seg_ends
        ch.gemm_flops = gemm_flops
        ch.gemm_bytes = dict(getattr(model, "last_gemm_bytes", {}))
        rb = cnt * 16
        native.call("pf_chain_add_copy", ch.h, self._results.ptr, rb, loss.data_ptr(), rb, rb, 1, 2)
        ch.finalize()
        ch.seg_ends[-1] = len(ch.units)
        native.call("pf_chain_set_desc", ch.h, self._desc.data_ptr())
        native.call("pf_chain_set_stamps", ch.h, self._stamps.data_ptr())
        base = self._ctl.data_ptr()
        ch.build_graph(flag, base if flag else None, base + 4 * _CURSOR0 if flag else None, base + 4)
        self._chains[key] = ch
        return ch

    def _record_tp_chain(self, key: tuple, kind: str, pidx: int, cnt: int, flag: Optional[int],
                         ws: dict) -> _Chain:
        """One phase of one batch of partitioned training (ResNetTrainPartitioned.record_phase):
        input from the images (partition 0) or the partition's input store, gradient of its
        output from the next partition's store, output / input gradient to the stores,
        labels in and per-sample losses out for the loss phase."""
        model = self.model
        part = self.plan.partitions[pidx]
        k = len(self.plan.partitions)
        ch = _Chain()
        ctx = ExecContext(self.stream, ws, chain=ch.h)
        node = 0
        if pidx == 0:
            nb = cnt * model.input_bytes()
            native.call("pf_chain_add_copy", ch.h, self.in_dev.data_ptr(), nb, self._in_host.ptr, nb, nb, 1, 1)
            x = self.in_dev[:cnt]
            node += 1
        else:
            x = self._tp_act[pidx][:cnt]
        labels = loss = None
        if kind == "L":
            ab = cnt * self._aux_host.tensor[0].numel() * self._aux_host.tensor.element_size()
            native.call("pf_chain_add_copy", ch.h, self.aux_dev.data_ptr(), ab, self._aux_host.ptr, ab, ab, 1, 3)
            node += 1
            labels = self.aux_dev[:cnt]
            loss = ctx.fbuf("loss", cnt * 4).view(cnt, 4)
        dout = self._tp_din[pidx + 1][:cnt] if kind == "B" else None
        ctx.node = node
        seg_ends, flops, nbytes, out = model.record_phase(kind, part.lo, part.hi, x, dout, labels, loss, ctx)
        ch.seg_ends, ch.gemm_flops, ch.gemm_bytes = list(seg_ends), flops, nbytes
        if kind == "F":  # the output boundary for the next partition
            dst = self._tp_act[pidx + 1][:cnt]
            nb = dst.numel() * 2
            native.call("pf_chain_add_copy", ch.h, dst.data_ptr(), nb, out.data_ptr(), nb, nb, 1, 0)
        elif pidx > 0:  # the gradient of the partition's input for the previous partition
            dst = self._tp_din[pidx][:cnt]
            nb = dst.numel() * 2
            native.call("pf_chain_add_copy", ch.h, dst.data_ptr(), nb, out.data_ptr(), nb, nb, 1, 0)
        if kind == "L":
            rb = cnt * 16
            native.call("pf_chain_add_copy", ch.h, self._results.ptr, rb, loss.data_ptr(), rb, rb, 1, 2)
        _ = k
        ch.finalize()
        ch.seg_ends[-1] = len(ch.units)
        native.call("pf_chain_set_desc", ch.h, self._desc.data_ptr())
        native.call("pf_chain_set_stamps", ch.h, self._stamps.data_ptr())
        base = self._ctl.data_ptr()
        ch.build_graph(flag, base if flag else None, base + 4 * _CURSOR0 if flag else None, base + 4)
        self._chains[key] = ch
        return ch

    def _write_back(self, part: int = 0) -> None:
        """Training jobs: copy the trained state of every module of partition `part` back to
        its pinned host blob (copy stream, after the fill stream), so the next range -- or a
        restage after an eviction -- continues from it."""
        p = self.plan.partitions[part]
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_stream(self.stream)
            for i in range(p.lo, p.hi):
                mod = self.model[i]
                if mod.host is not None and mod.weight_bytes():
                    native.call("pf_stage_d2h", mod.host.ptr, self._module_ptr(part, i), mod.weight_bytes(),
                                self.copy_stream.cuda_stream)
                    self.d2h_bytes += mod.weight_bytes()
        self.copy_stream.synchronize()

    def _drop_chains(self) -> None:
        # safe with launches in flight: kernel parameters are copied at launch time
        for ch in self._chains.values():
            ch.close()
        self._chains = {}

    def prewarm(self, flag_ptr: Optional[int] = None) -> None:
        """Record the current partition's chains and graphs for the plan's batch sizes
        now — when the Coordinator hands over the WorkItem — instead of at the first
        bubble, where recording would eat into the bubble."""
        if flag_ptr is not None:
            self._last_flag = flag_ptr or None
        if self.item is None or self.progress.finished:
            return
        if self._tp:
            for kind, pidx in self._tp_phases():
                self._chain((kind, pidx), self._tp_batch(), self._last_flag)
            return
        for pidx, part in enumerate(self.plan.partitions):  # every partition: switches record nothing
            for e in part.per_bubble:
                if e.num_batches and (self._loan_buf is not None or e.batch_size <= self._base_b.get(pidx, 1 << 30)):
                    self._chain(pidx, e.batch_size, self._last_flag)

    # ------------------------------------------------------------------ bubbles

    @property
    def busy(self) -> bool:
        return self.item is not None and not self.progress.finished

    def fill(self, slot: BubbleSlot) -> Optional[BubbleRecord]:
        """Enqueue this bubble's planned batches (asynchronously). The previous
        bubble is settled first. Returns the settled record of the previous bubble."""
        prev = self.settle() if self.pending is not None else None
        if not self.busy and self.work_source is not None:
            nxt = self.work_source()
            if nxt is not None:
                self.load(*nxt)
        if not self.busy:
            return prev
        if self._tp:
            self._fill_tp(slot)
            return prev
        if self._greedy is not None:
            self._fill_greedy(slot)
            return prev
        pr = self.progress
        if self._on_loan(pr.part) and self._loan is None:
            return prev  # loan-resident partition, loan not held: nothing to run
        if self._staged_part != pr.part:  # a run-ahead staged the next partition over this one
            self._stage_partition(pr.part)
        if (pr.resume is not None and pr.resume[1] > self._base_b.get(pr.part, pr.resume[1])
                and (self._loan is None or pr.resume_epoch != self._loan_epoch)):
            # a batch yielded on the loan, which has been returned since: its workspace is
            # gone, so it restarts from its first node (cursors are re-zeroed by the chain)
            pr.next_sample, pr.resume, pr.resume_zero = pr.resume[0], None, None
            self.loan_rollbacks += 1
        part = self.plan.partitions[pr.part]
        entry = part.per_bubble[slot.index] if slot.index < len(part.per_bubble) else None
        n_total = self.item.entry.size
        batches: list[tuple[int, int, int]] = []
        if entry is None or entry.num_batches == 0:
            return prev  # the plan gives this partition no work in this bubble (e.g. zero-length)
        if pr.resume is not None:
            batches.append(pr.resume)
        start = pr.next_sample
        if entry.num_batches > 0:
            bsz, nb = self._batch_cap(pr.part, entry.batch_size, entry.num_batches)
            for _ in range(nb - (1 if pr.resume is not None else 0)):
                if start >= n_total:
                    break
                cnt = min(bsz, n_total - start)
                batches.append((start, cnt, 0))
                start += cnt
        if not batches:
            return prev
        parts = [pr.part] * len(batches)
        ahead = pr.part + 1
        if (self.run_ahead and not self.model.is_training and start >= n_total and ahead < len(self.plan.partitions)
                and len(batches) < MAX_BATCHES and not self._on_loan(pr.part) and not self._on_loan(ahead)):
            nxt = self.plan.partitions[ahead]
            e2 = nxt.per_bubble[slot.index] if slot.index < len(nxt.per_bubble) else None
            s2 = 0
            if e2 is not None:
                bsz2, nb2 = self._batch_cap(ahead, e2.batch_size, e2.num_batches)
                for _ in range(min(nb2, MAX_BATCHES - len(batches))):
                    if s2 >= n_total:
                        break
                    cnt = min(bsz2, n_total - s2)
                    batches.append((s2, cnt, 0))
                    parts.append(ahead)
                    s2 += cnt
        model = self.model
        res_b = self._results.tensor.element_size() * _numel(model.result_shape())
        aux_b = 0 if self._aux_host is None else self._aux_host.tensor[0].numel() * self._aux_host.tensor.element_size()

        def io_bytes(pi: int) -> tuple[int, int]:
            pp = self.plan.partitions[pi]
            ib = model.input_bytes() if pp.lo == 0 else model.boundary_elems(pp.lo) * model.act_bytes()
            ob = res_b if pp.hi == len(model) else model.boundary_elems(pp.hi) * model.act_bytes()
            return ib, ob
        st = self.stream
        base = self._ctl.data_ptr()
        abort_ptr, done_ptr = base, base + 4
        cursors = base + 4 * _CURSOR0
        flag = slot.flag_ptr or None
        self._last_flag = flag
        launches = 0
        # device batch descriptors: batch k of this bubble reads its input / output slice
        # offsets from desc[k] (k = the bubble's done counter when it starts)
        dh = self._desc_host.tensor
        for k, (first, cnt, node) in enumerate(batches):
            pp = self.plan.partitions[parts[k]]
            in_b, out_b = io_bytes(parts[k])
            dh[k, 0] = first * in_b
            dh[k, 1] = first * out_b
            dh[k, 2] = first * aux_b
            if node == 0 and aux_b:
                self.h2d_bytes += cnt * aux_b
            if node == 0 and (pp.lo == 0 or self._store_host is not None):
                self.h2d_bytes += cnt * in_b
            if pp.hi == len(model) or self._store_host is not None:
                self.d2h_bytes += cnt * out_b
        with torch.cuda.stream(st):
            if slot.start_event is not None:
                st.wait_event(slot.start_event)
            if self._staged_event is not None:
                st.wait_event(self._staged_event)
            on_loan = sum(1 for k, (_, c, _) in enumerate(batches) if c > self._base_b.get(parts[k], c))
            if on_loan:
                self.loan_batches += on_loan
                if self._loan_ready is not None:  # the main job's last use of the lent buffer
                    st.wait_event(self._loan_ready)
                    self._loan_ready = None
            self._ctl[:3].zero_()  # fresh bubble: abort word, done counter, run-ahead staged
            if pr.resume_zero is not None:
                self._ctl[_CURSOR0 + pr.resume_zero] = 0
                pr.resume_zero = None
            native.call("pf_stage_h2d", self._desc.data_ptr(), self._desc_host.ptr,
                        8 * DESC_WORDS * len(batches), st.cuda_stream)
            native.call("pf_read_globaltimer", base + 32, st.cuda_stream)
            for k, (first, cnt, node) in enumerate(batches):
                if parts[k] != pr.part and parts[k - 1] == pr.part:
                    self._stage_in_stream(parts[k], st)  # run-ahead: after this partition's batches
                ch = self._chain(parts[k], cnt, flag)
                if node > 0 or not self.use_graphs:  # resume a yielded batch at its first incomplete node
                    native.call("pf_chain_launch", ch.h, flag, abort_ptr if flag else None,
                                cursors if flag else None, done_ptr, node, 0, 0, st.cuda_stream)
                    launches += len(ch.units) - node + 1
                else:
                    native.call("pf_chain_graph_launch", ch.h, st.cuda_stream)
                    launches += len(ch.units) + len(ch.seg_ends) + 2
                if k == 0 and node == 0 and self.timing and len(batches) > 1 and ch.gemm_flops:
                    native.call("pf_stage_d2h", self._stamps_first_host.ptr, self._stamps.data_ptr(),
                                16 * len(ch.units), st.cuda_stream)
            native.call("pf_read_globaltimer", base + 40, st.cuda_stream)
            launches += 2
        ev = torch.cuda.Event()
        ev.record(st)
        self.pending = _Pending(slot, batches, ev, launches, pr.part, has_resume=pr.resume is not None,
                                parts=parts, progress_key=(pr.part, pr.next_sample, pr.resume, self._cursor_now),
                                loan_epoch=self._loan_epoch)
        self.kernel_launches += launches
        return prev

    # ------------------------------------------------------------------ Algorithm-1 plans

    def load_greedy(self, item: WorkItem, model: FillSequential, gplan: GreedyPlan, batch_size: int) -> None:
        """Run a WorkItem's sample range with an Algorithm-1 plan (planner.greedy_pack_model,
        the paper's Executor packer: partition.py:425-494) instead of its
        DP ExecutionPlan. Algorithm 1 replicates the node list `num_replicas` times (one batch
        of `batch_size` per replica) and cuts it into partitions; partition j runs in the j-th
        bubble of the sequence, i.e. in bubble kind j mod P. A partition is a run of whole or
        partial replicas: segment (replica r, layers [lo, hi)). A replica cut between two
        partitions keeps its activation in slot r of the activation store. All weights stay
        resident (one staging at load), so each node's memory fits as the plan assumed.
        Results are those of the DP plan bit for bit (each sample's rows run the same kernels)."""
        L = len(model)
        per = tuple(BubblePlanEntry(batch_size, 1) for _ in range(max(1, len(item.plan.partitions[0].per_bubble))))
        whole = PartitionPlan(0, L, per, item.plan.total_tps_us, 0)
        carrier = WorkItem(item.entry, ExecutionPlan((whole,), item.plan.period_us, item.plan.total_tps_us),
                           item.reuse, item.wall_s, item.busy_s)
        self.load(carrier, model)  # one partition [0, L): every weight resident, workspace at batch_size
        self.item = item
        R = max(1, gplan.num_replicas)
        parts = greedy_segments(gplan, L)
        bnd = max([model.boundary_elems(i) for i in range(1, L)] + [1])
        slot_b = batch_size * bnd * model.act_bytes()
        # per-replica activation slots, and the staging buffer a segment's input is copied to
        self._g_store = self.arena.alloc((max(1, R * slot_b // 2),), torch.bfloat16)
        self._g_in = self.arena.alloc((max(1, slot_b // 2),), torch.bfloat16)
        self._greedy = {"parts": parts, "R": R, "b": batch_size, "j": 0, "pass": 0, "resume": None,
                        "slot_bytes": slot_b, "P": len(per)}

    def _greedy_chain(self, lo: int, hi: int, cnt: int, flag: Optional[int]) -> _Chain:
        key = (("G", lo, hi), cnt, flag)
        ch = self._chains.get(key)
        if ch is not None:
            return ch
        model = self.model
        views, ws = self._part_layout(0)
        for i, dev in views.items():
            model[i].dev = dev
        ch = _Chain()
        ctx = ExecContext(self.stream, ws, chain=ch.h)
        store = self._g_store.data_ptr()
        if lo == 0:
            nb = cnt * model.input_bytes()
            native.call("pf_chain_add_copy", ch.h, self.in_dev.data_ptr(), nb, self._in_host.ptr, nb, nb, 1, 1)
            x = self.in_dev[:cnt]
        else:  # slot r of the store (desc in_off) -> the workspace
            shape = model.boundary_shape(lo)
            x = self._g_in[:cnt * model.boundary_elems(lo) * model.act_bytes() // 2].view(
                model.act_dtype()).view(cnt, *shape)
            nb = cnt * model.boundary_elems(lo) * model.act_bytes()
            native.call("pf_chain_add_copy", ch.h, x.data_ptr(), nb, store, nb, nb, 1, 1)
        ctx.node = 1
        for i in range(lo, hi):
            before = ctx.node
            x = model[i](x, ctx)
            for node, fl in model[i].gemm_node_flops(cnt):
                ch.gemm_flops[before + node] = fl
            if (i - lo + 1) % _SEG_MODULES == 0 or i == hi - 1:
                ch.seg_ends.append(ctx.node)
        if hi == len(model):
            src, spitch, width, rows = model.result_view(x, cnt)
            native.call("pf_chain_add_copy", ch.h, self._results.ptr, width, src, spitch, width, rows, 2)
        else:  # -> slot r of the store (desc out_off)
            nb = cnt * model.boundary_elems(hi) * model.act_bytes()
            native.call("pf_chain_add_copy", ch.h, store, nb, x.data_ptr(), nb, nb, 1, 2)
        ch.finalize()
        ch.seg_ends[-1] = len(ch.units)
        native.call("pf_chain_set_desc", ch.h, self._desc.data_ptr())
        native.call("pf_chain_set_stamps", ch.h, self._stamps.data_ptr())
        base = self._ctl.data_ptr()
        ch.build_graph(flag, base if flag else None, base + 4 * _CURSOR0 if flag else None, base + 4)
        self._chains[key] = ch
        return ch

    def _greedy_batch(self, r: int) -> tuple[int, int]:
        """(first sample, count) of replica r of the current pass (0 count past the range)."""
        g = self._greedy
        first = (g["pass"] * g["R"] + r) * g["b"]
        return first, max(0, min(g["b"], self.item.entry.size - first))

    def _fill_greedy(self, slot: BubbleSlot) -> None:
        """Enqueue partition j's segments if this bubble is its bubble kind (j mod P);
        partitions of zero-length bubbles are empty and are skipped."""
        g = self._greedy
        while g["j"] < len(g["parts"]) and not g["parts"][g["j"]]:
            g["j"] += 1  # an empty partition (Algorithm 1 emits them for zero-length bubbles)
        if g["j"] >= len(g["parts"]):
            g["j"], g["pass"] = 0, g["pass"] + 1
        if g["pass"] * g["R"] * g["b"] >= self.item.entry.size and g["resume"] is None:
            self.progress.finished = True  # the last pass's remaining partitions hold no samples
            return
        if slot.index != g["j"] % g["P"]:
            return
        segs = g["parts"][g["j"]]
        start = 0 if g["resume"] is None else g["resume"][0]
        queue = []
        for k in range(start, len(segs)):
            r, lo, hi = segs[k]
            first, cnt = self._greedy_batch(r)
            node = g["resume"][1] if (g["resume"] is not None and k == start) else 0
            if cnt > 0:
                queue.append((k, r, lo, hi, first, cnt, node))
        if not queue:
            g["j"] += 1
            g["resume"] = None
            return
        model, st, base = self.model, self.stream, self._ctl.data_ptr()
        flag = slot.flag_ptr or None
        self._last_flag = flag
        res_b = self._results.tensor.element_size() * _numel(model.result_shape())
        dh = self._desc_host.tensor
        for q, (k, r, lo, hi, first, cnt, node) in enumerate(queue):
            dh[q, 0] = first * model.input_bytes() if lo == 0 else r * g["slot_bytes"]
            dh[q, 1] = first * res_b if hi == len(model) else r * g["slot_bytes"]
            dh[q, 2] = 0
            if lo == 0 and node == 0:
                self.h2d_bytes += cnt * model.input_bytes()
            if hi == len(model):
                self.d2h_bytes += cnt * res_b
        launches = 0
        with torch.cuda.stream(st):
            if slot.start_event is not None:
                st.wait_event(slot.start_event)
            if self._staged_event is not None:
                st.wait_event(self._staged_event)
            self._ctl[:3].zero_()
            if self.progress.resume_zero is not None:
                self._ctl[_CURSOR0 + self.progress.resume_zero] = 0
                self.progress.resume_zero = None
            native.call("pf_stage_h2d", self._desc.data_ptr(), self._desc_host.ptr, 8 * DESC_WORDS * len(queue),
                        st.cuda_stream)
            native.call("pf_read_globaltimer", base + 32, st.cuda_stream)
            for k, r, lo, hi, first, cnt, node in queue:
                ch = self._greedy_chain(lo, hi, cnt, flag)
                if node > 0 or not self.use_graphs:
                    native.call("pf_chain_launch", ch.h, flag, base if flag else None,
                                base + 4 * _CURSOR0 if flag else None, base + 4, node, 0, 0, st.cuda_stream)
                    launches += len(ch.units) - node + 1
                else:
                    native.call("pf_chain_graph_launch", ch.h, st.cuda_stream)
                    launches += len(ch.units) + len(ch.seg_ends) + 2
            native.call("pf_read_globaltimer", base + 40, st.cuda_stream)
            launches += 2
        ev = torch.cuda.Event()
        ev.record(st)
        self.pending = _Pending(slot, [(first, cnt, node) for _, _, _, _, first, cnt, node in queue], ev, launches, 0,
                                progress_key=(g["pass"], g["j"], g["resume"], self._cursor_now), greedy=list(queue))
        self.kernel_launches += launches

    def _settle_greedy(self, pend: _Pending, w: torch.Tensor, aborted: bool, done: int) -> BubbleRecord:
        g = self._greedy
        queue = pend.greedy
        ts = w[8:12].view(torch.int64)
        rec = BubbleRecord(pend.slot.index, len(queue), done, 0, aborted, int(ts[0]), int(ts[1]), pend.launches, 0,
                           1.0, tag=pend.slot.tag)
        L = len(self.model)
        prof = getattr(self.model, "profile", None)
        cost = ([prof.layers[i].exec_time_ms[max(prof.batch_sizes)] for i in range(L)]
                if prof is not None and len(prof.layers) == L else [self.model[i].flops_per_sample() for i in range(L)])
        total = sum(cost) or 1.0
        g_resume = None
        for q, (k, r, lo, hi, first, cnt, node) in enumerate(queue):
            if q < done:
                rec.sample_eq += cnt * sum(cost[lo:hi]) / total
                rec.samples_done += cnt
                if hi == L:
                    rec.samples_completed += cnt
                continue
            if q == done and aborted:
                ch = self._chains[(("G", lo, hi), cnt, pend.slot.flag_ptr or None)]
                rec.last_work_end_ns = self._last_work_end(ch)
                cur = w[_CURSOR0:_CURSOR0 + len(ch.units)]
                resume_node = len(ch.units)
                for j, (u, _) in enumerate(ch.units):
                    if int(cur[j]) < u:
                        resume_node = j
                        break
                if resume_node >= len(ch.units):  # every node finished; only the end marker was skipped
                    rec.sample_eq += cnt * sum(cost[lo:hi]) / total
                    if hi == L:
                        rec.samples_completed += cnt
                    g_resume = (k + 1, 0) if k + 1 < len(g["parts"][g["j"]]) else None
                else:
                    g_resume = (k, max(resume_node, node))
                    if not ch.units[resume_node][1]:
                        self.progress.resume_zero = resume_node
                break
        if g_resume is None and (done >= len(queue) or (aborted and done < len(queue) and
                                                        queue[done][0] + 1 >= len(g["parts"][g["j"]]))):
            g["j"] += 1  # partition j finished in this bubble
            g["resume"] = None
        else:
            g["resume"] = g_resume
        self.samples_completed += rec.samples_completed
        self.starved = self.starved + 1 if (done == 0 and aborted and g["resume"] == pend.progress_key[2]) else 0
        if g["j"] >= len(g["parts"]):
            g["j"], g["pass"] = 0, g["pass"] + 1
        if g["pass"] * g["R"] * g["b"] >= self.item.entry.size and g["resume"] is None:
            self.progress.finished = True
        self.records.append(rec)
        if self.starved >= STARVE_LIMIT:
            raise FillStarvation(f"no fill progress in {self.starved} consecutive bubbles (greedy plan, "
                                 f"partition {g['j']}, resume {g['resume']})")
        return rec

    # ------------------------------------------------------------------ partitioned training

    def _tp_phases(self) -> list[tuple[str, int]]:
        """Phases of one batch over k partitions: F_0 .. F_{k-2}, L_{k-1}, B_{k-2} .. B_0."""
        k = len(self.plan.partitions)
        return [("F", p) for p in range(k - 1)] + [("L", k - 1)] + [("B", p) for p in range(k - 2, -1, -1)]

    def _tp_batch(self) -> int:
        """Every phase runs at the plan's largest batch size (one batch = one SGD step)."""
        return max([e.batch_size for p in self.plan.partitions for e in p.per_bubble] + [8])

    def _tp_cost(self, kind: str, pidx: int, b: int) -> float:
        """Estimated phase time (us) from the profile: a partition's training time is its
        layers' sum; a forward phase is a third of it, a loss / backward phase (forward
        recomputed + backward + SGD) all of it."""
        prof = getattr(self.model, "profile", None)
        p = self.plan.partitions[pidx]
        if prof is None or len(prof.layers) != len(self.model):
            return 1.0
        t = sum(prof.layers[i].exec_time_us(b) if b in prof.layers[i].exec_time_ms else 1 for i in range(p.lo, p.hi))
        return t / 3.0 if kind == "F" else float(t)

    def _tp_swap(self, old: int, new: int, dirty: bool, st: torch.cuda.Stream) -> None:
        """Gated in-stream swap of the resident partition: write `old`'s state back to its
        pinned blobs (when a backward phase updated it), then stage `new` in. Skipped on the
        device if an earlier phase of this bubble yielded (pf_staging gate)."""
        key = ("tp", old, new, dirty)
        g = self._gated.get(key)
        if g is None:
            dst, src, nb = [], [], []
            if dirty:
                po = self.plan.partitions[old]
                for i in range(po.lo, po.hi):
                    if self.model[i].weight_bytes():
                        dst.append(self.model[i].host.ptr)
                        src.append(self._module_ptr(old, i))
                        nb.append(self.model[i].weight_bytes())
            pn = self.plan.partitions[new]
            for i in range(pn.lo, pn.hi):
                if self.model[i].weight_bytes():
                    dst.append(self._module_ptr(new, i))
                    src.append(self.model[i].host.ptr)
                    nb.append(self.model[i].weight_bytes())
            n = len(dst)
            g = ctypes.c_void_p()
            base = self._ctl.data_ptr()
            native.call("pf_staging_create", ctypes.byref(g), (ctypes.c_void_p * max(n, 1))(*dst),
                        (ctypes.c_void_p * max(n, 1))(*src), (ctypes.c_uint64 * max(n, 1))(*nb), n, base, base + 8)
            self._gated[key] = g
        native.call("pf_staging_launch", g, st.cuda_stream)
        self.h2d_bytes += sum(self.model[i].weight_bytes() for i in range(self.plan.partitions[new].lo,
                                                                           self.plan.partitions[new].hi))
        if dirty:
            self.d2h_bytes += sum(self.model[i].weight_bytes() for i in range(self.plan.partitions[old].lo,
                                                                              self.plan.partitions[old].hi))

    def _fill_tp(self, slot: BubbleSlot) -> None:
        """Enqueue this bubble's phases of partitioned training: a resumed phase first, then
        phases (swapping partitions in-stream when one changes) while the plan's time budget
        for this bubble lasts."""
        ts, phases, b = self._tp_state, self._tp_phases(), self._tp_batch()
        budget = sum(e.num_batches * self._tp_cost("B", pi, b) for pi, p in enumerate(self.plan.partitions)
                     for e in p.per_bubble[slot.index:slot.index + 1] if e.num_batches)
        if budget <= 0:
            return
        n_total = self.item.entry.size
        n_batches = -(-n_total // b)
        pr = self.progress
        queue: list[tuple[int, int, int]] = []  # (batch, phase, start node)
        bi, ph = pr.next_sample // b, ts["phase"]
        spent = 0.0
        if pr.resume is not None:
            queue.append((bi, ph, pr.resume[2]))
            spent += self._tp_cost(*phases[ph], b)
            ph += 1
            if ph == len(phases):
                bi, ph = bi + 1, 0
        while bi < n_batches and len(queue) < MAX_BATCHES and (not queue or spent < budget):
            queue.append((bi, ph, 0))
            spent += self._tp_cost(*phases[ph], b)
            ph += 1
            if ph == len(phases):
                bi, ph = bi + 1, 0
        st = self.stream
        base = self._ctl.data_ptr()
        flag = slot.flag_ptr or None
        self._last_flag = flag
        dh = self._desc_host.tensor
        in_b = self.model.input_bytes()
        aux_b = self._aux_host.tensor[0].numel() * self._aux_host.tensor.element_size()
        for q, (bj, pj, node) in enumerate(queue):
            first = bj * b
            dh[q, 0], dh[q, 1], dh[q, 2] = first * in_b, first * 16, first * aux_b
        launches = 0
        with torch.cuda.stream(st):
            if slot.start_event is not None:
                st.wait_event(slot.start_event)
            if self._staged_event is not None:
                st.wait_event(self._staged_event)
            self._ctl[:3].zero_()
            if pr.resume_zero is not None:
                self._ctl[_CURSOR0 + pr.resume_zero] = 0
                pr.resume_zero = None
            native.call("pf_stage_h2d", self._desc.data_ptr(), self._desc_host.ptr, 8 * DESC_WORDS * len(queue),
                        st.cuda_stream)
            native.call("pf_read_globaltimer", base + 32, st.cuda_stream)
            resident, dirty = ts["resident"], ts["dirty"]
            for q, (bj, pj, node) in enumerate(queue):
                kind, pidx = phases[pj]
                if pidx != resident:
                    self._tp_swap(resident, pidx, dirty, st)
                    resident, dirty = pidx, False
                    launches += 2
                ch = self._chain((kind, pidx), b, flag)
                if node > 0 or not self.use_graphs:
                    native.call("pf_chain_launch", ch.h, flag, base if flag else None,
                                base + 4 * _CURSOR0 if flag else None, base + 4, node, 0, 0, st.cuda_stream)
                    launches += len(ch.units) - node + 1
                else:
                    native.call("pf_chain_graph_launch", ch.h, st.cuda_stream)
                    launches += len(ch.units) + len(ch.seg_ends) + 2
                dirty = dirty or kind != "F"
            native.call("pf_read_globaltimer", base + 40, st.cuda_stream)
            launches += 2
        ev = torch.cuda.Event()
        ev.record(st)
        self.pending = _Pending(slot, [(bj * b, b, node) for bj, _, node in queue], ev, launches, pr.part,
                                has_resume=pr.resume is not None, parts=[phases[pj][1] for _, pj, _ in queue],
                                progress_key=(pr.part, pr.next_sample, pr.resume, self._cursor_now),
                                tp=list(queue))
        self.kernel_launches += launches

    def _settle_tp(self, pend: _Pending, w: torch.Tensor, aborted: bool, done: int) -> BubbleRecord:
        """Advance partitioned training: the first `done` phases completed; an interrupted
        phase resumes at its first incomplete node; the resident partition is the one of the
        last phase that started (a swap runs only behind completed phases)."""
        ts, phases, b = self._tp_state, self._tp_phases(), self._tp_batch()
        pr = self.progress
        queue = pend.tp
        ts0 = dict(ts)
        ts1 = (ts0["resident"], ts0["dirty"])
        rec = BubbleRecord(pend.slot.index, len(queue), done, 0, aborted, int(w[8:12].view(torch.int64)[0]),
                           int(w[8:12].view(torch.int64)[1]), pend.launches, pend.part, 1.0, tag=pend.slot.tag)
        k = len(self.plan.partitions)
        frac = self._flops_frac
        resident, dirty = ts1
        for q, (bj, pj, node) in enumerate(queue):
            kind, pidx = phases[pj]
            if q > done:
                break
            if q == done and not aborted:
                break
            if pidx != resident:
                resident, dirty = pidx, False
            if q < done:
                dirty = dirty or kind != "F"
                # a phase's share of the step: forward a third of the partition, loss/backward two thirds
                rec.sample_eq += b * frac[pidx] * (1.0 / 3.0 if kind == "F" else 2.0 / 3.0)
                pr.resume = None
                ph = pj + 1
                if ph == len(phases):  # the batch's last phase: the SGD step is complete
                    rec.samples_done += b
                    rec.samples_completed += b
                    pr.next_sample = (bj + 1) * b
                    ph = 0
                ts["phase"] = ph
            else:  # the phase that yielded
                ch = self._chains[((kind, pidx), b, pend.slot.flag_ptr or None)]
                rec.last_work_end_ns = self._last_work_end(ch)
                cur = w[_CURSOR0:_CURSOR0 + len(ch.units)]
                resume_node = len(ch.units)
                for j, (u, _) in enumerate(ch.units):
                    if int(cur[j]) < u:
                        resume_node = j
                        break
                dirty = dirty or (kind != "F" and resume_node > 0)
                if resume_node >= len(ch.units):  # every node finished; only the end marker was skipped
                    rec.sample_eq += b * frac[pidx] * (1.0 / 3.0 if kind == "F" else 2.0 / 3.0)
                    pr.resume = None
                    ph = pj + 1
                    if ph == len(phases):
                        rec.samples_done += b
                        rec.samples_completed += b
                        pr.next_sample = (bj + 1) * b
                        ph = 0
                    ts["phase"] = ph
                else:
                    pr.resume = (bj * b, b, max(resume_node, node))
                    if not ch.units[resume_node][1]:
                        pr.resume_zero = resume_node
                    ts["phase"] = pj
                    pr.next_sample = bj * b
        if self.timing and done > 0 and not aborted:
            # in-kernel stamps of the bubble's last phase: (FLOPs, ms, tag, batch, bytes) per GEMM node
            bj, pj, _ = queue[done - 1]
            ch = self._chains.get((phases[pj], b, pend.slot.flag_ptr or None))
            if ch is not None and ch.gemm_flops:
                native.call("pf_stage_d2h", self._stamps_host.ptr, self._stamps.data_ptr(), 16 * len(ch.units),
                            self.stream.cuda_stream)
                self.stream.synchronize()
                sh = self._stamps_host.tensor
                for nd, fl in ch.gemm_flops.items():
                    t0, t1 = int(sh[nd, 0]), int(sh[nd, 1])
                    if 0 < t0 < t1:
                        self.gemm_samples.append((fl, (t1 - t0) / 1e6, pend.slot.tag, b, ch.gemm_bytes.get(nd, 0.0)))
        ts["resident"], ts["dirty"] = resident, dirty
        self._staged_part = resident
        views, wsd = self._part_layout(resident)
        for i in range(self.plan.partitions[resident].lo, self.plan.partitions[resident].hi):
            self.model[i].dev = views[i]
        self.ws = wsd
        self._dev_views = dict(views)
        self.samples_completed += rec.samples_completed
        key_after = (pr.part, pr.next_sample, pr.resume, self._resume_cursor(pend, [], w))
        self.starved = self.starved + 1 if (done == 0 and aborted and key_after == pend.progress_key) else 0
        self._cursor_now = key_after[3]
        n_total = self.item.entry.size
        if pr.resume is None and pr.next_sample >= n_total:
            pr.finished = True
            if ts["dirty"]:
                self._write_back(ts["resident"])
                ts["dirty"] = False
        self.records.append(rec)
        if self.starved >= STARVE_LIMIT:
            raise FillStarvation(f"no fill progress in {self.starved} consecutive bubbles (partitioned training, "
                                 f"phase {ts['phase']}, resume point {pr.resume})")
        return rec

    def _stage_in_stream(self, part: int, st: torch.cuda.Stream) -> None:
        """Run-ahead staging: copy partition `part`'s weights into the region on the fill
        stream itself, ordered after the previous partition's batches, as a gated graph
        (pf_staging_*): the copies run only if none of those batches yielded (abort word
        0), else the region keeps the current partition's weights and the yielded batch's
        workspace, and settle() rolls the host-side layout back. Not gated by the flag:
        a copy that outlives the bubble only uses PCIe."""
        p = self.plan.partitions[part]
        views, ws = self._part_layout(part)
        g = self._gated.get(part)
        if g is None:
            mods = [i for i in range(p.lo, p.hi) if self.model[i].weight_bytes()]
            n = len(mods)
            dst = (ctypes.c_void_p * max(n, 1))(*[self._module_ptr(part, i) for i in mods])
            src = (ctypes.c_void_p * max(n, 1))(*[self.model[i].host.ptr for i in mods])
            nb = (ctypes.c_uint64 * max(n, 1))(*[self.model[i].weight_bytes() for i in mods])
            g = ctypes.c_void_p()
            base = self._ctl.data_ptr()
            native.call("pf_staging_create", ctypes.byref(g), dst, src, nb, n, base, base + 8)
            self._gated[part] = g
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        native.call("pf_staging_launch", g, st.cuda_stream)
        staged = sum(self.model[i].weight_bytes() for i in range(p.lo, p.hi))
        self.h2d_bytes += staged
        for i in range(p.lo, p.hi):
            self.model[i].dev = views[i]
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(st)
        self._staged_event = ev
        self._staged_part = part
        self.stagings.append((staged, e0, ev))
        self._ahead_staging = len(self.stagings) - 1
        self.ws = ws
        self._dev_views = dict(views)

    def _rollback_ahead_staging(self, part: int) -> None:
        """The gated run-ahead staging was skipped on the device: partition `part` is still
        resident; restore its host-side views and uncount the copy."""
        views, ws = self._part_layout(part)
        for i in range(self.plan.partitions[part].lo, self.plan.partitions[part].hi):
            self.model[i].dev = views[i]
        self.ws = ws
        self._dev_views = dict(views)
        self._staged_part = part
        k = self._ahead_staging
        if k is not None and k < len(self.stagings):
            b, e0, e1 = self.stagings[k]
            self.h2d_bytes -= b
            self.stagings[k] = (0, e0, e1)
        self._ahead_staging = None

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
                    self.stream.cuda_stream)
        self.stream.synchronize()
        w = words.tensor
        aborted = int(w[0]) != 0
        done = int(w[1])
        if pend.tp is not None:
            return self._settle_tp(pend, w, aborted, done)
        if pend.greedy is not None:
            return self._settle_greedy(pend, w, aborted, done)
        ts = w[8:12].view(torch.int64)
        pr = self.progress
        rec = BubbleRecord(pend.slot.index, len(pend.batches), done, 0, aborted, int(ts[0]), int(ts[1]),
                           pend.launches, pend.part, self._flops_frac[pend.part], tag=pend.slot.tag)
        if self.timing and done > 0 and len(pend.batches) > 1 and pend.batches[0][2] == 0:
            # the first batch's GEMM stamps (copied out after it ran, see fill)
            ch0 = self._chains.get(((pend.parts or [pend.part])[0], pend.batches[0][1], pend.slot.flag_ptr or None))
            if ch0 is not None and ch0.gemm_flops:
                sh = self._stamps_first_host.tensor
                for node, fl in ch0.gemm_flops.items():
                    t0, t1 = int(sh[node, 0]), int(sh[node, 1])
                    if 0 < t0 < t1:
                        self.gemm_samples.append((fl, (t1 - t0) / 1e6, pend.slot.tag, pend.batches[0][1],
                                                  ch0.gemm_bytes.get(node, 0.0), t1))
        if self.timing and done > 0 and not aborted:
            # in-kernel stamps of the bubble's last batch: (FLOPs, ms) of every GEMM node
            last_cnt = pend.batches[len(pend.batches) - 1][1]
            last_part = (pend.parts or [pend.part])[-1]  # a run-ahead's last batch is in part + 1
            ch = self._chains.get((last_part, last_cnt, pend.slot.flag_ptr or None))
            if ch is not None and ch.gemm_flops:
                n = len(ch.units)
                native.call("pf_stage_d2h", self._stamps_host.ptr, self._stamps.data_ptr(), 16 * n,
                            self.stream.cuda_stream)
                self.stream.synchronize()
                sh = self._stamps_host.tensor
                for node, fl in ch.gemm_flops.items():
                    t0, t1 = int(sh[node, 0]), int(sh[node, 1])
                    if 0 < t0 < t1:
                        self.gemm_samples.append((fl, (t1 - t0) / 1e6, pend.slot.tag, last_cnt,
                                                  ch.gemm_bytes.get(node, 0.0), t1))
        n_total = self.item.entry.size
        samples = 0
        parts = pend.parts or [pend.part] * len(pend.batches)
        rec.ran_ahead = any(p_ != pend.part for p_ in parts)
        if rec.ran_ahead and int(w[2]) == 0:  # a batch of this partition yielded: staging skipped
            self._rollback_ahead_staging(pend.part)
        last_part = len(self.plan.partitions) - 1
        completed_last = 0
        for k, (first, cnt, node) in enumerate(pend.batches):
            if parts[k] != pr.part and k <= done:
                # the run-ahead reached the next partition: the current one is complete
                if pr.resume is not None or pr.next_sample < n_total:
                    break  # (cannot happen: stream order) keep the current partition
                pr.part = parts[k]
                pr.next_sample = 0
                pr.resume = None
            if k < done:
                samples += cnt
                rec.sample_eq += cnt * self._flops_frac[parts[k]]
                if parts[k] == last_part:
                    completed_last += cnt
                if k == 0 and pend.has_resume:  # the resumed batch completed
                    pr.resume = None
                else:
                    pr.next_sample = max(pr.next_sample, first + cnt)
            elif k == done and aborted:
                ch = self._chains[(parts[k], cnt, pend.slot.flag_ptr or None)]
                rec.last_work_end_ns = self._last_work_end(ch)
                cur = w[_CURSOR0:_CURSOR0 + len(ch.units)]
                resume_node = len(ch.units)
                for j, (u, _) in enumerate(ch.units):
                    if int(cur[j]) < u:
                        resume_node = j
                        break
                if not (k == 0 and pend.has_resume):
                    pr.next_sample = max(pr.next_sample, first + cnt)
                if resume_node >= len(ch.units):
                    pr.resume = None  # every node finished; only the end marker was skipped
                    samples += cnt
                    rec.sample_eq += cnt * self._flops_frac[parts[k]]
                    if parts[k] == last_part:
                        completed_last += cnt
                else:
                    pr.resume = (first, cnt, max(resume_node, node))
                    pr.resume_epoch = pend.loan_epoch
                    if not ch.units[resume_node][1]:
                        pr.resume_zero = resume_node  # atomic: re-run the whole node
                break
            else:
                break
        rec.samples_done = samples
        rec.samples_completed = completed_last
        self.samples_completed += completed_last
        key_after = (pr.part, pr.next_sample, pr.resume, self._resume_cursor(pend, parts, w))
        self.starved = self.starved + 1 if (done == 0 and aborted and key_after == pend.progress_key) else 0
        self._cursor_now = key_after[3]
        if pr.resume is None and pr.next_sample >= n_total:
            if pr.part == len(self.plan.partitions) - 1:
                pr.finished = True
                if self.model.is_training:
                    self._write_back()
            else:
                pr.part += 1
                pr.next_sample = 0
                self._stage_partition(pr.part)
                self.prewarm()
        self.records.append(rec)
        if self.starved >= STARVE_LIMIT:
            raise FillStarvation(f"no fill progress in {self.starved} consecutive bubbles (partition "
                                 f"{pr.part}, resume point {pr.resume}): bubbles shorter than one unit")
        return rec

    def _resume_cursor(self, pend: _Pending, parts: list, w: torch.Tensor) -> int:
        """Cursor of the resume node (its claimed units) -- progress inside one node."""
        pr = self.progress
        if pr.resume is None:
            return -1
        first, cnt, node = pr.resume
        ch = self._chains.get((pr.part, cnt, pend.slot.flag_ptr or None))
        if ch is None or node >= len(ch.units):
            return -1
        return int(w[_CURSOR0 + node])

    def _last_work_end(self, ch: _Chain) -> int:
        """Latest in-kernel end stamp over the GEMM nodes of the batch that yielded. Later
        launches of the aborted chain exit before stamping and chain_begin leaves the stamps
        alone once the abort word is set, so these are the yielded batch's own."""
        nodes = sorted(ch.gemm_flops)
        if not nodes:
            return 0
        n = len(ch.units)
        native.call("pf_stage_d2h", self._stamps_host.ptr, self._stamps.data_ptr(), 16 * n,
                    self.stream.cuda_stream)
        self.stream.synchronize()
        sh = self._stamps_host.tensor
        ends = [int(sh[i, 1]) for i in nodes if 0 < int(sh[i, 0]) <= int(sh[i, 1])]
        return max(ends) if ends else 0

    def staging_stats(self, since: int = 0) -> dict:
        """H2D weight staging since `self.stagings[since]`: bytes, device ms (copy-stream
        events around each partition's pinned copies) and GB/s."""
        nbytes, ms = 0, 0.0
        for b, e0, e1 in self.stagings[since:]:
            e1.synchronize()
            nbytes += b
            ms += e0.elapsed_time(e1)
        return {"stagings": len(self.stagings) - since, "bytes": nbytes, "ms": ms,
                "gbs": nbytes / ms / 1e6 if ms > 0 else None}

    def results(self) -> torch.Tensor:
        """[N, *result_shape] bf16 results of the current range (host, pinned): BERT [CLS]
        embeddings, ResNet logits."""
        return self._results.tensor[: self.item.entry.size]

    def close(self) -> None:
        """Release everything: graphs and chains of every cached executable, their pinned
        host buffers, the control-block mirrors and the arena."""
        self.settle()
        torch.cuda.synchronize()
        if self._layout_key is not None:
            self._save_layout()
            self._layout_key = None
        for saved in self._layouts.values():
            _close_layout(saved)
        self._layouts = {}
        self._chains = {}
        self._gated = {}
        for buf in (self._ctl_host, self._desc_host, self._stamps_host, self._stamps_first_host):
            buf.close()
        self.arena.close()


def greedy_segments(gplan: GreedyPlan, num_layers: int) -> list[list[tuple[int, int, int]]]:
    """Segments (replica r, layers [lo, hi)) of every partition of an Algorithm-1 plan: the
    plan's partitions cut the node list replicated `num_replicas` times (partition.py:453-479)
    into consecutive runs, so partition j covers positions [p_j, p_j+1) of that list."""
    L = num_layers
    R = max(1, gplan.num_replicas)
    parts, pos = [], 0
    for nodes in gplan.partitions:
        segs: list[tuple[int, int, int]] = []
        for k, n in enumerate(nodes):
            r, node = divmod(pos + k, L)
            if node != n:
                raise ValueError(f"greedy partition node {n} at position {pos + k} of a {L}-node list")
            if segs and segs[-1][0] == r and segs[-1][2] == node:
                segs[-1] = (r, segs[-1][1], node + 1)
            else:
                segs.append((r, node, node + 1))
        parts.append(segs)
        pos += len(nodes)
    if pos != R * L:
        raise ValueError(f"greedy plan covers {pos} of {R} x {L} nodes")
    return parts


def _close_layout(saved: dict) -> None:
    """Destroy one cached executable: its chains / graphs and its pinned host buffers."""
    for ch in saved["_chains"].values():
        ch.close()
    for g in saved.get("_gated", {}).values():
        native.call("pf_staging_destroy", g)
    for name in ("_in_host", "_results", "_aux_host"):
        buf = saved.get(name)
        if buf is not None:
            buf.close()
    for buf in saved.get("_store_host") or []:
        buf.close()


def _pad256(n: int) -> int:
    return (n + 255) // 256 * 256


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= int(d)
    return n
