"""Measure a fill model's LayerProfile on B200 (the planner's input).

The reference only synthesizes profiles from a cost model (workload.py:216-271);
PipeFill "relies on profiles of the fill job model's layer execution times and
memory consumption". Here each module k of the fill
nn.Sequential is timed on the device with CUDA events inside a full-model
chain (so inter-kernel gaps are charged to the module that follows them), at
every batch size, and its memory is the arena bytes the executor really uses
(weights + the module's workspace + activation buffers). The result is a
ModelProfile whose layer k is module k, serialized with model_to_json — the
reference's profile wire format.
"""

from __future__ import annotations

from typing import Sequence

import torch

from .arena import Arena
from .fillmodels import ExecContext, FillSequential
from .profiles import JobKind, LayerProfile, ModelProfile

FIXED_TRANSIENT_BYTES = 1 << 20  # control block, cursors, alignment slack


def _module_mem(model: FillSequential, i: int, b: int) -> tuple[int, int]:
    """(weight bytes, transient bytes at batch b) of module i as the executor lays it
    out. A partition's workspace is the union (per buffer name, the largest size) of
    its modules' buffers, so every module is charged the union over the whole model:
    then "weights + max transient" of any partition -- the planner's peak
    (partition.py:143-150) -- bounds the executor's partition region. Plus the
    partition-input buffer, the batch's inputs and results, and the control block."""
    w = model[i].weight_bytes()
    ws = sum(2 * v for v in model.workspace(0, len(model), b).values())
    res = b * torch.tensor([], dtype=model.result_dtype()).element_size()
    for d in model.result_shape():
        res *= d
    act = model.act_bytes() * b * model.boundary_elems(i) + res + b * model.input_bytes()
    return w, ws + act + FIXED_TRANSIENT_BYTES


def measure_profile(model: FillSequential, batch_sizes: Sequence[int], reps: int = 5,
                    warmup: int = 2, name: str | None = None) -> ModelProfile:
    cfg = model.cfg
    bmax = max(batch_sizes)
    weights = sum((model[i].weight_bytes() + 255) // 256 * 256 for i in range(len(model)))
    need = model.workspace(0, len(model), bmax)
    in_dtype, in_shape = model.input_spec()
    arena = Arena(weights + 2 * sum(need.values()) + bmax * model.input_bytes() + (64 << 20))
    stream = torch.cuda.Stream()
    try:
        for mod in model:
            mod.stage(arena, stream)
        ws = {k: arena.alloc((v,), torch.bfloat16) for k, v in need.items()}
        in_dev = arena.alloc((bmax, *in_shape), in_dtype)
        times: dict[int, list[float]] = {}
        for b in sorted(batch_sizes):
            in_dev[:b].copy_(model.make_inputs(0, 0, b))
            per_rep = []
            for r in range(warmup + reps):
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(model) + 1)]
                with torch.cuda.stream(stream):
                    ctx = ExecContext(stream, ws)
                    x = in_dev[:b]
                    evs[0].record(stream)
                    for i, mod in enumerate(model):
                        x = mod(x, ctx)
                        evs[i + 1].record(stream)
                stream.synchronize()
                if r >= warmup:
                    per_rep.append([evs[i].elapsed_time(evs[i + 1]) for i in range(len(model))])
            med = []
            for i in range(len(model)):
                col = sorted(p[i] for p in per_rep)
                med.append(col[len(col) // 2])
            times[b] = med
    finally:
        torch.cuda.synchronize()
        for mod in model:
            mod.unstage()
        arena.close()

    layers = []
    sizes = sorted(batch_sizes)
    for i in range(len(model)):
        w, _ = _module_mem(model, i, 1)
        exec_ms, mem = {}, {}
        prev_t, prev_m = 0.0, 0
        for b in sizes:
            # enforce the profile contract (non-decreasing in batch size) against timer noise
            t = max(times[b][i], prev_t, 1e-3)
            m = max(w + _module_mem(model, i, b)[1], prev_m)
            exec_ms[b], mem[b] = t, m
            prev_t, prev_m = t, m
        flops = _module_flops(model, i)
        layers.append(LayerProfile(exec_time_ms=exec_ms, mem_bytes=mem, weight_bytes=w,
                                   flops_per_sample=flops))
    params = sum(model[i].weight_bytes() // 2 for i in range(len(model)))
    prof = ModelProfile(name=name or f"{cfg.name}-infer-b200", layers=tuple(layers), param_count=params,
                        kind_allowed=frozenset({JobKind.BATCH_INFERENCE}))
    model.profile = prof  # the executor weighs partitions by measured time share
    return prof


def _module_flops(model: FillSequential, i: int) -> float:
    """Algorithmic forward FLOPs of module i per sample (BERT: 24*s*h^2 + 4*s^2*h per
    layer; ResNet: 2 * MACs of its convolutions and classifier)."""
    return model[i].flops_per_sample()


def _is_module_buffer(name: str, i: int) -> bool:
    """Workspace buffers that belong to module i alone (its saved activations, statistics,
    output and gradient buffers); every other name is scratch shared across modules."""
    return name.startswith(f"s{i}.") or name == f"out{i}" or name.startswith(f"g{i}.")


def _module_own_bytes(model, i: int, batch: int) -> int:
    need = model.workspace(i, i + 1, batch)
    return sum(2 * v for k, v in need.items() if _is_module_buffer(k, i))


def measure_train_profile(model: FillSequential, batch_sizes: Sequence[int], reps: int = 4,
                          warmup: int = 2, name: str | None = None) -> ModelProfile:
    """Profile of a training fill job (forward + loss + backward + SGD per batch).

    A training step is one recorded chain over the whole model, so it is timed whole:
    the executor runs `warmup + reps` steps at each batch size, one per (unbounded)
    bubble, and the step time is the median of the in-kernel %globaltimer span of the
    bubble's work. Module k is charged the step time x its share of the step's FLOPs
    (the planner only sums layers for a training plan). Memory: module k's optimizer
    state (fp32 master + momentum + bf16 working copy) plus, as transient, the step's
    whole workspace (saved activations, gradients, scratch) and its inputs/results --
    a training step keeps every module's activations alive until its backward."""
    from fractions import Fraction  # noqa: F401  (plan types below use exact rationals)

    from . import schedule as S
    from .coordinator import Coordinator
    from .executor import BubbleSlot, Executor
    from .profiles import JobSpec

    flops = [model[i].flops_per_sample() for i in range(len(model))]
    total_f = sum(flops) or 1.0
    sizes = sorted(batch_sizes)
    step_ms: dict[int, float] = {}
    for b in sizes:
        layers = tuple(LayerProfile({b: 0.001}, {b: model[i].weight_bytes() + 1}, model[i].weight_bytes(), 1.0)
                       for i in range(len(model)))
        prof = ModelProfile("probe", layers, 1, frozenset({JobKind.TRAINING}))
        cyc = S.BubbleCycle((S.BubbleSpec(10**6, 10**6, 10**12, S.BubbleKind.FWD_BWD),
                             S.BubbleSpec(0, 0, 10**12, S.BubbleKind.FILL_DRAIN)), 2 * 10**6, 0)
        coord = Coordinator(0, cyc, 1, batch_sizes=[b], max_batches_per_bubble=1)
        coord.admit(JobSpec("probe", 0.0, prof, JobKind.TRAINING, b * (warmup + reps)))
        item = coord.request_work(0, 0.0)
        need = model.workspace(0, len(model), b)
        arena_bytes = sum((model[i].weight_bytes() + 255) // 256 * 256 for i in range(len(model))) \
            + 2 * sum((2 * v + 255) // 256 * 256 for v in need.values()) + b * model.input_bytes() + (256 << 20)
        ex = Executor(arena_bytes)
        try:
            ex.load(item, model)
            spans = []
            for k in range(warmup + reps):
                ex.fill(BubbleSlot(0, None, 0))
                rec = ex.settle()
                if k >= warmup and rec is not None and rec.fill_end_ns > rec.fill_start_ns:
                    spans.append((rec.fill_end_ns - rec.fill_start_ns) / 1e6)
            spans.sort()
            step_ms[b] = spans[len(spans) // 2]
        finally:
            ex.close()
    layers = []
    partitioned = getattr(model, "partitioned", False)
    for i in range(len(model)):
        w = model[i].weight_bytes()
        exec_ms, mem = {}, {}
        prev_t = 0.0
        if partitioned:
            # a partition keeps the saved activations and gradients of all its modules until its
            # backward: charge them to the module's batch-independent bytes (at the largest batch
            # size, conservative below it), so the planner's peak (sum of weight_bytes + the
            # largest transient, partition.py:143-150) bounds what the executor carves
            own = _module_own_bytes(model, i, sizes[-1])
            w_plan = w + own
        for b in sizes:
            if partitioned:
                need = model.workspace(i, i + 1, b)
                shared = sum(2 * v for k, v in need.items() if not _is_module_buffer(k, i))
                bnd = 2 * 2 * b * model.boundary_elems(i)  # input boundary + its gradient
                transient = shared + bnd + b * model.input_bytes() + FIXED_TRANSIENT_BYTES
            else:
                need = model.workspace(0, len(model), b)
                transient = sum(2 * v for v in need.values()) + b * model.input_bytes() + FIXED_TRANSIENT_BYTES
            t = max(step_ms[b] * flops[i] / total_f, prev_t, 1e-3)
            exec_ms[b] = t
            mem[b] = (w_plan if partitioned else w) + transient
            prev_t = t
        layers.append(LayerProfile(exec_time_ms=exec_ms, mem_bytes=mem, weight_bytes=w_plan if partitioned else w,
                                   flops_per_sample=flops[i]))
    params = sum(model[i].weight_bytes() // 10 for i in range(len(model)))
    prof = ModelProfile(name=name or f"{model.cfg.name}-train-b200", layers=tuple(layers), param_count=params,
                        kind_allowed=frozenset({JobKind.TRAINING}))
    model.profile = prof
    return prof
