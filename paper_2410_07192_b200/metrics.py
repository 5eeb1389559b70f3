"""Fill metrics from device timestamps, and their reduction over ranks.

The reference computes its metrics from simulated time (sim.py:266-322:
busy/wall, recovered TFLOPS, bubble ratio). Here the same quantities come from
%globaltimer stamps of the real run: each bubble's flag-set / flag-clear times,
and the fill stream's first/last kernel times inside it.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, fields
from typing import Iterable, Sequence


@dataclass
class FillStats:
    sample_equivalents: float = 0.0  # completed batches x FLOP share of their partition
    samples_completed: float = 0.0  # samples that left the last partition
    fill_busy_ns: float = 0.0  # fill-stream busy time inside bubbles
    bubble_ns: float = 0.0  # measured fillable bubble time (flag set -> cleared)
    idle_ns: float = 0.0  # analytic total idle incl. 1F1B's unfillable gaps
    gemm_flops: float = 0.0
    gemm_ms: float = 0.0
    launches: float = 0.0
    wall_s: float = 0.0  # host wall clock of the timed region   (max over ranks)
    device_s: float = 0.0  # device time of the timed iterations   (max over ranks)

    SUMMED = ("sample_equivalents", "samples_completed", "fill_busy_ns", "bubble_ns", "idle_ns",
              "gemm_flops", "gemm_ms", "launches")

    @property
    def value(self) -> float:
        return self.sample_equivalents / self.device_s if self.device_s > 0 else 0.0

    @property
    def bubble_filled(self) -> float:
        return self.fill_busy_ns / self.bubble_ns if self.bubble_ns else 0.0

    @property
    def idle_filled(self) -> float:
        return self.fill_busy_ns / self.idle_ns if self.idle_ns else 0.0

    @property
    def gemm_tflops(self) -> float:
        return self.gemm_flops / (self.gemm_ms / 1e3) / 1e12 if self.gemm_ms > 0 else 0.0

    def as_dict(self) -> dict:
        return asdict(self)


def busy_in_bubbles(bubbles: Sequence[tuple[int, int]],
                    fills: Sequence[tuple[int, int]]) -> int:
    """Sum over bubbles of |fill interval ∩ bubble interval| (ns). `bubbles` are
    (flag set, flag cleared) and `fills` the matching (fill start, fill end) —
    (0, 0) for a bubble that got no work."""
    busy = 0
    for (b0, b1), (f0, f1) in zip(bubbles, fills):
        if f1 <= 0:
            continue
        busy += max(0, min(f1, b1) - max(f0, b0))
    return busy


def aggregate(stats: FillStats, device=None) -> FillStats:
    """Whole-job stats: work summed over ranks, times as the max over ranks."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return stats
    names = [f.name for f in fields(FillStats)]
    vals = torch.tensor([getattr(stats, n) for n in names], dtype=torch.float64, device=device)
    sums, maxs = vals.clone(), vals.clone()
    dist.all_reduce(sums, op=dist.ReduceOp.SUM)
    dist.all_reduce(maxs, op=dist.ReduceOp.MAX)
    out = FillStats()
    for i, n in enumerate(names):
        setattr(out, n, float(sums[i] if n in FillStats.SUMMED else maxs[i]))
    return out


def mean_slowdown(on: dict[int, Iterable[float]], off: dict[int, Iterable[float]]) -> float | None:
    """Mean over stages of (mean iteration time with fill) / (without) - 1."""
    import statistics

    vals = []
    for s, v in on.items():
        if s in off:
            vals.append(statistics.mean(v) / statistics.mean(off[s]) - 1.0)
    return statistics.mean(vals) if vals else None


def slowdown_stats(on: dict[int, Sequence[float]], off: dict[int, Sequence[float]]) -> dict:
    """Main-job slowdown from interleaved fill-on / fill-off iterations of every stage.

    In a pipeline the slowest stage paces all of them, so the headline `max` is the
    maximum over stages of mean(on) / mean(off) - 1 (the reference's OverheadModel is one
    factor for the whole job, sim.py:32-56); `mean` is kept as a secondary figure.
    `noise_floor` is the same statistic between the two halves of the fill-off iterations
    (off[0::2] vs off[1::2]) -- what the measurement reports when nothing changed."""
    import statistics

    per_stage, noise = {}, {}
    for s in sorted(on):
        if s not in off or not on[s] or not off[s]:
            continue
        per_stage[s] = statistics.mean(on[s]) / statistics.mean(off[s]) - 1.0
        a, b = list(off[s])[0::2], list(off[s])[1::2]
        if a and b:
            noise[s] = abs(statistics.mean(a) / statistics.mean(b) - 1.0)
    if not per_stage:
        return {"max": None, "mean": None, "argmax_stage": None, "noise_floor": None, "per_stage": {}}
    worst = max(per_stage, key=lambda s: per_stage[s])
    return {"max": per_stage[worst], "mean": statistics.mean(per_stage.values()), "argmax_stage": worst,
            "noise_floor": max(noise.values()) if noise else None,
            "per_stage": {str(s): v for s, v in per_stage.items()},
            "per_stage_noise": {str(s): v for s, v in noise.items()},
            "iterations": {"fill_on": sum(len(v) for v in on.values()),
                           "fill_off": sum(len(v) for v in off.values())}}


def distribution(values: Sequence[float]) -> dict:
    """n, p50, p99 and max of a sample (nearest-rank percentiles)."""
    v = sorted(values)
    if not v:
        return {"n": 0, "p50": None, "p99": None, "max": None}

    def rank(q: float) -> float:
        return v[min(len(v) - 1, max(0, int(-(-q * len(v) // 1)) - 1))]
    return {"n": len(v), "p50": rank(0.50), "p99": rank(0.99), "max": v[-1]}
