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
