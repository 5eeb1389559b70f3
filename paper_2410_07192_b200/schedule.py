"""Main-job pipeline schedule, bubble characterization and the BUBBLE instruction.

Drop-in for the reference's `bubblefill.pipeline` (pkg/src/bubblefill/pipeline.py).
Public names and arithmetic are kept identical so that every downstream plan is
bit-exact:

* durations are integer microseconds; ms -> us uses Python's round-half-even
  (pipeline.py:81-86),
* usable bubble time is ``math.floor(duration_us * fill_fraction)`` evaluated
  in IEEE double (pipeline.py:205),
* bubble fractions are exact ``Fraction`` values (pipeline.py:38-45).

B200 additions (no reference counterpart): :func:`stage_program` emits the
per-stage instruction list *with* BUBBLE instructions — the list the engine in
``engine.py`` executes — and :func:`cycle_from_measurements` builds a
``BubbleCycle`` from measured bubble durations / free memory instead of the
analytic model.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from fractions import Fraction
from typing import NamedTuple, Sequence

US_PER_MS = 1000
TIMELINE_ORACLE_CAP = 10_000
DEFAULT_FILL_FRACTION = 0.68
DEFAULT_FREE_MEM = 4_500_000_000


class ScheduleKind(Enum):
    GPIPE = "gpipe"
    ONE_F_ONE_B = "1f1b"


class BubbleKind(Enum):
    FWD_BWD = "fwd_bwd"
    FILL_DRAIN = "fill_drain"


def _ms_to_us(ms: float) -> int:
    # Python's round() is round-half-even, exactly as the reference converts.
    return round(ms * US_PER_MS)


def bubble_fraction(p: int, m: int) -> Fraction:
    """(p - 1) / (m + p - 1): idle share of one iteration (pipeline.py:38-45)."""
    if p < 1 or m < 1:
        raise ValueError(f"need p >= 1 and m >= 1, got p={p}, m={m}")
    return Fraction(p - 1, p - 1 + m)


@dataclass(frozen=True)
class PipelineConfig:
    """Main-job shape and per-microbatch stage timings (pipeline.py:48-97)."""

    num_stages: int
    num_microbatches: int
    t_fwd_ms: float
    t_bwd_ms: float
    schedule: ScheduleKind = ScheduleKind.GPIPE
    fwd_free_mem: int = DEFAULT_FREE_MEM
    drain_free_mem: int = DEFAULT_FREE_MEM
    fill_fraction: float = DEFAULT_FILL_FRACTION

    def __post_init__(self) -> None:
        if self.num_stages < 1:
            raise ValueError(f"num_stages must be >= 1, got {self.num_stages}")
        if self.num_microbatches < 1:
            raise ValueError(f"num_microbatches must be >= 1, got {self.num_microbatches}")
        if min(self.t_fwd_us, self.t_bwd_us) < 1:
            raise ValueError("t_fwd_ms and t_bwd_ms must round to >= 1 microsecond")
        if not (0.0 < self.fill_fraction <= 1.0):
            raise ValueError(f"fill_fraction must be in (0, 1], got {self.fill_fraction}")
        if min(self.fwd_free_mem, self.drain_free_mem) < 0:
            raise ValueError("free memory must be >= 0")

    @property
    def t_fwd_us(self) -> int:
        return _ms_to_us(self.t_fwd_ms)

    @property
    def t_bwd_us(self) -> int:
        return _ms_to_us(self.t_bwd_ms)

    @property
    def period_us(self) -> int:
        step = self.t_fwd_us + self.t_bwd_us
        return step * (self.num_microbatches + self.num_stages - 1)

    @property
    def stage_idle_us(self) -> int:
        return (self.t_fwd_us + self.t_bwd_us) * (self.num_stages - 1)


@dataclass(frozen=True)
class BubbleSpec:
    """One bubble: raw idle span, the fill-usable part, free bytes, kind."""

    duration_us: int
    usable_us: int
    free_mem_bytes: int
    kind: BubbleKind

    def __post_init__(self) -> None:
        if self.duration_us < 0 or self.free_mem_bytes < 0:
            raise ValueError("bubble duration and free memory must be >= 0")
        if self.usable_us < 0 or self.usable_us > self.duration_us:
            raise ValueError("usable_us must be within [0, duration_us]")

    @property
    def duration_ms(self) -> float:
        return self.duration_us / US_PER_MS


@dataclass(frozen=True)
class BubbleCycle:
    """A stage's repeating bubble sequence plus its never-filled scattered idle."""

    bubbles: tuple[BubbleSpec, ...]
    period_us: int
    stage_id: int
    unfillable_us: int = 0

    def __post_init__(self) -> None:
        if self.total_idle_us > self.period_us:
            raise ValueError("bubble durations exceed the iteration period")

    @property
    def period_ms(self) -> float:
        return self.period_us / US_PER_MS

    @property
    def total_idle_us(self) -> int:
        return self.unfillable_us + sum(b.duration_us for b in self.bubbles)

    @property
    def idle_fraction(self) -> Fraction:
        return Fraction(self.total_idle_us, self.period_us)


def _validate_stage(config: PipelineConfig, stage_id: int) -> None:
    if stage_id < 0 or stage_id >= config.num_stages:
        raise ValueError(f"stage_id {stage_id} out of range [0, {config.num_stages})")


def fwd_bwd_bubble_duration_us(config: PipelineConfig, stage_id: int) -> int:
    """GPipe: (p-s-1)(tf+tb); 1F1B: (p-s-1)tb + max(0, p-s-m)tf (pipeline.py:160-172)."""
    _validate_stage(config, stage_id)
    downstream = config.num_stages - stage_id - 1
    if config.schedule is ScheduleKind.GPIPE:
        return downstream * (config.t_fwd_us + config.t_bwd_us)
    extra = max(0, config.num_stages - stage_id - config.num_microbatches)
    return downstream * config.t_bwd_us + extra * config.t_fwd_us


def fill_drain_bubble_duration_us(config: PipelineConfig, stage_id: int) -> int:
    """s (tf + tb) for both schedules (pipeline.py:175-185)."""
    _validate_stage(config, stage_id)
    return stage_id * (config.t_fwd_us + config.t_bwd_us)


def unfillable_duration_us(config: PipelineConfig, stage_id: int) -> int:
    """Scattered idle outside the two bubbles; 0 for GPipe (pipeline.py:188-197)."""
    _validate_stage(config, stage_id)
    rest = (config.stage_idle_us - fwd_bwd_bubble_duration_us(config, stage_id)
            - fill_drain_bubble_duration_us(config, stage_id))
    if rest < 0:  # pragma: no cover - closed forms guarantee rest >= 0
        raise AssertionError("negative scattered idle")
    return rest


def _bubble(duration_us: int, free_mem: int, kind: BubbleKind, fill_fraction: float) -> BubbleSpec:
    # float multiply then floor, exactly as pipeline.py:205
    return BubbleSpec(duration_us, math.floor(duration_us * fill_fraction), free_mem, kind)


def build_bubble_cycle(config: PipelineConfig, stage_id: int) -> BubbleCycle:
    """Analytic bubble characterization of one stage (pipeline.py:200-216)."""
    _validate_stage(config, stage_id)
    ff = config.fill_fraction
    return BubbleCycle(
        bubbles=(
            _bubble(fwd_bwd_bubble_duration_us(config, stage_id), config.fwd_free_mem,
                    BubbleKind.FWD_BWD, ff),
            _bubble(fill_drain_bubble_duration_us(config, stage_id), config.drain_free_mem,
                    BubbleKind.FILL_DRAIN, ff),
        ),
        period_us=config.period_us,
        stage_id=stage_id,
        unfillable_us=unfillable_duration_us(config, stage_id),
    )


def cycle_from_measurements(
    stage_id: int,
    period_us: int,
    durations_us: Sequence[int],
    free_mem_bytes: Sequence[int],
    fill_fraction: float = DEFAULT_FILL_FRACTION,
    unfillable_us: int = 0,
) -> BubbleCycle:
    """BubbleCycle from *measured* bubble durations and free memory (fwd-bwd first,
    fill-drain second), using the reference's usable-time rule (pipeline.py:205)."""
    if len(durations_us) != len(free_mem_bytes) or not durations_us:
        raise ValueError("need one free-memory value per measured bubble")
    kinds = (BubbleKind.FWD_BWD, BubbleKind.FILL_DRAIN)
    bubbles = tuple(
        _bubble(int(d), int(m), kinds[min(i, 1)], fill_fraction)
        for i, (d, m) in enumerate(zip(durations_us, free_mem_bytes))
    )
    return BubbleCycle(bubbles, int(period_us), stage_id, int(unfillable_us))


def with_cooldown(cycle: BubbleCycle, cooldown_us: int, min_duration_us: int = 0,
                  max_fraction: float = 1.0) -> BubbleCycle:
    """The same cycle with the usable time of every bubble longer than min_duration_us capped
    at duration - min(cooldown_us, max_fraction * duration).

    Power-aware usable time: under the board power cap the SM clock the main
    job resumes at depends on the power the end of the preceding bubble drew. An idle tail
    before the recv lets the power controller raise the clock again. The controller needs
    ~40 ms to react, so a short bubble gains nothing from a tail and is filled whole. The
    reference's usable rule (pipeline.py:205, floor(duration * fill_fraction)) applies first."""
    if cooldown_us <= 0:
        return cycle
    bubbles = tuple(b if b.duration_us <= min_duration_us else
                    BubbleSpec(b.duration_us,
                               max(0, min(b.usable_us, b.duration_us - int(min(cooldown_us,
                                                                             max_fraction * b.duration_us)))),
                               b.free_mem_bytes, b.kind) for b in cycle.bubbles)
    return BubbleCycle(bubbles, cycle.period_us, cycle.stage_id, cycle.unfillable_us)


# ---------------------------------------------------------------------------
# instruction streams


class Instr(NamedTuple):
    """One pipeline instruction: op in {"F", "B", "BUBBLE"}; microbatch index for
    F/B; the BubbleKind for BUBBLE."""

    op: str
    mb: int = -1
    kind: BubbleKind | None = None


def _fb_order(config: PipelineConfig, stage_id: int) -> list[tuple[str, int]]:
    m = config.num_microbatches
    if config.schedule is ScheduleKind.GPIPE:
        return [("F", j) for j in range(m)] + [("B", j) for j in range(m)]
    warm = min(m, config.num_stages - stage_id - 1)
    order = [("F", j) for j in range(warm)]
    for j in range(m - warm):
        order.extend((("F", warm + j), ("B", j)))
    order.extend(("B", j) for j in range(m - warm, m))
    return order


def _instruction_sequences(config: PipelineConfig) -> list[list[tuple[str, int]]]:
    """Per-stage F/B order (pipeline.py:219-234)."""
    return [_fb_order(config, s) for s in range(config.num_stages)]


def stage_program(config: PipelineConfig, stage_id: int) -> list[Instr]:
    """The stage's instruction list for one iteration, with PipeFill's BUBBLE
    instruction inserted where the large bubbles occur: right
    before the first backward (fwd-bwd bubble) and after the last backward
    (the fill-drain wrap-around gap). A BUBBLE is emitted only for a bubble of
    nonzero analytic duration."""
    _validate_stage(config, stage_id)
    prog: list[Instr] = []
    first_b_seen = False
    fwd_bwd = fwd_bwd_bubble_duration_us(config, stage_id)
    for op, j in _fb_order(config, stage_id):
        if op == "B" and not first_b_seen:
            first_b_seen = True
            if fwd_bwd > 0:
                prog.append(Instr("BUBBLE", kind=BubbleKind.FWD_BWD))
        prog.append(Instr(op, j))
    if fill_drain_bubble_duration_us(config, stage_id) > 0:
        prog.append(Instr("BUBBLE", kind=BubbleKind.FILL_DRAIN))
    return prog


def _busy_spans(config: PipelineConfig) -> list[list[tuple[int, int, str]]]:
    """Dependency replay of all stages (the semantics of pipeline.py:237-278):
    F j on s waits for F j on s-1; B j waits for B j on s+1, or for the stage's
    own F j on the last stage. Evaluated in one topological pass."""
    p, m = config.num_stages, config.num_microbatches
    tf, tb = config.t_fwd_us, config.t_bwd_us
    orders = _instruction_sequences(config)
    done: dict[tuple[str, int, int], int] = {}  # (op, stage, mb) -> end time
    pos = [0] * p
    clock = [0] * p
    spans: list[list[tuple[int, int, str]]] = [[] for _ in range(p)]
    pending = sum(len(o) for o in orders)
    while pending:
        advanced = False
        for s in range(p):
            while pos[s] < len(orders[s]):
                op, j = orders[s][pos[s]]
                if op == "F":
                    dep = None if s == 0 else ("F", s - 1, j)
                else:
                    dep = ("F", s, j) if s == p - 1 else ("B", s + 1, j)
                if dep is not None and dep not in done:
                    break
                ready = 0 if dep is None else done[dep]
                start = max(clock[s], ready)
                end = start + (tf if op == "F" else tb)
                done[(op, s, j)] = end
                spans[s].append((start, end, op))
                clock[s] = end
                pos[s] += 1
                pending -= 1
                advanced = True
        if not advanced:  # pragma: no cover - valid schedules never deadlock
            raise AssertionError("dependency deadlock: invalid schedule")
    if max(clock) != config.period_us:  # pragma: no cover
        raise AssertionError("iteration span disagrees with the closed-form period")
    return spans


_enumerate_busy_spans = _busy_spans


def replay_makespan(config: PipelineConfig, duration) -> float:
    """One iteration's makespan of the p-stage pipeline when op (stage, op, mb) takes
    `duration(stage, op, mb)` (any unit): the dependency replay of _busy_spans with
    per-op instead of uniform times. Used to compose a pipeline iteration time from the
    per-op device timings measured on each stage (bench.py: main-job slowdown)."""
    p = config.num_stages
    orders = _instruction_sequences(config)
    done: dict[tuple[str, int, int], float] = {}
    pos = [0] * p
    clock = [0.0] * p
    pending = sum(len(o) for o in orders)
    while pending:
        advanced = False
        for s in range(p):
            while pos[s] < len(orders[s]):
                op, j = orders[s][pos[s]]
                if op == "F":
                    dep = None if s == 0 else ("F", s - 1, j)
                else:
                    dep = ("F", s, j) if s == p - 1 else ("B", s + 1, j)
                if dep is not None and dep not in done:
                    break
                start = max(clock[s], 0.0 if dep is None else done[dep])
                clock[s] = done[(op, s, j)] = start + duration(s, op, j)
                pos[s] += 1
                pending -= 1
                advanced = True
        if not advanced:  # pragma: no cover - valid schedules never deadlock
            raise AssertionError("dependency deadlock: invalid schedule")
    return max(clock)


def brute_force_schedule_timeline(config: PipelineConfig) -> list[list[tuple[int, int]]]:
    """Per-stage idle intervals of one iteration window (pipeline.py:281-305)."""
    if config.num_stages * config.num_microbatches > TIMELINE_ORACLE_CAP:
        raise ValueError(
            f"p*m = {config.num_stages * config.num_microbatches} exceeds the oracle cap "
            f"{TIMELINE_ORACLE_CAP}"
        )
    out = []
    for stage_spans in _busy_spans(config):
        gaps = []
        cursor = 0
        for start, end, _ in stage_spans:
            if start > cursor:
                gaps.append((cursor, start))
            cursor = end
        if cursor < config.period_us:
            gaps.append((cursor, config.period_us))
        out.append(gaps)
    return out


def timeline_bubble_spans(config: PipelineConfig, stage_id: int) -> tuple[int, int, int]:
    """(fwd_bwd, fill_drain, unfillable) from the enumerated timeline (pipeline.py:308-333)."""
    _validate_stage(config, stage_id)
    if config.num_stages * config.num_microbatches > TIMELINE_ORACLE_CAP:
        raise ValueError("oracle cap exceeded")
    spans = _busy_spans(config)[stage_id]
    period = config.period_us
    wrap = spans[0][0] + (period - spans[-1][1])
    k = next(i for i, sp in enumerate(spans) if sp[2] == "B")
    before_first_b = spans[k][0] - spans[k - 1][1]
    idle = period - sum(e - s for s, e, _ in spans)
    return before_first_b, wrap, idle - before_first_b - wrap


def program_timeline(config: PipelineConfig, stage_id: int) -> list[tuple[Instr, int, int]]:
    """The stage program with the analytic start/end time (us, within one
    iteration window) of every instruction; a BUBBLE spans the idle gap it marks
    (the fill-drain BUBBLE spans the tail of this window plus the head of the next)."""
    spans = _busy_spans(config)[stage_id]
    prog = stage_program(config, stage_id)
    out: list[tuple[Instr, int, int]] = []
    k = 0
    for ins in prog:
        if ins.op == "BUBBLE":
            if ins.kind is BubbleKind.FWD_BWD:
                out.append((ins, spans[k - 1][1], spans[k][0]))
            else:
                tail_start = spans[-1][1]
                out.append((ins, tail_start, config.period_us + spans[0][0]))
        else:
            s, e, _ = spans[k]
            out.append((ins, s, e))
            k += 1
    return out


def steady_state_timeline(config: PipelineConfig, stage_id: int) -> list[tuple[Instr, int, int]]:
    """program_timeline re-based to the stage's steady-state window: the window opens
    at the stage's first compute instruction and closes at the next iteration's, so it
    is exactly one period long. The idle head before the first F (s * t_fwd under
    1F1B/GPipe) is the tail of the previous iteration's fill-drain BUBBLE, which
    program_timeline already spans into the next window; re-basing keeps it from being
    idled a second time at the start of every emulated iteration (engine.StageEngine)."""
    tl = program_timeline(config, stage_id)
    head = min(s for ins, s, _ in tl if ins.op != "BUBBLE")
    return [(ins, s - head, e - head) for ins, s, e in tl]
