"""Multi-job fill service: Placer + per-stage Coordinators driving real Executors.

Reference counterpart: the simulator's event loop ``run_sim`` /
``compute_metrics`` (pkg/src/bubblefill/sim.py:200-322) and the CLI report
(cli.py:47,80-99). The simulator advances a clock by the plan's time model
(``WorkItem.wall_s`` = period x sum ceil(N / samples-per-cycle),
partition.py:118-124). Here the same Placer (``routing``) and Coordinators
(``coordinator``) hand WorkItems to one ``Executor`` per pipeline stage, and the
ranges really run in the stages' bubbles on the GPU:

* virtual time advances one pipeline iteration (``period_us`` of the
  PipelineConfig built from the measured t_fwd / t_bwd) per round; in round r
  every stage runs one main-job iteration with its bubbles filled. At N=1 the
  stages of a round run one after the other on the GPU (time-multiplexed
  emulation, artificial neighbours); their bubbles are the same ones a
  dedicated GPU per stage would see;
* a job is routed at its arrival time (``route_avg_jct`` etc. with
  now_s = arrival_s, as sim.py:240-252); WorkItems are dispatched to an idle
  stage worker at the start of a round and a range completes at the end of the
  round in which its last batch left the last partition, so measured JCTs are
  period-quantised exactly like the simulator's;
* per-job busy time is the device time its batches ran inside bubbles
  (executor BubbleRecords, %globaltimer stamps), not the plan's estimate.

``write_report`` emits the reference's ``jobs.csv`` columns and ``summary.json``
scalars (cli.py:47,80-99), plus the simulator's prediction of every JCT for the
same jobs, cycles and policies.
"""

from __future__ import annotations

import csv
import json
import math
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional, Sequence

from .coordinator import FIFO, Coordinator, OrderingPolicy
from .planner import Infeasible
from .profiles import JobSpec, isolated_throughput
from .routing import route_avg_jct, route_makespan_min, route_round_robin, route_shortest_queue
from .schedule import BubbleCycle, PipelineConfig, bubble_fraction, build_bubble_cycle

JOBS_CSV_COLUMNS = ["id", "arrival_s", "start_s", "completion_s", "coordinator", "flops"]
ROUTING = ("avg_jct", "makespan", "round_robin", "shortest_queue")


@dataclass(frozen=True)
class ServiceConfig:
    """The SimConfig fields that shape a real run (sim.py:60-70)."""

    pipeline: PipelineConfig
    routing: str = "avg_jct"
    ordering: OrderingPolicy = FIFO
    batch_sizes: Optional[tuple[int, ...]] = None
    max_batches_per_bubble: int = 16

    def __post_init__(self) -> None:
        if self.routing not in ROUTING:
            raise ValueError(f"routing must be one of {ROUTING}, got {self.routing!r}")


@dataclass
class JobResult:
    job_id: str
    model: str
    samples: int
    arrival_s: float
    start_s: float
    completion_s: float
    coordinator: int
    fill_flops: float
    busy_s: float  # measured device time of the job's batches inside bubbles
    rel_perf: float
    predicted_completion_s: Optional[float] = None  # the reference simulator's

    @property
    def jct_s(self) -> float:
        return self.completion_s - self.arrival_s


@dataclass
class ServiceReport:
    per_job: dict[str, JobResult]
    rejected: list[str]
    unfinished: list[str]
    rounds: int
    period_s: float
    bubble_ns: int = 0
    fill_busy_ns: int = 0
    samples_completed: int = 0
    scalars_extra: dict = field(default_factory=dict)
    gpus: int = 1  # pipeline stages served (one worker each)
    stage_iterations: int = 0  # stage iterations actually run (a stage with nothing to fill is skipped)

    def scalars(self) -> dict:
        done = sorted(self.per_job.values(), key=lambda r: r.job_id)
        jcts = sorted(r.jct_s for r in done)
        makespan = max((r.completion_s for r in done), default=0.0)
        span = makespan - min((r.arrival_s for r in done), default=0.0)
        flops = sum(r.fill_flops for r in done)
        busy = sum(r.busy_s for r in done)
        pred = [r.predicted_completion_s - r.arrival_s for r in done if r.predicted_completion_s is not None]
        out = {
            "avg_jct_s": sum(jcts) / len(jcts) if jcts else 0.0,
            "p99_jct_s": jcts[max(0, math.ceil(0.99 * len(jcts)) - 1)] if jcts else 0.0,
            "makespan_s": makespan,
            "completed": len(done),
            "rejected": len(self.rejected),
            "unfinished": len(self.unfinished),
            "recovered_tflops_active": flops / busy / 1e12 if busy > 0 else 0.0,
            "fill_samples_per_s": sum(r.samples for r in done) / span if span > 0 else 0.0,
            "mean_rel_perf": sum(r.rel_perf for r in done) / len(done) if done else 0.0,
            "bubble_time_filled": self.fill_busy_ns / self.bubble_ns if self.bubble_ns else 0.0,
            "predicted_avg_jct_s": sum(pred) / len(pred) if pred else None,
            "rounds": self.rounds,
            "period_s": self.period_s,
        }
        # the reference's SimReport.scalars keys (sim.py:139-153), from measured quantities:
        # bubble_ratio = measured bubble time / stage time, wall-clock TFLOP/s over all GPUs,
        # GPU-hours = measured busy time (sim.py:119-120), gpus_saved (sim.py:156-159)
        stage_ns = (self.stage_iterations or self.rounds * max(1, self.gpus)) * self.period_s * 1e9
        ratio = self.bubble_ns / stage_ns if stage_ns > 0 else 0.0
        out.update({
            "bubble_ratio": ratio,
            "recovered_tflops_wallclock": flops / (span * max(1, self.gpus)) / 1e12 if span > 0 else 0.0,
            "mean_fill_gpu_hours": busy / 3600.0 / len(done) if done else 0.0,
            "gpus_saved": max(1, self.gpus) * ratio * out["mean_rel_perf"],
            "main_job_slowdown": None,
        })
        out.update(self.scalars_extra)
        return out


class FillService:
    """Placer + one Coordinator and one Executor per stage, driven round by round.

    ``run_iteration(stage, executor)`` runs one main-job iteration of that stage
    with its BUBBLE instructions handed to `executor` and returns the engine's
    timing dict (``record_timing``: start, main_end, step_end, bubbles)."""

    def __init__(self, config: ServiceConfig, models: dict, executors: Sequence,
                 run_iteration: Callable[[int, object], dict],
                 cycles: Optional[Sequence[BubbleCycle]] = None,
                 flag_of: Optional[Callable[[int], int]] = None):
        p = config.pipeline.num_stages
        if len(executors) != p:
            raise ValueError("one executor per stage")
        self.config = config
        self.models = models  # ModelProfile.name -> FillSequential
        self.executors = list(executors)
        self.run_iteration = run_iteration
        self.flag_of = flag_of
        self.cycles = list(cycles) if cycles is not None else [
            build_bubble_cycle(config.pipeline, s) for s in range(p)]
        self.coordinators = [
            Coordinator(s, self.cycles[s], 1, config.ordering, config.batch_sizes,
                        config.max_batches_per_bubble) for s in range(p)]
        self.period_s = config.pipeline.period_us / 1e6
        self.rr_counter = 0

    def _route(self, job: JobSpec, now_s: float) -> Optional[int]:
        cs, r = self.coordinators, self.config.routing
        if r == "avg_jct":
            return route_avg_jct(cs, job, now_s)
        if r == "makespan":
            return route_makespan_min(cs, job, now_s)
        if r == "shortest_queue":
            return route_shortest_queue(cs)
        idx = route_round_robin(self.rr_counter, len(cs))
        self.rr_counter += 1
        return idx

    def run(self, jobs: Sequence[JobSpec], max_rounds: int = 1000) -> ServiceReport:
        for a, b in zip(jobs, jobs[1:]):
            if a.arrival_s > b.arrival_s:
                raise ValueError("jobs must be sorted by arrival time")
        by_id = {j.id: j for j in jobs}
        pending = list(jobs)
        assigned: dict[str, int] = {}
        start_s: dict[str, float] = {}
        busy_ns: dict[str, int] = {}
        completion: dict[str, float] = {}
        rejected: list[str] = []
        inflight: list = [None] * len(self.coordinators)
        bubble_ns = fill_ns = 0
        rounds = stage_iters = 0
        from .metrics import busy_in_bubbles

        for r in range(max_rounds):
            t0 = r * self.period_s
            t1 = t0 + self.period_s
            # causality: a job is routed and dispatched at the first round start at or after its
            # arrival (a job arriving mid-round waits for the next round, as a real service
            # dispatching at iteration boundaries would); 1 ns of slack absorbs the float
            # rounding of arrivals placed exactly on an iteration boundary
            while pending and pending[0].arrival_s <= t0 + 1e-9:
                job = pending.pop(0)
                cidx = self._route(job, max(job.arrival_s, t0))
                ok = False
                if cidx is not None:
                    try:
                        self.coordinators[cidx].admit(job)
                        ok = True
                    except Infeasible:
                        ok = False
                if ok:
                    assigned[job.id] = cidx
                else:
                    rejected.append(job.id)
            if not pending and all(x is None for x in inflight) and not any(c.queue for c in self.coordinators):
                break
            rounds = r + 1
            for s, (coord, ex) in enumerate(zip(self.coordinators, self.executors)):
                if inflight[s] is None:
                    item = coord.request_work(0, t0)
                    if item is not None:
                        jid = item.entry.job_id
                        start_s.setdefault(jid, t0)
                        inflight[s] = item
                        if self.flag_of is not None:
                            ex.prewarm(self.flag_of(s))  # chains recorded at load gate on this flag
                        ex.load(item, self.models[by_id[jid].model.name])
                if inflight[s] is None:
                    continue  # nothing to fill: the stage's iteration is not needed
                n0 = len(ex.records)
                stage_iters += 1
                t = self.run_iteration(s, ex)
                ex.settle()
                recs = {rec.tag: rec for rec in ex.records[n0:]}
                bubbles, fills = [], []
                for _kind, b0, b1, tag in t["bubbles"]:
                    rec = recs.get(tag)
                    bubbles.append((b0, b1))
                    fills.append((rec.fill_start_ns, rec.fill_end_ns) if rec is not None else (0, 0))
                bubble_ns += sum(b1 - b0 for b0, b1 in bubbles)
                used = busy_in_bubbles(bubbles, fills)
                fill_ns += used
                jid = inflight[s].entry.job_id
                busy_ns[jid] = busy_ns.get(jid, 0) + used
                if not ex.busy:  # the range left the last partition in this round
                    done = coord.on_range_done(0, inflight[s], t1)
                    inflight[s] = None
                    if done is not None:
                        completion[done] = t1

        per_job: dict[str, JobResult] = {}
        for jid, t_done in completion.items():
            job = by_id[jid]
            busy = busy_ns.get(jid, 0) / 1e9
            iso = isolated_throughput(job.model, job.kind)
            rel = (job.samples / busy) / iso if busy > 0 and iso > 0 else 0.0
            per_job[jid] = JobResult(jid, job.model.name, job.samples, job.arrival_s, start_s[jid], t_done,
                                     assigned[jid], job.samples * job.model.flops_per_sample, busy, rel)
        unfinished = [j.id for j in jobs if j.id not in completion and j.id not in rejected]
        samples = sum(r.samples for r in per_job.values())
        return ServiceReport(per_job, rejected, unfinished, rounds, self.period_s, bubble_ns, fill_ns, samples,
                             gpus=len(self.coordinators), stage_iterations=stage_iters)


def predict(config: ServiceConfig, jobs: Sequence[JobSpec],
            cycles: Optional[Sequence[BubbleCycle]] = None) -> dict[str, float]:
    """The plan time model's completion time of every job: the simulator's event loop
    (sim.py:213-261) over fresh Coordinators with the same cycles and policies --
    arrivals routed at arrival time, a worker's range done at now + wall_s, ties by
    (time, completions first, sequence). Returns {job_id: completion_s}."""
    import heapq

    p = config.pipeline.num_stages
    cyc = list(cycles) if cycles is not None else [build_bubble_cycle(config.pipeline, s) for s in range(p)]
    cs = [Coordinator(s, cyc[s], 1, config.ordering, config.batch_sizes, config.max_batches_per_bubble)
          for s in range(p)]
    shell = FillService.__new__(FillService)
    shell.coordinators, shell.config, shell.rr_counter = cs, config, 0
    by_id = {j.id: j for j in jobs}
    heap: list[tuple] = []
    seq = 0
    for job in jobs:
        heapq.heappush(heap, (job.arrival_s, 1, seq, "arrival", job.id))
        seq += 1
    done: dict[str, float] = {}

    def dispatch(cidx: int, now_s: float) -> None:
        nonlocal seq
        c = cs[cidx]
        for w in range(c.workers):
            if c.worker_job[w] is not None:
                continue
            item = c.request_work(w, now_s)
            if item is None:
                break
            heapq.heappush(heap, (now_s + item.wall_s, 0, seq, "range_done", (cidx, w, item)))
            seq += 1

    while heap:
        now_s, _, _, kind, payload = heapq.heappop(heap)
        if kind == "arrival":
            job = by_id[payload]
            cidx = shell._route(job, now_s)
            if cidx is None:
                continue
            try:
                cs[cidx].admit(job)
            except Infeasible:
                continue
            dispatch(cidx, now_s)
        else:
            cidx, w, item = payload
            jid = cs[cidx].on_range_done(w, item, now_s)
            if jid is not None:
                done[jid] = now_s
            dispatch(cidx, now_s)
    return done


TOOL_VERSION = "b200-0.1.0"
# sweep.csv columns after the variant and its axes (cli.py:137-151)
SWEEP_CSV_FIXED = ["bubble_ratio", "avg_jct_s", "p99_jct_s", "makespan_s", "completed", "rejected",
                   "recovered_tflops_wallclock", "recovered_tflops_active", "mean_rel_perf",
                   "mean_fill_gpu_hours", "gpus_saved", "main_job_slowdown"]


def write_manifest(out_dir: str | Path, subcommand: str, seed: int, config: Optional[dict] = None) -> None:
    """manifest.json with the reference's keys (cli.py:62-74); the run is configured in code,
    so the config is recorded inline (config_path / trace_path are None)."""
    doc = {"tool_version": TOOL_VERSION, "subcommand": subcommand, "seed": seed, "config_path": None,
           "config_sha256": None, "trace_path": None, "trace_sha256": None}
    if config is not None:
        doc["config"] = config
    Path(out_dir).mkdir(parents=True, exist_ok=True)
    (Path(out_dir) / "manifest.json").write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def write_report(out_dir: str | Path, report: ServiceReport, extra: Optional[dict] = None,
                 seed: Optional[int] = None) -> None:
    """jobs.csv (the reference's columns + model, samples, measured busy, JCT and the
    time model's predicted completion), summary.json (cli.py:80-99) and, with a seed,
    manifest.json (cli.py:62-74)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    with open(out / "jobs.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(JOBS_CSV_COLUMNS + ["model", "samples", "busy_s", "jct_s", "predicted_completion_s"])
        for jid in sorted(report.per_job):
            rec = report.per_job[jid]
            w.writerow([rec.job_id, repr(rec.arrival_s), repr(rec.start_s), repr(rec.completion_s),
                        rec.coordinator, repr(rec.fill_flops), rec.model, rec.samples, repr(rec.busy_s),
                        repr(rec.jct_s), repr(rec.predicted_completion_s)])
    summary = dict(report.scalars())
    summary["tool_version"] = TOOL_VERSION
    summary["rejected_ids"] = sorted(report.rejected)
    summary["unfinished_ids"] = sorted(report.unfinished)
    if extra:
        summary.update(extra)
    (out / "summary.json").write_text(json.dumps(summary, indent=2, sort_keys=True) + "\n")
    if seed is not None:
        write_manifest(out, "serve", seed, extra)


def write_sweep(out_dir: str | Path, rows: Sequence[tuple[str, dict, dict]], seed: int = 0) -> None:
    """sweep.csv in the reference's layout (cli.py:153-185): one row per variant, its axes,
    then SWEEP_CSV_FIXED from that variant's scalars (floats as repr); plus manifest.json.
    `rows` = (variant name, {axis: value}, scalars)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    axis_names = list(rows[0][1]) if rows else []
    with open(out / "sweep.csv", "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["variant", *axis_names, *SWEEP_CSV_FIXED])
        for name, axes, sc in rows:
            w.writerow([name, *[axes[a] for a in axis_names]]
                       + [repr(sc[k]) if isinstance(sc[k], float) else sc[k] for k in SWEEP_CSV_FIXED])
    write_manifest(out, "sweep", seed)


def write_plan(out_dir: str | Path, plan, model_name: str, stage: int, algo: str = "dp") -> None:
    """plan.json as the reference's `partition` subcommand writes it (cli.py:214-236):
    {algo, model, stage, plan_to_dict(plan)..., tool_version}."""
    from .planner import plan_to_dict

    doc: dict = {"algo": algo, "model": model_name, "stage": stage}
    doc.update(plan_to_dict(plan))
    doc["tool_version"] = TOOL_VERSION
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    (out / "plan.json").write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")