"""Multi-job fill service (Placer + per-stage SJF Coordinators + executors).

* ``service.predict`` restates the simulator's dispatch loop
  (pkg/src/bubblefill/sim.py:213-261) over this package's Coordinators and
  Placer; where the reference tree is mounted it is compared with the
  reference's own ``run_sim`` on the same jobs (completion times with ==).
* ``FillService.run`` is driven with stand-in executors that complete a range in
  exactly the plan's number of cycles (wall_s / period): with arrivals on
  iteration boundaries its measured completions must equal the prediction.
"""

import json
import os
import subprocess
import sys

import pytest

import paper_2410_07192_b200 as pf
from paper_2410_07192_b200.coordinator import SJF
from paper_2410_07192_b200.executor import BubbleRecord
from paper_2410_07192_b200.service import FillService, ServiceConfig, predict, write_report

REF_SRC = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (template, samples, arrival in periods, kind)
JOBS = [("bert_base", 6000, 0.0, "batch_inference"), ("xlm_roberta_xl", 2500, 0.0, "batch_inference"),
        ("bert_large", 800, 1.0, "batch_inference"), ("efficientnet", 40000, 2.0, "batch_inference"),
        ("bert_base", 3000, 2.0, "training"), ("swin_large", 1200, 5.0, "batch_inference"),
        ("bert_large", 15000, 7.0, "batch_inference"), ("efficientnet", 9000, 9.0, "training")]
PIPE = dict(p=8, m=8, tf=7.2, tb=16.1, sched="1f1b", fmem=4_500_000_000, dmem=4_500_000_000, ff=0.68)

_REF_SCRIPT = r"""
import json, sys
sys.path.insert(0, %(src)r)
from bubblefill import coordinator, pipeline, sim, workload
P = %(pipe)r
cfg = pipeline.PipelineConfig(P["p"], P["m"], P["tf"], P["tb"], pipeline.ScheduleKind(P["sched"]),
                              P["fmem"], P["dmem"], P["ff"])
jobs = []
for i, (t, n, a, k) in enumerate(%(jobs)r):
    kind = workload.JobKind(k)
    prof = workload.synth_profile(workload.ModelTemplate.by_name(t), kind=kind)
    jobs.append(workload.JobSpec(f"j{i}", a * cfg.period_us / 1e6, prof, kind, n))
out = {}
for routing in ("avg_jct", "makespan", "round_robin", "shortest_queue"):
    sc = sim.SimConfig(cfg, routing=routing, ordering=coordinator.SJF)
    rep = sim.run_sim(sc, jobs)
    out[routing] = {j: r.completion_s for j, r in rep.per_job.items()}
print(json.dumps(out))
"""


def _pipeline():
    P = PIPE
    return pf.PipelineConfig(P["p"], P["m"], P["tf"], P["tb"], pf.ScheduleKind(P["sched"]),
                             P["fmem"], P["dmem"], P["ff"])


def _jobs(cfg):
    out = []
    for i, (t, n, a, k) in enumerate(JOBS):
        kind = pf.JobKind(k)
        prof = pf.synth_profile(pf.ModelTemplate.by_name(t), kind=kind)
        out.append(pf.JobSpec(f"j{i}", a * cfg.period_us / 1e6, prof, kind, n))
    return out


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not mounted")
def test_predict_matches_reference_run_sim():
    script = _REF_SCRIPT % {"src": REF_SRC, "pipe": PIPE, "jobs": JOBS}
    res = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    ref = json.loads(res.stdout)
    cfg = _pipeline()
    jobs = _jobs(cfg)
    for routing, expected in ref.items():
        got = predict(ServiceConfig(cfg, routing=routing, ordering=SJF), jobs)
        assert got == expected, routing


class _StandIn:
    """Completes a range in exactly wall_s / period iterations (the plan's cycles)."""

    def __init__(self, period_s):
        self.period_s = period_s
        self.records, self.item, self.left, self.loads = [], None, 0, []

    @property
    def busy(self):
        return self.item is not None and self.left > 0

    def load(self, item, model):
        self.item = item
        self.left = round(item.wall_s / self.period_s)
        self.loads.append((item.entry.job_id, model))

    def prewarm(self, flag=None):
        pass

    def settle(self):
        return None


def test_service_measured_completions_equal_prediction(tmp_path):
    cfg = _pipeline()
    jobs = _jobs(cfg)
    scfg = ServiceConfig(cfg, routing="avg_jct", ordering=SJF)
    period = cfg.period_us / 1e6
    exs = [_StandIn(period) for _ in range(cfg.num_stages)]
    clock = {"n": 0}

    def run_iteration(stage, ex):
        clock["n"] += 1
        tag = (stage, clock["n"])
        ex.left -= 1
        ex.records.append(BubbleRecord(0, 1, 1, 1, False, 100, 900, tag=tag))
        return {"start": 0, "main_end": 1000, "step_end": 1000, "bubbles": [(0, 0, 1000, tag)]}

    models = {j.model.name: f"model:{j.model.name}" for j in jobs}
    svc = FillService(scfg, models, exs, run_iteration)
    rep = svc.run(jobs, max_rounds=10_000)
    expected = predict(scfg, jobs)
    assert not rep.unfinished and not rep.rejected
    got = {j: r.completion_s for j, r in rep.per_job.items()}
    assert set(got) == set(expected)
    for j in got:
        assert got[j] == pytest.approx(expected[j], rel=1e-12, abs=1e-9), j
    # every stage executor loaded the model object the registry maps the profile to
    assert all(m == f"model:{jobs[int(j[1:])].model.name}" for ex in exs for j, m in ex.loads)
    # busy time comes from the executors' bubble records (100..900 inside 0..1000)
    assert rep.fill_busy_ns == 800 * clock["n"] and rep.bubble_ns == 1000 * clock["n"]
    write_report(tmp_path, rep, {"stages": cfg.num_stages})
    summary = json.loads((tmp_path / "summary.json").read_text())
    assert summary["completed"] == len(jobs)
    header = (tmp_path / "jobs.csv").read_text().splitlines()[0].split(",")
    assert header[:6] == ["id", "arrival_s", "start_s", "completion_s", "coordinator", "flops"]
    # the reference's SimReport.scalars keys are all reported (sim.py:139-153)
    for k in ("bubble_ratio", "recovered_tflops_wallclock", "recovered_tflops_active", "mean_rel_perf",
              "mean_fill_gpu_hours", "gpus_saved", "main_job_slowdown", "avg_jct_s", "p99_jct_s", "makespan_s"):
        assert k in summary, k


def test_report_files_follow_reference_layout(tmp_path):
    """manifest.json / sweep.csv / plan.json carry the reference CLI's keys and columns
    (cli.py:62-74, 137-185, 214-236); plan.json's body is plan_to_dict of the executed plan."""
    from paper_2410_07192_b200.planner import dp_optimal_plan, plan_to_dict
    from paper_2410_07192_b200.service import SWEEP_CSV_FIXED, write_manifest, write_plan, write_sweep

    cfg = _pipeline()
    jobs = _jobs(cfg)
    scfg = ServiceConfig(cfg, routing="avg_jct", ordering=SJF)
    exs = [_StandIn(cfg.period_us / 1e6) for _ in range(cfg.num_stages)]

    def run_iteration(stage, ex):
        ex.left -= 1
        ex.records.append(BubbleRecord(0, 1, 1, 1, False, 100, 900, tag=(stage,)))
        return {"start": 0, "main_end": 1000, "step_end": 1000, "bubbles": [(0, 0, 1000, (stage,))]}

    rep = FillService(scfg, {j.model.name: j.model.name for j in jobs}, exs, run_iteration).run(jobs, 10_000)
    write_report(tmp_path / "v0", rep, {"free_mem_gb": 4.5}, seed=7)
    man = json.loads((tmp_path / "v0" / "manifest.json").read_text())
    assert set(man) >= {"tool_version", "subcommand", "seed", "config_path", "config_sha256", "trace_path",
                        "trace_sha256"} and man["seed"] == 7
    sc = rep.scalars()
    assert 0.0 < sc["bubble_ratio"] <= 1.0 and sc["gpus_saved"] >= 0.0
    write_sweep(tmp_path, [("v0", {"free_mem_gb": 4.5}, sc), ("v1", {"free_mem_gb": 8.0}, sc)])
    lines = (tmp_path / "sweep.csv").read_text().splitlines()
    assert lines[0].split(",") == ["variant", "free_mem_gb", *SWEEP_CSV_FIXED] and len(lines) == 3
    if os.path.isdir(REF_SRC):  # same fixed columns as the reference CLI's sweep.csv
        out = subprocess.run([sys.executable, "-c", f"import sys; sys.path.insert(0, {REF_SRC!r}); "
                              "from bubblefill import cli; print(','.join(cli.SWEEP_CSV_FIXED[1:]))"],
                             capture_output=True, text=True, check=True).stdout.strip()
        assert out.split(",") == SWEEP_CSV_FIXED
    plan = dp_optimal_plan(jobs[0].model, pf.build_bubble_cycle(cfg, 3))
    write_plan(tmp_path / "plan", plan, jobs[0].model.name, 3)
    doc = json.loads((tmp_path / "plan" / "plan.json").read_text())
    assert doc["algo"] == "dp" and doc["stage"] == 3 and doc["model"] == jobs[0].model.name
    assert {k: doc[k] for k in plan_to_dict(plan)} == json.loads(json.dumps(plan_to_dict(plan)))
    write_manifest(tmp_path / "m", "serve", 0, {"x": 1})
    assert json.loads((tmp_path / "m" / "manifest.json").read_text())["config"] == {"x": 1}


def test_service_never_starts_a_job_before_it_arrives():
    """Arrivals in the middle of an iteration are dispatched at the next iteration start:
    start_s >= arrival_s for every job, and no job waits more than one period to start
    when a stage is idle (sim.py:213-261 orders events by time; here time is quantised)."""
    cfg = _pipeline()
    period = cfg.period_us / 1e6
    jobs = [pf.JobSpec(j.id, (i * 0.37 + 0.11) * period, j.model, j.kind, j.samples)
            for i, j in enumerate(_jobs(cfg))]
    scfg = ServiceConfig(cfg, routing="avg_jct", ordering=SJF)
    exs = [_StandIn(period) for _ in range(cfg.num_stages)]

    def run_iteration(stage, ex):
        ex.left -= 1
        ex.records.append(BubbleRecord(0, 1, 1, 1, False, 100, 900, tag=(stage,)))
        return {"start": 0, "main_end": 1000, "step_end": 1000, "bubbles": [(0, 0, 1000, (stage,))]}

    rep = FillService(scfg, {j.model.name: j.model.name for j in jobs}, exs, run_iteration).run(jobs, 10_000)
    assert not rep.unfinished and not rep.rejected
    for r in rep.per_job.values():
        assert r.start_s >= r.arrival_s, r
        assert r.completion_s > r.start_s
    first = min(rep.per_job.values(), key=lambda r: r.arrival_s)
    assert first.start_s - first.arrival_s < period + 1e-9
