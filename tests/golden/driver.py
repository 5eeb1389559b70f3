"""Control-plane scenario driver shared by the golden generator and the parity tests.

Every function takes ``ns`` — an object with attributes ``pipeline``, ``workload``,
``partition``, ``coordinator``, ``placer`` — and plain-data inputs, and returns
plain data (ints, exact float reprs, Fractions as "num/den"). make_golden.py runs
it with ns = the reference package (bubblefill, imported from /root/reference);
tests run it with ns = this package through the compat aliases, and compare
outputs with ==.
"""

from __future__ import annotations

import math
from fractions import Fraction


def frac(x: Fraction) -> str:
    return f"{x.numerator}/{x.denominator}"


def fnum(x: float):
    if isinstance(x, float) and not math.isfinite(x):
        return repr(x)
    return x


# ---------------------------------------------------------------- builders


def make_cycle(ns, spec: dict):
    P = ns.pipeline
    bubbles = tuple(P.BubbleSpec(d, u, m, P.BubbleKind(k)) for d, u, m, k in spec["bubbles"])
    return P.BubbleCycle(bubbles=bubbles, period_us=spec["period"], stage_id=spec["stage"],
                         unfillable_us=spec.get("unfillable", 0))


def cycle_to_spec(c) -> dict:
    return {
        "bubbles": [[b.duration_us, b.usable_us, b.free_mem_bytes, b.kind.value] for b in c.bubbles],
        "period": c.period_us,
        "stage": c.stage_id,
        "unfillable": c.unfillable_us,
    }


def make_config(ns, cfg: dict):
    P = ns.pipeline
    return P.PipelineConfig(cfg["p"], cfg["m"], cfg["tf"], cfg["tb"], P.ScheduleKind(cfg["sched"]),
                            cfg["fmem"], cfg["dmem"], cfg["ff"])


# ---------------------------------------------------------------- pipeline


def run_pipeline(ns, cfg: dict) -> dict:
    P = ns.pipeline
    c = make_config(ns, cfg)
    out = {
        "period": c.period_us,
        "tf_us": c.t_fwd_us,
        "tb_us": c.t_bwd_us,
        "fraction": frac(P.bubble_fraction(c.num_stages, c.num_microbatches)),
        "stages": [],
    }
    for s in range(c.num_stages):
        cyc = P.build_bubble_cycle(c, s)
        rec = cycle_to_spec(cyc)
        rec["idle"] = frac(cyc.idle_fraction)
        if c.num_stages * c.num_microbatches <= 256:
            rec["timeline"] = list(P.timeline_bubble_spans(c, s))
        out["stages"].append(rec)
    if c.num_stages * c.num_microbatches <= 256:
        out["idle_intervals"] = [[list(g) for g in st] for st in P.brute_force_schedule_timeline(c)]
    return out


# ---------------------------------------------------------------- planner


def plan_record(Pa, plan) -> dict:
    return {
        "dict": Pa.plan_to_dict(plan),
        "total": frac(plan.total_tps_us),
        "parts": [[p.lo, p.hi, [[e.batch_size, e.num_batches] for e in p.per_bubble],
                   frac(p.tps_us), p.busy_us_per_cycle] for p in plan.partitions],
        "wall": [plan.range_wall_us(n) for n in (1, 7, 32, 100, 1000)],
        "busy": [plan.range_busy_us(n) for n in (1, 7, 32, 100, 1000)],
    }


def run_planner(ns, inst: dict) -> dict:
    W, Pa = ns.workload, ns.partition
    model = W.model_from_json(inst["model"])
    cycle = make_cycle(ns, inst["cycle"])
    sizes = inst.get("sizes")
    cap = inst.get("cap", 16)
    out: dict = {}
    try:
        out["dp"] = plan_record(Pa, Pa.dp_optimal_plan(model, cycle, sizes, cap))
    except Pa.Infeasible as exc:
        out["dp"] = {"infeasible": str(exc)}
    try:
        out["fixed"] = plan_record(Pa, Pa.fixed_batch_baseline(model, cycle, sizes, cap))
    except Pa.Infeasible as exc:
        out["fixed"] = {"infeasible": str(exc)}
    greedy = {}
    for b in model.batch_sizes:
        try:
            g = Pa.greedy_pack_model(model, cycle, b)
            greedy[str(b)] = [[list(p) for p in g.partitions], g.num_replicas]
        except Pa.Infeasible as exc:
            greedy[str(b)] = {"infeasible": str(exc)}
        except ValueError as exc:
            greedy[str(b)] = {"value_error": str(exc)}
    out["greedy"] = greedy
    tps = []
    for lo, hi, entries in inst.get("tps_queries", []):
        plan = [Pa.BubblePlanEntry(b, n) for b, n in entries]
        r = Pa.partition_tps(model, lo, hi, plan, cycle)
        tps.append(None if r is None else frac(r))
    out["tps"] = tps
    if inst.get("oracle"):
        try:
            out["oracle_total"] = frac(Pa.brute_force_plan_oracle(model, cycle, sizes, min(cap, 8)).total_tps_us)
        except Pa.Infeasible as exc:
            out["oracle_total"] = {"infeasible": str(exc)}
    out["fingerprint_len"] = len(model.fingerprint()[2])
    out["peak"] = [model.peak_mem_bytes(b) for b in model.batch_sizes]
    out["exec"] = [model.exec_time_us(b) for b in model.batch_sizes]
    return out


# ---------------------------------------------------------------- coordinator + placer


def run_scenario(ns, sc: dict) -> dict:
    """Event-driven multi-stage scenario: jobs arrive, are routed, admitted, and
    dispatched to workers; every decision and prediction is logged."""
    W, C, Pl, Pa = ns.workload, ns.coordinator, ns.placer, ns.partition
    models = {name: W.model_from_json(text) for name, text in sc["models"].items()}
    if sc["ordering"][0] == "concurrent":
        ordering = C.OrderingPolicy("concurrent", sc["ordering"][1])
    else:
        ordering = C.OrderingPolicy(sc["ordering"][0])
    coords = [C.Coordinator(i, make_cycle(ns, spec), sc["workers"], ordering,
                            sc.get("sizes"), sc.get("cap", 16))
              for i, spec in enumerate(sc["cycles"])]
    log: list = []
    events = []  # (time, prio, seq, payload)
    seq = 0
    for j in sc["jobs"]:
        events.append((j["arrival"], 1, seq, ("arrival", j)))
        seq += 1
    rr = 0
    import heapq

    heapq.heapify(events)

    def dispatch(ci: int, now: float):
        nonlocal seq
        c = coords[ci]
        for w in range(c.workers):
            if c.worker_job[w] is not None:
                continue
            item = c.request_work(w, now)
            if item is None:
                break
            log.append(["dispatch", ci, w, item.entry.job_id, item.entry.lo, item.entry.hi,
                        item.reuse, fnum(item.wall_s), fnum(item.busy_s)])
            heapq.heappush(events, (now + item.wall_s, 0, seq, ("done", ci, w, item)))
            seq += 1

    while events:
        now, _, _, payload = heapq.heappop(events)
        if payload[0] == "arrival":
            j = payload[1]
            job = W.JobSpec(j["id"], j["arrival"], models[j["model"]], W.JobKind(j["kind"]), j["samples"])
            # plan-query predictions of every coordinator, before routing
            for ci, c in enumerate(coords):
                q, jct = c.hypothetical_plan(job, now)
                log.append(["hyp", ci, job.id, [[e.job_id, e.lo, e.hi] for e in q],
                            [[k, fnum(v)] for k, v in jct.items()]])
            mode = sc["routing"]
            if mode == "avg_jct":
                ci = Pl.route_avg_jct(coords, job, now)
            elif mode == "makespan":
                ci = Pl.route_makespan_min(coords, job, now)
            elif mode == "shortest_queue":
                ci = Pl.route_shortest_queue(coords)
            else:
                ci = Pl.route_round_robin(rr, len(coords))
                rr += 1
            log.append(["route", job.id, ci])
            if ci is None:
                continue
            try:
                coords[ci].admit(job)
            except Pa.Infeasible as exc:
                log.append(["reject", job.id, str(exc)])
                continue
            log.append(["admit", ci, job.id, fnum(coords[ci].proc_key[job.id][0]),
                        [[e.job_id, e.lo, e.hi] for e in coords[ci].queue]])
            dispatch(ci, now)
        else:
            _, ci, w, item = payload
            done = coords[ci].on_range_done(w, item, now)
            if done is not None:
                log.append(["complete", ci, done, fnum(now)])
            for jid in sorted(coords[ci].jobs):
                if jid not in coords[ci].completed_at_s:
                    log.append(["jct", ci, jid, fnum(coords[ci].estimate_jct(jid, now))])
            dispatch(ci, now)
    views = []
    for ci, c in enumerate(coords):
        views.append([fnum(t) for t in c.rem_times_s(0.0)])
    return {"log": log, "rem": views}


def run_policies(ns, pol: dict) -> dict:
    Pl = ns.placer
    out = []
    for case in pol["cases"]:
        view = Pl.JobView(tuple(case["proc"]), case["arrival"])
        rem = case["rem"]
        scores = []
        for i in range(len(rem)):
            scores.append([fnum(Pl.executor_score(Pl.Sjf(), view, rem, i)),
                           fnum(Pl.executor_score(Pl.MakespanMin(), view, rem, i)),
                           fnum(Pl.executor_score(Pl.Composite(((0.3, Pl.Sjf()), (0.7, Pl.MakespanMin()))),
                                                  view, rem, i))])
        jobs = [(f"q{k}", Pl.JobView(tuple(p), a)) for k, (p, a) in enumerate(case["queue"])]
        picks = [Pl.pick_next_job(Pl.MakespanMin(), jobs, rem, i) for i in range(len(rem))]
        picks_sjf = [Pl.pick_next_job(Pl.Sjf(), jobs, rem, i) for i in range(len(rem))]
        out.append({"scores": scores, "picks": picks, "picks_sjf": picks_sjf})
    return {"cases": out}
