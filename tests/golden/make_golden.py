"""Generate control-plane golden vectors by running the REFERENCE implementation.

    python tests/golden/make_golden.py        (needs /root/reference; build container only)

Imports the reference package `bubblefill` from /root/reference/pkg/src, feeds it
seeded plain-data inputs (pipeline configs, model profiles + bubble cycles,
multi-stage job scenarios, policy cases) through tests/golden/driver.py, and writes
inputs and outputs to tests/golden/control_plane.json.gz. The parity tests replay
the same inputs on this package and compare with ==.
"""

import gzip
import json
import os
import random
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, HERE)

import bubblefill  # noqa: E402  (the reference)
from bubblefill import coordinator, partition, pipeline, placer, workload  # noqa: E402

import driver  # noqa: E402

assert os.path.realpath(bubblefill.__file__).startswith(REF_SRC), bubblefill.__file__
REF = types.SimpleNamespace(pipeline=pipeline, workload=workload, partition=partition,
                            coordinator=coordinator, placer=placer)
GB = 1_000_000_000


def pipeline_inputs():
    out = []
    for p in (1, 2, 3, 4, 8, 16):
        for m in (1, 2, 3, 8, 16):
            for tf, tb in ((1.0, 2.0), (0.0015, 0.0025), (1.2345, 2.0005), (3.3, 0.7)):
                for sched in ("gpipe", "1f1b"):
                    for ff in (0.68, 0.7):
                        out.append({"p": p, "m": m, "tf": tf, "tb": tb, "sched": sched,
                                    "fmem": 4_500_000_000, "dmem": 2_000_000_000, "ff": ff})
    return out


def rand_model(rng, n_layers, sizes, name, zero_us=False):
    W = workload
    layers = []
    for _ in range(n_layers):
        base = rng.choice([0.0004, 0.01, 0.1, 0.5, 1.0, 2.5]) if zero_us else rng.uniform(0.05, 3.0)
        slope = rng.uniform(0.0, 1.0)
        weight = rng.choice([0, rng.randint(1, 3 * GB)])
        trans1 = rng.randint(1, GB)
        tgrow = rng.uniform(1.0, 2.0)
        exec_ms, mem = {}, {}
        for k, b in enumerate(sizes):
            exec_ms[b] = round(base * (1 + slope * k), 6)
            mem[b] = weight + int(trans1 * (tgrow ** k))
        layers.append(W.LayerProfile(exec_ms, mem, weight, rng.uniform(1e8, 1e10)))
    return W.model_to_json(W.ModelProfile(name, tuple(layers), rng.randint(1, 10**9),
                                          frozenset({W.JobKind.BATCH_INFERENCE, W.JobKind.TRAINING})))


def rand_cycle(rng, stage=0):
    period = rng.randint(20_000, 200_000)
    d1 = rng.randint(0, period // 3)
    d2 = rng.randint(0, period // 3)
    u1 = rng.randint(0, d1) if rng.random() < 0.7 else d1
    u2 = rng.randint(0, d2) if rng.random() < 0.7 else d2
    m1 = rng.choice([rng.randint(0, 4 * GB), 8 * GB, 500_000_000])
    m2 = rng.choice([rng.randint(0, 4 * GB), 8 * GB, 500_000_000])
    return {"bubbles": [[d1, u1, m1, "fwd_bwd"], [d2, u2, m2, "fill_drain"]], "period": period,
            "stage": stage, "unfillable": rng.randint(0, period - d1 - d2)}


def planner_inputs():
    rng = random.Random(2410_07192)
    out = []
    # desk-scale instances, also checked against the exhaustive oracle
    for i in range(160):
        sizes = rng.choice([(1,), (1, 2), (1, 2, 4), (2, 4)])
        n = rng.randint(1, 6)
        model = rand_model(rng, n, sizes, f"toy{i}")
        cyc = rand_cycle(rng)
        cyc["bubbles"][0][1] = rng.randint(1000, 60_000)
        cyc["bubbles"][0][0] = max(cyc["bubbles"][0][0], cyc["bubbles"][0][1])
        cyc["bubbles"][1][1] = rng.randint(0, 60_000)
        cyc["bubbles"][1][0] = max(cyc["bubbles"][1][0], cyc["bubbles"][1][1])
        cyc["period"] = max(cyc["period"], cyc["bubbles"][0][0] + cyc["bubbles"][1][0])
        cyc["unfillable"] = 0
        q = []
        for _ in range(4):
            lo = rng.randrange(n)
            hi = rng.randint(lo + 1, n)
            q.append([lo, hi, [[b, rng.randint(1, 4)] if rng.random() < 0.8 else [0, 0]
                               for b in (rng.choice(sizes), rng.choice(sizes))]])
        out.append({"model": model, "cycle": cyc, "sizes": None, "cap": rng.choice([4, 8]),
                    "tps_queries": q, "oracle": True})
    # larger random instances, including exec times that round to 0 us
    for i in range(120):
        sizes = rng.choice([(1, 2, 4, 8), (1, 2, 4, 8, 16, 32), (4, 8, 16)])
        n = rng.randint(1, 48)
        model = rand_model(rng, n, sizes, f"rand{i}", zero_us=rng.random() < 0.3)
        out.append({"model": model, "cycle": rand_cycle(rng, rng.randint(0, 7)),
                    "sizes": list(sizes[: rng.randint(1, len(sizes))]) if rng.random() < 0.3 else None,
                    "cap": rng.choice([1, 3, 16])})
    # the catalog's synthetic profiles on the configs' analytic cycles
    W, P = workload, pipeline
    for tmpl in W.ModelTemplate:
        for kind in (W.JobKind.BATCH_INFERENCE, W.JobKind.TRAINING):
            for sizes in ((1, 2, 4, 8), (1, 2, 4, 8, 16, 32)):
                try:
                    m = W.synth_profile(tmpl, batch_sizes=sizes, kind=kind)
                except ValueError:
                    continue
                for cfg in (P.PipelineConfig(4, 8, 1.0, 2.0, P.ScheduleKind.ONE_F_ONE_B),
                            P.PipelineConfig(8, 8, 1.0, 2.0, P.ScheduleKind.ONE_F_ONE_B),
                            P.PipelineConfig(8, 8, 1.0, 2.0, P.ScheduleKind.GPIPE,
                                             fwd_free_mem=500_000_000, drain_free_mem=1_000_000_000)):
                    for s in range(cfg.num_stages):
                        out.append({"model": W.model_to_json(m),
                                    "cycle": driver.cycle_to_spec(P.build_bubble_cycle(cfg, s)),
                                    "sizes": None, "cap": 16})
    return out


def scenario_inputs():
    W, P = workload, pipeline
    rng = random.Random(7192)
    models = {}
    for tmpl, kind in ((W.ModelTemplate.BERT_BASE, W.JobKind.BATCH_INFERENCE),
                       (W.ModelTemplate.BERT_LARGE, W.JobKind.BATCH_INFERENCE),
                       (W.ModelTemplate.EFFICIENTNET, W.JobKind.TRAINING),
                       (W.ModelTemplate.XLM_ROBERTA_XL, W.JobKind.BATCH_INFERENCE)):
        m = W.synth_profile(tmpl, kind=kind)
        models[m.name] = W.model_to_json(m)
    names = sorted(models)
    kinds = {n: ("training" if n.endswith("train") else "batch_inference") for n in names}
    out = []
    cfgs = [P.PipelineConfig(4, 8, 1.0, 2.0, P.ScheduleKind.ONE_F_ONE_B),
            P.PipelineConfig(4, 8, 1.0, 2.0, P.ScheduleKind.GPIPE, fwd_free_mem=2 * GB,
                             drain_free_mem=6 * GB)]
    for routing in ("avg_jct", "makespan", "shortest_queue", "round_robin"):
        for ordering in (["fifo"], ["sjf"], ["concurrent", 4000]):
            cfg = cfgs[len(out) % 2]
            workers = 1 + (len(out) % 3)
            t = 0.0
            jobs = []
            for k in range(18):
                t += rng.expovariate(1 / 3.0)
                nm = rng.choice(names)
                jobs.append({"id": f"j{k:03d}", "arrival": round(t, 3), "model": nm,
                             "kind": kinds[nm], "samples": rng.choice([1, 5, 64, 999, 20_000, 123_457])})
            out.append({"models": models, "ordering": ordering, "routing": routing, "workers": workers,
                        "cycles": [driver.cycle_to_spec(P.build_bubble_cycle(cfg, s))
                                   for s in range(cfg.num_stages)],
                        "jobs": jobs})
    return out


def policy_inputs():
    rng = random.Random(55)
    cases = []
    for _ in range(60):
        n = rng.randint(1, 6)
        cases.append({
            "proc": [rng.choice([rng.uniform(0.1, 50), float("inf")]) if k else rng.uniform(0.1, 50)
                     for k in range(n)],
            "arrival": rng.uniform(0, 10),
            "rem": [rng.choice([0.0, rng.uniform(0, 30)]) for _ in range(n)],
            "queue": [([rng.uniform(0.5, 20) for _ in range(n)], rng.choice([0.0, 1.0, 2.5]))
                      for _ in range(rng.randint(1, 5))],
        })
    return {"cases": cases}


def main():
    doc = {"generator": "tests/golden/make_golden.py", "reference": "bubblefill " + bubblefill.__version__}
    pins = pipeline_inputs()
    doc["pipeline"] = [{"in": c, "out": driver.run_pipeline(REF, c)} for c in pins]
    plans = planner_inputs()
    doc["planner"] = [{"in": p, "out": driver.run_planner(REF, p)} for p in plans]
    scen = scenario_inputs()
    doc["scenarios"] = [{"in": s, "out": driver.run_scenario(REF, s)} for s in scen]
    pol = policy_inputs()
    doc["policies"] = {"in": pol, "out": driver.run_policies(REF, pol)}
    text = json.dumps(doc, sort_keys=True, allow_nan=True)
    path = os.path.join(HERE, "control_plane.json.gz")
    with gzip.open(path, "wt") as fh:
        fh.write(text)
    print(f"wrote {path}: {len(pins)} pipeline configs, {len(plans)} plan instances, "
          f"{len(scen)} scenarios, {len(pol['cases'])} policy cases ({len(text)/1e6:.1f} MB raw)")


if __name__ == "__main__":
    main()
