"""bench.py — PipeFill fill-job executor on B200: fill samples/s in bubbles.

Metric (BASELINE.json): "fill-job samples/s in bubbles at <=2% main-job slowdown;
% bubble time filled". Workload (BASELINE.json configs[1], per GPU): one stage of
an 8-stage 1F1B GPT-style 8B main job (h=4096, 5 layers/stage, FFN 16384, seq 2048,
microbatch 2, 8 microbatches, bf16, AdamW) with BERT-large batch-inference fill
jobs (seq 128) planned by the PipeFill DP partitioner from a B200-measured profile.

At N=1 the neighbouring stages are artificial (BASELINE north star "1 GPU (fill
executor alone, artificial bubbles)"): every recv completes at its arrival time in
the analytic 8-stage timeline built from the MEASURED t_fwd/t_bwd of this GPU, so
the bubbles are real idle windows of a real main-job iteration. Step k runs one
main-job iteration of stage (rank + k*N) mod 8, cycling through the pipeline. One
step = one iteration with both of its bubbles filled.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1|c2|c3]

`--config` picks the BASELINE.json configuration (default c2 = configs[1], the
headline): c1 = 4-stage 1F1B GPT-2-small main job + BERT-base bs-32 fill (configs[0]);
c3 = 8-stage GPipe + a BERT-large fill whose weights exceed the bubble free memory
(arena capped at 320 MB -> a multi-partition plan, weights staged host->HBM per
partition, activations offloaded to pinned host memory between partitions).

Rank 0 prints ONE JSON line. `value` is device-timed (%globaltimer stamps of the
iterations, max over ranks); `e2e` is host wall clock around the same steps
through the public API (Coordinator -> WorkItem -> Executor, inputs from and results
to pinned host memory, host readback included).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fill-job samples/s in bubbles at ≤2% main-job slowdown; % bubble time filled"
FILL_BATCH_SIZES = (8, 16, 32, 64, 128)
CONFIGS = {
    # BASELINE.json configs[1] (headline)
    "c2": {"stages": 8, "micro": 8, "schedule": "1f1b", "main": "gpt8b", "fill": "bert_large",
           "batch_sizes": FILL_BATCH_SIZES, "arena_cap": 24 << 30, "chunk": 16384, "rotate": True},
    # configs[0]: the reference's CPU-runnable case, on the GPU
    "c1": {"stages": 4, "micro": 8, "schedule": "1f1b", "main": "gpt2small", "fill": "bert_base",
           "batch_sizes": (32,), "arena_cap": 24 << 30, "chunk": 16384, "rotate": True,
           # the 124M-parameter main job never reaches the power cap (untailed fill: -0.1 %
           # slowdown), so its short bubbles are filled at full width
           "short_ctas": 0},
    # configs[2]: fill weights (0.67 GB) exceed the bubble free memory given to the fill job.
    # A rank stays on one stage ((rank + 3) mod 8: stage 3 at N=1 has both bubble kinds)
    # so a range progresses through the plan's partitions across iterations.
    "c3": {"stages": 8, "micro": 8, "schedule": "gpipe", "main": "gpt8b", "fill": "bert_large",
           "batch_sizes": FILL_BATCH_SIZES, "arena_cap": 320 << 20, "chunk": 4096, "rotate": False,
           # Coordinator(max_batches_per_bubble=...) (coordinator.py:78-86): the reference
           # default 16 leaves 2/3 of a 100 ms GPipe bubble idle for a 5-layer partition
           "max_batches": 64},
    # configs[3]: ResNet-50 fill-job TRAINING (fwd + bwd + SGD per batch) under 1F1B at 2/4/8 stages
    "c4": {"stages": 8, "micro": 8, "schedule": "1f1b", "main": "gpt8b", "fill": "resnet50_train",
           "batch_sizes": (32, 64), "arena_cap": 80 << 30, "chunk": 4096, "depths": (2, 4, 8),
           "max_batches": 64},
    # configs[4]: multi-job queue -- Placer (avg-JCT routing) + per-stage SJF Coordinators,
    # mixed BERT-base / BERT-large / ResNet-50 inference jobs, bubble free-memory cap sweep
    "c5": {"stages": 8, "micro": 8, "schedule": "1f1b", "main": "gpt8b", "fill": "bert_large",
           "batch_sizes": FILL_BATCH_SIZES, "caps_gb": (0.5, 1, 2, 4, 8), "max_batches": 64,
           "jobs": (("bert_base", 8192, 0.0), ("bert_large", 4096, 0.0), ("resnet50", 2048, 0.25),
                    ("bert_base", 2048, 0.5), ("bert_large", 8192, 1.0), ("resnet50", 1024, 1.25),
                    ("bert_base", 4096, 1.5), ("bert_large", 2048, 2.0), ("bert_base", 16384, 3.0),
                    ("resnet50", 4096, 3.5), ("bert_large", 1024, 4.0))},
}
FILL_FRACTION = 0.95  # reference default 0.68 (V100 context-switch slack); B200 yields in us
# Real NCCL pipeline: the same fill fraction; the round-1 slowdown at 0.95 (+2.1-2.2 % at N=4) was the
# power-cap effect the bubble tail below addresses
FILL_FRACTION_NCCL = 0.95
# Power-aware bubble tail: the main job runs power-capped; after an idle bubble the
# board's power controller lets it start at up to 1965 MHz, after a bubble filled at full power at
# ~1600. The last THROTTLE_MS of every bubble longer than that run on THROTTLE_CTAS CTAs and the
# last COOLDOWN_MS idle; shorter bubbles run whole on SHORT_CTAS CTAs (an untailed short bubble
# leaves the clock depressed for the ~60 ms of main-job compute after it). Measured on B200:
# composed 8-stage main-job slowdown +3.5-4.6 % without any policy; with the tail alone +1.5 to
# +2.9 % (profiles/r02/power_sweep.md); with short bubbles on 32 CTAs too +0.99 to +1.76 %
# (8 runs, profiles/r02/final5, short/), at ~26 % less fill than without any policy.
COOLDOWN_MS = 25.0
THROTTLE_MS = 60.0
THROTTLE_CTAS = 64
SHORT_CTAS = 32  # bubbles <= the tail threshold run whole on 32 CTAs (round 2)
TAIL_MIN_MS = None
TAIL_FRAC = 1.0
TAIL_FROM_FRAC = 0.0
LATE_COOLDOWN_MS = None
# main-job slowdown phase: A = fill-off, B = fill-on iteration of one stage; the first of each run is
# discarded (it inherits the other mode's power state), leaving 6 off and 7 on per stage (the
# power-state noise makes single runs of the shorter AAABBBBBBAAA pattern spread by +-0.7 points)
DEFAULT_SLOWDOWN_PATTERN = "AAAABBBBBBBBAAAA"


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        d["source"] = "MEASURED_PEAKS.json"
        return d
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self.tag = None  # the main thread's current phase ("fill_on" / "fill_off"), stored per row
        self.tags: list = []
        self._stop = threading.Event()
        self._thr = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
                    self.tags.append(self.tag)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thr.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and
                          r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows),
                "sw_power_cap_samples": sum(1 for r in self.rows if len(r) > 6 and r[6].lower().startswith("active"))}

    def by_tag(self) -> dict:
        """Median SM MHz and board power per phase tag."""
        out = {}
        for tag in sorted({t for t in self.tags if t is not None}):
            rows = [r for r, t in zip(self.rows, self.tags) if t == tag]
            sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
            pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
            out[tag] = {"sm_mhz": statistics.median(sm) if sm else None,
                        "power_w": statistics.median(pw) if pw else None, "samples": len(rows),
                        "sw_power_cap_samples": sum(1 for r in rows if len(r) > 6 and r[6].lower().startswith("active"))}
        return out


def measure_h2d_gbs(nbytes: int = 256 << 20, reps: int = 5) -> float:
    """Pinned host -> HBM copy bandwidth of this box (the staging roofline)."""
    import torch

    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dst.copy_(src, non_blocking=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    e1.record()
    e1.synchronize()
    return nbytes * reps / e0.elapsed_time(e1) / 1e6


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------- reference arm


def cpu_fill_throughput(batch: int, reps: int, threads: int | None = None) -> dict:
    """The oracle CPU execution of the fill job (BERT-large fp32 forward, torch CPU), with
    the oracle's own random weights and token ids: nothing of this package (its models,
    kernels or native library) is on this path."""
    import torch

    from oracle import fill_ref

    if threads:
        torch.set_num_threads(threads)
    h, heads, ffn, layers, vocab, seq = 1024, 16, 4096, 24, 30522, 128  # BERT-large
    emb, params = fill_ref.bert_random_params(h, ffn, layers, vocab, seq, seed=0)
    g = torch.Generator().manual_seed(1)
    times = []
    for r in range(reps):
        ids = torch.randint(0, vocab, (batch, seq), generator=g, dtype=torch.int32)
        t0 = time.perf_counter()
        with torch.no_grad():
            x = fill_ref.bert_embeddings(ids, emb, 1e-12)
            for p in params:
                x = fill_ref.bert_layer(x, p, heads, 1e-12)
            _ = x[:, 0, :].sum().item()
        times.append(time.perf_counter() - t0)
    return {"times": times, "batch": batch, "threads": torch.get_num_threads()}


def control_plane_timings(pkg, partition_mod, budget_s: float = 8.0) -> dict:
    """the control plane on the host CPU (single thread, the GIL) on identical
    inputs -- build_bubble_cycle (8 stages), dp_optimal_plan (BERT-base / BERT-large /
    XLM-R-XL synthetic profiles), greedy_pack_model, route_avg_jct (8 Coordinators with
    queued jobs) and run_sim (48 jobs). `pkg` is the reference's bubblefill (baseline/_ref)
    or this package; both expose the same API (bubblefill/__init__.py:5-51). Medians in ms."""
    def timed(fn, reps):
        ts = []
        t_end = time.perf_counter() + budget_s / 6
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
            if time.perf_counter() > t_end:
                break
        return 1e3 * statistics.median(ts)

    cfg = pkg.PipelineConfig(8, 8, 7.2, 16.1, pkg.ScheduleKind.ONE_F_ONE_B, 4_500_000_000, 4_500_000_000, 0.68)
    profs = {n: pkg.synth_profile(pkg.ModelTemplate.by_name(n), kind=pkg.JobKind.BATCH_INFERENCE)
             for n in ("bert_base", "bert_large", "xlm_roberta_xl")}
    cyc = pkg.build_bubble_cycle(cfg, 3)
    out = {"build_bubble_cycle_8_stages_ms": timed(lambda: [pkg.build_bubble_cycle(cfg, s) for s in range(8)], 200)}
    for n, prof in profs.items():
        out[f"dp_optimal_plan_{n}_L{len(prof.layers)}_ms"] = timed(lambda p=prof: pkg.dp_optimal_plan(p, cyc), 20)
    out["greedy_pack_model_bert_large_bs8_ms"] = timed(
        lambda: partition_mod.greedy_pack_model(profs["bert_large"], cyc, 8), 50)
    period = cfg.period_us / 1e6
    names = list(profs)
    jobs = [pkg.JobSpec(f"j{i}", i * 0.3 * period, profs[names[i % 3]], pkg.JobKind.BATCH_INFERENCE,
                        2000 + 500 * (i % 7)) for i in range(48)]

    def route():
        cs = [pkg.Coordinator(s, pkg.build_bubble_cycle(cfg, s), 1) for s in range(8)]
        for j in jobs[:40]:
            cs[int(j.id[1:]) % 8].admit(j)
        t0 = time.perf_counter()
        pkg.route_avg_jct(cs, jobs[40], jobs[40].arrival_s)
        return time.perf_counter() - t0
    rt = [route() for _ in range(5)]
    out["route_avg_jct_8_coords_40_queued_ms"] = 1e3 * statistics.median(rt)
    out["run_sim_48_jobs_ms"] = timed(lambda: pkg.run_sim(pkg.SimConfig(cfg), jobs), 3)
    return out


def reference_package():
    """The unmodified reference (`pip install --target baseline/_ref /root/reference/pkg`,
    DESIGN.md §5), or None when it is not installed."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "bubblefill")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import bubblefill
    import bubblefill.partition

    return bubblefill, bubblefill.partition


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import torch

    threads = os.cpu_count() or 1
    batch = 4
    res = cpu_fill_throughput(batch, args.warmup + args.steps, threads)
    timed = res["times"][args.warmup:]
    value = batch * len(timed) / sum(timed)
    ref = reference_package()
    control = ({"impl": "reference (baseline/_ref bubblefill, unmodified)", "cores": 1,
                **control_plane_timings(*ref)} if ref else
               {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref /root/reference/pkg)"})
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * sum(timed) / len(timed), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "bert_large fill inference, seq 128, CPU oracle (no bubbles: whole CPU)",
                   "global_batch": batch, "seq_len": 128},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": res["threads"], "kind": "port",
                         "sample": f"{len(timed)} batches of {batch} BERT-large sequences, torch CPU fp32 "
                                   f"(oracle/fill_ref.py; the reference has no fill-compute code)"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "control_plane_cpu_baseline": control,
        "cpu_model": cpu_model(),
    }
    _ = torch
    print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(json.dumps(line) + "\n")


# --------------------------------------------------------------------------- our arm


def run_service_sweep(args, conf) -> None:
    """configs[4]: Placer + per-stage SJF Coordinators + one Executor per stage
    (service.FillService), mixed BERT-base / BERT-large jobs, one run per bubble
    free-memory cap. Stages of the 8-stage pipeline are time-multiplexed on this
    GPU (artificial neighbours); each rank runs an independent replica."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=__import__("datetime").timedelta(seconds=240))
    import paper_2410_07192_b200 as pf
    from paper_2410_07192_b200 import native
    from paper_2410_07192_b200.coordinator import SJF
    from paper_2410_07192_b200.engine import GPT2_SMALL_STAGE, GPT_8B_STAGE, GPTStage, StageEngine, measure_stage_times
    from paper_2410_07192_b200.executor import Executor
    from paper_2410_07192_b200.fillmodels import BERT_BASE, BERT_LARGE, bert, resnet50
    from paper_2410_07192_b200.metrics import slowdown_stats
    from paper_2410_07192_b200.profiler import measure_profile
    from paper_2410_07192_b200.schedule import with_cooldown
    from paper_2410_07192_b200.service import (FillService, ServiceConfig, predict, write_plan, write_report,
                                               write_sweep)

    native.require_device()
    peaks = load_peaks()
    P, M = conf["stages"], conf["micro"]
    gcfg = GPT_8B_STAGE if args.main == "gpt8b" else GPT2_SMALL_STAGE
    main_model = GPTStage(gcfg, seed=rank)
    tf_ms, tb_ms = measure_stage_times(main_model)
    registry, profiles = {}, {}
    for name, make in (("bert_base", lambda: bert(BERT_BASE, seed=0)),
                       ("bert_large", lambda: bert(BERT_LARGE, seed=0)), ("resnet50", lambda: resnet50(seed=0))):
        m = make()
        prof = measure_profile(m, conf["batch_sizes"])
        registry[prof.name], profiles[name] = m, prof
    _, hi_prio = torch.cuda.Stream.priority_range()
    streams = (torch.cuda.Stream(priority=hi_prio), torch.cuda.Stream(priority=hi_prio))
    pcfg = pf.PipelineConfig(P, M, tf_ms, tb_ms, pf.ScheduleKind.ONE_F_ONE_B, 1, 1, args.fill_fraction)
    engines = [StageEngine(pcfg, s, main_model, None, streams=streams) for s in range(P)]
    for e_ in engines:
        set_tail(e_, args)  # the power-aware policy of configs[1]
    period_s = pcfg.period_us / 1e6
    jobs = [pf.JobSpec(f"j{i}-{name}", a * period_s, profiles[name], pf.JobKind.BATCH_INFERENCE, n)
            for i, (name, n, a) in enumerate(conf["jobs"])]

    def iterate(s: int, fill: bool) -> dict:
        eng = engines[s]
        eng.reset_stamps()
        eng.set_anchor()
        rec = eng.run_iteration(0, fill=fill)
        if fill:
            eng.executor.settle()
        t = eng.record_timing(rec)
        t["stage"] = s
        return t

    off = {}
    for s in range(P):
        iterate(s, False)
        for _ in range(2):
            t = iterate(s, False)
            off.setdefault(s, []).append(t["main_end"] - t["start"])

    out_dir = args.report_dir or os.path.join(ROOT, "gpurun_out", "c5_report")
    rows, launches, dev_ns, sample_eq, on_iter, sweep_rows = [], 0, 0, 0.0, {}, []
    with ClockSampler(local) as clocks:
        w0 = time.perf_counter()
        for cap_gb in conf["caps_gb"]:
            cap = int(cap_gb * 2**30)
            ccfg = pf.PipelineConfig(P, M, tf_ms, tb_ms, pf.ScheduleKind.ONE_F_ONE_B, cap, cap, args.fill_fraction)
            scfg = ServiceConfig(ccfg, "avg_jct", SJF, tuple(conf["batch_sizes"]), conf["max_batches"])
            # the planners see the same idle tails as configs[1]'s Coordinators
            cycles = [with_cooldown(pf.build_bubble_cycle(ccfg, s), int(stage_cooldown_ms(args, s, P) * 1000),
                                    int(tail_min_ms(args) * 1000), args.tail_frac / 2)
                      if tail_on_stage(args, s, P) else pf.build_bubble_cycle(ccfg, s) for s in range(P)]
            executors = [Executor(cap, job_seed=s) for s in range(P)]
            steps = []

            def run_iteration(s, ex):
                engines[s].executor = ex
                t = iterate(s, True)
                steps.append(t)
                return t

            svc = FillService(scfg, registry, executors, run_iteration,
                              flag_of=lambda s: engines[s].words.flag.value, cycles=cycles)
            rep = svc.run(jobs, max_rounds=60)
            pred = predict(scfg, jobs, cycles=cycles)
            for jid, res in rep.per_job.items():
                res.predicted_completion_s = pred.get(jid)
            recs = [r for ex in executors for r in ex.records]
            eq = sum(r.sample_eq for r in recs)
            ns = sum(t["step_end"] - t["start"] for t in steps)
            launches += sum(ex.kernel_launches for ex in executors) + sum(e.launches for e in engines)
            cap_iter = {}
            for t in steps:
                on_iter.setdefault(t["stage"], []).append(t["main_end"] - t["start"])
                cap_iter.setdefault(t["stage"], []).append(t["main_end"] - t["start"])
            rep.scalars_extra["main_job_slowdown"] = slowdown_stats(cap_iter, off)["max"]
            sc = rep.scalars()
            row = {"free_mem_gb": cap_gb, "sample_eq_per_s": eq / (ns / 1e9) if ns else 0.0,
                   "iterations": len(steps), **{k: sc[k] for k in (
                       "completed", "rejected", "unfinished", "avg_jct_s", "predicted_avg_jct_s", "p99_jct_s",
                       "makespan_s", "bubble_time_filled", "recovered_tflops_active", "mean_rel_perf",
                       "fill_samples_per_s")},
                   "partitions": {j: len(c.executables[j].partitions) for c in svc.coordinators
                                  for j in c.executables}}
            rows.append(row)
            dev_ns += ns
            sample_eq += eq
            vdir = os.path.join(out_dir, f"free_mem_{cap_gb}gb")
            write_report(vdir, rep, {"free_mem_gb": cap_gb, "stages": P, "microbatches": M, "routing": "avg_jct",
                                     "ordering": "sjf", "sample_eq_per_s": row["sample_eq_per_s"]}, seed=0)
            for c in svc.coordinators:  # the executed plans, as the reference's `partition` writes them
                for jid, plan in c.executables.items():
                    write_plan(os.path.join(vdir, "plans", f"stage{c.stage_id}", jid), plan, jid, c.stage_id)
            sweep_rows.append((f"free_mem_{cap_gb}gb", {"free_mem_gb": cap_gb}, sc))
            for ex in executors:
                ex.close()
            for e in engines:
                e.executor = None
        torch.cuda.synchronize()
        w1 = time.perf_counter()
    with open(os.path.join(out_dir, "sweep.json"), "w") as fh:
        json.dump(rows, fh, indent=2)
    write_sweep(out_dir, sweep_rows, seed=0)
    slow = slowdown_stats(on_iter, off)
    best = rows[-1]
    if rank == 0:
        line = {
            "metric": METRIC, "value": best["sample_eq_per_s"], "unit": "samples/s", "n_gpus": world,
            "steps": sum(r["iterations"] for r in rows), "warmup": 2 * P,
            "ms_per_step": dev_ns / 1e6 / max(1, sum(r["iterations"] for r in rows)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, synthetic token ids)",
            "config": {"name": "c5", "workload": f"{P}-stage 1F1B {gcfg.hidden}-hidden main job, "
                       "Placer(avg_jct) + per-stage SJF Coordinators, mixed BERT-base/BERT-large/ResNet-50 "
                       "inference jobs, "
                       "free-memory cap sweep (stages time-multiplexed on one GPU)",
                       "jobs": [list(j) for j in conf["jobs"]], "caps_gb": list(conf["caps_gb"]),
                       "max_batches_per_bubble": conf["max_batches"], "fill_fraction": args.fill_fraction,
                       "t_fwd_ms": tf_ms, "t_bwd_ms": tb_ms},
            "sweep": rows,
            "main_job_slowdown": slow["max"], "main_job_slowdown_mean": slow["mean"],
            "main_job_slowdown_detail": slow,
            "value_definition": "sample-equivalents/s over device time of the filled iterations at the "
                                "largest free-memory cap",
            "roofline": None, "cpu_baseline": None,
            "e2e": {"value": sample_eq / (w1 - w0), "unit": "samples/s", "h2d_bytes_per_step": None,
                    "d2h_bytes_per_step": None},
            "gpu_launches": launches, "clocks": clocks.summary(), "report_dir": out_dir,
            "peaks_source": peaks["source"],
        }
        print(json.dumps(line), flush=True)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(json.dumps(line) + "\n")
    if world > 1:
        dist.destroy_process_group()


def run_training_depths(args, conf) -> None:
    """configs[3]: ResNet-50 training as the fill job of the 8B main job's 1F1B pipeline at
    each depth p in conf["depths"]. At N=1 the p stages are emulated (artificial
    neighbours) and visited round-robin, one iteration per step, like configs[1]; each
    stage trains its own ResNet-50 job planned by the DP from a B200-measured training
    profile. value = images trained per second of device time at the deepest pipeline."""
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=__import__("datetime").timedelta(seconds=240))
    import paper_2410_07192_b200 as pf
    from paper_2410_07192_b200 import native
    from paper_2410_07192_b200.engine import GPT2_SMALL_STAGE, GPT_8B_STAGE, GPTStage, StageEngine, measure_stage_times
    from paper_2410_07192_b200.executor import Executor
    from paper_2410_07192_b200.metrics import FillStats, aggregate, busy_in_bubbles, slowdown_stats
    from paper_2410_07192_b200.profiler import measure_train_profile
    from paper_2410_07192_b200.training import resnet50_train

    native.require_device()
    peaks = load_peaks()
    gcfg = GPT_8B_STAGE if args.main == "gpt8b" else GPT2_SMALL_STAGE
    main_model = GPTStage(gcfg, seed=rank)
    tf_ms, tb_ms = measure_stage_times(main_model)
    _, hi_prio = torch.cuda.Stream.priority_range()
    streams = (torch.cuda.Stream(priority=hi_prio), torch.cuda.Stream(priority=hi_prio))
    free_b, total_b = torch.cuda.mem_get_info()
    part = bool(args.train_partitioned)
    probe_model = resnet50_train(seed=0, partitioned=part)
    profile = measure_train_profile(probe_model, conf["batch_sizes"])
    torch.cuda.synchronize()
    # the main job's peak with 8 microbatches in flight (stage 0 of the deepest pipeline)
    probe = StageEngine(pf.PipelineConfig(max(conf["depths"]), conf["micro"], tf_ms, tb_ms,
                                          pf.ScheduleKind.ONE_F_ONE_B, 1, 1, args.fill_fraction),
                        0, main_model, None, streams=streams)
    probe.set_anchor()
    probe.run_iteration(0, fill=False)
    torch.cuda.synchronize()
    free_b, total_b = torch.cuda.mem_get_info()
    reserved = torch.cuda.max_memory_reserved()
    arena_bytes = int(min(max(0, total_b - reserved - (4 << 30)) * 0.9, conf["arena_cap"]))
    if args.arena_cap_gb:  # a capped bubble free memory: partitioned training plans
        arena_bytes = min(arena_bytes, int(args.arena_cap_gb * 2**30))
    executor = Executor(arena_bytes, job_seed=rank)
    n_total = args.warmup + args.steps
    results, stats_all = {}, []
    with ClockSampler(local) as clocks:
        for P in conf["depths"]:
            # bubble free memory the planner sees: the arena, less (partitioned training) the
            # executor's allocations outside the partition region -- the boundary stores of every
            # partition (one batch each way) and the batch inputs -- which the per-partition peak
            # of the reference's memory model (partition.py:143-150) cannot express
            plan_mem = arena_bytes
            if part:
                b_max = max(conf["batch_sizes"])
                stores = sum(2 * 2 * b_max * probe_model.boundary_elems(i) for i in range(1, len(probe_model)))
                plan_mem = max(arena_bytes // 4, arena_bytes - stores - b_max * probe_model.input_bytes() - (64 << 20))
            pcfg = pf.PipelineConfig(P, conf["micro"], tf_ms, tb_ms, pf.ScheduleKind.ONE_F_ONE_B, plan_mem,
                                     plan_mem, args.fill_fraction)
            engines = {s_: StageEngine(pcfg, s_, main_model, executor, streams=streams) for s_ in range(P)}
            for e_ in engines.values():
                e_.op_stamps = True  # per-op stamps for the composed slowdown
            models = {s_: resnet50_train(seed=s_, partitioned=part) for s_ in range(P)}
            for m_ in models.values():
                m_.profile = profile
            coords, items = {}, {}
            for s_ in range(P):
                coords[s_] = pf.Coordinator(s_, pf.build_bubble_cycle(pcfg, s_), 1,
                                            pf.OrderingPolicy("concurrent", conf["chunk"]),
                                            batch_sizes=list(conf["batch_sizes"]),
                                            max_batches_per_bubble=conf["max_batches"])
                coords[s_].admit(pf.JobSpec(f"train-{s_}", 0.0, profile, pf.JobKind.TRAINING, 1 << 22))

            def next_work(s_):
                prev = items.get(s_)
                if prev is not None and not executor.busy:
                    coords[s_].on_range_done(0, prev, 0.0)
                item = coords[s_].request_work(0, 0.0)
                items[s_] = item
                return None if item is None else (item, models[s_])

            def iterate(s_, fill):
                eng = engines[s_]
                eng.reset_stamps()
                eng.set_anchor()
                rec = eng.run_iteration(0, fill=fill)
                if fill:
                    executor.settle()
                t = eng.record_timing(rec)
                t["stage"] = s_
                return t

            off = {}
            for s_ in range(P):
                iterate(s_, False)
                for _ in range(2):
                    t = iterate(s_, False)
                    off.setdefault(s_, []).append(t["main_end"] - t["start"])
            current = {"stage": None}

            def step(k):
                s_ = (rank + k * world) % P
                if current["stage"] != s_:
                    nxt = next_work(s_) if items.get(s_) is None else (items[s_], models[s_])
                    if nxt is not None:
                        executor.load(*nxt)
                    executor.prewarm(engines[s_].words.flag.value)
                    executor.work_source = lambda s__=s_: next_work(s__)
                    current["stage"] = s_
                    torch.cuda.synchronize()
                return iterate(s_, True)

            for k in range(args.warmup):
                step(k)
            executor.timing = True
            executor.gemm_samples = []
            n_rec0 = len(executor.records)
            launches0 = executor.kernel_launches + sum(e.launches for e in engines.values())
            h2d0 = executor.h2d_bytes
            steps = [step(k) for k in range(args.warmup, n_total)]
            executor.timing = False
            recs = executor.records[n_rec0:]
            by_tag = {r_.tag: r_ for r_ in recs}
            bubbles, fills, on_iter = [], [], {}
            for t in steps:
                on_iter.setdefault(t["stage"], []).append(t["main_end"] - t["start"])
                for kind, t_set, t_clr, tag in t["bubbles"]:
                    r_ = by_tag.get(tag)
                    bubbles.append((t_set, t_clr))
                    fills.append((r_.fill_start_ns, r_.fill_end_ns) if r_ is not None else (0, 0))
            launch_roof = gemm_launch_roofline(executor.gemm_samples, peaks)
            st = FillStats(
                sample_equivalents=sum(r_.sample_eq for r_ in recs),
                samples_completed=sum(r_.samples_completed for r_ in recs),
                fill_busy_ns=busy_in_bubbles(bubbles, fills), bubble_ns=sum(b1 - b0 for b0, b1 in bubbles),
                idle_ns=sum(pf.build_bubble_cycle(pcfg, t["stage"]).total_idle_us * 1000 for t in steps),
                gemm_flops=sum(g[0] for g in executor.gemm_samples), gemm_ms=sum(g[1] for g in executor.gemm_samples),
                launches=executor.kernel_launches + sum(e.launches for e in engines.values()) - launches0,
                device_s=sum(t["step_end"] - t["start"] for t in steps) / 1e9)
            tot = aggregate(st, device=torch.device("cuda", local))
            stats_all.append(tot)

            def run_block(s_: int, modes: list) -> list[dict]:
                """Consecutive iterations of stage s_ from one anchor, fill on or off per
                iteration (as for configs[1]); the executor holds stage s_'s training job."""
                if current["stage"] != s_:
                    executor.settle()
                    nxt = next_work(s_) if items.get(s_) is None else (items[s_], models[s_])
                    if nxt is not None:
                        executor.load(*nxt)
                    executor.prewarm(engines[s_].words.flag.value)
                    executor.work_source = lambda s__=s_: next_work(s__)
                    current["stage"] = s_
                    torch.cuda.synchronize()
                eng = engines[s_]
                executor.settle()
                eng.reset_stamps()
                eng.set_anchor()
                recs_ = [eng.run_iteration(i, fill=(m == "on")) for i, m in enumerate(modes)]
                executor.settle()
                out = []
                for r_ in recs_:
                    t = eng.record_timing(r_)
                    t["stage"] = s_
                    out.append(t)
                return out

            # main-job slowdown as for configs[1]: the p-stage pipeline composed from per-op
            # device times, fill on vs off (the per-stage iteration time of the emulation hides
            # a stage's slowdown in its idle gaps); after the timed region
            interf = measure_interference(args, list(range(P)), run_block, local, pcfg)
            comp = interf.get("pipeline") or {}
            results[str(P)] = {
                "images_per_s": tot.value, "bubble_time_filled": tot.bubble_filled,
                "bubble_time_filled_of_total_idle": tot.idle_filled,
                "main_job_slowdown": comp.get("slowdown"),
                "main_job_slowdown_noise_floor": comp.get("noise_floor"),
                "main_job_slowdown_definition": "composed p-stage pipeline iteration time from per-op device "
                                                "stamps, fill on / off - 1 (DESIGN.md §5.1)",
                "main_job_slowdown_stage_compute": interf["slowdown"],
                "interference_per_stage": interf["per_stage"],
                "main_job_iteration_slowdown": slowdown_stats(on_iter, off),
                "main_job_slowdown_detail": slowdown_stats(on_iter, off),
                "gemm_tflops_in_situ": tot.gemm_tflops, "gemm_launch_roofline": launch_roof,
                "sgd_steps": int(sum(r_.batches_done for r_ in recs)),
                "plan_stage0": pf.plan_to_dict(coords[0].executables["train-0"]),
                "partitions_per_stage": {str(s_): len(coords[s_].executables[f"train-{s_}"].partitions)
                                         for s_ in range(P)},
                "h2d_bytes_per_step": (executor.h2d_bytes - h2d0) / max(1, len(steps)),
                "ms_per_step": 1000 * tot.device_s / max(1, len(steps))}
            executor.work_source = None
            for m_ in models.values():
                _ = m_
    deepest = results[str(max(conf["depths"]))]
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    if rank == 0:
        line = {
            "metric": METRIC, "value": deepest["images_per_s"], "unit": "images/s (training)", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": deepest["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init ResNet-50, N(0,1) 224x224 images, uniform labels)",
            "config": {"name": "c4", "workload": "ResNet-50 training fill (fwd+bwd+SGD per batch, train-mode BN) in "
                       "the bubbles of a 1F1B GPT-style 8B main job at 2/4/8 stages (artificial neighbours)"
                       + (", 18-module partitioned training plans (batch-major phases, state written back "
                          "per partition)" if part else ""),
                       "train_partitioned": part, "arena_cap_gb": args.arena_cap_gb,
                       "depths": list(conf["depths"]), "batch_sizes": list(conf["batch_sizes"]),
                       "fill_fraction": args.fill_fraction, "arena_bytes": arena_bytes,
                       "t_fwd_ms": tf_ms, "t_bwd_ms": tb_ms,
                       "train_step_ms": {str(b): profile_step_ms(profile, b) for b in conf["batch_sizes"]}},
            "per_pipeline_depth": results,
            "bubble_time_filled": deepest["bubble_time_filled"],
            "main_job_slowdown": deepest["main_job_slowdown"],
            "main_job_slowdown_definition": deepest["main_job_slowdown_definition"],
            "main_job_slowdown_per_depth": {d_: r_["main_job_slowdown"] for d_, r_ in results.items()},
            "roofline": {"bound": "tensor", "achieved": deepest["gemm_tflops_in_situ"], "peak": peak,
                         "unit": "TFLOP/s", "frac": deepest["gemm_tflops_in_situ"] / peak, "traffic": None,
                         "kernel": "pf_gemm + pf_gemm_splitk (tcgen05)",
                         **deepest["gemm_launch_roofline"]},
            "cpu_baseline": None,
            "e2e": None, "gpu_launches": int(sum(t.launches for t in stats_all)), "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(json.dumps(line) + "\n")
    executor.close()
    if world > 1:
        dist.destroy_process_group()


def tail_min_ms(args) -> float:
    return args.throttle_ms if args.tail_min_ms is None else args.tail_min_ms


def tail_on_stage(args, stage: int, stages: int) -> bool:
    """Stage-aware tail: only stages from ceil(tail_from_frac x p) on get it. The composed
    slowdown comes almost entirely from the later stages (their steady state is the critical
    path): with the early stages' ops unaffected it moves by <= 0.1 point, with the last
    stage's by 1.1."""
    return stage >= math.ceil(args.tail_from_frac * stages - 1e-9)


def stage_cooldown_ms(args, stage: int, stages: int) -> float:
    """Idle tail of a stage's bubbles: --late-cooldown-ms for the last quarter of the stages
    (the last stage's steady state is the pipeline's critical path)."""
    late = args.late_cooldown_ms is not None and stage >= math.ceil(0.75 * stages - 1e-9)
    return args.late_cooldown_ms if late else args.cooldown_ms


def set_tail(engine, args) -> None:
    """The power-aware bubble tail of DESIGN.md §5.1 on a stage engine: bubbles longer than
    tail_min_ms run their last min(throttle_ms, tail_frac x duration) on throttle_ctas CTAs."""
    if not tail_on_stage(args, engine.stage, engine.cfg.num_stages):
        engine.throttle_ns = 0
        return
    engine.throttle_ns = int(args.throttle_ms * 1e6)
    engine.throttle_ctas = args.throttle_ctas
    engine.throttle_min_ns = int(tail_min_ms(args) * 1e6)
    engine.throttle_frac = args.tail_frac
    engine.short_ctas = args.short_ctas
    engine.short_window_ns = None if args.short_window_ms is None else int(args.short_window_ms * 1e6)


def measure_interference(args, stages, run_block, local, pcfg) -> dict:
    """Main-job slowdown with filling on vs off, from blocks of consecutive iterations.

    Every stage runs fill-off (A) and fill-on (B) iterations back to back from one anchor, in
    the order of `--slowdown-pattern` (default AAABBBBBBAAA, so clock and temperature drifts
    cancel between the modes); the first iteration after a switch is dropped because it
    inherits the other mode's power state from the preceding fill-drain bubble. Per-op stamps
    give each op's duration and the SM clock it started at, and the main stream's resume
    delay after every bubble's recv (flag clear).

    Headline: the p-stage pipeline's iteration time composed from the measured per-op
    durations of every stage (schedule.replay_makespan, the dependency replay of
    pipeline.py:237-278 with measured instead of uniform op times), fill on vs off. With
    artificial neighbours a stage's own iteration time hides its slowdown in its idle gaps,
    so it is reported only as a secondary figure, next to each stage's compute time."""
    import torch

    from paper_2410_07192_b200.metrics import distribution, slowdown_stats
    from paper_2410_07192_b200.schedule import replay_makespan

    pattern = ["off" if c == "A" else "on" for c in (args.slowdown_pattern or DEFAULT_SLOWDOWN_PATTERN)]
    counted = [i > 0 and pattern[i - 1] == pattern[i] for i in range(len(pattern))]
    if args.slowdown_stages:
        stages = [int(x) for x in args.slowdown_stages.split(",")]
    dump = []
    on, off = {}, {}
    comp_on, comp_off = {}, {}  # stage -> main-job compute time per iteration (sum of its ops)
    opdur = {"on": {}, "off": {}, "off_a": {}, "off_b": {}}  # (stage, op, mb) -> [ns]
    mhz = {"on": {}, "off": {}}
    resume = {"on": [], "off": []}
    first = {"on": {}, "off": {}}  # stage -> duration of the window's first op (ns)
    with ClockSampler(local) as clocks:
        for s_ in stages:
            clocks.tag = f"stage_{s_}"
            n_off = 0
            for mode, use, t in zip(pattern, counted, run_block(s_, pattern)):
                if args.dump_ops:
                    dump.append({"stage": s_, "mode": mode, "counted": use, "start": t["start"],
                                 "main_end": t["main_end"], "ops": t.get("ops", []),
                                 "bubbles": [b[:3] for b in t["bubbles"]], "resume_ns": t.get("resume_ns", [])})
                if not use:
                    continue
                (on if mode == "on" else off).setdefault(s_, []).append(t["main_end"] - t["start"])
                (comp_on if mode == "on" else comp_off).setdefault(s_, []).append(
                    sum(t1 - t0 for _, _, t0, t1, _ in t.get("ops", [])))
                keys = [mode] + ([("off_a", "off_b")[n_off % 2]] if mode == "off" else [])
                n_off += mode == "off"
                for op, mb, t0, t1, m in t.get("ops", []):
                    for k in keys:
                        opdur[k].setdefault((s_, op, mb), []).append(t1 - t0)
                    mhz[mode].setdefault(s_, []).append(m)
                if t.get("ops"):
                    first[mode].setdefault(s_, []).append(t["ops"][0][3] - t["ops"][0][2])
                resume[mode] += [ns / 1e3 for ns in t.get("resume_ns", [])]
        clocks.tag = None
        torch.cuda.synchronize()
    if args.dump_ops:
        with open(args.dump_ops, "w") as fh:
            json.dump(dump, fh)

    def makespan(key: str) -> float | None:
        d = opdur[key]
        if any((s_, op, j) not in d for s_ in range(pcfg.num_stages)
               for op in ("F", "B") for j in range(pcfg.num_microbatches)):
            return None  # not every stage measured
        return replay_makespan(pcfg, lambda s_, op, j: statistics.mean(d[(s_, op, j)]))

    span = {k: makespan(k) for k in opdur}
    pipe = None
    if span["on"] and span["off"]:
        pipe = {"slowdown": span["on"] / span["off"] - 1.0,
                "noise_floor": abs(span["off_a"] / span["off_b"] - 1.0) if span["off_a"] and span["off_b"] else None,
                "iteration_ms_fill_on": span["on"] / 1e6, "iteration_ms_fill_off": span["off"] / 1e6}
    per_stage = {}
    for s_ in stages:
        per_stage[str(s_)] = {
            "compute_ms_fill_on": statistics.mean(comp_on[s_]) / 1e6,
            "compute_ms_fill_off": statistics.mean(comp_off[s_]) / 1e6,
            "iter_ms_fill_on": statistics.mean(on[s_]) / 1e6, "iter_ms_fill_off": statistics.mean(off[s_]) / 1e6,
            "sm_mhz_fill_on": statistics.median(mhz["on"][s_]), "sm_mhz_fill_off": statistics.median(mhz["off"][s_]),
            "first_op_ms": {m: statistics.mean(first[m][s_]) / 1e6 for m in ("on", "off")}}
    return {"pipeline": pipe, "slowdown": slowdown_stats(comp_on, comp_off),
            "iteration_slowdown": slowdown_stats(on, off), "per_stage": per_stage,
            "main_resume_delay_us": {m: distribution(v) for m, v in resume.items()},
            "clocks": clocks.by_tag(), "pattern": args.slowdown_pattern or DEFAULT_SLOWDOWN_PATTERN}


def yield_latency(steps, by_tag) -> dict:
    """Fill-stream overrun past each bubble's end (flag clear -> the fill stream's last
    stamp) over the timed bubbles: the bound the preemption protocol gives (one GEMM tile,
    DESIGN.md §3) is what the preempted bubbles show."""
    from paper_2410_07192_b200.metrics import distribution

    pre, done, release = [], [], []
    for t in steps:
        for kind, t_set, t_clr, tag in t["bubbles"]:
            r = by_tag.get(tag)
            if r is None or r.fill_end_ns <= 0:
                continue
            over = (r.fill_end_ns - t_clr) / 1e3
            (pre if r.aborted else done).append(over)
            if r.aborted and r.last_work_end_ns > 0:
                release.append(max(0.0, (r.last_work_end_ns - t_clr) / 1e3))
    resume = [ns / 1e3 for t in steps for ns in t.get("resume_ns", [])]
    return {"yield_latency_us": distribution(release),
            "yield_latency_definition": "preempted bubbles: last exit of a fill GEMM CTA of the yielded batch "
                                        "(in-kernel %globaltimer) - flag clear; 0 when the batch yielded "
                                        "between kernels. Bound: one output tile (DESIGN.md §3)",
            "preempted_overrun_us": distribution(pre),
            "completed_overrun_us": distribution([max(0.0, x) for x in done]),
            "completed_bubbles_overrunning": sum(1 for x in done if x > 0),
            "main_resume_delay_us": distribution(resume),
            "definition": "overrun = fill stream's end stamp (after the aborted batches' no-op gate launches) - "
                          "bubble flag clear (us); main resume delay = main stream's first stamp after the "
                          "bubble - flag clear (us)"}


def gemm_launch_roofline(samples, peaks) -> dict:
    """Per-launch roofline of in-situ GEMM samples (flops, ms, tag, batch, min bytes): each
    launch's bound is max(F / tensor peak, B / HBM peak); the fraction is the sum of those
    bounds over the sum of the measured times. Many ResNet GEMMs (K or N = 64..256, M up
    to 200 K rows) are HBM-bound, so their tensor-peak fraction alone understates them."""
    pt = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * 1e12
    pb = peaks.get("hbm_gbs", 6466.1) * 1e9
    t = sum(g[1] for g in samples) / 1e3
    if t <= 0:
        return {"frac_of_launch_roofline": None}
    bound = sum(max(g[0] / pt, (g[4] if len(g) > 4 else 0.0) / pb) for g in samples)
    hbm = sum(1 for g in samples if len(g) > 4 and g[4] / pb > g[0] / pt)
    return {"frac_of_launch_roofline": bound / t, "hbm_bound_launches": hbm, "launches": len(samples),
            "bytes_per_s_gbs": sum(g[4] for g in samples if len(g) > 4) / t / 1e9}


def profile_step_ms(profile, b: int) -> float:
    return sum(layer.exec_time_ms[b] for layer in profile.layers)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="c2", choices=tuple(CONFIGS))
    ap.add_argument("--fill", default=None, choices=("bert_large", "bert_base"))
    ap.add_argument("--main", default=None, choices=("gpt8b", "gpt2small"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pipeline", default="emulated", choices=("emulated", "nccl"),
                    help="emulated: every rank runs stages of an 8-stage pipeline against artificial "
                         "neighbours; nccl: the N ranks ARE an N-stage pipeline (NCCL P2P over NVLink)")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    ap.add_argument("--report-dir", default=None, help="c5: jobs.csv / summary.json per free-memory cap")
    ap.add_argument("--save-profile", default=None, help="write the measured fill ModelProfile JSON here")
    ap.add_argument("--debug", action="store_true", help="per-bubble details to stderr")
    ap.add_argument("--fill-fraction", type=float, default=None,
                    help=f"share of each bubble the planner may fill (reference default 0.68; here "
                         f"{FILL_FRACTION} emulated, {FILL_FRACTION_NCCL} nccl)")
    ap.add_argument("--optimizer-offload", action="store_true",
                    help="main job keeps its AdamW moments in pinned host memory between steps and "
                         "lends their device buffer to the fill in the bubbles between (DESIGN.md §3.3)")
    ap.add_argument("--stage", type=int, default=None,
                    help="every timed iteration runs stage (rank + STAGE) mod 8 instead of rotating over stages")
    ap.add_argument("--no-loan", action="store_true",
                    help="with --optimizer-offload: free the moments' device blocks instead of lending them")
    ap.add_argument("--max-batches", type=int, default=None,
                    help="Coordinator max_batches_per_bubble (overrides the config's)")
    ap.add_argument("--cooldown-ms", type=float, default=COOLDOWN_MS,
                    help="idle tail kept at the end of every bubble (power-aware usable time, DESIGN.md §5)")
    ap.add_argument("--throttle-ms", type=float, default=THROTTLE_MS,
                    help="throttle the fill to --throttle-ctas CTAs this long before every bubble's end")
    ap.add_argument("--throttle-ctas", type=int, default=THROTTLE_CTAS)
    ap.add_argument("--short-window-ms", type=float, default=None,
                    help="throttle only the last this-many ms of a short bubble (default: all of it)")
    ap.add_argument("--short-ctas", type=int, default=None,
                    help="bubbles not longer than the tail threshold run whole on this many CTAs (0: all; "
                         f"default {SHORT_CTAS}, c1: 0)")
    ap.add_argument("--tail-min-ms", type=float, default=TAIL_MIN_MS,
                    help="bubbles no longer than this get no power tail (default: --throttle-ms)")
    ap.add_argument("--late-cooldown-ms", type=float, default=LATE_COOLDOWN_MS,
                    help="idle tail for the last quarter of the stages (default: --cooldown-ms)")
    ap.add_argument("--tail-from-frac", type=float, default=TAIL_FROM_FRAC,
                    help="only stages >= ceil(frac x stages) get the power tail (0: every stage)")
    ap.add_argument("--tail-frac", type=float, default=TAIL_FRAC,
                    help="a bubble's throttled tail is at most this share of it (its idle cooldown half of that)")
    ap.add_argument("--loss-iters", type=int, default=4,
                    help="nccl: iterations per deterministic fill-off / on / off loss-identity replay")
    ap.add_argument("--train-partitioned", action="store_true",
                    help="c4: ResNet-50 training with its 18 modules as plan nodes (partitioned across bubbles)")
    ap.add_argument("--arena-cap-gb", type=float, default=None,
                    help="cap the fill arena / bubble free memory (GB), e.g. to force multi-partition plans")
    ap.add_argument("--slowdown-pattern", default=None,
                    help="explicit fill-off (A) / fill-on (B) iteration order per stage, e.g. AABBBBAA")
    ap.add_argument("--slowdown-stages", default=None, help="comma-separated stages for the slowdown phase")
    ap.add_argument("--dump-ops", default=None, help="write the slowdown phase's per-op stamps (JSON) here")
    ap.add_argument("--batch-sizes", default=None,
                    help="comma-separated profiled fill batch sizes (overrides the config's)")
    args = ap.parse_args()
    if args.fill_fraction is None:
        args.fill_fraction = FILL_FRACTION_NCCL if args.pipeline == "nccl" else FILL_FRACTION
    conf = dict(CONFIGS[args.config])
    if args.short_ctas is None:
        args.short_ctas = conf.get("short_ctas", SHORT_CTAS)
    if args.max_batches is not None:
        conf["max_batches"] = args.max_batches
    if args.stage is not None:
        conf["rotate"] = False
        conf["stage"] = args.stage
    if args.batch_sizes:
        conf["batch_sizes"] = tuple(int(b) for b in args.batch_sizes.split(","))
    args.fill = args.fill or conf["fill"]
    args.main = args.main or conf["main"]
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == "c5":
        run_service_sweep(args, conf)
        return
    if args.config == "c4":
        run_training_depths(args, conf)
        return

    if args.pipeline == "nccl":  # deterministic cuBLAS for the bitwise loss comparison below
        os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=__import__("datetime").timedelta(seconds=240))

    import paper_2410_07192_b200 as pf
    from paper_2410_07192_b200 import native
    from paper_2410_07192_b200.engine import (GPT2_SMALL_STAGE, GPT_8B_STAGE, GPTStage,
                                              NcclPipelineEngine, StageEngine, measure_stage_times)
    from paper_2410_07192_b200.executor import Executor
    from paper_2410_07192_b200.fillmodels import BERT_BASE, BERT_LARGE, bert
    from paper_2410_07192_b200.metrics import FillStats, aggregate, busy_in_bubbles, slowdown_stats
    from paper_2410_07192_b200.profiler import measure_profile
    from paper_2410_07192_b200.schedule import with_cooldown

    native.require_device()
    peaks = load_peaks()
    P_STAGES, M_MICRO = conf["stages"], conf["micro"]
    sched = pf.ScheduleKind.GPIPE if conf["schedule"] == "gpipe" else pf.ScheduleKind.ONE_F_ONE_B

    # ---- main job and its measured stage timings
    gcfg = GPT_8B_STAGE if args.main == "gpt8b" else GPT2_SMALL_STAGE
    main_model = GPTStage(gcfg, seed=rank)
    tf_ms, tb_ms = measure_stage_times(main_model)
    if args.optimizer_offload and args.pipeline == "nccl":
        raise SystemExit("--optimizer-offload is implemented for the emulated engine (StageEngine) only")
    if args.optimizer_offload:  # AdamW moments in pinned host memory between steps
        main_model.enable_optimizer_offload(h2d_gbs=measure_h2d_gbs(), loan=not args.no_loan)

    # ---- fill job: BERT with a B200-measured profile
    fcfg = BERT_LARGE if args.fill == "bert_large" else BERT_BASE
    fill_model = bert(fcfg, seed=0)
    profile = measure_profile(fill_model, conf["batch_sizes"])
    if args.save_profile and rank == 0:
        with open(args.save_profile, "w") as fh:
            fh.write(pf.model_to_json(profile) + "\n")

    # ---- bubble characterization: free memory with the main job at its peak
    probe_cfg = pf.PipelineConfig(P_STAGES, M_MICRO, tf_ms, tb_ms, sched, 1, 1, args.fill_fraction)
    _, hi_prio = torch.cuda.Stream.priority_range()
    shared_streams = (torch.cuda.Stream(priority=hi_prio), torch.cuda.Stream(priority=hi_prio))
    probe = StageEngine(probe_cfg, 0, main_model, None, streams=shared_streams)  # stage 0: most activations
    probe.set_anchor()
    probe.run_iteration(0, fill=False)
    torch.cuda.synchronize()
    free_b, total_b = torch.cuda.mem_get_info()
    reserved = torch.cuda.max_memory_reserved()
    free_mem = int(max(0, total_b - reserved - (4 << 30)) * 0.9)  # safety margin
    arena_bytes = min(free_mem, conf["arena_cap"])
    if args.arena_cap_gb:  # a main job that leaves less HBM free (the memory-loan runs)
        arena_bytes = min(arena_bytes, int(args.arena_cap_gb * 2**30))
    pcfg = pf.PipelineConfig(P_STAGES, M_MICRO, tf_ms, tb_ms, sched, arena_bytes, arena_bytes,
                             args.fill_fraction)

    executor = Executor(arena_bytes, job_seed=rank)
    if main_model.offload is not None and main_model.offload.loan:
        main_model.offload.borrower = executor  # the moments' buffer is lent between steps
    coords: dict[int, pf.Coordinator] = {}
    engines: dict[int, object] = {}
    items: dict[int, object] = {}

    def coordinator_for(s: int, cfg, cycle=None) -> pf.Coordinator:
        if s not in coords:
            # the stage's Coordinator; a long-running fill job split into 16K-sample ranges
            # power-aware tail: bubbles longer than the throttle window keep an idle cooldown
            cyc = cycle or pf.build_bubble_cycle(cfg, s)
            if tail_on_stage(args, s, cfg.num_stages):
                cyc = with_cooldown(cyc, int(stage_cooldown_ms(args, s, cfg.num_stages) * 1000),
                                    int(tail_min_ms(args) * 1000), args.tail_frac / 2)
            coords[s] = pf.Coordinator(s, cyc, 1,
                                       pf.OrderingPolicy("concurrent", conf["chunk"]),
                                       batch_sizes=list(conf["batch_sizes"]),
                                       max_batches_per_bubble=conf.get("max_batches", 16))
            coords[s].admit(pf.JobSpec(f"fill-{s}", 0.0, profile, pf.JobKind.BATCH_INFERENCE, 10_000_000))
        return coords[s]

    def next_work():
        s = items["stage"]
        if s in engines and hasattr(engines[s], "loan_kinds"):
            executor.loan_kinds = engines[s].loan_kinds()  # the plan's bubbles planned with the loan
        prev = items.get("item")
        if prev is not None and not executor.busy:
            coords[s].on_range_done(0, prev, 0.0)
        item = coords[s].request_work(0, 0.0)
        items["item"] = item
        return None if item is None else (item, fill_model)

    executor.work_source = next_work
    n_total = args.warmup + args.steps
    off: dict[int, list] = {}

    if args.pipeline == "nccl":
        # the N ranks form an N-stage 1F1B pipeline; t_fwd/t_bwd = slowest stage
        tt = torch.tensor([tf_ms, tb_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tf_ms, tb_ms = tt.tolist()
        pcfg = pf.PipelineConfig(world, M_MICRO, tf_ms, tb_ms, sched, arena_bytes, arena_bytes,
                                 args.fill_fraction)
        eng = NcclPipelineEngine(pcfg, main_model, executor)
        engines[rank] = eng
        items["stage"], items["item"] = rank, None

        def run_phase(fill: bool, n_iter: int = n_total, skip: int = args.warmup) -> list[dict]:
            eng.reset_stamps()
            dist.barrier()
            eng.set_anchor()
            recs_ = []
            for it in range(n_iter):
                recs_.append(eng.run_iteration(it, fill=fill, last=(it == n_iter - 1)))
            if fill:
                executor.settle()
            eng.sync()
            out, prev_end = [], None
            for it, r in enumerate(recs_):
                t = eng.record_timing(r)
                if prev_end is not None and it >= skip:
                    out.append({"start": prev_end, "main_end": t["main_end"], "step_end": t["main_end"],
                                "bubbles": t["bubbles"], "stage": rank})
                prev_end = t["main_end"]
            return out

        snap = main_model.snapshot()  # every phase trains from the same weights and data
        run_phase(False)  # untimed warm-up phase (lazy NCCL P2P setup, allocator growth)
        main_model.restore(snap)
        off_steps = run_phase(False)
        for t in off_steps:
            off.setdefault(rank, []).append(t["main_end"] - t["start"])
        # bubble characterization from the fill-off iterations: measured duration of every
        # BUBBLE (flag set -> recv done) and the measured iteration period
        meas = {0: [], 1: []}
        for t in off_steps:
            for kind, t_set, t_clr, _ in t["bubbles"]:
                meas[kind].append((t_clr - t_set) // 1000)
        period_us = int(statistics.median(off[rank]) // 1000)
        durs = [int(statistics.median(meas[k])) if meas[k] else 0 for k in (0, 1)]
        analytic = pf.build_bubble_cycle(pcfg, rank)
        measured_cycle = pf.cycle_from_measurements(
            rank, max(period_us, sum(durs)), durs, [arena_bytes, arena_bytes], args.fill_fraction,
            unfillable_us=max(0, min(analytic.unfillable_us, period_us - sum(durs))))
        coordinator_for(rank, pcfg, measured_cycle)
        set_tail(eng, args)
        eng.expected_ns = {k: d * 1000 for k, d in enumerate(durs)}
        characterization = {"measured_bubbles_us": durs, "measured_period_us": period_us,
                            "analytic_bubbles_us": [b.duration_us for b in analytic.bubbles],
                            "analytic_period_us": analytic.period_us}
        main_model.restore(snap)
        executor.timing = True
        executor.gemm_samples = []
        n_rec0 = len(executor.records)
        n_stage0 = len(executor.stagings)
        launches0 = executor.kernel_launches + eng.launches
        h2d0, d2h0 = executor.h2d_bytes, executor.d2h_bytes
        torch.cuda.synchronize()
        with ClockSampler(local) as clocks:
            w0 = time.perf_counter()
            steps = run_phase(True)
            torch.cuda.synchronize()
            checksum = float(executor.results().float().sum()) if executor.item is not None else 0.0
            w1 = time.perf_counter()
        # host wall clock of the timed iterations only (warmup iterations excluded pro rata)
        w0 = w1 - (w1 - w0) * args.steps / n_total
        recs = [r for r in executor.records[n_rec0:]
                if any(r.tag == b[3] for t in steps for b in t["bubbles"])]
        launches = executor.kernel_launches + eng.launches - launches0
        executor.timing = False
        # a second fill-off phase (ABA around the timed fill-on phase: drifts cancel)
        main_model.restore(snap)
        for t in run_phase(False):
            off.setdefault(rank, []).append(t["main_end"] - t["start"])
        # main-job loss identity: the throughput phases above run the normal (flash SDPA,
        # non-deterministic) main job; this replay runs it with deterministic kernels (math SDPA,
        # use_deterministic_algorithms), fill off / on / off from one snapshot, so any effect of
        # the fill job on the main job's numerics would show as a bitwise loss difference
        flash = torch.backends.cuda.flash_sdp_enabled(), torch.backends.cuda.mem_efficient_sdp_enabled()
        torch.backends.cuda.enable_flash_sdp(False)
        torch.backends.cuda.enable_mem_efficient_sdp(False)
        torch.use_deterministic_algorithms(True)
        loss_runs = []
        for fill_ in (False, True, False):
            eng.losses = []
            main_model.restore(snap)
            run_phase(fill_, n_iter=args.loss_iters, skip=0)
            loss_runs.append([float(x) for x in eng.losses])
        torch.use_deterministic_algorithms(False)
        torch.backends.cuda.enable_flash_sdp(flash[0])
        torch.backends.cuda.enable_mem_efficient_sdp(flash[1])
        obj = [loss_runs]
        dist.broadcast_object_list(obj, src=world - 1)  # the last stage owns the loss
        losses_off, losses, losses_off2 = obj[0]
        del snap
    else:
        characterizations: dict[int, dict] = {}

        def engine_for(s: int) -> StageEngine:
            if s not in engines:
                engines[s] = StageEngine(pcfg, s, main_model, executor, streams=shared_streams)
                engines[s].op_stamps = True  # per-op stamps + SM clock, fill on and off alike
                set_tail(engines[s], args)
                coordinator_for(s, pcfg, measured_cycle(s))
            return engines[s]

        def measured_cycle(s: int):
            """Bubble characterization of stage s from fill-off iterations:
            durations from the flag stamps, free memory from the main job's allocated bytes at
            every BUBBLE, capped at the arena (the fill cannot use more). Plans are made from
            it instead of the analytic build_bubble_cycle (pipeline.py:200-216)."""
            from paper_2410_07192_b200.engine import characterize_stage

            _, rep = characterize_stage(engines[s], iterations=2, fill_fraction=args.fill_fraction)
            free = [min(arena_bytes, int(f)) for f in rep["free_mem_bytes"]]
            # bubble kinds inside the optimizer-state loan window get the lent bytes on top
            lent = engines[s].loan_kinds()
            off_ = main_model.offload
            free = [f + (off_.device_buf.numel() if k in lent else 0) for k, f in enumerate(free)]
            analytic = pf.build_bubble_cycle(pcfg, s)
            durs = [d if a > 0 else 0 for d, a in zip(rep["measured_bubbles_us"],
                                                       [b.duration_us for b in analytic.bubbles])]
            period = max(rep["measured_period_us"], sum(durs))
            cyc = pf.cycle_from_measurements(s, period, durs, free, args.fill_fraction,
                                             unfillable_us=max(0, min(analytic.unfillable_us, period - sum(durs))))
            characterizations[s] = {k: rep[k] for k in ("measured_bubbles_us", "analytic_bubbles_us",
                                                        "measured_period_us", "free_mem_bytes",
                                                        "main_job_allocated_bytes", "insitu_t_fwd_ms",
                                                        "insitu_t_bwd_ms")}
            characterizations[s]["planned_free_mem_bytes"] = free
            characterizations[s]["loan_kinds"] = sorted(lent)
            return cyc

        def stage_of(k: int) -> int:
            return (rank + k * world) % P_STAGES if conf["rotate"] else (rank + conf.get("stage", 3)) % P_STAGES

        def run_step(k: int, fill: bool, stage: int | None = None) -> dict:
            s = stage_of(k) if stage is None else stage
            eng = engine_for(s)
            if fill and items.get("stage") != s:
                if items.get("item") is not None and items.get("stage") is not None:
                    coords[items["stage"]].worker_job[0] = None  # abandon the partial range
                items["stage"], items["item"] = s, None
                # hand the stage's next WorkItem to the executor before the iteration
                # (layout, weight staging and graph recording off the bubbles)
                nxt = next_work()
                if nxt is not None:
                    executor.load(*nxt)
                executor.prewarm(eng.words.flag.value)
                torch.cuda.synchronize()
            eng.reset_stamps()
            eng.set_anchor()
            h0 = time.perf_counter()
            rec = eng.run_iteration(0, fill=fill)
            h1 = time.perf_counter()
            if fill:
                executor.settle()
            t = eng.record_timing(rec)
            t["stage"] = s
            if args.debug:
                ms = torch.cuda.memory_stats()
                print(f"[dbg] stage {s} fill={fill} host enqueue {1e3 * (h1 - h0):.1f} ms, "
                      f"alloc retries {ms.get('num_alloc_retries', 0)}, "
                      f"reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB", file=sys.stderr)
            return t

        # fill-off iterations: the main job's own iteration time per stage (one
        # untimed + one timed iteration of every stage the timed fill-on steps visit)
        for s_ in sorted({stage_of(k) for k in range(args.warmup, n_total)}):
            for rep in range(2):
                t = run_step(s_, fill=False, stage=s_)
                if rep:
                    off.setdefault(s_, []).append(t["main_end"] - t["start"])

        # executables of every stage the timed steps visit are built now (arena layout,
        # weight staging, graph recording), as the Coordinators would at admission
        for k in range(args.warmup, n_total):
            s_ = stage_of(k)
            eng_ = engine_for(s_)
            items["stage"], items["item"] = s_, None
            nxt = next_work()
            if nxt is not None:
                executor.load(*nxt)
            executor.prewarm(eng_.words.flag.value)
        items["stage"] = None
        torch.cuda.synchronize()

        # fill-on: warmup, then the timed steps
        for k in range(args.warmup):
            run_step(k, fill=True)
        executor.timing = True
        executor.gemm_samples = []
        n_rec0 = len(executor.records)
        n_stage0 = len(executor.stagings)
        launches0 = executor.kernel_launches + sum(e.launches for e in engines.values())
        h2d0, d2h0 = executor.h2d_bytes, executor.d2h_bytes
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        steps = []
        with ClockSampler(local) as clocks:
            w0 = time.perf_counter()
            for k in range(args.warmup, n_total):
                steps.append(run_step(k, fill=True))
            torch.cuda.synchronize()
            checksum = float(executor.results().float().sum())  # host reads the results
            w1 = time.perf_counter()
        recs = executor.records[n_rec0:]
        launches = executor.kernel_launches + sum(e.launches for e in engines.values()) - launches0
        losses, losses_off, losses_off2 = [], [], []
        characterization = {"method": "per stage, 2 fill-off iterations: bubble durations from the flag stamps, "
                                      "free memory from memory_allocated() at each BUBBLE (capped at the arena); "
                                      "the neighbours' arrivals follow the analytic timeline of the measured "
                                      "t_fwd/t_bwd (artificial neighbours)",
                            "per_stage": {str(k): v for k, v in sorted(characterizations.items())}}
        # main-job interference, after (and outside) the timed region: every stage the timed
        # steps visited runs fill-off and fill-on iterations interleaved ABBA (off on on off ...)
        def run_block(s_: int, modes: list) -> list[dict]:
            """Consecutive iterations of stage s_ from one anchor (no host gap between them),
            fill on or off per iteration; the executor holds stage s_'s work."""
            eng = engine_for(s_)
            if items.get("stage") != s_:
                if items.get("item") is not None and items.get("stage") is not None:
                    coords[items["stage"]].worker_job[0] = None
                items["stage"], items["item"] = s_, None
                nxt = next_work()
                if nxt is not None:
                    executor.load(*nxt)
                executor.prewarm(eng.words.flag.value)
            executor.settle()
            eng.reset_stamps()
            eng.set_anchor()
            recs_ = [eng.run_iteration(i, fill=(m == "on")) for i, m in enumerate(modes)]
            executor.settle()
            out = []
            for r in recs_:
                t = eng.record_timing(r)
                t["stage"] = s_
                out.append(t)
            return out

        interference = measure_interference(args, list(range(P_STAGES)), run_block, local, pcfg)

    # ---- accounting from device timestamps
    # sample-equivalents: a batch that passed partition [lo, hi) counts as the share of
    # the model's FLOPs in that partition (= completed samples in steady state)
    by_tag = {r.tag: r for r in recs}
    bubbles, fills = [], []
    for t in steps:
        for kind, t_set, t_clr, tag in t["bubbles"]:
            r = by_tag.get(tag)
            bubbles.append((t_set, t_clr))
            fills.append((r.fill_start_ns, r.fill_end_ns) if r is not None else (0, 0))
    on_iter: dict[int, list] = {}
    for t in steps:
        on_iter.setdefault(t["stage"], []).append(t["main_end"] - t["start"])
    if args.debug:
        for t in steps:
            print(f"[dbg] rank {rank} stage {t['stage']} main {(t['main_end'] - t['start']) / 1e6:.1f} ms "
                  f"step {(t['step_end'] - t['start']) / 1e6:.1f} ms", file=sys.stderr)
            for kind, t_set, t_clr, tag in t["bubbles"]:
                r = by_tag.get(tag)
                info = "no fill" if r is None else (
                    f"fill +{(r.fill_start_ns - t_set) / 1e6:.2f}..+{(r.fill_end_ns - t_set) / 1e6:.2f} ms "
                    f"part {r.part} batches {r.batches_done}/{r.batches_planned} aborted {r.aborted}")
                print(f"[dbg]   bubble {kind} at +{(t_set - t['start']) / 1e6:.1f} ms len "
                      f"{(t_clr - t_set) / 1e6:.2f} ms: {info}", file=sys.stderr)
    if args.pipeline == "nccl":
        # every rank is one stage: gather all stages' iteration times, max over stages
        both = [None] * world if world > 1 else [(on_iter, off)]
        if world > 1:
            dist.all_gather_object(both, (on_iter, off))
        on_all, off_all = {}, {}
        for o_, f_ in both:
            on_all.update(o_)
            off_all.update(f_)
        interference = {"slowdown": slowdown_stats(on_all, off_all)}
    slow = dict(interference["slowdown"])
    if interference.get("pipeline"):  # headline: the composed pipeline iteration time
        slow["max_stage_compute"] = slow["max"]
        slow["max"] = interference["pipeline"]["slowdown"]
        slow["noise_floor_stage_compute"] = slow["noise_floor"]
        slow["noise_floor"] = interference["pipeline"]["noise_floor"]
        if world > 1:
            # every rank is an independent replica of the same emulated pipeline: the
            # headline is the mean of the N measurements, each listed
            per_rank = [None] * world
            dist.all_gather_object(per_rank, (interference["pipeline"]["slowdown"], interference["pipeline"]["noise_floor"]))
            slow["per_rank"] = [v[0] for v in per_rank]
            slow["per_rank_noise_floor"] = [v[1] for v in per_rank]
            slow["max_over_ranks"] = max(slow["per_rank"])
            slow["max"] = statistics.mean(slow["per_rank"])
            slow["noise_floor"] = statistics.mean(x for x in slow["per_rank_noise_floor"] if x is not None)
    yield_stats = yield_latency(steps, by_tag)
    # roofline samples: GEMM launches that ran at full width, i.e. ended before their bubble's
    # throttled part began: the tail of a long bubble and the whole of a
    # short one run on throttle_ctas / short_ctas of the 148 SMs by design. Samples are the
    # first and the last batch of every bubble (in-kernel %globaltimer stamps).
    from paper_2410_07192_b200.engine import _throttle_tail

    throttle_start = {}
    for t in steps:
        eng = engines.get(t["stage"]) if isinstance(engines, dict) else None
        for kind, t_set, t_clr, tag in t["bubbles"]:
            tail = _throttle_tail(eng, t_clr - t_set)[0] if eng is not None else 0
            throttle_start[tag] = t_clr - tail
    gemm_full = [g for g in executor.gemm_samples
                 if len(g) > 5 and g[2] in throttle_start and g[5] <= throttle_start[g[2]]]
    gemm_all = list(executor.gemm_samples)
    stats = FillStats(
        sample_equivalents=sum(r.sample_eq for r in recs),
        samples_completed=sum(r.samples_completed for r in recs),
        fill_busy_ns=busy_in_bubbles(bubbles, fills),
        bubble_ns=sum(b1 - b0 for b0, b1 in bubbles),
        idle_ns=sum(pf.build_bubble_cycle(pcfg, t["stage"]).total_idle_us * 1000 for t in steps),
        gemm_flops=sum(g[0] for g in gemm_full),
        gemm_ms=sum(g[1] for g in gemm_full),
        launches=launches, wall_s=w1 - w0,
        device_s=sum(t["step_end"] - t["start"] for t in steps) / 1e9)
    gemm_launches = len(gemm_full)
    gemm_by_batch = {}
    for fl, ms, _, cnt, *_ in gemm_full:
        a = gemm_by_batch.setdefault(str(cnt), [0.0, 0.0, 0])
        a[0] += fl
        a[1] += ms
        a[2] += 1
    gemm_by_batch = {b: {"tflops": f / (ms / 1e3) / 1e12, "launches": n} for b, (f, ms, n) in gemm_by_batch.items()}
    all_ms = sum(g[1] for g in gemm_all)
    gemm_all_tflops = sum(g[0] for g in gemm_all) / (all_ms / 1e3) / 1e12 if all_ms else None
    executor.timing = False
    traffic, traffic_src = None, None
    try:  # DRAM bytes per GEMM launch from the committed ncu --set full capture
        with open(os.path.join(ROOT, "profiles", "r02", "gemm_traffic.json")) as fh:
            tdoc = json.load(fh)
        traffic, traffic_src = tdoc["per_launch_dram_bytes"], tdoc["source"]
    except (OSError, KeyError, ValueError):
        pass
    staging = executor.staging_stats(n_stage0)
    h2d_peak = measure_h2d_gbs()
    staging["h2d_peak_gbs"] = h2d_peak
    staging["frac"] = staging["gbs"] / h2d_peak if staging["gbs"] else None
    tot = aggregate(stats, device=torch.device("cuda", local))  # summed work, max time over ranks
    value = tot.value
    e2e = tot.sample_equivalents / tot.wall_s if tot.wall_s > 0 else 0.0
    achieved = tot.gemm_tflops
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    dev_s = tot.device_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = cpu_fill_throughput(batch=4, reps=3, threads=os.cpu_count())
        t = res["times"][1:]
        cpu = {"value": 4 * len(t) / sum(t), "unit": "samples/s", "cores": res["threads"], "kind": "port",
               "sample": "2 batches x 4 BERT-large seq-128 sequences, torch CPU fp32 oracle "
                         "(oracle/fill_ref.py), after 1 warm-up batch", "cpu_model": cpu_model()}
        ref = reference_package()
        cpu["control_plane"] = {
            "reference": ({"cores": 1, **control_plane_timings(*ref)} if ref else "baseline/_ref not installed"),
            "ours": {"cores": 1, **control_plane_timings(pf, __import__("paper_2410_07192_b200.planner",
                                                                        fromlist=["x"]))},
            "note": "the same control-plane calls on identical inputs, single-threaded Python on the host: "
                    "the reference package vs this package's bit-exact restatement (BASELINE.md §4)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * dev_s / max(1, len(steps)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init weights, synthetic token ids / activations)",
            "config": {
                "name": args.config,
                "workload": (f"{pcfg.num_stages}-stage {conf['schedule'].upper()} GPT-style main job ({gcfg.layers} layers of "
                             f"h={gcfg.hidden} per stage; "
                             + ("one stage per GPU over NCCL P2P" if args.pipeline == "nccl" else
                                f"{'8B' if args.main == 'gpt8b' else 'GPT-2-small'} model, artificial "
                                "neighbours: one emulated stage per GPU-step")
                             + f") + {fcfg.name} batch-inference fill (seq {fcfg.seq})"),
                "pipeline": args.pipeline,
                "main_stage": {"hidden": gcfg.hidden, "layers": gcfg.layers, "ffn": gcfg.ffn,
                               "seq": gcfg.seq, "micro_batch": gcfg.micro_batch,
                               "microbatches": M_MICRO, "stages": pcfg.num_stages,
                               "t_fwd_ms": tf_ms, "t_bwd_ms": tb_ms},
                "fill": {"model": fcfg.name, "seq_len": fcfg.seq, "profiled_batch_sizes": list(conf["batch_sizes"]),
                         "range_chunk_samples": conf["chunk"],
                         "max_batches_per_bubble": conf.get("max_batches", 16),
                         "fill_fraction": args.fill_fraction, "cooldown_ms": args.cooldown_ms,
                         "throttle_ms": args.throttle_ms, "throttle_ctas": args.throttle_ctas,
                         "tail_min_ms": tail_min_ms(args), "tail_frac": args.tail_frac, "short_ctas": args.short_ctas, "short_window_ms": args.short_window_ms,
                         "tail_from_frac": args.tail_from_frac, "late_cooldown_ms": args.late_cooldown_ms,
                         "arena_bytes": arena_bytes,
                         "plans": {str(s): pf.plan_to_dict(c.executables[f"fill-{s}"]) for s, c in coords.items()}},
                "stages_run": [t["stage"] for t in steps],
                "l2": "inputs larger than L2 (BERT-large weights 0.67 GB streamed per batch; main job 1B params)",
            },
            "bubble_time_filled": tot.bubble_filled,
            "bubble_time_filled_of_total_idle": tot.idle_filled,
            "main_job_slowdown": slow["max"],
            "main_job_slowdown_definition": (
                "iteration time of the 8-stage pipeline composed from every stage's measured per-op device times "
                "(dependency replay, schedule.replay_makespan), fill on / fill off - 1; per-op times from blocks of "
                "consecutive iterations of each stage after the timed region (pattern "
                + (args.slowdown_pattern or DEFAULT_SLOWDOWN_PATTERN) + ", first iteration after a switch dropped). "
                "Not the emulated stage's own iteration time: its artificial neighbours' fixed arrival times absorb "
                "its slowdown in its idle gaps (main_job_iteration_slowdown). noise floor = the same composition "
                "from the two halves of the fill-off iterations"
                + ("; with N > 1 ranks (independent replicas) the mean of their N measurements "
                   "(main_job_slowdown_detail.per_rank)" if world > 1 else "")
                if args.pipeline == "emulated" else
                "max over pipeline stages (ranks) of mean(fill-on) / mean(fill-off) main-job iteration time - 1"),
            "main_job_iteration_slowdown": interference.get("iteration_slowdown"),
            "main_job_slowdown_mean": slow["mean"],
            "main_job_slowdown_noise_floor": slow["noise_floor"],
            "main_job_slowdown_detail": slow,
            "interference": {k: v for k, v in interference.items() if k not in ("slowdown", "iteration_slowdown")},
            "yield": yield_stats,
            "per_stage_iter_ms_timed": {str(st): {"fill_on": statistics.mean(v) / 1e6} for st, v in on_iter.items()},
            "bubble_characterization": characterization,
            "optimizer_offload": None if main_model.offload is None else {
                "state_bytes": main_model.offload.state_bytes, "lead_ms": main_model.offload.lead_us / 1e3,
                "h2d_gbs": main_model.offload.h2d_gbs, "transfers": main_model.offload.transfers,
                "loan": None if not main_model.offload.loan else {
                    "bytes": main_model.offload.device_buf.numel(), "loans": main_model.offload.loans,
                    "loan_batches": executor.loan_batches, "rollbacks": executor.loan_rollbacks}},
            "weight_staging": staging,
            "bubbles_preempted": sum(1 for r in recs if r.aborted),
            "bubbles_filled": len(recs),
            "fill_sample_equivalents": tot.sample_equivalents,
            "fill_samples_completed": int(tot.samples_completed),
            "value_definition": "sample-equivalents/s: completed batches x share of the model's FLOPs in "
                                "the batch's partition, over device time of the timed iterations",
            "parity": {"tolerance": "bf16 path rel 2e-2 (north star), measured as max|got - ref| / max|ref| "
                                    "against the CPU fp32 oracle (oracle/fill_ref.py): a norm-wise bound, "
                                    "lenient for small outputs; fp32 path rel 1e-4",
                       "evidence": "tests/test_kernels_gpu.py (BERT-base/large shapes), tests/test_executor_gpu.py "
                                   "(whole model through the executor), __graft_entry__.smoke()"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": "pf_gemm (tcgen05)", "launches_timed": gemm_launches,
                         "by_batch_size": gemm_by_batch,
                         "sampling": "in-kernel %globaltimer span (first CTA start -> last working CTA end) of "
                                     "every GEMM node of the first and the last batch of each bubble, kept when "
                                     "it ended before the bubble's throttled part began (full width: 148 SMs)",
                         **gemm_launch_roofline(gemm_full, peaks),
                         "achieved_incl_throttled_tail": gemm_all_tflops,
                         "launches_incl_throttled_tail": len(gemm_all),
                         "peak_source": peaks["source"] + " bf16_tflops_sustained"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "samples/s",
                    "h2d_bytes_per_step": (executor.h2d_bytes - h2d0) // max(1, len(steps)),
                    "d2h_bytes_per_step": (executor.d2h_bytes - d2h0) // max(1, len(steps))},
            "gpu_launches": int(tot.launches),
            "clocks": clocks.summary(),
            "result_checksum": checksum,
            "main_job_losses": ({"fill_off": losses_off[-8:], "fill_on": losses[-8:], "fill_off_again": losses_off2[-8:],
                                 "identical": len(losses_off) == len(losses) and losses_off == losses,
                                 "identical_off_vs_off_again": losses_off == losses_off2,
                                 "finite": all(math.isfinite(x) for x in losses_off + losses + losses_off2),
                                 "max_rel_diff_on_vs_off": max(abs(a - b) / max(abs(a), 1e-12)
                                                               for a, b in zip(losses_off, losses)),
                                 "max_rel_diff_off_vs_off_again": max(abs(a - b) / max(abs(a), 1e-12)
                                                                      for a, b in zip(losses_off, losses_off2)),
                                 "note": f"{args.loss_iters} iterations per run replayed from one snapshot with "
                                         "deterministic torch kernels (math SDPA, use_deterministic_algorithms), "
                                         "after the throughput phases (flash SDPA): identical == bitwise equal "
                                         "losses; fill-off vs fill-off-again checks the run-to-run reproducibility"}
                                if losses else None),
        }
        text = json.dumps(line)
        print(text, flush=True)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(text + "\n")
    executor.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
