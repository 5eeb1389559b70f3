"""Host-side measurement helpers (CPU): the composed pipeline makespan, the slowdown
statistics (max over stages, noise floor), percentiles and the power-aware usable time."""

import math

import paper_2410_07192_b200 as pf
from paper_2410_07192_b200.metrics import distribution, slowdown_stats
from paper_2410_07192_b200.schedule import replay_makespan, with_cooldown


def test_replay_makespan_equals_the_closed_form_period_for_uniform_ops():
    for sched in (pf.ScheduleKind.ONE_F_ONE_B, pf.ScheduleKind.GPIPE):
        for p, m in ((2, 4), (4, 8), (8, 8), (8, 16), (3, 1)):
            cfg = pf.PipelineConfig(p, m, 1.5, 2.25, sched)
            got = replay_makespan(cfg, lambda s, op, j: cfg.t_fwd_us if op == "F" else cfg.t_bwd_us)
            assert got == cfg.period_us


def test_replay_makespan_sees_one_slow_stage():
    """A stage whose ops are 10 % slower slows the whole pipeline (the slowest stage paces
    it); a slowdown in a stage's idle gaps only would not show in its own iteration time."""
    cfg = pf.PipelineConfig(8, 8, 1.0, 2.0, pf.ScheduleKind.ONE_F_ONE_B)
    base = replay_makespan(cfg, lambda s, op, j: 1000.0 if op == "F" else 2000.0)
    slow = replay_makespan(cfg, lambda s, op, j: (1000.0 if op == "F" else 2000.0) * (1.1 if s == 3 else 1.0))
    assert base < slow <= 1.1 * base
    assert slow / base - 1 > 0.02


def test_slowdown_stats_reports_the_worst_stage_and_a_noise_floor():
    on = {0: [101.0, 101.0], 7: [105.0, 105.0]}
    off = {0: [100.0, 100.0, 100.0, 100.0], 7: [100.0, 101.0, 100.0, 101.0]}
    st = slowdown_stats(on, off)
    assert st["argmax_stage"] == 7
    assert math.isclose(st["max"], 105.0 / 100.5 - 1)
    assert math.isclose(st["mean"], (0.01 + 105.0 / 100.5 - 1) / 2)
    assert math.isclose(st["noise_floor"], 1 - 100.0 / 101.0)  # off[0::2] = 100, off[1::2] = 101 at stage 7
    assert slowdown_stats({}, {})["max"] is None


def test_distribution_nearest_rank():
    d = distribution(list(range(1, 201)))
    assert (d["n"], d["p50"], d["p99"], d["max"]) == (200, 100, 198, 200)
    assert distribution([])["p99"] is None


def test_with_cooldown_caps_usable_time_only():
    cfg = pf.PipelineConfig(8, 8, 7.0, 16.0, pf.ScheduleKind.ONE_F_ONE_B, fill_fraction=0.95)
    for s in range(8):
        cyc = pf.build_bubble_cycle(cfg, s)
        cd = with_cooldown(cyc, 10_000)
        assert cd.period_us == cyc.period_us and cd.unfillable_us == cyc.unfillable_us
        for a, b in zip(cyc.bubbles, cd.bubbles):
            assert (a.duration_us, a.free_mem_bytes, a.kind) == (b.duration_us, b.free_mem_bytes, b.kind)
            assert b.usable_us == max(0, min(a.usable_us, a.duration_us - 10_000))
    assert with_cooldown(cyc, 0) is cyc
    # bubbles no longer than min_duration_us are filled whole
    cyc = pf.build_bubble_cycle(cfg, 6)  # fwd-bwd 16 ms, fill-drain 138 ms
    cd = with_cooldown(cyc, 10_000, 50_000)
    assert cd.bubbles[0] == cyc.bubbles[0]
    assert cd.bubbles[1].usable_us == cyc.bubbles[1].duration_us - 10_000


def test_greedy_segments_cut_replicas_at_partition_boundaries():
    from paper_2410_07192_b200.executor import greedy_segments
    from paper_2410_07192_b200.planner import GreedyPlan, greedy_pack

    g = GreedyPlan(((0, 1, 2, 3, 0, 1, 2, 3, 0), (1, 2, 3)), 3)
    assert greedy_segments(g, 4) == [[(0, 0, 4), (1, 0, 4), (2, 0, 1)], [(2, 1, 4)]]
    # empty partitions (zero-length bubbles) stay empty; every node is covered once
    plan = greedy_pack([500, 0, 300], [10**9] * 3, [(100, 1)] * 5)
    segs = greedy_segments(plan, 5)
    covered = sorted((r, i) for part in segs for r, lo, hi in part for i in range(lo, hi))
    assert covered == [(r, i) for r in range(plan.num_replicas) for i in range(5)]
    assert any(part == [] for part in segs)


def test_power_tail_rules():
    import argparse

    import bench
    from paper_2410_07192_b200.engine import _throttle_tail

    args = argparse.Namespace(tail_from_frac=0.375, throttle_ms=50.0, throttle_ctas=64, tail_min_ms=None,
                              tail_frac=1.0, cooldown_ms=20.0)
    assert [bench.tail_on_stage(args, s, 8) for s in range(8)] == [False] * 3 + [True] * 5
    assert [bench.tail_on_stage(args, s, 4) for s in range(4)] == [False, False, True, True]

    class E:
        throttle_ns, throttle_ctas, throttle_min_ns, throttle_frac = 50_000_000, 64, None, 1.0
    assert _throttle_tail(E, 40_000_000) == (0, 0)  # shorter than the window: not throttled
    assert _throttle_tail(E, 120_000_000) == (50_000_000, 64)
    E.short_ctas = 32  # ... unless short bubbles run whole on fewer CTAs
    assert _throttle_tail(E, 40_000_000) == (40_000_000, 32)
    E.short_window_ns = 30_000_000  # ... or only their last 30 ms
    assert _throttle_tail(E, 40_000_000) == (30_000_000, 32)
    assert _throttle_tail(E, 20_000_000) == (20_000_000, 32)
    assert _throttle_tail(E, 120_000_000) == (50_000_000, 64)  # long bubbles: unchanged
    E.short_ctas, E.short_window_ns = 0, None
    E.throttle_min_ns, E.throttle_frac = 20_000_000, 0.6
    assert _throttle_tail(E, 40_000_000) == (24_000_000, 64)
