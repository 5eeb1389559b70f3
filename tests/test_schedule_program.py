"""BUBBLE instruction placement and the per-instruction timeline the engine executes."""

import itertools

import pytest

from paper_2410_07192_b200.schedule import (
    BubbleKind,
    PipelineConfig,
    ScheduleKind,
    build_bubble_cycle,
    cycle_from_measurements,
    program_timeline,
    stage_program,
    steady_state_timeline,
    timeline_bubble_spans,
)


def cfgs():
    for p, m, sched, (tf, tb) in itertools.product(range(1, 9), (1, 2, 3, 8, 16), ScheduleKind,
                                                   ((1.0, 2.0), (0.7, 1.9))):
        yield PipelineConfig(p, m, tf, tb, sched)


def test_bubbles_sit_before_first_backward_and_after_last():
    for c in cfgs():
        for s in range(c.num_stages):
            prog = stage_program(c, s)
            ops = [i.op for i in prog]
            cyc = build_bubble_cycle(c, s)
            fb, fd = cyc.bubbles
            assert ops.count("F") == c.num_microbatches == ops.count("B")
            if fb.duration_us > 0:
                k = ops.index("BUBBLE")
                assert prog[k].kind is BubbleKind.FWD_BWD and ops[k + 1] == "B" and "B" not in ops[:k]
            else:
                assert all(i.kind is not BubbleKind.FWD_BWD for i in prog)
            if fd.duration_us > 0:
                assert prog[-1].op == "BUBBLE" and prog[-1].kind is BubbleKind.FILL_DRAIN
            else:
                assert prog[-1].op == "B"


def test_timeline_bubbles_match_analytic_durations():
    """The engine's BUBBLE windows equal the closed-form bubble durations (pipeline.py:160-216)."""
    for c in cfgs():
        for s in range(c.num_stages):
            cyc = build_bubble_cycle(c, s)
            tl = program_timeline(c, s)
            spans = {ins.kind: end - start for ins, start, end in tl if ins.op == "BUBBLE"}
            fb, fd = cyc.bubbles
            assert spans.get(BubbleKind.FWD_BWD, 0) == fb.duration_us
            assert spans.get(BubbleKind.FILL_DRAIN, 0) == fd.duration_us
            # compute ops are back to back with the analytic durations
            for ins, start, end in tl:
                if ins.op == "F":
                    assert end - start == c.t_fwd_us
                elif ins.op == "B":
                    assert end - start == c.t_bwd_us
            assert timeline_bubble_spans(c, s)[:2] == (fb.duration_us, fd.duration_us)


def test_busy_plus_idle_is_period():
    for c in cfgs():
        for s in range(c.num_stages):
            tl = program_timeline(c, s)
            busy = sum(e - b for i, b, e in tl if i.op != "BUBBLE")
            cyc = build_bubble_cycle(c, s)
            assert busy + cyc.total_idle_us == c.period_us


def test_steady_state_window_is_one_period():
    """The emulated engine's window: first compute at 0, the fill-drain BUBBLE closes at
    exactly one period, bubble durations and instruction order unchanged."""
    for c in cfgs():
        for s in range(c.num_stages):
            tl, ss = program_timeline(c, s), steady_state_timeline(c, s)
            assert [i for i, _, _ in tl] == [i for i, _, _ in ss]
            assert [e - b for _, b, e in tl] == [e - b for _, b, e in ss]
            assert min(b for i, b, _ in ss if i.op != "BUBBLE") == 0
            assert max(e for _, _, e in ss) <= c.period_us
            for i, b, e in ss:
                if i.op == "BUBBLE" and i.kind is BubbleKind.FILL_DRAIN:
                    assert e == c.period_us


def test_cycle_from_measurements_uses_reference_usable_rule():
    cyc = cycle_from_measurements(3, 45_000, [14_000, 9_001], [4_000_000_000, 2_000_000_000], 0.7)
    assert cyc.bubbles[0].usable_us == int(14_000 * 0.7) and cyc.bubbles[1].usable_us == 6300
    assert cyc.bubbles[1].kind is BubbleKind.FILL_DRAIN and cyc.stage_id == 3
    with pytest.raises(ValueError):
        cycle_from_measurements(0, 10, [20], [1])  # bubbles exceed the period


def test_loan_window_kinds_8_stage_1f1b():
    """Optimizer-state loan window (engine.loan_window_kinds): the fwd-bwd
    bubble of stages 0-6 opens after the previous step's copy-out and before the copy-back;
    the fill-drain bubble opens at the step, before the copy-out has finished."""
    import paper_2410_07192_b200 as pf
    from paper_2410_07192_b200.engine import loan_window_kinds
    from paper_2410_07192_b200.schedule import steady_state_timeline

    cfg = pf.PipelineConfig(8, 8, 12.0, 24.0, pf.ScheduleKind.ONE_F_ONE_B, 1, 1, 0.9)
    got = [loan_window_kinds(steady_state_timeline(cfg, s), cfg.period_us, 94_000) for s in range(8)]
    assert got == [{0}] * 7 + [set()]
    # a copy-back issued earlier than the fwd-bwd bubble closes the window for it
    got = [loan_window_kinds(steady_state_timeline(cfg, s), cfg.period_us, 400_000) for s in range(8)]
    assert all(0 not in g for g in got[:3]), got
    # no transfer time: the fill-drain bubble right after the step is inside too
    assert loan_window_kinds(steady_state_timeline(cfg, 3), cfg.period_us, 0) == {0, 1}
