"""N>1 host logic on CPU with the gloo backend (world size 2): per-rank fill stats are
summed (work) and maxed (time) exactly as bench.py does over NCCL."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2410_07192_b200.metrics import FillStats, aggregate, busy_in_bubbles, mean_slowdown


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st = FillStats(sample_equivalents=100.0 * (rank + 1), samples_completed=64 * rank,
                   fill_busy_ns=1e6 * (rank + 1), bubble_ns=2e6, idle_ns=3e6, gemm_flops=1e12,
                   gemm_ms=1.0 + rank, launches=10, wall_s=1.0 + rank, device_s=0.5 + rank)
    out = aggregate(st)
    q.put((rank, out.as_dict()))
    dist.destroy_process_group()


def test_aggregate_over_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        d = res[r]
        assert d["sample_equivalents"] == 300.0 and d["samples_completed"] == 64
        assert d["fill_busy_ns"] == 3e6 and d["bubble_ns"] == 4e6 and d["launches"] == 20
        assert d["wall_s"] == 2.0 and d["device_s"] == 1.5  # max over ranks
    st = FillStats(**res[0])
    assert st.value == 200.0 and st.bubble_filled == 0.75


def test_busy_in_bubbles_clips_to_bubble_windows():
    bubbles = [(100, 200), (300, 400), (500, 600)]
    fills = [(110, 190), (350, 450), (0, 0)]
    assert busy_in_bubbles(bubbles, fills) == 80 + 50


def test_mean_slowdown():
    assert mean_slowdown({0: [102.0], 1: [99.0]}, {0: [100.0], 1: [100.0]}) == pytest.approx(0.005)
    assert mean_slowdown({}, {}) is None
