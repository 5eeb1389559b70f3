"""The Executor running Coordinator WorkItems on B200: numerics vs the CPU fp32 oracle,
multi-partition plans (weight staging + activation offload), and preemption/resume."""

import ctypes
import math

import pytest
import torch

from oracle import fill_ref

pytestmark = pytest.mark.gpu

REL_TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def pf():
    import paper_2410_07192_b200 as pf
    from paper_2410_07192_b200 import native

    native.require_device()
    return pf


def tiny_cfg():
    from paper_2410_07192_b200.fillmodels import BertConfig

    return BertConfig("bert_tiny", vocab=1000, hidden=256, heads=4, ffn=1024, layers=3)


def oracle_cls(model, ids):
    x = fill_ref.bert_embeddings(ids, model.oracle_params(0), model.cfg.eps)
    for i in range(1, len(model)):
        x = fill_ref.bert_layer(x, model.oracle_params(i), model.cfg.heads, model.cfg.eps)
    return x[:, 0, :]


def plan_item(pf, model, samples, free_mem, sizes=(4, 8)):
    from paper_2410_07192_b200.profiles import JobSpec, LayerProfile, ModelProfile, JobKind

    layers = []
    for i in range(len(model)):
        w = model[i].weight_bytes()
        layers.append(LayerProfile({b: 0.01 * b for b in sizes}, {b: w + 1_000_000 * b for b in sizes}, w, 1.0))
    prof = ModelProfile("tiny", tuple(layers), 1, frozenset({JobKind.BATCH_INFERENCE}))
    cyc = pf.BubbleCycle((pf.BubbleSpec(1000, 1000, free_mem, pf.BubbleKind.FWD_BWD),
                          pf.BubbleSpec(500, 500, free_mem, pf.BubbleKind.FILL_DRAIN)), 10_000, 0)
    coord = pf.Coordinator(0, cyc, 1)
    job = JobSpec("j0", 0.0, prof, JobKind.BATCH_INFERENCE, samples)
    plan = coord.admit(job)
    return coord.request_work(0, 0.0), plan


def run_to_completion(ex, bubbles_fn, max_bubbles=500):
    k = 0
    while ex.busy and k < max_bubbles:
        ex.fill(bubbles_fn(k))
        k += 1
    ex.settle()
    torch.cuda.synchronize()
    assert not ex.busy
    return k


def test_executor_single_partition_matches_oracle(pf):
    from paper_2410_07192_b200.executor import BubbleSlot, Executor
    from paper_2410_07192_b200.fillmodels import bert, synthetic_ids

    model = bert(tiny_cfg(), seed=3)
    item, plan = plan_item(pf, model, samples=37, free_mem=8_000_000_000)
    assert len(plan.partitions) == 1
    ex = Executor(256 << 20, job_seed=5)
    ex.load(item, model)
    run_to_completion(ex, lambda k: BubbleSlot(k % 2, None, 0))
    got = ex.results().float()
    ids = synthetic_ids(5, 0, 37, model.cfg.seq, model.cfg.vocab)
    ref = oracle_cls(model, ids)
    err = ((got - ref).abs().max() / ref.abs().max()).item()
    assert err < REL_TOL_BF16, err
    assert ex.samples_completed == 37
    ex.close()


def test_executor_multi_partition_offload_matches_single(pf):
    """A memory cap forces a multi-partition plan: weights are staged per partition and
    activations offloaded/reloaded through pinned host memory; results must be
    bit-identical to the single-partition run."""
    from paper_2410_07192_b200.executor import BubbleSlot, Executor
    from paper_2410_07192_b200.fillmodels import bert

    model = bert(tiny_cfg(), seed=4)
    item1, plan1 = plan_item(pf, model, samples=20, free_mem=8_000_000_000)
    w_emb = model[0].weight_bytes()
    w_layer = model[1].weight_bytes()
    # room for the embedding alone or two layers -> >= 2 partitions
    item2, plan2 = plan_item(pf, model, samples=20, free_mem=max(w_emb, 2 * w_layer) + 4_000_000)
    assert len(plan2.partitions) >= 2, plan2
    outs = []
    for item in (item1, item2):
        ex = Executor(256 << 20, job_seed=9)
        ex.load(item, model)
        run_to_completion(ex, lambda k: BubbleSlot(k % 2, None, 0))
        outs.append(ex.results().clone())
        ex.close()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("multi", [False, True])
def test_executor_preemption_resume_is_exact(pf, multi):
    """Bubbles that close mid-batch (timer-cleared flag) must yield, resume at the
    first incomplete kernel, and produce results identical to an unpreempted run --
    also for a multi-partition plan, where a bubble that finishes a partition runs
    ahead into the next one (in-stream weight staging) and may be preempted there."""
    from paper_2410_07192_b200 import native
    from paper_2410_07192_b200.executor import BubbleSlot, Executor
    from paper_2410_07192_b200.fillmodels import bert

    model = bert(tiny_cfg(), seed=6)
    free = 8_000_000_000
    if multi:
        free = max(model[0].weight_bytes(), 2 * model[1].weight_bytes()) + 17_000_000
    item, plan = plan_item(pf, model, samples=48, free_mem=free, sizes=(8, 16))
    if multi:
        assert len(plan.partitions) > 1
    ex0 = Executor(256 << 20, job_seed=2)
    ex0.load(item, model)
    run_to_completion(ex0, lambda k: BubbleSlot(k % 2, None, 0))
    ref = ex0.results().clone()
    ex0.close()

    flag = ctypes.c_void_p()
    native.call("pf_flag_create", ctypes.byref(flag))
    anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
    comm = torch.cuda.Stream()
    ex = Executor(256 << 20, job_seed=2)
    ex.load(item, model)

    def bubble(k):
        # the "main job" busy for a while (host enqueues the fill meanwhile), then
        # open the bubble and close it 50-350 us later
        with torch.cuda.stream(comm):
            torch.cuda._sleep(400_000)
        native.call("pf_read_globaltimer", anchor.data_ptr(), comm.cuda_stream)
        native.call("pf_flag_write_on_stream", flag, 1, comm.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(comm)
        native.call("pf_flag_clear_at", flag, anchor.data_ptr(), 50_000 + 100_000 * (k % 4), None,
                    comm.cuda_stream)
        return BubbleSlot(k % 2, ev, flag.value)

    n = run_to_completion(ex, bubble, max_bubbles=2000)
    aborted = sum(r.aborted for r in ex.records)
    assert aborted > 0, "bubbles were long enough to never preempt; shorten them"
    assert torch.equal(ex.results(), ref), (n, aborted)
    if multi:  # some bubble ran ahead into the next partition
        assert any(r.ran_ahead for r in ex.records)
    ex.close()
    native.call("pf_flag_destroy", flag)


@pytest.mark.parametrize("preempt", [False, True])
def test_greedy_algorithm1_plan_matches_the_dp_plan(pf, preempt):
    """An Algorithm-1 plan (planner.greedy_pack_model, partition.py:425-494)
    executed for real: 3 replicas of the node list packed into two bubbles, partitions that
    cut a replica in the middle (its activation kept in a store slot), partition j in bubble
    kind j mod 2. Results equal the DP single-partition run bit for bit -- also when timer-
    closed bubbles preempt segments mid-way."""
    from paper_2410_07192_b200.executor import BubbleSlot, Executor
    from paper_2410_07192_b200.fillmodels import bert
    from paper_2410_07192_b200.planner import greedy_pack_model
    from paper_2410_07192_b200.profiles import JobKind, JobSpec, LayerProfile, ModelProfile

    model = bert(tiny_cfg(), seed=8)
    b, n = 8, 60
    layers = tuple(LayerProfile({b: 0.01}, {b: model[i].weight_bytes() + (8 << 20)}, model[i].weight_bytes(), 1.0)
                   for i in range(len(model)))
    prof = ModelProfile("tiny-greedy", layers, 1, frozenset({JobKind.BATCH_INFERENCE}))
    cyc = pf.BubbleCycle((pf.BubbleSpec(100, 100, 8_000_000_000, pf.BubbleKind.FWD_BWD),
                          pf.BubbleSpec(60, 60, 8_000_000_000, pf.BubbleKind.FILL_DRAIN)), 10_000, 0)
    gplan = greedy_pack_model(prof, cyc, b)
    assert gplan.num_replicas == 3 and len(gplan.partitions) >= 2, gplan
    coord = pf.Coordinator(0, cyc, 1, batch_sizes=[b])
    coord.admit(JobSpec("g", 0.0, prof, JobKind.BATCH_INFERENCE, n))
    item = coord.request_work(0, 0.0)

    ex0 = Executor(256 << 20, job_seed=4)
    ex0.load(item, model)
    run_to_completion(ex0, lambda k: BubbleSlot(k % 2, None, 0))
    ref = ex0.results().clone()
    ex0.close()

    ex = Executor(256 << 20, job_seed=4)
    ex.load_greedy(item, model, gplan, b)
    if preempt:
        flag = ctypes.c_void_p()
        native_call = __import__("paper_2410_07192_b200.native", fromlist=["call"]).call
        native_call("pf_flag_create", ctypes.byref(flag))
        anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
        comm = torch.cuda.Stream()

        def bubble(k):
            with torch.cuda.stream(comm):
                torch.cuda._sleep(400_000)
            native_call("pf_read_globaltimer", anchor.data_ptr(), comm.cuda_stream)
            native_call("pf_flag_write_on_stream", flag, 1, comm.cuda_stream)
            ev = torch.cuda.Event()
            ev.record(comm)
            native_call("pf_flag_clear_at", flag, anchor.data_ptr(), 60_000 + 120_000 * (k % 4), None,
                        comm.cuda_stream)
            return BubbleSlot(k % 2, ev, flag.value)
        run_to_completion(ex, bubble, max_bubbles=3000)
        assert sum(r.aborted for r in ex.records) > 0
    else:
        run_to_completion(ex, lambda k: BubbleSlot(k % 2, None, 0))
    assert ex.samples_completed == n
    assert torch.equal(ex.results(), ref)
    ex.close()
    if preempt:
        native_call("pf_flag_destroy", flag)


def plan_item_per_kind(pf, model, samples, free_fwd, free_drain, sizes=(4, 16)):
    """plan_item with a different free memory per bubble kind (the loan's effect)."""
    from paper_2410_07192_b200.profiles import JobSpec, LayerProfile, ModelProfile, JobKind

    layers = []
    for i in range(len(model)):
        w = model[i].weight_bytes()
        layers.append(LayerProfile({b: 0.005 + 0.0005 * b for b in sizes}, {b: w + 1_000_000 * b for b in sizes}, w, 1.0))
    prof = ModelProfile("tiny", tuple(layers), 1, frozenset({JobKind.BATCH_INFERENCE}))
    cyc = pf.BubbleCycle((pf.BubbleSpec(1000, 1000, free_fwd, pf.BubbleKind.FWD_BWD),
                          pf.BubbleSpec(500, 500, free_drain, pf.BubbleKind.FILL_DRAIN)), 10_000, 0)
    coord = pf.Coordinator(0, cyc, 1)
    plan = coord.admit(JobSpec("j0", 0.0, prof, JobKind.BATCH_INFERENCE, samples))
    return coord.request_work(0, 0.0), plan


@pytest.mark.parametrize("resident", [False, True])
def test_executor_memory_loan_is_exact_and_returned(pf, resident):
    """Memory loan: the fwd-bwd bubbles are planned with more free memory
    (a lent buffer). resident=False: they run larger batches whose workspace lives in the
    loan; the fill-drain bubbles run region-sized batches. resident=True: the arena cannot
    hold the model at all, so the plan's one partition runs only in the fwd-bwd bubbles
    with its weights and workspace in the loan, restaged at every grant. The lender takes
    the buffer back after every fwd-bwd bubble (revoke) and scribbles over it; bubbles
    close mid-batch, so loan batches yield and must restart. Results equal an
    unpreempted, loan-free run bit for bit."""
    from paper_2410_07192_b200 import native
    from paper_2410_07192_b200.executor import BubbleSlot, Executor
    from paper_2410_07192_b200.fillmodels import bert

    model = bert(tiny_cfg(), seed=8)
    w = sum(model[i].weight_bytes() for i in range(len(model)))
    item, plan = plan_item_per_kind(pf, model, samples=96, free_fwd=8_000_000_000,
                                    free_drain=(w // 4) if resident else w + 8_000_000)
    assert len(plan.partitions) == 1
    want = [16, 0] if resident else [16, 4]
    assert [e.batch_size for e in plan.partitions[0].per_bubble] == want, plan
    ex0 = Executor(256 << 20, job_seed=4)
    ex0.load(item, model)
    run_to_completion(ex0, lambda k: BubbleSlot(k % 2, None, 0))
    ref = ex0.results().clone()
    ex0.close()

    flag = ctypes.c_void_p()
    native.call("pf_flag_create", ctypes.byref(flag))
    anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
    comm = torch.cuda.Stream()
    lender = torch.cuda.Stream()
    loan = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    ex = Executor((w // 2) if resident else (256 << 20), job_seed=4)
    ex.loan_kinds = {0}
    ex.load(item, model)
    assert ex._on_loan(0) == resident

    def bubble(k):
        kind = k % 2
        if kind == 0:  # the lender's copy-out done: lend for the fwd-bwd bubble
            ready = torch.cuda.Event()
            ready.record(lender)
            ready.synchronize()
            ex.lend(loan, ready)
        with torch.cuda.stream(comm):
            torch.cuda._sleep(300_000)
        native.call("pf_read_globaltimer", anchor.data_ptr(), comm.cuda_stream)
        native.call("pf_flag_write_on_stream", flag, 1, comm.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(comm)
        native.call("pf_flag_clear_at", flag, anchor.data_ptr(), 60_000 + 90_000 * (k % 5), None, comm.cuda_stream)
        return BubbleSlot(kind, ev, flag.value)

    k = 0
    while ex.busy and k < 3000:
        ex.fill(bubble(k))
        if k % 2 == 0:  # take the buffer back and overwrite it (the moments' copy-back)
            lender.wait_event(ex.revoke())
            with torch.cuda.stream(lender):
                loan.fill_(0xA5)
        k += 1
    ex.settle()
    torch.cuda.synchronize()
    assert not ex.busy
    assert ex.loan_batches > 0
    assert ex.loan_rollbacks > 0, "no loan batch yielded across a revoke; vary the bubbles"
    assert torch.equal(ex.results(), ref), (k, ex.loan_batches, ex.loan_rollbacks)
    if resident:  # the weights were staged into every loan the fill used
        assert len(ex.stagings) > 3, len(ex.stagings)
    ex.close()
    native.call("pf_flag_destroy", flag)
