"""Main-job optimizer-state offload (engine.OptimizerOffload).

The bubble before the first backward sees the AdamW moments' bytes as free HBM. The main
job's parameters after several iterations are bitwise those of a run without offload, also
when the moments' device buffer is lent to a filling executor between steps (loan mode).
The comparison runs in a subprocess with deterministic kernels (math SDPA, deterministic
cuBLAS), because the default flash SDPA backward is not bitwise reproducible."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch
torch.backends.cuda.enable_flash_sdp(False); torch.backends.cuda.enable_mem_efficient_sdp(False)
torch.backends.cuda.enable_math_sdp(True)
torch.use_deterministic_algorithms(True)
import paper_2410_07192_b200 as pf
from paper_2410_07192_b200 import native
from paper_2410_07192_b200.engine import GPT2_SMALL_STAGE, GPTStage, StageEngine, measure_stage_times
native.require_device()
tf, tb = measure_stage_times(GPTStage(GPT2_SMALL_STAGE, seed=0))
cfg = pf.PipelineConfig(4, 8, tf, tb, pf.ScheduleKind.ONE_F_ONE_B, 1, 1, 0.68)
out = {}
for offload in (False, True):
    model = GPTStage(GPT2_SMALL_STAGE, seed=0)
    off = model.enable_optimizer_offload() if offload else None
    eng = StageEngine(cfg, 0, model, None)  # stage 0 of 4: a 3*t_bwd fwd-bwd bubble
    mems = []
    for k in range(4):
        eng.reset_stamps()
        eng.set_anchor()
        rec = eng.run_iteration(0, fill=False)
        torch.cuda.synchronize()
        mems.append(dict(rec.bubble_mem)[0])
    flat = torch.cat([p.detach().float().flatten() for p in model.parameters()])
    out[str(offload)] = {"mems": mems, "sum": float(flat.double().sum()),
                         "state_bytes": off.state_bytes if off else 0,
                         "transfers": off.transfers if off else 0}
    torch.save(flat.cpu(), os.path.join(os.environ["OUT"], f"params_{offload}.pt"))

# loan: the moments' device buffer is lent to a filling executor between steps
from paper_2410_07192_b200.executor import Executor
from paper_2410_07192_b200.fillmodels import BertConfig, bert
from paper_2410_07192_b200.profiles import JobKind, JobSpec, LayerProfile, ModelProfile
model = GPTStage(GPT2_SMALL_STAGE, seed=0)
off = model.enable_optimizer_offload(loan=True)
ex = Executor(256 << 20, job_seed=1)
off.borrower = ex
eng = StageEngine(cfg, 0, model, ex)
fill = bert(BertConfig("bert_tiny", vocab=1000, hidden=256, heads=4, ffn=1024, layers=3), seed=2)
for k in range(4):
    if k == 1:  # states exist: plan the fill (fwd-bwd bubbles with the loan: batch 16, else 4)
        kinds = eng.loan_kinds()
        sizes = (4, 16)
        w = sum(fill[i].weight_bytes() for i in range(len(fill)))
        layers = tuple(LayerProfile({b: 0.005 + 0.0005 * b for b in sizes}, {b: fill[i].weight_bytes() + 1_000_000 * b
                                                                  for b in sizes}, fill[i].weight_bytes(), 1.0)
                       for i in range(len(fill)))
        prof = ModelProfile("tiny", layers, 1, frozenset({JobKind.BATCH_INFERENCE}))
        cyc = pf.BubbleCycle((pf.BubbleSpec(1000, 1000, 8_000_000_000, pf.BubbleKind.FWD_BWD),
                              pf.BubbleSpec(500, 500, w + 8_000_000, pf.BubbleKind.FILL_DRAIN)), 10_000, 0)
        coord = pf.Coordinator(0, cyc, 1)
        coord.admit(JobSpec("j", 0.0, prof, JobKind.BATCH_INFERENCE, 1_000_000))
        ex.loan_kinds = {0} & kinds
        ex.load(coord.request_work(0, 0.0), fill)
        ex.prewarm(eng.words.flag.value)
    eng.reset_stamps()
    eng.set_anchor()
    eng.run_iteration(0, fill=k > 0)
    if k > 0:
        ex.settle()
    torch.cuda.synchronize()
flat = torch.cat([p.detach().float().flatten() for p in model.parameters()])
out["loan"] = {"kinds": sorted(kinds), "loans": off.loans, "loan_batches": ex.loan_batches,
               "rollbacks": ex.loan_rollbacks, "samples": ex.samples_completed}
torch.save(flat.cpu(), os.path.join(os.environ["OUT"], "params_loan.pt"))
print(json.dumps(out))
"""


@pytest.mark.gpu
def test_optimizer_offload_frees_bubble_memory_and_keeps_the_main_job_exact(tmp_path):
    import torch

    env = dict(os.environ, ROOT=ROOT, OUT=str(tmp_path), CUBLAS_WORKSPACE_CONFIG=":4096:8")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    on, offr = res["True"], res["False"]
    a = torch.load(tmp_path / "params_False.pt")
    b = torch.load(tmp_path / "params_True.pt")
    assert torch.equal(a, b), "optimizer offload changed the main job's parameters"
    sb = on["state_bytes"]
    # GPT-2-small stage: 3 layers, ~21 M parameters -> two bf16 moments ~85 MB
    assert sb > 50e6, res
    assert on["transfers"] >= 6, res  # an evict and a prefetch per optimizer step
    # iteration 0's bubble comes before any gradient or optimizer state exists; from
    # iteration 1 on, the offloading run's fwd-bwd bubble has grown by the moments' bytes
    # less than the resident run's (deltas, since both runs share one process)
    for k in (1, 2, 3):
        grew_resident = offr["mems"][k] - offr["mems"][0]
        grew_offload = on["mems"][k] - on["mems"][0]
        assert grew_resident - grew_offload >= 0.95 * sb, res
    # the lent buffer: the fill ran loan-sized batches in the fwd-bwd bubbles between the
    # copy-out and the copy-back, and the main job's parameters are still bitwise exact
    loan = res["loan"]
    assert 0 in loan["kinds"] and loan["loans"] >= 3 and loan["loan_batches"] > 0, res
    assert loan["samples"] > 0, res
    assert torch.equal(a, torch.load(tmp_path / "params_loan.pt")), "the loan changed the main job's parameters"
