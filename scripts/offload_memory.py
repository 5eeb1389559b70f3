"""Main-job memory with and without optimizer-state offload: the peak torch
reserves over a stage-0 iteration of the 8-stage 8B pipeline (what bounds the fill arena),
and the allocated bytes at each BUBBLE. python scripts/offload_memory.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_07192_b200 as pf  # noqa: E402
from paper_2410_07192_b200.engine import GPT_8B_STAGE, GPTStage, StageEngine, measure_stage_times  # noqa: E402

out = {}
for offload in (False, True):
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    model = GPTStage(GPT_8B_STAGE, seed=0)
    tf, tb = measure_stage_times(model, warm_ms=200)
    if offload:
        model.enable_optimizer_offload()
    cfg = pf.PipelineConfig(8, 8, tf, tb, pf.ScheduleKind.ONE_F_ONE_B, 1, 1, 0.95)
    eng = StageEngine(cfg, 0, model, None)
    for it in range(3):
        eng.reset_stamps()
        eng.set_anchor()
        rec = eng.run_iteration(0, fill=False)
        torch.cuda.synchronize()
        if it == 0:
            torch.cuda.reset_peak_memory_stats()
    free, total = torch.cuda.mem_get_info()
    out["offload" if offload else "resident"] = {
        "max_reserved_gb": torch.cuda.max_memory_reserved() / 2**30,
        "max_allocated_gb": torch.cuda.max_memory_allocated() / 2**30,
        "bubble_allocated_gb": [(k, a / 2**30) for k, a in rec.bubble_mem],
        "free_after_gb": free / 2**30,
        "state_bytes_gb": (model.offload.state_bytes / 2**30) if model.offload else None}
    print(json.dumps(out), flush=True)
    del eng, model
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
