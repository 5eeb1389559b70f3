"""2-rank check of main-job losses with filling off / off again / on, bench-like main job
(non-deterministic kernels): torchrun --nproc-per-node 2 scripts/nccl_loss_check.py"""
import json, os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
if os.environ.get("DETERMINISTIC") == "1":
    torch.backends.cuda.enable_flash_sdp(False); torch.backends.cuda.enable_mem_efficient_sdp(False)
    torch.use_deterministic_algorithms(True)
import paper_2410_07192_b200 as pf
from paper_2410_07192_b200.engine import GPT_8B_STAGE, GPTStage, NcclPipelineEngine, measure_stage_times
from paper_2410_07192_b200.executor import Executor
from paper_2410_07192_b200.fillmodels import BERT_LARGE, bert
from paper_2410_07192_b200.profiler import measure_profile
model = GPTStage(GPT_8B_STAGE, seed=rank)
tf, tb = measure_stage_times(model)
tt = torch.tensor([tf, tb], device="cuda"); dist.all_reduce(tt, op=dist.ReduceOp.MAX)
pcfg = pf.PipelineConfig(world, 8, tt[0].item(), tt[1].item(), pf.ScheduleKind.ONE_F_ONE_B, 8 << 30, 8 << 30, 0.95)
fill = bert(BERT_LARGE, seed=0)
prof = measure_profile(fill, (32, 64, 128))
coord = pf.Coordinator(rank, pf.build_bubble_cycle(pcfg, rank), 1, pf.OrderingPolicy("concurrent", 16384))
coord.admit(pf.JobSpec("j", 0.0, prof, pf.JobKind.BATCH_INFERENCE, 10_000_000))
ex = Executor(8 << 30)
ex.work_source = lambda: (coord.request_work(0, 0.0), fill)
eng = NcclPipelineEngine(pcfg, model, ex)
snap = model.snapshot()
out = {}
n = int(os.environ.get("ITERS", "6"))
for name, on in (("off", False), ("off2", False), ("on", True)):
    model.restore(snap); eng.losses = []
    eng.reset_stamps(); dist.barrier(); eng.set_anchor()
    for it in range(n):
        eng.run_iteration(it, fill=on, last=(it == n - 1))
    ex.settle(); eng.sync()
    out[name] = [round(float(x), 5) for x in eng.losses]
print("RESULT", rank, json.dumps(out), flush=True)
ex.close()
dist.destroy_process_group()
