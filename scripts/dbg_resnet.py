import sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2410_07192_b200 as pf
from paper_2410_07192_b200 import native
from paper_2410_07192_b200.executor import Executor
from paper_2410_07192_b200.fillmodels import resnet50
from test_resnet_gpu import _item, _run, _oracle_logits
native.require_device()
model = resnet50(seed=5)
n = 10
want = _oracle_logits(model, model.make_inputs(4, 0, n))
res = {}
for name, cap, store in (("single", 8_000_000_000, "auto"),
                         ("multi-host", max(model[i].weight_bytes() for i in range(len(model))) + 2_000_000 * 8 + 4_000_000, "host"),
                         ("multi-dev", max(model[i].weight_bytes() for i in range(len(model))) + 2_000_000 * 8 + 4_000_000, "auto")):
    item, plan = _item(pf, model, n, cap)
    print(name, [(p.lo, p.hi, [(e.batch_size, e.num_batches) for e in p.per_bubble]) for p in plan.partitions])
    ex = Executor(2 << 30, job_seed=4, activation_store=store)
    got = _run(ex, item, model).float()
    ex.close()
    res[name] = got
    print(name, "err vs oracle per row", [round(((got[r] - want[r]).norm() / want[r].norm()).item(), 4) for r in range(n)])
for k in ("multi-host", "multi-dev"):
    print(k, "rows equal to single:", [bool(torch.equal(res[k][r], res["single"][r])) for r in range(n)])
