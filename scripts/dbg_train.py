import sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2410_07192_b200 as pf
from paper_2410_07192_b200 import native
from paper_2410_07192_b200.executor import BubbleSlot, Executor
from paper_2410_07192_b200.fillmodels import ResNetConfig
from paper_2410_07192_b200.training import resnet50_train, synthetic_labels
from test_train_gpu import _plan_item, _torchvision_from
native.require_device()
cfg = ResNetConfig(image=int(sys.argv[1]) if len(sys.argv) > 1 else 64)
model = resnet50_train(cfg, seed=7)
batch, n, seed = 8, 8, 3
tv, blocks = _torchvision_from(model)
item = _plan_item(pf, model, n, batch)
ex = Executor(8 << 30, job_seed=seed)
ex.load(item, model)
ex.fill(BubbleSlot(0, None, 0)); ex.settle(); torch.cuda.synchronize()
L = len(model)
img = model.make_inputs(seed, 0, batch).float().permute(0, 3, 1, 2)
tv.train()
acts = {}
with torch.no_grad():
    x = tv.maxpool(tv.relu(tv.bn1(tv.conv1(img)))); acts[0] = x
    i = 1
    for layer in (tv.layer1, tv.layer2, tv.layer3, tv.layer4):
        for blk in layer:
            x = blk(x); acts[i] = x; i += 1
    logits = tv.fc(torch.flatten(tv.avgpool(x), 1))
def rel(a, b): return ((a - b).norm() / b.norm()).item()
for i in range(L - 1):
    b, h, w, c = batch, *model[i].out_shape()
    got = ex.ws[f"out{i}"].view(-1)[:b*h*w*c].view(b, h, w, c).float().cpu().permute(0, 3, 1, 2)
    print(i, "rel", round(rel(got, acts[i]), 4))
got = ex.ws[f"s{L-1}.logits"].view(-1)[:batch*1000].view(batch, 1000).float().cpu()
print("logits rel", rel(got, logits))
lab = synthetic_labels(seed, 0, batch, 1000)[:, 0].long()
print("loss gpu", ex.results()[:8, 0].tolist())
print("loss ref", torch.nn.functional.cross_entropy(logits, lab, reduction="none").tolist())
