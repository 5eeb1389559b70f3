"""bf16 precision floor of one ResNet bottleneck backward: torchvision's block in fp32 vs the
same block with every tensor rounded to bf16 at the points the B200 kernels store bf16
(conv outputs, BN outputs, ReLU outputs, and the gradients between them). Prints the
relative differences of dx, a conv weight gradient and a BN gamma gradient (~7-8 %),
the bound tests/test_train_gpu.py holds its gradient tolerance against."""
import torch, torchvision
import torch.nn.functional as F
torch.manual_seed(0)
tv = torchvision.models.resnet50(weights=None).train()
blk = tv.layer1[1]
x = torch.relu(torch.randn(8, 256, 16, 16))
dout = torch.randn(8, 256, 16, 16)
class R(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t): return t.to(torch.bfloat16).float()
    @staticmethod
    def backward(ctx, g): return g.to(torch.bfloat16).float()
def bn(t, m): return F.batch_norm(t, None, None, m.weight, m.bias, training=True, eps=1e-5)
def run(e):
    r = R.apply if e else (lambda t: t)
    for p in blk.parameters(): p.grad = None
    xi = r(x.clone()).detach().requires_grad_(True)
    a = r(F.relu(r(bn(r(blk.conv1(xi)), blk.bn1))))
    a = r(F.relu(r(bn(r(blk.conv2(a)), blk.bn2))))
    y = r(F.relu(r(bn(r(blk.conv3(a)), blk.bn3)) + xi))
    y.backward(r(dout) if e else dout)
    return xi.grad.clone(), blk.conv2.weight.grad.clone(), blk.bn1.weight.grad.clone()
a = run(False); b = run(True)
rel = lambda u, v: ((u - v).norm() / v.norm()).item()
print("emulated bf16 vs fp32: dx", rel(b[0], a[0]), "dW2", rel(b[1], a[1]), "dgamma1", rel(b[2], a[2]))
