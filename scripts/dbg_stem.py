import sys, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2410_07192_b200 import native, kernels as K
from paper_2410_07192_b200.fillmodels import resnet50
from test_resnet_gpu import _ref_im2col
native.require_device()
model = resnet50(seed=5)
b = 8
img = model.make_inputs(4, 0, b)
x = img.cuda()
col = K.im2col(x, 7, 7, 2, 3, 152)
torch.cuda.synchronize()
ref_col = _ref_im2col(img, 7, 7, 2, 3, 152)
c = col.cpu()
bad = (c != ref_col).any(dim=1)
print("im2col rows differing:", int(bad.sum()), "first", int(bad.nonzero()[0]) if bad.any() else None)
p = model.oracle_params(0)
w = model[0].host_params["w"].cuda(); bb = model[0].host_params["b"].cuda()
y = K.linear(col, w, bb, relu=True)
torch.cuda.synchronize()
ref = torch.relu(ref_col.float() @ p["w"].T + p["b"])
err = (y.float().cpu() - ref).norm(dim=1) / ref.norm(dim=1).clamp_min(1e-6)
per = err.view(b, -1).max(dim=1).values
print("gemm per-sample max row err", [round(v, 4) for v in per.tolist()])
y2 = K.linear(ref_col.cuda(), w, bb, relu=True)
torch.cuda.synchronize()
print("gemm on ref col equal:", bool(torch.equal(y2, y)))
for M in (100352, 50176, 25088):
    y3 = K.linear(ref_col[:M].cuda(), w, bb, relu=True); torch.cuda.synchronize()
    e3 = ((y3.float().cpu() - ref[:M]).norm(dim=1) / ref[:M].norm(dim=1).clamp_min(1e-6)).view(-1, 12544).max(dim=1).values
    print(M, [round(v, 4) for v in e3.tolist()])
