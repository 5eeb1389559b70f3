import torch, sys
sys.path.insert(0, "/root/repo")
from paper_2410_07192_b200 import kernels as K, native
native.require_device()
g = torch.Generator().manual_seed(0)
for (n, k) in [(512, 1024), (2048, 512), (512, 4608), (64, 152), (256, 64), (1000, 2048)]:
    x = torch.randn(1568, k, generator=g).to(torch.bfloat16).cuda()
    w = (torch.randn(n, k, generator=g) * k ** -0.5).to(torch.bfloat16).cuda()
    b = torch.randn(n, generator=g).to(torch.bfloat16).cuda()
    outs = {}
    for m in (1568, 784, 392, 196, 98):
        outs[m] = K.linear(x[:m], w, b, relu=True)
    ref = outs[1568]
    print(n, k, {m: bool(torch.equal(o, ref[:m])) for m, o in outs.items()}, {m: K.gemm_units(m, n, k) for m in outs})
