"""ResNet-50 fill jobs on B200: image kernels (im2col / pooling / ReLU-epilogue GEMM)
and the whole partitioned forward through the Executor, against the CPU fp32 oracle
(oracle/fill_ref.py, itself pinned to torchvision in test_oracle_pinned.py)."""

import pytest
import torch

from oracle import fill_ref

pytestmark = pytest.mark.gpu

REL_TOL_BF16 = 2e-2


@pytest.fixture(scope="module")
def K():
    from paper_2410_07192_b200 import kernels, native

    native.require_device()
    return kernels


def _ref_im2col(x, kh, kw, stride, pad, kp):
    """NHWC im2col with (ky, kx, c) column order, zero padding, pad columns."""
    b, h, w, c = x.shape
    ho, wo = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    xp = torch.zeros(b, h + 2 * pad, w + 2 * pad, c, dtype=x.dtype)
    xp[:, pad:pad + h, pad:pad + w] = x
    cols = []
    for ky in range(kh):
        for kx in range(kw):
            cols.append(xp[:, ky:ky + stride * (ho - 1) + 1:stride, kx:kx + stride * (wo - 1) + 1:stride, :])
    col = torch.cat(cols, dim=-1).reshape(b * ho * wo, kh * kw * c)
    out = torch.zeros(b * ho * wo, kp, dtype=x.dtype)
    out[:, :kh * kw * c] = col
    return out


@pytest.mark.parametrize("shape,k,stride,pad,kp", [
    ((2, 37, 37, 3), 7, 2, 3, 152),     # stem: scalar path, pad columns
    ((3, 14, 14, 64), 3, 1, 1, 576),    # 3x3 stride 1
    ((2, 15, 15, 128), 3, 2, 1, 1152),  # 3x3 stride 2, odd size
    ((2, 14, 14, 256), 1, 2, 0, 256),   # 1x1 stride-2 projection gather
])
def test_im2col_is_exact(K, shape, k, stride, pad, kp):
    g = torch.Generator().manual_seed(0)
    x = torch.randn(*shape, generator=g).to(torch.bfloat16)
    got = K.im2col(x.cuda(), k, k, stride, pad, kp).cpu()
    assert torch.equal(got, _ref_im2col(x, k, k, stride, pad, kp))


def test_maxpool_and_avgpool(K):
    g = torch.Generator().manual_seed(1)
    x = torch.randn(3, 29, 29, 64, generator=g).to(torch.bfloat16)
    got = K.maxpool(x.cuda(), 3, 2, 1).cpu()
    want = torch.nn.functional.max_pool2d(x.float().permute(0, 3, 1, 2), 3, 2, 1).permute(0, 2, 3, 1)
    assert torch.equal(got, want.to(torch.bfloat16))  # a max of bf16 values is exact
    y = torch.randn(4, 7, 7, 2048, generator=g).to(torch.bfloat16)
    got = K.avgpool(y.cuda()).float().cpu()
    want = y.float().mean(dim=(1, 2))
    assert ((got - want).abs().max() / want.abs().max()).item() < 1e-2


@pytest.mark.parametrize("m,n,k,res", [(3136, 64, 576, False), (784, 512, 128, True), (200, 1000, 2048, False)])
def test_gemm_relu_epilogue(K, m, n, k, res):
    g = torch.Generator().manual_seed(2)
    x = torch.randn(m, k, generator=g).to(torch.bfloat16)
    w = (torch.randn(n, k, generator=g) * k ** -0.5).to(torch.bfloat16)
    b = (torch.randn(n, generator=g) * 0.1).to(torch.bfloat16)
    r = torch.randn(m, n, generator=g).to(torch.bfloat16) if res else None
    got = K.linear(x.cuda(), w.cuda(), b.cuda(), residual=None if r is None else r.cuda(), relu=True).float().cpu()
    want = torch.relu(fill_ref.linear(x, w, b, residual=r))
    assert (got >= 0).all()
    err = ((got - want).abs().max() / want.abs().max()).item()
    assert err < REL_TOL_BF16, err


def _oracle_logits(model, img):
    params = [model.oracle_params(i) for i in range(len(model))]
    x = fill_ref.resnet_stem(img, params[0])
    for i in range(1, len(model) - 1):
        x = fill_ref.bottleneck(x, params[i], model[i].stride)
    return fill_ref.resnet_head(x, params[-1])


def _item(pf, model, samples, free_mem, sizes=(4, 8)):
    from paper_2410_07192_b200.profiles import JobKind, JobSpec, LayerProfile, ModelProfile

    layers = []
    for i in range(len(model)):
        w = model[i].weight_bytes()
        layers.append(LayerProfile({b: 0.001 * b for b in sizes}, {b: w + 2_000_000 * b for b in sizes}, w, 1.0))
    prof = ModelProfile("resnet-test", tuple(layers), 1, frozenset({JobKind.BATCH_INFERENCE}))
    cyc = pf.BubbleCycle((pf.BubbleSpec(2000, 2000, free_mem, pf.BubbleKind.FWD_BWD),
                          pf.BubbleSpec(1000, 1000, free_mem, pf.BubbleKind.FILL_DRAIN)), 20_000, 0)
    coord = pf.Coordinator(0, cyc, 1)
    plan = coord.admit(JobSpec("r0", 0.0, prof, JobKind.BATCH_INFERENCE, samples))
    return coord.request_work(0, 0.0), plan


def _run(ex, item, model):
    from paper_2410_07192_b200.executor import BubbleSlot

    ex.load(item, model)
    k = 0
    while ex.busy and k < 2000:
        ex.fill(BubbleSlot(k % 2, None, 0))
        k += 1
    ex.settle()
    torch.cuda.synchronize()
    assert not ex.busy
    return ex.results().clone()


def test_resnet50_executor_matches_oracle_and_partitions_agree():
    """Full ResNet-50 (224x224) through the Executor: single-partition logits within
    rel 2e-2 of the CPU fp32 oracle; a memory-capped multi-partition plan (weights
    staged per partition, NHWC activations offloaded between partitions) gives
    bit-identical logits."""
    import paper_2410_07192_b200 as pf
    from paper_2410_07192_b200 import native
    from paper_2410_07192_b200.executor import Executor
    from paper_2410_07192_b200.fillmodels import resnet50

    native.require_device()
    model = resnet50(seed=5)
    n = 10
    item1, plan1 = _item(pf, model, n, 8_000_000_000)
    assert len(plan1.partitions) == 1
    ex = Executor(2 << 30, job_seed=4)
    got = _run(ex, item1, model).float()
    ex.close()
    img = model.make_inputs(4, 0, n)
    want = _oracle_logits(model, img)
    err = ((got - want).norm() / want.norm()).item()
    assert err < REL_TOL_BF16, err
    # room for the largest block's weights plus a batch of 8 of transients, not for all
    # 51 MB of weights -> a multi-partition plan
    cap = max(model[i].weight_bytes() for i in range(len(model))) + 2_000_000 * 8 + 4_000_000
    item2, plan2 = _item(pf, model, n, cap)
    assert len(plan2.partitions) >= 2, plan2
    ex = Executor(2 << 30, job_seed=4, activation_store="host")
    got2 = _run(ex, item2, model)
    ex.close()
    assert torch.equal(got2.float(), got)
