"""Training kernels (ResNet-50 fill training) against CPU fp32 torch references:
split-K GEMM, transpose, BatchNorm batch statistics / apply / backward, col2im,
pooling backward, softmax cross-entropy and the SGD update."""

import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

REL = 2e-2


@pytest.fixture(scope="module")
def K():
    from paper_2410_07192_b200 import kernels, native

    native.require_device()
    return kernels


def rel(got, want):
    got, want = got.float().cpu(), want.float().cpu()
    return ((got - want).norm() / want.norm().clamp_min(1e-12)).item()


def bf(*shape, gen, scale=1.0):
    return (torch.randn(*shape, generator=gen) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("m,n,k,splits", [(64, 576, 25088, 16), (256, 64, 6272, 8), (1000, 2048, 64, 4),
                                          (200, 136, 1000, 3)])
def test_gemm_splitk(K, m, n, k, splits):
    g = torch.Generator().manual_seed(0)
    x, w = bf(m, k, gen=g), bf(n, k, gen=g, scale=k ** -0.5)
    parts = K.gemm_splitk(x.cuda(), w.cuda(), splits)
    s = K.gemm_splitk_splits(k, splits)
    assert parts.shape == (s, m, n)
    assert rel(parts.float().sum(0), x.float() @ w.float().T) < REL


def test_transpose_exact(K):
    g = torch.Generator().manual_seed(1)
    x = bf(1000, 72, gen=g)
    assert torch.equal(K.transpose(x.cuda()).cpu(), x.T.contiguous())


def _bn_forward(K, z, gamma, beta, eps=1e-5, residual=None, relu=True):
    m, c = z.shape
    dev = z.device
    partial = torch.empty(1024, 2 * c, device=dev)
    p = K.colstats(z, partial)
    mean, invstd, scale, shift = (torch.empty(c, device=dev) for _ in range(4))
    K.bn_finalize(partial, p, m, gamma, beta, eps, mean, invstd, scale, shift)
    y = torch.empty_like(z)
    K.bn_apply(z, scale, shift, y, residual=residual, relu=relu)
    return y, mean, invstd


def test_batchnorm_forward_backward(K):
    """Train-mode BatchNorm + residual + ReLU forward and its backward against torch
    autograd (F.batch_norm(training=True)) in fp32."""
    g = torch.Generator().manual_seed(2)
    m, c = 6272, 256
    z = bf(m, c, gen=g, scale=2.0) + 0.5
    r = bf(m, c, gen=g)
    gamma = torch.rand(c, generator=g) + 0.5
    beta = torch.randn(c, generator=g) * 0.1
    dy = bf(m, c, gen=g)
    zc, rc, gc, bc = z.cuda(), r.cuda(), gamma.cuda(), beta.cuda()
    y, mean, invstd = _bn_forward(K, zc, gc, bc, residual=rc)
    # reference
    zt = z.float().requires_grad_(True)
    gt = gamma.clone().requires_grad_(True)
    btt = beta.clone().requires_grad_(True)
    yt = torch.relu(F.batch_norm(zt, None, None, gt, btt, training=True, eps=1e-5) + r.float())
    assert rel(y, yt.detach()) < REL
    yt.backward(dy.float())
    # backward: stats partials of (dA, dA*xhat), dA = dy*[y>0]
    dev = zc.device
    partial = torch.empty(1024, 2 * c, device=dev)
    p = K.colstats(zc, partial, g=dy.cuda(), ymask=y, mean=mean, invstd=invstd)
    dgamma, dbeta = torch.empty(c, device=dev), torch.empty(c, device=dev)
    K.bn_bwd_finalize(partial, p, c, dgamma, dbeta)
    dz = torch.empty_like(zc)
    da = torch.empty_like(zc)
    K.bn_bwd_apply(zc, dy.cuda(), mean, invstd, gc, dgamma, dbeta, dz, ymask=y, da=da)
    assert rel(dgamma, gt.grad) < REL
    assert rel(dbeta, btt.grad) < REL
    assert rel(dz, zt.grad) < REL
    assert rel(da, dy.float() * (yt.detach() > 0)) < 1e-2


def _ref_im2col(x, kh, kw, stride, pad, kp):
    b, h, w, c = x.shape
    ho, wo = (h + 2 * pad - kh) // stride + 1, (w + 2 * pad - kw) // stride + 1
    xp = F.pad(x, (0, 0, pad, pad, pad, pad))
    cols = [xp[:, ky:ky + stride * (ho - 1) + 1:stride, kx:kx + stride * (wo - 1) + 1:stride, :]
            for ky in range(kh) for kx in range(kw)]
    col = torch.cat(cols, dim=-1).reshape(b * ho * wo, kh * kw * c)
    return F.pad(col, (0, kp - kh * kw * c))


@pytest.mark.parametrize("shape,k,stride,pad", [((2, 14, 14, 64), 3, 1, 1), ((2, 15, 15, 32), 3, 2, 1),
                                                ((3, 8, 8, 128), 1, 2, 0)])
def test_col2im_is_the_adjoint_of_im2col(K, shape, k, stride, pad):
    g = torch.Generator().manual_seed(3)
    b, h, w, c = shape
    kp = (k * k * c + 7) // 8 * 8
    x = torch.randn(*shape, generator=g, requires_grad=True)
    col = _ref_im2col(x, k, k, stride, pad, kp)
    dcol = bf(*col.shape, gen=g)
    (col * dcol.float()).sum().backward()
    r = bf(*shape, gen=g)
    got = K.col2im(dcol.cuda(), b, h, w, c, k, k, stride, pad, residual=r.cuda())
    assert rel(got, x.grad + r.float()) < 1e-2


def test_pool_backward(K):
    g = torch.Generator().manual_seed(4)
    x = bf(2, 28, 28, 64, gen=g)
    xt = x.float().permute(0, 3, 1, 2).requires_grad_(True)
    yt = F.max_pool2d(xt, 3, 2, 1)
    dy = bf(*yt.permute(0, 2, 3, 1).shape, gen=g)
    yt.backward(dy.float().permute(0, 3, 1, 2))
    got = K.maxpool_bwd(x.cuda(), dy.cuda())
    assert rel(got, xt.grad.permute(0, 2, 3, 1)) < 1e-2
    d = bf(4, 2048, gen=g)
    got = K.avgpool_bwd(d.cuda(), 49)
    assert rel(got, (d.float() / 49)[:, None, :].expand(4, 49, 2048)) < 1e-2


@pytest.mark.parametrize("shape", [(2, 28, 28, 64), (3, 17, 15, 16), (64, 112, 112, 64)])
def test_maxpool_argmax_path_is_bit_identical(K, shape):
    """pf_maxpool_argmax writes the same pooled output as pf_maxpool plus the first-maximum
    window positions; pf_maxpool_bwd_argmax (reads 8 index bytes per window) equals
    pf_maxpool_bwd (re-scans every window) bit for bit, ties included."""
    from paper_2410_07192_b200 import native

    g = torch.Generator().manual_seed(9)
    b, h, w, c = shape
    x = bf(b, h, w, c, gen=g)
    x[0, :4, :4, :8] = 1.0  # ties inside windows: the first maximum wins in both paths
    x = x.cuda()
    ho, wo = (h + 2 - 3) // 2 + 1, (w + 2 - 3) // 2 + 1
    y_ref = K.maxpool(x, 3, 2, 1) if hasattr(K, "maxpool") else None
    y = torch.empty(b, ho, wo, c, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(b * ho * wo * c, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    native.call("pf_maxpool_argmax", x.data_ptr(), y.data_ptr(), idx.data_ptr(), b, h, w, c, 3, 2, 1, None, s)
    if y_ref is not None:
        assert torch.equal(y, y_ref)
    dy = bf(b, ho, wo, c, gen=g).cuda()
    dx = torch.empty_like(x)
    native.call("pf_maxpool_bwd_argmax", idx.data_ptr(), dy.data_ptr(), dx.data_ptr(), b, h, w, c, 3, 2, 1, None, s)
    torch.cuda.synchronize()
    assert torch.equal(dx, K.maxpool_bwd(x, dy))


def test_softmax_cross_entropy(K):
    g = torch.Generator().manual_seed(5)
    b, n = 24, 1000
    z = bf(b, n, gen=g, scale=3.0)
    labels = torch.randint(0, n, (b,), generator=g)
    lab4 = torch.zeros(b, 4, dtype=torch.int32)
    lab4[:, 0] = labels
    loss4 = torch.empty(b, 4, device="cuda")
    dz = torch.empty(b, n, dtype=torch.bfloat16, device="cuda")
    K.softmax_xent(z.cuda(), lab4.cuda(), loss4, dz, 1.0 / b)
    zt = z.float().requires_grad_(True)
    lt = F.cross_entropy(zt, labels, reduction="none")
    lt.mean().backward()
    assert rel(loss4[:, 0], lt.detach()) < 1e-3
    assert rel(dz, zt.grad) < REL


def test_sgd_update_and_splitk_sum(K):
    g = torch.Generator().manual_seed(6)
    n1, n2 = 10_000, 3_000
    w1, w2 = torch.randn(n1, generator=g).cuda(), torch.randn(n2, generator=g).cuda()
    v1, v2 = torch.randn(n1, generator=g).cuda(), torch.zeros(n2).cuda()
    parts = bf(3, n1, gen=g).cuda()
    g2 = torch.randn(n2, generator=g).cuda()
    work1 = torch.empty(n1, dtype=torch.bfloat16, device="cuda")
    e1 = (w1.clone(), v1.clone(), w2.clone(), v2.clone())
    K.sgd_update([dict(master=w1.data_ptr(), momentum=v1.data_ptr(), work=work1.data_ptr(), grad=parts.data_ptr(),
                       n=n1, split_stride=n1, splits=3, grad_kind=0, weight_decay=1e-4),
                  dict(master=w2.data_ptr(), momentum=v2.data_ptr(), grad=g2.data_ptr(), n=n2, grad_kind=1)],
                 lr=0.1, momentum=0.9)
    torch.cuda.synchronize()
    gsum = parts.float().sum(0) + 1e-4 * e1[0]
    ev1 = 0.9 * e1[1] + gsum
    assert torch.allclose(v1, ev1, rtol=1e-5, atol=1e-5)
    assert torch.allclose(w1, e1[0] - 0.1 * ev1, rtol=1e-5, atol=1e-5)
    assert torch.equal(work1, w1.to(torch.bfloat16))
    assert torch.allclose(w2, e1[2] - 0.1 * (0.9 * e1[3] + g2), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("m,n,k,res", [(6272, 576, 64, False), (1000, 2048, 1000, True), (200, 136, 96, True)])
def test_gemm_nn_mn_major_b(K, m, n, k, res):
    """Data-gradient GEMM with W read MN-major: x[M,K] @ w[K,N] (+ residual)."""
    g = torch.Generator().manual_seed(7)
    x, w = bf(m, k, gen=g), bf(k, n, gen=g, scale=k ** -0.5)
    r = bf(m, n, gen=g) if res else None
    got = K.gemm_nn(x.cuda(), w.cuda(), residual=None if r is None else r.cuda())
    want = x.float() @ w.float() + (r.float() if res else 0)
    assert rel(got, want) < REL


@pytest.mark.parametrize("k,m,n,splits", [(25088, 64, 576, 16), (6272, 256, 64, 8), (64, 1000, 2048, 1),
                                          (1000, 200, 136, 3)])
def test_gemm_splitk_tn_mn_major_both(K, k, m, n, splits):
    """Weight-gradient GEMM straight from row-major activations: a[K,M]^T @ b[K,N]."""
    g = torch.Generator().manual_seed(8)
    a, b = bf(k, m, gen=g), bf(k, n, gen=g, scale=k ** -0.5)
    parts = K.gemm_splitk_tn(a.cuda(), b.cuda(), splits)
    assert rel(parts.float().sum(0), a.float().T @ b.float()) < REL
