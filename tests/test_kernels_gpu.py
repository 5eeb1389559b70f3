"""Parity of every sm_100a kernel against the CPU fp32 oracle (bf16 path, rel 2e-2)."""

import pytest
import torch

from oracle import fill_ref

pytestmark = pytest.mark.gpu

REL_TOL_BF16 = 2e-2  # north star: bf16 path within rel 2e-2 of the CPU fp32 execution


def rel_err(got: torch.Tensor, ref: torch.Tensor) -> float:
    got = got.float().cpu()
    ref = ref.float().cpu()
    return ((got - ref).abs().max() / ref.abs().max().clamp_min(1e-6)).item()


@pytest.fixture(scope="module")
def K():
    from paper_2410_07192_b200 import kernels, native

    native.require_device()
    return kernels


def _bf16(*shape, scale=1.0, gen=None):
    return (torch.randn(*shape, generator=gen) * scale).to(torch.bfloat16)


@pytest.mark.parametrize(
    "m,n,k,bias,gelu,res",
    [
        (4096, 3072, 768, True, True, False),   # BERT-base FFN1
        (4096, 768, 3072, True, False, True),   # FFN2 + residual
        (4096, 2304, 768, True, False, False),  # QKV
        (4096, 768, 768, True, False, True),    # attention out + residual
        (4096, 4096, 1024, True, True, False),  # BERT-large FFN1
        (128, 128, 64, False, False, False),
        (200, 264, 136, True, True, True),      # ragged M/N/K tails
        (65536, 64, 152, True, False, False),   # short K, ~4 tiles per CTA: epilogue staging reuse
        (1, 8, 8, False, False, False),
        (16384, 1024, 1024, True, False, True),  # 512 tiles: last wave of 68 run as 136 half tiles
        (16384, 1024, 4096, True, False, True),  # BERT-large FFN2 (tail halves, long K)
        (16384, 3072, 1024, True, False, False),  # QKV: 1536 tiles, 56-tile tail
        (19200, 1024, 256, True, True, False),   # ragged: 150 x 4 tiles, tail of 12 with GELU
    ],
)
def test_gemm(K, m, n, k, bias, gelu, res):
    g = torch.Generator().manual_seed(m * 7 + n * 3 + k)
    x = _bf16(m, k, gen=g)
    w = _bf16(n, k, scale=k ** -0.5, gen=g)
    b = _bf16(n, gen=g) if bias else None
    r = _bf16(m, n, gen=g) if res else None
    ref = fill_ref.linear(x.float(), w.float(), None if b is None else b.float(), gelu=gelu,
                          residual=None if r is None else r.float())
    cu = lambda t: None if t is None else t.cuda()
    got = K.linear(x.cuda(), w.cuda(), cu(b), gelu=gelu, residual=cu(r))
    torch.cuda.synchronize()
    assert rel_err(got, ref) < REL_TOL_BF16


@pytest.mark.parametrize("rows,cols,res", [(4096, 768, True), (4096, 1024, False), (33, 2048, True), (5, 8, False),
                                           (16384, 1024, True), (7001, 1024, False)])
def test_layernorm(K, rows, cols, res):
    g = torch.Generator().manual_seed(rows + cols)
    x = _bf16(rows, cols, gen=g)
    r = _bf16(rows, cols, gen=g) if res else None
    gamma = (1 + 0.1 * torch.randn(cols, generator=g)).to(torch.bfloat16)
    beta = (0.1 * torch.randn(cols, generator=g)).to(torch.bfloat16)
    ref = fill_ref.layernorm(x.float() + (r.float() if r is not None else 0), gamma.float(), beta.float(), 1e-12)
    got = K.layernorm(x.cuda(), gamma.cuda(), beta.cuda(), 1e-12, residual=None if r is None else r.cuda())
    torch.cuda.synchronize()
    assert rel_err(got, ref) < REL_TOL_BF16


def test_rmsnorm(K):
    g = torch.Generator().manual_seed(3)
    x = _bf16(1000, 4096 // 2, gen=g)
    gamma = (1 + 0.1 * torch.randn(2048, generator=g)).to(torch.bfloat16)
    ref = fill_ref.rmsnorm(x.float(), gamma.float(), 1e-6)
    got = K.rmsnorm(x.cuda(), gamma.cuda(), 1e-6)
    torch.cuda.synchronize()
    assert rel_err(got, ref) < REL_TOL_BF16


@pytest.mark.parametrize("rows,cols", [(384 * 128, 128), (100, 1000), (7, 2048)])
def test_softmax(K, rows, cols):
    g = torch.Generator().manual_seed(rows)
    x = _bf16(rows, cols, scale=3.0, gen=g)
    ref = fill_ref.softmax(x.float(), 0.5)
    got = K.softmax(x.cuda(), 0.5)
    torch.cuda.synchronize()
    assert rel_err(got, ref) < REL_TOL_BF16


@pytest.mark.parametrize("batch,seq,heads,masked", [(32, 128, 12, False), (4, 128, 16, True), (3, 77, 2, False),
                                                     (2, 1, 1, False), (128, 128, 16, False), (40, 128, 16, True),
                                                     (37, 100, 12, False)])
def test_attention(K, batch, seq, heads, masked):
    g = torch.Generator().manual_seed(batch * seq + heads)
    hidden = heads * 64
    qkv = _bf16(batch, seq, 3 * hidden, gen=g)
    mask = None
    if masked:
        keep = torch.rand(batch, seq, generator=g) > 0.3
        keep[:, 0] = True
        mask = torch.where(keep, 0.0, -10000.0).float()
    ref = fill_ref.attention(qkv.float(), heads, mask)
    got = K.attention(qkv.cuda(), heads, mask_add=None if mask is None else mask.cuda())
    torch.cuda.synchronize()
    assert rel_err(got, ref) < REL_TOL_BF16


def test_embedding_ln(K):
    g = torch.Generator().manual_seed(11)
    vocab, hidden, batch, seq = 30522, 768, 4, 128
    word = _bf16(vocab, hidden, scale=0.02, gen=g)
    pos = _bf16(512, hidden, scale=0.02, gen=g)
    typ = _bf16(2, hidden, scale=0.02, gen=g)
    gamma = torch.ones(hidden, dtype=torch.bfloat16)
    beta = torch.zeros(hidden, dtype=torch.bfloat16)
    ids = torch.randint(0, vocab, (batch, seq), generator=g, dtype=torch.int32)
    ref = fill_ref.embedding_ln(ids, word.float(), pos.float(), typ.float(), gamma.float(), beta.float(), 1e-12)
    got = K.embedding_ln(ids.cuda(), word.cuda(), pos.cuda(), typ.cuda(), gamma.cuda(), beta.cuda(), 1e-12)
    torch.cuda.synchronize()
    assert rel_err(got, ref) < REL_TOL_BF16


def test_gemm_preemption_protocol(K):
    """Flag 0: nothing claimed, abort set. Flag 1: all tiles claimed, resumable prefix."""
    m, n, k = 4096, 3072, 768
    x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda") * k ** -0.5).to(torch.bfloat16)
    words = torch.zeros(8, dtype=torch.int32, device="cuda")
    flag, abort, cursor = (words[i:i + 1] for i in range(3))
    ctl = K.KernelCtl(flag.data_ptr(), abort.data_ptr(), cursor.data_ptr())
    y = torch.zeros(m, n, dtype=torch.bfloat16, device="cuda")
    K.linear(x, w, out=y, ctl=ctl)
    torch.cuda.synchronize()
    assert abort.item() == 1 and cursor.item() == 0 and y.abs().max().item() == 0
    # chain aborted: even with the flag set, the launch must not start
    flag.fill_(1)
    K.linear(x, w, out=y, ctl=ctl)
    torch.cuda.synchronize()
    assert cursor.item() == 0
    abort.zero_()
    K.linear(x, w, out=y, ctl=ctl)
    torch.cuda.synchronize()
    assert cursor.item() >= K.gemm_units(m, n, k) and abort.item() == 0
    ref = x.float() @ w.float().T
    assert rel_err(y, ref) < REL_TOL_BF16


def test_attention_preemption_protocol(K):
    """Persistent attention: flag 0 -> no CTA counts itself, abort set, output untouched;
    flag 1 -> every CTA counts itself (units = CTAs launched) and the result is correct."""
    batch, seq, heads = 64, 128, 16  # 1024 units over <= 296 CTAs: several units per CTA
    g = torch.Generator().manual_seed(5)
    qkv = _bf16(batch, seq, 3 * heads * 64, gen=g).cuda()
    words = torch.zeros(8, dtype=torch.int32, device="cuda")
    flag, abort, cursor = (words[i:i + 1] for i in range(3))
    ctl = K.KernelCtl(flag.data_ptr(), abort.data_ptr(), cursor.data_ptr())
    out = torch.zeros(batch, seq, heads * 64, dtype=torch.bfloat16, device="cuda")
    K.attention(qkv, heads, out=out, ctl=ctl)
    torch.cuda.synchronize()
    assert abort.item() == 1 and cursor.item() == 0 and out.abs().max().item() == 0
    abort.zero_()
    flag.fill_(1)
    K.attention(qkv, heads, out=out, ctl=ctl)
    torch.cuda.synchronize()
    units = K.attention_units(batch, seq, heads, 64)
    assert abort.item() == 0 and cursor.item() == units and units <= batch * heads
    ref = fill_ref.attention(qkv.float().cpu(), heads, None)
    assert rel_err(out, ref) < REL_TOL_BF16


def test_layernorm_preemption_protocol(K):
    """Persistent LayerNorm: flag 0 -> nothing written, abort set, cursor 0; flag 1 -> every
    CTA counts itself (units = CTAs launched) and the rows are exact re-runs."""
    rows, cols = 9000, 1024
    g = torch.Generator().manual_seed(3)
    x = _bf16(rows, cols, gen=g).cuda()
    gamma = torch.ones(cols, dtype=torch.bfloat16, device="cuda")
    beta = torch.zeros(cols, dtype=torch.bfloat16, device="cuda")
    words = torch.zeros(8, dtype=torch.int32, device="cuda")
    flag, abort, cursor = (words[i:i + 1] for i in range(3))
    ctl = K.KernelCtl(flag.data_ptr(), abort.data_ptr(), cursor.data_ptr())
    out = torch.zeros_like(x)
    K.layernorm(x, gamma, beta, 1e-12, out=out, ctl=ctl)
    torch.cuda.synchronize()
    assert abort.item() == 1 and cursor.item() == 0 and out.abs().max().item() == 0
    abort.zero_()
    flag.fill_(1)
    K.layernorm(x, gamma, beta, 1e-12, out=out, ctl=ctl)
    torch.cuda.synchronize()
    assert abort.item() == 0 and cursor.item() == K.norm_units(rows, cols)
    assert torch.equal(out, K.layernorm(x, gamma, beta, 1e-12))


@pytest.mark.parametrize("m,n,k,variant", [(16384, 1024, 1024, "tail"), (16384, 1024, 4096, "pair"),
                                           (16384, 4096, 1024, "pair")])
def test_gemm_tail_halves_resume_exact(K, m, n, k, variant):
    """Resume from a claimed prefix (cursor preset, as the executor resumes a yielded node):
    for the single-CTA kernel whose last wave runs as half tiles and for the CTA-pair kernel
    (the default for long-K / wide-N GEMMs) the resumed launch writes exactly the reference's
    values for the units it runs, and a full launch equals an uninterrupted one bit for bit."""
    g = torch.Generator().manual_seed(21)
    x = _bf16(m, k, gen=g).cuda()
    w = _bf16(n, k, scale=k ** -0.5, gen=g).cuda()
    b = _bf16(n, gen=g).cuda()
    units = K.gemm_units(m, n, k)
    if variant == "tail":
        assert units > (m // 128) * (n // 256), "expected the half-tile tail for this shape"
    else:  # 256 x 256 CTA-pair tiles, the N = 1024 shape with a half-tile tail wave
        assert units >= (m // 256) * (n // 256), "expected 256 x 256 CTA-pair tiles for this shape"
    ref = K.linear(x, w, b)
    words = torch.zeros(8, dtype=torch.int32, device="cuda")
    flag, abort, cursor = (words[i:i + 1] for i in range(3))
    ctl = K.KernelCtl(flag.data_ptr(), abort.data_ptr(), cursor.data_ptr())
    y = torch.zeros(m, n, dtype=torch.bfloat16, device="cuda")
    for start in (units - 150, units - 7, 0):  # early, in the last wave, whole
        y.zero_()
        words.zero_()
        flag.fill_(1)
        cursor.fill_(start)
        K.linear(x, w, b, out=y, ctl=ctl)  # runs units [start, units)
        torch.cuda.synchronize()
        assert abort.item() == 0 and cursor.item() >= units
        mask = y != 0
        assert mask.any() and torch.equal(y[mask], ref[mask])
    assert torch.equal(y, ref)


@pytest.mark.parametrize("m,n,k,v", [(16384, 1024, 1024, 8), (16384, 4096, 1024, 16), (4096, 3072, 768, 2),
                                     (16384, 4096, 1024, 3)])
def test_gemm_throttled_flag_is_exact(K, m, n, k, v):
    """Flag value v >= 2 (power-aware bubble tail): at most v CTAs (v / 2 CTA pairs) claim
    tiles, no abort is raised, every unit still runs once, and the result equals the
    unthrottled launch bit for bit -- single-CTA (tail halves) and CTA-pair variants."""
    g = torch.Generator().manual_seed(31)
    x = _bf16(m, k, gen=g).cuda()
    w = _bf16(n, k, scale=k ** -0.5, gen=g).cuda()
    b = _bf16(n, gen=g).cuda()
    ref = K.linear(x, w, b, gelu=True)
    words = torch.zeros(8, dtype=torch.int32, device="cuda")
    flag, abort, cursor = (words[i:i + 1] for i in range(3))
    ctl = K.KernelCtl(flag.data_ptr(), abort.data_ptr(), cursor.data_ptr())
    y = torch.zeros(m, n, dtype=torch.bfloat16, device="cuda")
    flag.fill_(v)
    K.linear(x, w, b, gelu=True, out=y, ctl=ctl)
    torch.cuda.synchronize()
    assert abort.item() == 0 and cursor.item() >= K.gemm_units(m, n, k)
    assert torch.equal(y, ref)


def test_flag_throttle_at_respects_a_closed_bubble(K):
    """pf_flag_throttle_at: 1 -> v at the deadline; a flag already cleared (0) stays 0."""
    import ctypes

    from paper_2410_07192_b200 import native

    s = torch.cuda.current_stream().cuda_stream
    for start, want in ((1, 7), (0, 0)):
        flag = ctypes.c_void_p()
        native.call("pf_flag_create", ctypes.byref(flag))
        native.call("pf_flag_write_on_stream", flag, start, s)
        anchor = torch.zeros(1, dtype=torch.int64, device="cuda")
        native.call("pf_read_globaltimer", anchor.data_ptr(), s)
        native.call("pf_flag_throttle_at", flag, anchor.data_ptr(), 20_000, 7, s)
        val = torch.full((1,), -1, dtype=torch.int32).pin_memory()
        native.call("pf_stage_d2h", val.data_ptr(), flag, 4, s)
        torch.cuda.synchronize()
        native.call("pf_flag_destroy", flag)
        assert int(val.item()) == want
