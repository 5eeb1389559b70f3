"""The fp32 fill path (north star: fp32 path within rel 1e-4 of the CPU torch execution):
fp32 kernels against CPU fp32 torch / the oracle, and a whole fp32 BERT through the
Executor, single- and multi-partition."""

import pytest
import torch

from oracle import fill_ref

pytestmark = pytest.mark.gpu

REL_TOL_FP32 = 1e-4  # north star: fp32 path rel 1e-4


def rel(got, want):
    got, want = got.float().cpu(), want.float().cpu()
    return ((got - want).abs().max() / want.abs().max().clamp_min(1e-12)).item()


@pytest.fixture(scope="module")
def K():
    from paper_2410_07192_b200 import kernels, native

    native.require_device()
    return kernels


@pytest.mark.parametrize("m,n,k,gelu,res", [(300, 264, 136, True, True), (1024, 768, 768, False, True),
                                            (96, 3072, 1024, True, False)])
def test_gemm_f32(K, m, n, k, gelu, res):
    g = torch.Generator().manual_seed(0)
    x = torch.randn(m, k, generator=g)
    w = torch.randn(n, k, generator=g) * k ** -0.5
    b = torch.randn(n, generator=g) * 0.1
    r = torch.randn(m, n, generator=g) if res else None
    got = K.linear(x.cuda(), w.cuda(), b.cuda(), gelu=gelu, residual=None if r is None else r.cuda())
    want = fill_ref.linear(x, w, b, gelu=gelu, residual=r)
    assert got.dtype == torch.float32
    assert rel(got, want) < 1e-5


def test_layernorm_attention_embedding_f32(K):
    g = torch.Generator().manual_seed(1)
    x, r = torch.randn(512, 768, generator=g), torch.randn(512, 768, generator=g)
    gam, bet = torch.rand(768, generator=g) + 0.5, torch.randn(768, generator=g) * 0.1
    got = K.layernorm(x.cuda(), gam.cuda(), bet.cuda(), 1e-12, residual=r.cuda())
    assert rel(got, fill_ref.layernorm(x + r, gam, bet, 1e-12)) < 1e-5
    qkv = torch.randn(3, 100, 3 * 256, generator=g)
    got = K.attention(qkv.cuda(), 4)
    assert rel(got, fill_ref.attention(qkv, 4)) < 1e-5
    ids = torch.randint(0, 1000, (2, 128), generator=g, dtype=torch.int32)
    word, pos, typ = torch.randn(1000, 256, generator=g), torch.randn(512, 256, generator=g), torch.randn(2, 256,
                                                                                                        generator=g)
    gam, bet = torch.ones(256), torch.zeros(256)
    got = K.embedding_ln(ids.cuda(), word.cuda(), pos.cuda(), typ.cuda(), gam.cuda(), bet.cuda(), 1e-12)
    assert rel(got, fill_ref.embedding_ln(ids, word, pos, typ, gam, bet, 1e-12)) < 1e-5


def test_bert_fp32_executor_matches_oracle():
    import paper_2410_07192_b200 as pf
    from paper_2410_07192_b200 import native
    from paper_2410_07192_b200.executor import BubbleSlot, Executor
    from paper_2410_07192_b200.fillmodels import BertConfig, bert, synthetic_ids
    from test_executor_gpu import oracle_cls, plan_item, run_to_completion

    native.require_device()
    cfg = BertConfig("bert_tiny_fp32", vocab=1000, hidden=256, heads=4, ffn=1024, layers=3, precision="fp32")
    model = bert(cfg, seed=3)
    n = 21
    item1, plan1 = plan_item(pf, model, samples=n, free_mem=8_000_000_000)
    assert len(plan1.partitions) == 1
    ex = Executor(256 << 20, job_seed=5)
    ex.load(item1, model)
    run_to_completion(ex, lambda k: BubbleSlot(k % 2, None, 0))
    got = ex.results().clone()
    ex.close()
    assert got.dtype == torch.float32
    ref = oracle_cls(model, synthetic_ids(5, 0, n, cfg.seq, cfg.vocab))
    assert rel(got, ref) < REL_TOL_FP32
    # memory cap -> multi-partition plan, fp32 activations offloaded between partitions
    w_emb, w_layer = model[0].weight_bytes(), model[1].weight_bytes()
    item2, plan2 = plan_item(pf, model, samples=n, free_mem=max(w_emb, 2 * w_layer) + 4_000_000)
    assert len(plan2.partitions) >= 2
    ex = Executor(256 << 20, job_seed=5, activation_store="host")
    ex.load(item2, model)
    run_to_completion(ex, lambda k: BubbleSlot(k % 2, None, 0))
    got2 = ex.results().clone()
    ex.close()
    assert torch.equal(got2, got)
