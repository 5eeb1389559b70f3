"""Pin the CPU fp32 fill oracle (oracle/fill_ref.py) against torch's own, independently
written BERT-style encoder (nn.TransformerEncoderLayer, post-LN, exact GELU).

The reference has no tensor code, so the oracle cannot be pinned to
reference golden vectors; this checks it restates standard BERT semantics."""

import torch
from torch import nn

from oracle import fill_ref


def test_bert_layer_matches_torch_transformer_encoder_layer():
    torch.manual_seed(0)
    h, heads, f, b, s = 64, 4, 256, 3, 16
    ref = nn.TransformerEncoderLayer(h, heads, f, dropout=0.0, activation="gelu", batch_first=True,
                                     norm_first=False, layer_norm_eps=1e-12).eval()
    p = {
        "qkv_w": ref.self_attn.in_proj_weight.detach(), "qkv_b": ref.self_attn.in_proj_bias.detach(),
        "out_w": ref.self_attn.out_proj.weight.detach(), "out_b": ref.self_attn.out_proj.bias.detach(),
        "ln1_g": ref.norm1.weight.detach(), "ln1_b": ref.norm1.bias.detach(),
        "ffn1_w": ref.linear1.weight.detach(), "ffn1_b": ref.linear1.bias.detach(),
        "ffn2_w": ref.linear2.weight.detach(), "ffn2_b": ref.linear2.bias.detach(),
        "ln2_g": ref.norm2.weight.detach(), "ln2_b": ref.norm2.bias.detach(),
    }
    # nn.MultiheadAttention packs in_proj as [q; k; v] with heads contiguous inside each:
    # exactly the (3, heads, d) layout fill_ref and the kernels use
    x = torch.randn(b, s, h)
    with torch.no_grad():
        want = ref(x)
    got = fill_ref.bert_layer(x, p, heads, 1e-12)
    assert torch.allclose(got, want, rtol=1e-4, atol=1e-4), (got - want).abs().max()


def test_attention_mask_and_softmax():
    torch.manual_seed(1)
    qkv = torch.randn(2, 8, 3 * 32)
    mask = torch.zeros(2, 8)
    mask[1, 5:] = -1e4
    o = fill_ref.attention(qkv, 2, mask)
    # masked keys get ~0 weight: dropping them must not change the output
    o2 = fill_ref.attention(qkv[1:, :5].contiguous(), 2)
    assert torch.allclose(o[1, :5], o2[0], atol=1e-5)
    p = fill_ref.softmax(torch.randn(5, 7), 0.3)
    assert torch.allclose(p.sum(-1), torch.ones(5))
