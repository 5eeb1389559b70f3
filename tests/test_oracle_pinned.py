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


def _torchvision_resnet50_from(model):
    """torchvision's ResNet-50 (eval) carrying the fill model's folded weights: every
    BatchNorm is the identity scale (gamma 1, running var 1 - eps, mean 0) with the
    folded shift as beta, so conv + BN == the folded conv the kernels run."""
    import torchvision

    tv = torchvision.models.resnet50(weights=None).eval()
    params = [model.oracle_params(i) for i in range(len(model))]

    def load(conv, bn, w, b):
        from oracle.fill_ref import conv_weight
        k = conv.kernel_size[0]
        conv.weight.data.copy_(conv_weight(w, conv.in_channels, k, k))
        bn.weight.data.fill_(1.0)
        bn.bias.data.copy_(b.float())
        bn.running_mean.data.zero_()
        bn.running_var.data.fill_(1.0 - bn.eps)

    load(tv.conv1, tv.bn1, params[0]["w"], params[0]["b"])
    i = 1
    for layer in (tv.layer1, tv.layer2, tv.layer3, tv.layer4):
        for blk in layer:
            p = params[i]
            load(blk.conv1, blk.bn1, p["w1"], p["b1"])
            load(blk.conv2, blk.bn2, p["w2"], p["b2"])
            load(blk.conv3, blk.bn3, p["w3"], p["b3"])
            if blk.downsample is not None:
                load(blk.downsample[0], blk.downsample[1], p["wd"], p["bd"])
            i += 1
    tv.fc.weight.data.copy_(params[i]["fc_w"].float())
    tv.fc.bias.data.copy_(params[i]["fc_b"].float())
    return tv, params


def test_resnet50_oracle_matches_torchvision():
    """The ResNet-50 oracle (folded-BN NCHW fp32, module by module as the fill model is
    partitioned) against torchvision.models.resnet50 with the same weights."""
    from paper_2410_07192_b200.fillmodels import ResNetConfig, resnet50

    cfg = ResNetConfig(image=64)
    model = resnet50(cfg, seed=3, pinned=False)
    tv, params = _torchvision_resnet50_from(model)
    img = model.make_inputs(11, 0, 2)  # NHWC bf16
    with torch.no_grad():
        want = tv(img.float().permute(0, 3, 1, 2))
        x = fill_ref.resnet_stem(img, params[0])
        for i in range(1, len(model) - 1):
            x = fill_ref.bottleneck(x, params[i], model[i].stride)
        got = fill_ref.resnet_head(x, params[-1])
    rel = ((got - want).norm() / want.norm()).item()
    assert rel < 1e-5, rel
