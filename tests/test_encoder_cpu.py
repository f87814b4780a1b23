"""CPU checks of the frozen-encoder oracle (oracle/encoder.py):
bidirectional attention against torch, the encoder pinned to HF transformers'
Qwen2.5-VL vision tower on identical weights, the window / position
conventions, the placeholder placement and the feature -> position mapping
used by the step oracle."""
import math

import numpy as np
import torch

from oracle import encoder as oe
from oracle.model import bf16_round
from paper_2508_02317_b200.runtime import synthetic_batch, synthetic_images
from tests.step_common import tiny_dense, tiny_encoder


def _model():
    m = tiny_dense(layers=1, hidden=256, heads=2, kv=2, ffn=512, vocab=512)
    m["modules"].append(tiny_encoder(layers=2, hidden=160, heads=2, head_dim=80, ffn=256, patch_dim=40,
                                     tokens_per_item=16))
    return m


def test_attention_bidir_matches_torch():
    rng = np.random.default_rng(0)
    cu = [0, 5, 6, 19]
    q, k, v = (bf16_round(rng.standard_normal((19, 2, 80)).astype(np.float32)) for _ in range(3))
    o = oe.attention_bidir(q, k, v, cu, 1 / math.sqrt(80))
    for a, b in zip(cu[:-1], cu[1:]):
        t = [torch.from_numpy(x[a:b]).double().transpose(0, 1) for x in (q, k, v)]
        ref = torch.nn.functional.scaled_dot_product_attention(*t, scale=1 / math.sqrt(80))
        np.testing.assert_allclose(o[a:b], ref.transpose(0, 1).numpy(), rtol=1e-5, atol=1e-6)


def _hf_vision(ea, P):
    """HF transformers' Qwen2.5-VL vision tower (the module VeOmni trains
    around) with the oracle's weights, fp32, eager attention."""
    from transformers.models.qwen2_5_vl.configuration_qwen2_5_vl import Qwen2_5_VLVisionConfig
    from transformers.models.qwen2_5_vl.modeling_qwen2_5_vl import Qwen2_5_VisionTransformerPretrainedModel

    ps = int(round(math.sqrt(ea.patch_dim / 6)))
    assert 3 * 2 * ps * ps == ea.patch_dim
    cfg = Qwen2_5_VLVisionConfig(depth=ea.layers, hidden_size=ea.hidden, num_heads=ea.heads,
                                 intermediate_size=ea.ffn, out_hidden_size=ea.out_hidden, patch_size=ps,
                                 temporal_patch_size=2, in_channels=3, spatial_merge_size=2,
                                 window_size=ea.window_merge * 2 * ps, fullatt_block_indexes=ea.fullatt,
                                 hidden_act="silu")
    cfg._attn_implementation = "eager"
    m = Qwen2_5_VisionTransformerPretrainedModel(cfg).float().eval()
    sd = m.state_dict()
    for k in sd:
        src = P["visual." + k]
        sd[k] = torch.from_numpy(np.ascontiguousarray(src)).reshape(sd[k].shape).float()
    m.load_state_dict(sd)
    return m


def test_encoder_oracle_pinned_to_hf_qwen2_5_vl_vision():
    """oracle.encoder_fwd (round_operands=False) == HF Qwen2_5_VisionTransformer
    on the same weights: 2-D RoPE, windowed + full-attention blocks, biases,
    window permutation and its inverse, merger."""
    model = tiny_dense(layers=1, hidden=256, heads=2, kv=2, ffn=512, vocab=512)
    enc = tiny_encoder(layers=3, hidden=160, heads=2, head_dim=80, ffn=256, patch_dim=96, tokens_per_item=16)
    enc["arch"].update(window_merge=2, fullatt_blocks=[1])
    model["modules"].append(enc)
    ea = oe.EncArch.from_model_json(model)
    assert ea.fullatt == [1] and ea.window_merge == 2
    P = oe.init_encoder(ea, 2508)
    pix = np.random.default_rng(3).standard_normal((2, 64, 96)).astype(np.float32)
    hf = _hf_vision(ea, P)
    with torch.no_grad():
        ref = hf(torch.from_numpy(pix.reshape(-1, 96)), grid_thw=torch.tensor([[1, 8, 8]] * 2)).pooler_output
    ref = ref.numpy()
    got = oe.encoder_fwd(ea, P, pix, round_operands=False)
    assert got.shape == ref.shape == (32, 256)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-4, err
    # the executor's bf16 rounding points stay close to the fp32 module
    got16 = oe.encoder_fwd(ea, P, pix)
    assert np.abs(got16 - ref).max() / np.abs(ref).max() < 3e-2
    # windows matter: all-full attention gives different features
    ea_full = oe.EncArch(**{**ea.__dict__, "fullatt": [0, 1, 2]})
    assert np.abs(oe.encoder_fwd(ea_full, P, pix, round_operands=False) - ref).max() > 1e-3


def test_window_order_and_positions():
    order, lens = oe.window_order(8, 2)
    assert lens == [16, 16, 16, 16] and sorted(order) == list(range(16))
    assert list(order[:4]) == [0, 1, 4, 5]  # units (0,0),(0,1),(1,0),(1,1) of a 4x4 unit grid
    hp, wp = oe.patch_hw(4)
    assert list(zip(hp[:4], wp[:4])) == [(0, 0), (0, 1), (1, 0), (1, 1)]
    order, lens = oe.window_order(32, 4)  # Qwen2.5-VL 448 px image: 16 windows of 8x8 patches
    assert lens == [64] * 16


def test_placeholders_and_injection_map():
    model = _model()
    ea = oe.EncArch.from_model_json(model)
    b = synthetic_images(synthetic_batch(512, 256, 2, seed=7), tokens_per_item=16, patch_dim=40, items_per_row=2)
    img = b["img"]
    assert img["pixels"].shape == (len(img["row"]), 64, 40)
    order = list(zip(img["row"], img["pos"]))
    assert order == sorted(order)
    for r, p in order:
        assert (b["labels"][r, p - 1:p + 16] == -100).all()
        cu = b["cu_rows"][r]
        assert any(a < p and p + 16 <= c for a, c in zip(cu[:-1], cu[1:]))  # inside one sample
    P = oe.init_encoder(ea, 2508)
    mask, feats = oe.inject_for_rows(ea, P, img, range(1, 2), 256)
    sel = img["row"] == 1
    assert mask.sum() == 16 * sel.sum() and feats.shape == (mask.sum(), 256)
    want = oe.encoder_fwd(ea, P, img["pixels"][sel])
    np.testing.assert_array_equal(feats, want)  # one row: positions ascend with the items
