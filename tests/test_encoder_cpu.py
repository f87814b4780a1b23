"""CPU checks of the frozen-encoder oracle (oracle/encoder.py):
bidirectional attention against torch, the encoder against an independent
torch restatement with the same bf16 rounding points, the placeholder
placement and the feature -> position mapping used by the step oracle."""
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
                                     tokens_per_item=4))
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


def _torch_encoder(ea, P, pixels):
    """Independent restatement: torch fp64 with bf16 casts at the executor's
    rounding points (GEMM operands, bf16 GEMM outputs, the merger input)."""
    def r(x):
        return x.to(torch.bfloat16).double()

    def lin(x, w):
        return r(x) @ r(torch.from_numpy(P[w]).double()).T

    def norm(x, w):
        y = x * torch.rsqrt((x * x).mean(-1, keepdim=True) + ea.rms_eps)
        return y * r(torch.from_numpy(P[w]).double())

    n, Pp, pd = pixels.shape
    x = lin(torch.from_numpy(pixels.reshape(n * Pp, pd)).double(), "visual.patch_embed.proj.weight").float().double()
    h, d = ea.heads, ea.head_dim
    for i in range(ea.layers):
        p = f"visual.blocks.{i}."
        qkv = r(lin(norm(x, p + "norm1.weight"), p + "attn.qkv.weight"))
        q, k, v = (qkv[:, j * h * d:(j + 1) * h * d].reshape(n, Pp, h, d).transpose(1, 2) for j in range(3))
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v, scale=1 / math.sqrt(d))
        x = x + lin(o.transpose(1, 2).reshape(n * Pp, h * d), p + "attn.proj.weight")
        h2 = norm(x, p + "norm2.weight")
        x = x + lin(torch.nn.functional.silu(lin(h2, p + "mlp.gate_proj.weight")) * lin(h2, p + "mlp.up_proj.weight"),
                    p + "mlp.down_proj.weight")
    m = r(norm(x, "visual.merger.ln_q.weight")).reshape(n * Pp // 4, 4 * ea.hidden)
    y = torch.nn.functional.gelu(r(lin(m, "visual.merger.mlp.0.weight")))
    return r(lin(y, "visual.merger.mlp.2.weight")).numpy()


def test_encoder_matches_torch_restatement():
    model = _model()
    ea = oe.EncArch.from_model_json(model)
    assert (ea.hidden, ea.patch_dim, ea.out_hidden, ea.tokens_per_item) == (160, 40, 256, 4)
    P = oe.init_encoder(ea, 2508)
    pix = np.random.default_rng(1).standard_normal((3, 16, 40)).astype(np.float32)
    got = oe.encoder_fwd(ea, P, pix)
    ref = _torch_encoder(ea, P, pix)
    assert got.shape == (12, 256)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-2, err


def test_placeholders_and_injection_map():
    model = _model()
    ea = oe.EncArch.from_model_json(model)
    b = synthetic_images(synthetic_batch(512, 256, 2, seed=7), tokens_per_item=4, patch_dim=40, items_per_row=2)
    img = b["img"]
    assert img["pixels"].shape == (len(img["row"]), 16, 40)
    order = list(zip(img["row"], img["pos"]))
    assert order == sorted(order)
    for r, p in order:
        assert (b["labels"][r, p - 1:p + 4] == -100).all()
        cu = b["cu_rows"][r]
        assert any(a < p and p + 4 <= c for a, c in zip(cu[:-1], cu[1:]))  # inside one sample
    P = oe.init_encoder(ea, 2508)
    mask, feats = oe.inject_for_rows(ea, P, img, range(1, 2), 256)
    sel = img["row"] == 1
    assert mask.sum() == 4 * sel.sum() and feats.shape == (mask.sum(), 256)
    want = oe.encoder_fwd(ea, P, img["pixels"][sel])
    np.testing.assert_array_equal(feats, want)  # one row: positions ascend with the items
