"""CPU oracle for the frozen omni-modal encoder path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's reference arm, never by the product path.

What the reference fixes (omniplan only sizes the encoder):
  * step_graph.cpp:141-166 build_encoders: per micro-batch an `encoder.<mod>`
    compute node of 2 * active_params * tokens FLOPs over this rank's share
    (mix_fraction * local_tokens) of the modality tokens, then a
    `scatter.<mod>` all_to_all of tokens * hidden * dtype bytes into the SP
    group when tokens_per_item > 0; a frozen module (trainable = false) has no
    backward node.
  * comm.cpp:91-105 encoder_scatter_volume: feature_bytes * (sp - 1) / sp.
  * specs.hpp:66-75 ModuleSpec {name, kind, arch, trainable, tokens_per_item}.
The arithmetic lives in un-vendored VeOmni code around the HF Qwen2.5-VL vision
tower.  This oracle restates HF transformers 5.5
`Qwen2_5_VisionTransformerPretrainedModel` (models/qwen2_5_vl/
modeling_qwen2_5_vl.py:345-518) and is pinned against it in
tests/test_encoder_cpu.py (same weights, fp32, round_operands=False):

  patches [P, pd] of one item, P = 4 * tokens_per_item = g x g patches
  (processor order: 2x2 merge units row-major, patches inside a unit
  row-major; rot_pos_emb :382-409)
  x  = patches . W_patch^T                        (Conv3d as a matmul, no bias)
  window order: merge units regrouped into windows of `window_merge` x
  `window_merge` units (get_window_index :411-451); x and the rotary angles
  are permuted into it, the merger output is permuted back (:512-514)
  per block i:
     h = rmsnorm1(x);  q|k|v = h . W_qkv^T + b_qkv
     2-D RoPE on q, k (rotate_half over head_dim, angle of dim j < d/2:
       hpos * inv[j] for j < d/4, wpos * inv[j - d/4], inv from theta 1e4 over
       d/2 dims; apply_rotary_pos_emb_vision :164-175)
     attention bidirectional inside the item when i is a full-attention block
     (fullatt_blocks), else inside each window
     x += o . W_proj^T + b_proj
     x += down(silu(gate(h2)) * up(h2)) (+ biases), h2 = rmsnorm2(x)
  merger: m = rmsnorm_q(x) viewed as [P/4, 4 He]; feat = W2 . gelu(W1 . m + b1) + b2

Defaults follow Qwen2.5-VL-7B: window_merge 4 (112 px windows of 14 px
patches), full-attention blocks every 8th ({7, 15, 23, 31} at depth 32; the
last block of a shallower encoder).  The features replace the embeddings of
the item's tokens_per_item placeholder tokens (masked scatter); those
positions get no embedding gradient.  Weights and biases use the backbone's
deterministic init (model.init_values, HF names).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from oracle.model import F32, bf16_round, init_values, param_key, rmsnorm_fwd, silu


@dataclass
class EncArch:
    hidden: int
    layers: int
    heads: int
    head_dim: int
    ffn: int
    patch_dim: int
    out_hidden: int
    tokens_per_item: int
    rms_eps: float = 1e-6
    window_merge: int = 4
    fullatt: list = field(default_factory=list)
    rope_theta: float = 10000.0

    @staticmethod
    def from_model_json(m: dict) -> "EncArch | None":
        """The first encoder module with an arch; patch width = its arch.vocab;
        optional arch keys window_merge, fullatt_blocks, rope_theta."""
        fnd = next(x for x in m["modules"] if x.get("kind", "foundation") == "foundation")
        for mod in m["modules"]:
            if mod.get("kind") == "encoder" and "arch" in mod:
                a = mod["arch"]
                L = a["layers"]
                return EncArch(hidden=a["hidden"], layers=L, heads=a["heads"],
                               head_dim=a["head_dim"], ffn=a["ffn_dim"], patch_dim=a["vocab"],
                               out_hidden=fnd["arch"]["hidden"],
                               tokens_per_item=mod["tokens_per_item"],
                               window_merge=a.get("window_merge", 4),
                               fullatt=list(a.get("fullatt_blocks", default_fullatt(L))),
                               rope_theta=a.get("rope_theta", 10000.0))
        return None


def default_fullatt(layers: int):
    """Qwen2.5-VL-7B: blocks 7, 15, 23, 31 of 32 attend over the whole image."""
    return sorted({i for i in range(layers) if (i + 1) % 8 == 0} | {layers - 1})


def grid_of(e: EncArch) -> int:
    """Patch grid side g of one item (g x g = 4 * tokens_per_item, g even)."""
    P = 4 * e.tokens_per_item
    g = int(round(math.sqrt(P)))
    assert g * g == P and g % 2 == 0, "items must be square patch grids of even side"
    return g


def patch_hw(g: int):
    """(hpos, wpos) of every patch in processor order (rot_pos_emb :382-409)."""
    i = np.arange(g * g)
    unit, sub = i // 4, i % 4
    bh, bw = unit // (g // 2), unit % (g // 2)
    return bh * 2 + sub // 2, bw * 2 + sub % 2


def window_order(g: int, wm: int):
    """(window_index over merge units, window lengths in patches) as
    get_window_index :411-451 (padding windows dropped)."""
    lg = g // 2
    pad = wm - lg % wm
    nw = (lg + pad) // wm
    idx = np.full((nw * wm, nw * wm), -1, np.int64)
    idx[:lg, :lg] = np.arange(lg * lg).reshape(lg, lg)
    idx = idx.reshape(nw, wm, nw, wm).transpose(0, 2, 1, 3).reshape(nw * nw, wm * wm)
    order, lens = [], []
    for w in idx:
        v = w[w >= 0]
        if len(v):
            order += list(v)
            lens.append(4 * len(v))
    return np.array(order, np.int64), lens


def rope_angles(e: EncArch, g: int):
    """[P, d/2] rotary angles of every patch (processor order)."""
    d = e.head_dim
    half, quarter = d // 2, d // 4
    inv = (1.0 / (e.rope_theta ** (np.arange(0, half, 2, dtype=np.float64) / half))).astype(F32)
    hp, wp = patch_hw(g)
    ang = np.concatenate([hp[:, None].astype(F32) * inv[None, :quarter],
                          wp[:, None].astype(F32) * inv[None, :quarter]], axis=1)
    return ang.astype(F32)


def encoder_specs(e: EncArch):
    He, F = e.hidden, e.ffn
    W = e.heads * e.head_dim
    out = [("visual.patch_embed.proj.weight", (He, e.patch_dim), "normal")]
    for i in range(e.layers):
        p = f"visual.blocks.{i}."
        out += [(p + "norm1.weight", (He,), "ones"),
                (p + "attn.qkv.weight", (3 * W, He), "normal"),
                (p + "attn.qkv.bias", (3 * W,), "normal"),
                (p + "attn.proj.weight", (He, W), "normal"),
                (p + "attn.proj.bias", (He,), "normal"),
                (p + "norm2.weight", (He,), "ones"),
                (p + "mlp.gate_proj.weight", (F, He), "normal"),
                (p + "mlp.gate_proj.bias", (F,), "normal"),
                (p + "mlp.up_proj.weight", (F, He), "normal"),
                (p + "mlp.up_proj.bias", (F,), "normal"),
                (p + "mlp.down_proj.weight", (He, F), "normal"),
                (p + "mlp.down_proj.bias", (He,), "normal")]
    out += [("visual.merger.ln_q.weight", (He,), "ones"),
            ("visual.merger.mlp.0.weight", (4 * He, 4 * He), "normal"),
            ("visual.merger.mlp.0.bias", (4 * He,), "normal"),
            ("visual.merger.mlp.2.weight", (e.out_hidden, 4 * He), "normal"),
            ("visual.merger.mlp.2.bias", (e.out_hidden,), "normal")]
    return out


def init_encoder(e: EncArch, seed: int) -> dict:
    P = {}
    for name, shape, kind in encoder_specs(e):
        n = int(np.prod(shape))
        P[name] = np.ones(shape, F32) if kind == "ones" else init_values(param_key(name, seed), n).reshape(shape)
    return P


def _erf(x: np.ndarray) -> np.ndarray:
    from scipy.special import erf  # noqa: PLC0415

    return erf(x)


def gelu(x):
    return (0.5 * x * (1.0 + _erf(x.astype(np.float64) / math.sqrt(2.0)))).astype(F32)


def attention_bidir(q, k, v, cu, scale):
    """q/k/v [N, h, d] (bf16-valued), bidirectional inside [cu[i], cu[i+1])."""
    N, h, d = q.shape
    o = np.zeros((N, h, d), F32)
    for a, b in zip(cu[:-1], cu[1:]):
        qs, ks, vs = (t[a:b].astype(np.float64) for t in (q, k, v))
        s = np.einsum("qhd,khd->hqk", qs, ks) * scale
        s -= s.max(-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(-1, keepdims=True)
        o[a:b] = np.einsum("hqk,khd->qhd", p, vs).astype(F32)
    return o


def rope_rotate(x, ang):
    """rotate_half RoPE of x [N, h, d] with per-row angles [N, d/2] (fp32)."""
    half = x.shape[-1] // 2
    c, s = np.cos(ang.astype(np.float64)).astype(F32), np.sin(ang.astype(np.float64)).astype(F32)
    c, s = c[:, None, :], s[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], -1).astype(F32)


def encoder_fwd(e: EncArch, P: dict, pixels: np.ndarray, round_operands: bool = True) -> np.ndarray:
    """pixels [n_items, 4*tpi, pd] -> features [n_items * tpi, out_hidden] in
    processor (merge-unit) order.  round_operands: the executor's bf16
    rounding points (GEMM operands and bf16 GEMM outputs, q/k/v after RoPE,
    the merger input and GELU output); False = plain fp32/fp64 (HF pin)."""
    r = bf16_round if round_operands else (lambda x: np.asarray(x, F32))

    def mm(x, w, b=None):
        y = r(x).astype(np.float64) @ r(w).astype(np.float64).T
        if b is not None:
            y = y + r(b).astype(np.float64)
        return y.astype(F32)

    n, Pp, _ = pixels.shape
    assert Pp == 4 * e.tokens_per_item
    g = grid_of(e)
    worder, wlens = window_order(g, e.window_merge)
    perm = (worder[:, None] * 4 + np.arange(4)[None, :]).reshape(-1)  # patch rows in window order
    ang = rope_angles(e, g)[perm]
    nh, d = e.heads, e.head_dim
    out = []
    for it in range(n):
        x = mm(pixels[it], P["visual.patch_embed.proj.weight"])[perm]
        cu_full = [0, Pp]
        cu_win = list(np.cumsum([0] + wlens))
        for i in range(e.layers):
            p = f"visual.blocks.{i}."
            h, _ = rmsnorm_fwd(x, r(P[p + "norm1.weight"]), e.rms_eps)
            qkv = r(mm(h, P[p + "attn.qkv.weight"], P[p + "attn.qkv.bias"]))
            q = r(rope_rotate(qkv[:, : nh * d].reshape(Pp, nh, d), ang))
            k = r(rope_rotate(qkv[:, nh * d: 2 * nh * d].reshape(Pp, nh, d), ang))
            v = qkv[:, 2 * nh * d:].reshape(Pp, nh, d)
            o = attention_bidir(q, k, v, cu_full if i in e.fullatt else cu_win, 1.0 / math.sqrt(d))
            x = (x + mm(r(o).reshape(Pp, nh * d), P[p + "attn.proj.weight"], P[p + "attn.proj.bias"])).astype(F32)
            h2, _ = rmsnorm_fwd(x, r(P[p + "norm2.weight"]), e.rms_eps)
            gt = r(mm(h2, P[p + "mlp.gate_proj.weight"], P[p + "mlp.gate_proj.bias"]))
            up = r(mm(h2, P[p + "mlp.up_proj.weight"], P[p + "mlp.up_proj.bias"]))
            act = silu(gt) * up
            x = (x + mm(act, P[p + "mlp.down_proj.weight"], P[p + "mlp.down_proj.bias"])).astype(F32)
        m, _ = rmsnorm_fwd(x, r(P["visual.merger.ln_q.weight"]), e.rms_eps)
        m = r(m).reshape(Pp // 4, 4 * e.hidden)
        y = r(gelu(r(mm(m, P["visual.merger.mlp.0.weight"], P["visual.merger.mlp.0.bias"]))))
        f = r(mm(y, P["visual.merger.mlp.2.weight"], P["visual.merger.mlp.2.bias"]))
        out.append(f[np.argsort(worder)])
    return np.concatenate(out, 0)


def inject_for_rows(e: EncArch, P: dict, img: dict, rows: range, S: int):
    """(mask [len(rows)*S] bool, features [n_masked, H]) for the items placed in
    `rows` of the global batch (positions row-major over those rows)."""
    sel = [j for j in range(len(img["row"])) if img["row"][j] in rows]
    mask = np.zeros(len(rows) * S, bool)
    if not sel:
        return mask, np.zeros((0, e.out_hidden), F32)
    feats = encoder_fwd(e, P, img["pixels"][sel])
    tpi = e.tokens_per_item
    order = []
    for jj, j in enumerate(sel):
        base = (img["row"][j] - rows.start) * S + img["pos"][j]
        mask[base: base + tpi] = True
        order += [(base + t, jj * tpi + t) for t in range(tpi)]
    order.sort()
    return mask, feats[[f for _, f in order]]
