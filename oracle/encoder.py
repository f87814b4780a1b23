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
The arithmetic lives in un-vendored VeOmni / HF code (Qwen2.5-VL vision
tower), so the encoder math is defined here, and the
executor implements exactly this; "parity" for this row means the executor
against this definition (parity unpinned against VeOmni itself):

  patches [P, pd] of one item (P = 4 * tokens_per_item)
  x  = patches . W_patch^T                                    (fp32 residual)
  per block:  x += proj(attn(rmsnorm1(x)))   bidirectional inside the item,
                                              heads x head_dim, no RoPE
              x += down(silu(gate(h2)) * up(h2)),  h2 = rmsnorm2(x)
  merger:     m = rmsnorm_q(x) viewed as [P/4, 4 He] (2x2 spatial merge of
              consecutive patches); feat = W2 . gelu(W1 . m)  ->  [P/4, H]

Qwen2.5-VL's 2-D RoPE and windowed attention are omitted.  The features
replace the embeddings of the item's tokens_per_item placeholder tokens
(masked scatter); those positions get no embedding gradient.  Weights use the
same deterministic init as the backbone (model.init_values, HF names).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

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

    @staticmethod
    def from_model_json(m: dict) -> "EncArch | None":
        """The first encoder module with an arch; patch width = its arch.vocab."""
        fnd = next(x for x in m["modules"] if x.get("kind", "foundation") == "foundation")
        for mod in m["modules"]:
            if mod.get("kind") == "encoder" and "arch" in mod:
                a = mod["arch"]
                return EncArch(hidden=a["hidden"], layers=a["layers"], heads=a["heads"],
                               head_dim=a["head_dim"], ffn=a["ffn_dim"], patch_dim=a["vocab"],
                               out_hidden=fnd["arch"]["hidden"],
                               tokens_per_item=mod["tokens_per_item"])
        return None


def encoder_specs(e: EncArch):
    He, F = e.hidden, e.ffn
    out = [("visual.patch_embed.proj.weight", (He, e.patch_dim), "normal")]
    for i in range(e.layers):
        p = f"visual.blocks.{i}."
        out += [(p + "norm1.weight", (He,), "ones"),
                (p + "attn.qkv.weight", (3 * e.heads * e.head_dim, He), "normal"),
                (p + "attn.proj.weight", (He, e.heads * e.head_dim), "normal"),
                (p + "norm2.weight", (He,), "ones"),
                (p + "mlp.gate_proj.weight", (F, He), "normal"),
                (p + "mlp.up_proj.weight", (F, He), "normal"),
                (p + "mlp.down_proj.weight", (He, F), "normal")]
    out += [("visual.merger.ln_q.weight", (He,), "ones"),
            ("visual.merger.mlp.0.weight", (4 * He, 4 * He), "normal"),
            ("visual.merger.mlp.2.weight", (e.out_hidden, 4 * He), "normal")]
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


def encoder_fwd(e: EncArch, P: dict, pixels: np.ndarray) -> np.ndarray:
    """pixels [n_items, 4*tpi, pd] -> features [n_items * tpi, out_hidden]
    (bf16-valued fp32), with the executor's bf16 rounding points."""
    r = bf16_round

    def mm(x, w):
        return (r(x).astype(np.float64) @ r(w).astype(np.float64).T).astype(F32)

    n, Pp, _ = pixels.shape
    assert Pp == 4 * e.tokens_per_item
    N = n * Pp
    cu = np.arange(0, N + 1, Pp)
    x = mm(pixels.reshape(N, -1), P["visual.patch_embed.proj.weight"])
    nh, d = e.heads, e.head_dim
    for i in range(e.layers):
        p = f"visual.blocks.{i}."
        h, _ = rmsnorm_fwd(x, r(P[p + "norm1.weight"]), e.rms_eps)
        qkv = r(mm(h, P[p + "attn.qkv.weight"]))
        q = qkv[:, : nh * d].reshape(N, nh, d)
        k = qkv[:, nh * d: 2 * nh * d].reshape(N, nh, d)
        v = qkv[:, 2 * nh * d:].reshape(N, nh, d)
        o = attention_bidir(q, k, v, cu, 1.0 / math.sqrt(d))
        x = (x + mm(o.reshape(N, nh * d), P[p + "attn.proj.weight"])).astype(F32)
        h2, _ = rmsnorm_fwd(x, r(P[p + "norm2.weight"]), e.rms_eps)
        act = silu(mm(h2, P[p + "mlp.gate_proj.weight"])) * mm(h2, P[p + "mlp.up_proj.weight"])
        x = (x + mm(act, P[p + "mlp.down_proj.weight"])).astype(F32)
    m, _ = rmsnorm_fwd(x, r(P["visual.merger.ln_q.weight"]), e.rms_eps)
    m = r(m).reshape(N // 4, 4 * e.hidden)
    y = gelu(r(mm(m, P["visual.merger.mlp.0.weight"])))
    return r(mm(y, P["visual.merger.mlp.2.weight"]))


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
