"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the timed
CPU baseline.  The product path (libopx.so) never calls it.

numpy restatement (fp32 storage, fp64 accumulation in reductions) of one
fwd+bwd+AdamW training step of the decoder the reference models:

* block shapes and layer typing follow omniplan's accounting
  (proj/src/specs.cpp:36-55, proj/include/omniplan/specs.hpp:39-62): bias-free
  q/k/v/o, two RMSNorms per layer, gated MLP or MoE (router + E experts) on
  layers with (l+1) % stride == 0, untied embedding/head + final norm;
* Ulysses semantics and FSDP sharding over dp_shard*sp
  (plan.hpp:22-25) are reproduced by ``simulate_ranks`` which splits tokens
  the way the mesh does (plan.cpp:161-166: SP group = consecutive ranks) and
  sums parameter gradients in rank order;
* packed varlen isolation via cu_seqlens (packing.hpp:20-31);
* math conventions the reference leaves to third-party code are taken from
  HF transformers 5.5 Qwen2 / Qwen3-MoE (installed, not under /root/reference):
  RMSNorm rsqrt(mean(x^2)+eps)*w, rotate_half RoPE (theta 1e6), SwiGLU MLP,
  router softmax -> top-k -> renormalise (norm_topk_prob=True, the
  Qwen3-30B-A3B checkpoint setting), AdamW as torch.optim.AdamW.

Parity status: the reference computes no tensors (proj/README.md:22-23), so
nothing in /root/reference pins these numerics; tests/test_oracle.py pins this
oracle against HF transformers' Qwen2/Qwen3-MoE forward and torch autograd on
identical weights, and against the compiled reference planner for all
accounting values.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

F32 = np.float32
MASK64 = (1 << 64) - 1

# Accumulation dtype of the GEMMs, attention and reductions: fp64 (the
# checker).  bench.py's CPU baseline legs switch it to fp32 (set_accumulate)
# so the timed CPU path is an all-core fp32 BLAS implementation of the step.
_ACC = [np.float64]


def ACC():
    return _ACC[0]


def set_accumulate(dtype) -> None:
    _ACC[0] = np.dtype(dtype).type

# C helpers (oracle/c/oracle_init.c, built by oracle/Makefile): bit-identical
# restatements of init_values / bf16_round that only make large-width parity
# tests fast; the numpy code below is the definition and the fallback.
_CLIB = None


def _clib():
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os

        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "liboracle_init.so")
        _CLIB = False
        if os.path.exists(path) and not os.environ.get("ORACLE_NO_C"):
            L = ctypes.CDLL(path)
            L.oracle_init_values.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_double, ctypes.c_void_p]
            L.oracle_bf16_round.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
            _CLIB = L
    return _CLIB


# ----------------------------------------------------------------------------
# configuration
# ----------------------------------------------------------------------------
@dataclasses.dataclass
class Arch:
    layers: int
    hidden: int
    heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    experts: int = 0
    top_k: int = 0
    expert_ffn: int = 0
    moe_stride: int = 1
    rms_eps: float = 1e-6
    rope_theta: float = 1e6

    @staticmethod
    def from_model_json(m: dict) -> "Arch":
        f = [x for x in m["modules"] if x["kind"] == "foundation"][0]["arch"]
        moe = f.get("moe")
        return Arch(layers=f["layers"], hidden=f["hidden"], heads=f["heads"], kv_heads=f["kv_heads"],
                    head_dim=f["head_dim"], ffn=f["ffn_dim"], vocab=f["vocab"],
                    experts=moe["num_experts"] if moe else 0, top_k=moe["top_k"] if moe else 0,
                    expert_ffn=moe["expert_ffn_dim"] if moe else 0,
                    moe_stride=moe.get("moe_layer_stride", 1) if moe else 1)

    def is_moe(self, l: int) -> bool:
        return self.experts > 0 and (l + 1) % self.moe_stride == 0


# ----------------------------------------------------------------------------
# deterministic init (bit-identical to kernels/elementwise.cu init_kernel)
# ----------------------------------------------------------------------------
def fnv1a64(s: str) -> int:
    h = 0xCBF29CE484222325
    for ch in s.encode():
        h ^= ch
        h = (h * 0x100000001B3) & MASK64
    return h


def param_key(name: str, seed: int) -> int:
    return fnv1a64(name) ^ ((seed * 0x9E3779B97F4A7C15) & MASK64)


def _splitmix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        z = x
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def init_values(key: int, n: int, std: float = 0.02, start: int = 0) -> np.ndarray:
    L = _clib()
    if L and n > 4096:
        out = np.empty(n, F32)
        L.oracle_init_values(key & MASK64, n, start, std * math.sqrt(3.0) / 16777216.0,
                             out.ctypes.data)
        return out
    return init_values_np(key, n, std, start)


def init_values_np(key: int, n: int, std: float = 0.02, start: int = 0) -> np.ndarray:
    i = np.arange(start, start + n, dtype=np.uint64)
    k = np.uint64(key)
    c = np.uint64(0xD1B54A32D192ED03)
    with np.errstate(over="ignore"):
        z0 = _splitmix(k + (np.uint64(2) * i) * c)
        z1 = _splitmix(k + (np.uint64(2) * i + np.uint64(1)) * c)
    m24 = np.uint64(0xFFFFFF)
    s = ((z0 >> np.uint64(40)).astype(np.int64) + ((z0 >> np.uint64(8)) & m24).astype(np.int64)
         + (z1 >> np.uint64(40)).astype(np.int64) + ((z1 >> np.uint64(8)) & m24).astype(np.int64)
         - (1 << 25))
    cc = std * math.sqrt(3.0) / 16777216.0
    return (s.astype(np.float64) * cc).astype(F32)


def param_specs(a: Arch):
    """(hf_name, shape, kind) in HF naming; kind 'normal' or 'ones'."""
    H, d = a.hidden, a.head_dim
    out = [("model.embed_tokens.weight", (a.vocab, H), "normal")]
    for l in range(a.layers):
        p = f"model.layers.{l}."
        out += [(p + "input_layernorm.weight", (H,), "ones"),
                (p + "self_attn.q_proj.weight", (a.heads * d, H), "normal"),
                (p + "self_attn.k_proj.weight", (a.kv_heads * d, H), "normal"),
                (p + "self_attn.v_proj.weight", (a.kv_heads * d, H), "normal"),
                (p + "self_attn.o_proj.weight", (H, a.heads * d), "normal"),
                (p + "post_attention_layernorm.weight", (H,), "ones")]
        if a.is_moe(l):
            E, Fe = a.experts, a.expert_ffn
            out += [(p + "mlp.gate.weight", (E, H), "normal"),
                    (p + "mlp.experts.gate_proj", (E, Fe, H), "normal"),
                    (p + "mlp.experts.up_proj", (E, Fe, H), "normal"),
                    (p + "mlp.experts.down_proj", (E, H, Fe), "normal")]
        else:
            out += [(p + "mlp.gate_proj.weight", (a.ffn, H), "normal"),
                    (p + "mlp.up_proj.weight", (a.ffn, H), "normal"),
                    (p + "mlp.down_proj.weight", (H, a.ffn), "normal")]
    out += [("model.norm.weight", (H,), "ones"), ("lm_head.weight", (a.vocab, H), "normal")]
    return out


def init_params(a: Arch, seed: int) -> dict:
    P = {}
    for name, shape, kind in param_specs(a):
        n = int(np.prod(shape))
        if kind == "ones":
            P[name] = np.ones(shape, F32)
        else:
            P[name] = init_values(param_key(name, seed), n).reshape(shape)
    return P


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    x = np.ascontiguousarray(x, dtype=F32)
    L = _clib()
    if L and x.size > 4096:
        out = np.empty_like(x)
        L.oracle_bf16_round(x.ctypes.data, out.ctypes.data, x.size)
        return out
    return bf16_round_np(x)


def bf16_round_np(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=F32)
    u = x.view(np.uint32).astype(np.uint64)
    r = ((u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)) << np.uint64(16)
    out = r.astype(np.uint32).view(F32)
    return np.where(np.isnan(x), x, out)


# ----------------------------------------------------------------------------
# building blocks
# ----------------------------------------------------------------------------
def rmsnorm_fwd(x, w, eps):
    ms = (x.astype(ACC(), copy=False) ** 2).mean(-1, keepdims=True)
    rstd = (1.0 / np.sqrt(ms + eps)).astype(F32)
    return (x * rstd * w).astype(F32), rstd


def rmsnorm_bwd(dy, x, w, rstd):
    xh = x * rstd
    g = dy * w
    mean = (g.astype(ACC(), copy=False) * xh).mean(-1, keepdims=True).astype(F32)
    dx = rstd * (g - xh * mean)
    dw = (dy.astype(ACC(), copy=False) * xh).sum(0).astype(F32)
    return dx.astype(F32), dw


def rope_tables(pos, d, theta):
    inv = (1.0 / (theta ** (np.arange(0, d, 2, dtype=np.float64) / d))).astype(F32)
    ang = pos.astype(F32)[:, None] * inv[None, :]  # fp32 product, as on the GPU
    ang = ang.astype(np.float64)
    return np.cos(ang).astype(F32), np.sin(ang).astype(F32)


def rope_apply(x, cos, sin, inverse=False):
    """x [N, h, d]; rotate_half convention."""
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    c, s = cos[:, None, :], sin[:, None, :]
    if inverse:
        s = -s
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], -1).astype(F32)


def attention_fwd(q, k, v, cu, scale):
    """q [N,hq,d], k/v [N,hk,d]; causal within each [cu[i], cu[i+1])."""
    N, hq, d = q.shape
    hk = k.shape[1]
    G = hq // hk
    o = np.zeros_like(q)
    lse = np.zeros((hq, N), F32)
    for a, b in zip(cu[:-1], cu[1:]):
        L = b - a
        mask = np.tril(np.ones((L, L), bool))
        for h in range(hq):
            s = (q[a:b, h].astype(ACC(), copy=False) @ k[a:b, h // G].astype(ACC(), copy=False).T) * scale
            s = np.where(mask, s, -np.inf)
            m = s.max(-1, keepdims=True)
            e = np.exp(s - m)
            z = e.sum(-1, keepdims=True)
            o[a:b, h] = ((e / z) @ v[a:b, h // G]).astype(F32)
            lse[h, a:b] = (m + np.log(z))[:, 0]
    return o, lse


def attention_bwd(q, k, v, o, lse, do, cu, scale):
    N, hq, d = q.shape
    hk = k.shape[1]
    G = hq // hk
    dq = np.zeros_like(q)
    dk = np.zeros(k.shape, ACC())
    dv = np.zeros(v.shape, ACC())
    for a, b in zip(cu[:-1], cu[1:]):
        L = b - a
        mask = np.tril(np.ones((L, L), bool))
        for h in range(hq):
            kh = h // G
            qq, kk, vv = (t.astype(ACC(), copy=False) for t in (q[a:b, h], k[a:b, kh], v[a:b, kh]))
            s = np.where(mask, (qq @ kk.T) * scale, -np.inf)
            p = np.exp(s - lse[h, a:b, None].astype(ACC(), copy=False))
            dO = do[a:b, h].astype(ACC(), copy=False)
            dv[a:b, kh] += p.T @ dO
            dp = dO @ vv.T
            delta = (dO * o[a:b, h].astype(ACC(), copy=False)).sum(-1, keepdims=True)
            ds = p * (dp - delta)
            dq[a:b, h] = (ds @ kk * scale).astype(F32)
            dk[a:b, kh] += ds.T @ qq * scale
    return dq, dk.astype(F32), dv.astype(F32)


def silu(x):
    return x / (1.0 + np.exp(-x))


def router_logits(h_bf16, w_bf16):
    """fp32 logits in a defined summation order the GPU follows exactly
    (kernels/moe.cu router kernel): for H % 128 == 0 the K range is split in
    four quarters, each summed with k ascending -- every step rounds acc + h*w
    once (the bf16 x bf16 product is exact in fp32, so the kernel's fused
    multiply-add and this multiply-then-add agree bit for bit) -- and the
    partials are combined as (p0 + p1) + (p2 + p3); otherwise one sequential
    sum over all of K."""
    T, H = h_bf16.shape
    splits = 4 if H % 128 == 0 else 1
    q = H // splits
    parts = []
    for z in range(splits):
        acc = np.zeros((T, w_bf16.shape[0]), F32)
        for kk in range(z * q, (z + 1) * q):
            acc = (acc + (h_bf16[:, kk:kk + 1] * w_bf16[None, :, kk]).astype(F32)).astype(F32)
        parts.append(acc)
    if splits == 1:
        return parts[0]
    return ((parts[0] + parts[1]).astype(F32) + (parts[2] + parts[3]).astype(F32)).astype(F32)


def topk_route(logits, k):
    """Top-k on logits (softmax is monotone), ties -> lower expert index;
    weights = renormalised softmax over the selected experts."""
    T, E = logits.shape
    order = np.lexsort((np.broadcast_to(np.arange(E), (T, E)), -logits), axis=-1)
    idx = order[:, :k].astype(np.int32)
    sel = np.take_along_axis(logits, idx, -1).astype(np.float64)
    e = np.exp(sel - sel.max(-1, keepdims=True))
    w = (e / e.sum(-1, keepdims=True)).astype(F32)
    return idx, w


def permutation(idx, E):
    """Stable counting sort of (token, slot) pairs by expert: returns for each
    permuted row the flat pair index t*k+j, and per-expert counts."""
    flat = idx.reshape(-1)
    order = np.argsort(flat, kind="stable").astype(np.int32)
    counts = np.bincount(flat, minlength=E).astype(np.int32)
    return order, counts


# ----------------------------------------------------------------------------
# the model step
# ----------------------------------------------------------------------------
class Step:
    """One fwd+bwd on a packed batch.  All matmul operands are the bf16-rounded
    values the GPU feeds its tensor cores (weights and GEMM inputs), accumulation
    in fp64 and everything else in fp32, so GPU-vs-CPU differences are the
    GPU's rounding of intermediates only."""

    def __init__(self, a: Arch, params: dict, round_operands: bool = True, forced_routes=None):
        self.a = a
        self.P = params
        self.r = bf16_round if round_operands else (lambda x: x.astype(F32, copy=False))
        # {layer: [N, k] expert indices}: route with these instead of the
        # oracle's own top-k (the weights still come from the oracle's logits);
        # used to separate discrete routing flips from arithmetic differences.
        self.forced = forced_routes or {}
        self.flips = {}  # {layer: fraction of tokens whose expert set differs}

    def mm(self, x, w):  # x [N,K] . w[M,K]^T
        return (self.r(x).astype(ACC(), copy=False) @ self.r(w).astype(ACC(), copy=False).T).astype(F32)

    def run(self, ids, labels, pos, cu, n_valid, inject=None):
        """ids/labels/pos [N] (N = all tokens of the batch rows, concatenated);
        cu: global cu_seqlens over those tokens.  inject = (mask [N], feats):
        encoder features replacing the masked embeddings (oracle/encoder.py).
        Returns (loss_sum, grads)."""
        a, P = self.a, self.P
        H, d, nh, nk = a.hidden, a.head_dim, a.heads, a.kv_heads
        N = ids.shape[0]
        scale = 1.0 / math.sqrt(d)
        cos, sin = rope_tables(pos, d, a.rope_theta)
        G = {}
        x = self.r(P["model.embed_tokens.weight"])[ids].astype(F32)
        if inject is not None and inject[0].any():
            x[inject[0]] = inject[1]
        saved = []
        for l in range(a.layers):
            p = f"model.layers.{l}."
            st = {"x": x}
            h, st["r1"] = rmsnorm_fwd(x, self.r(P[p + "input_layernorm.weight"]), a.rms_eps)
            st["h"] = h
            q = self.mm(h, P[p + "self_attn.q_proj.weight"]).reshape(N, nh, d)
            k = self.mm(h, P[p + "self_attn.k_proj.weight"]).reshape(N, nk, d)
            v = self.mm(h, P[p + "self_attn.v_proj.weight"]).reshape(N, nk, d)
            qr, kr = rope_apply(q, cos, sin), rope_apply(k, cos, sin)
            qr, kr, v = self.r(qr), self.r(kr), self.r(v)
            o, lse = attention_fwd(qr, kr, v, cu, scale)
            st.update(qr=qr, kr=kr, v=v, o=o, lse=lse)
            o2 = o.reshape(N, nh * d)
            x2 = x + self.mm(o2, P[p + "self_attn.o_proj.weight"])
            st["x2"] = x2
            h2, st["r2"] = rmsnorm_fwd(x2, self.r(P[p + "post_attention_layernorm.weight"]), a.rms_eps)
            st["h2"] = h2
            if a.is_moe(l):
                y, st["moe"] = self.moe_fwd(l, h2)
            else:
                g = self.mm(h2, P[p + "mlp.gate_proj.weight"])
                u = self.mm(h2, P[p + "mlp.up_proj.weight"])
                act = silu(g) * u
                st.update(g=g, u=u, act=act)
                y = self.mm(act, P[p + "mlp.down_proj.weight"])
            x = (x2 + y).astype(F32)
            saved.append(st)
        hf, rf = rmsnorm_fwd(x, self.r(P["model.norm.weight"]), a.rms_eps)
        logits = self.mm(hf, P["lm_head.weight"]).astype(ACC(), copy=False)
        valid = labels >= 0
        m = logits.max(-1, keepdims=True)
        lse_v = (m + np.log(np.exp(logits - m).sum(-1, keepdims=True)))[:, 0]
        lab = np.where(valid, labels, 0)
        loss_rows = np.where(valid, lse_v - logits[np.arange(N), lab], 0.0)
        dlog = np.exp(logits - lse_v[:, None])
        dlog[np.arange(N), lab] -= 1.0
        dlog = (dlog * valid[:, None] / n_valid).astype(F32)
        # head backward
        G["lm_head.weight"] = (self.r(dlog).astype(ACC(), copy=False).T @ self.r(hf).astype(ACC(), copy=False)).astype(F32)
        dhf = (self.r(dlog).astype(ACC(), copy=False) @ self.r(P["lm_head.weight"]).astype(ACC(), copy=False)).astype(F32)
        dx, G["model.norm.weight"] = rmsnorm_bwd(dhf, x, self.r(P["model.norm.weight"]), rf)
        for l in reversed(range(a.layers)):
            p = f"model.layers.{l}."
            st = saved[l]
            if a.is_moe(l):
                dh2 = self.moe_bwd(l, st["h2"], st["moe"], dx, G)
            else:
                act = st["act"]
                G[p + "mlp.down_proj.weight"] = self.wgrad(dx, act)
                dact = self.dgrad(dx, P[p + "mlp.down_proj.weight"])
                g, u = self.r(st["g"]), self.r(st["u"])
                sg = 1.0 / (1.0 + np.exp(-g))
                dact = self.r(dact)
                du = dact * g * sg
                dg = dact * u * sg * (1.0 + g * (1.0 - sg))
                G[p + "mlp.gate_proj.weight"] = self.wgrad(dg, st["h2"])
                G[p + "mlp.up_proj.weight"] = self.wgrad(du, st["h2"])
                dh2 = self.dgrad(dg, P[p + "mlp.gate_proj.weight"]) + self.dgrad(du, P[p + "mlp.up_proj.weight"])
            ddx, G[p + "post_attention_layernorm.weight"] = rmsnorm_bwd(
                dh2.astype(F32), st["x2"], self.r(P[p + "post_attention_layernorm.weight"]), st["r2"])
            dx = (dx + ddx).astype(F32)
            o2 = st["o"].reshape(N, nh * d)
            G[p + "self_attn.o_proj.weight"] = self.wgrad(dx, o2)
            do = self.r(self.dgrad(dx, P[p + "self_attn.o_proj.weight"])).reshape(N, nh, d)
            dqr, dkr, dv = attention_bwd(st["qr"], st["kr"], st["v"], self.r(st["o"]), st["lse"], do, cu, scale)
            dq = rope_apply(dqr, cos, sin, inverse=True).reshape(N, nh * d)
            dk = rope_apply(dkr, cos, sin, inverse=True).reshape(N, nk * d)
            dv = dv.reshape(N, nk * d)
            h = st["h"]
            G[p + "self_attn.q_proj.weight"] = self.wgrad(dq, h)
            G[p + "self_attn.k_proj.weight"] = self.wgrad(dk, h)
            G[p + "self_attn.v_proj.weight"] = self.wgrad(dv, h)
            dh = (self.dgrad(dq, P[p + "self_attn.q_proj.weight"]) + self.dgrad(dk, P[p + "self_attn.k_proj.weight"])
                  + self.dgrad(dv, P[p + "self_attn.v_proj.weight"]))
            ddx, G[p + "input_layernorm.weight"] = rmsnorm_bwd(
                dh.astype(F32), st["x"], self.r(P[p + "input_layernorm.weight"]), st["r1"])
            dx = (dx + ddx).astype(F32)
        dE = np.zeros((a.vocab, H), ACC())
        if inject is not None:
            dx = np.where(inject[0][:, None], np.float32(0), dx)
        np.add.at(dE, ids, dx.astype(ACC(), copy=False))
        G["model.embed_tokens.weight"] = dE.astype(F32)
        self.loss_rows = loss_rows.astype(F32)
        return float(loss_rows.sum()), G

    def wgrad(self, dy, x):  # dW[M,K] = dy[N,M]^T x[N,K]
        return (self.r(dy).astype(ACC(), copy=False).T @ self.r(x).astype(ACC(), copy=False)).astype(F32)

    def dgrad(self, dy, w):  # dx[N,K] = dy[N,M] w[M,K]
        return (self.r(dy).astype(ACC(), copy=False) @ self.r(w).astype(ACC(), copy=False)).astype(F32)

    # -------------------------------------------------------------- MoE
    def moe_fwd(self, l, h2):
        a, P = self.a, self.P
        p = f"model.layers.{l}.mlp."
        hb = self.r(h2)
        logits = router_logits(hb, self.r(P[p + "gate.weight"]))
        idx, w = topk_route(logits, a.top_k)
        if l in self.forced:
            f = np.asarray(self.forced[l], np.int32).reshape(idx.shape)
            self.flips[l] = float(np.mean(np.any(np.sort(f, 1) != np.sort(idx, 1), 1)))
            idx = f
            sel = np.take_along_axis(logits, idx, -1).astype(np.float64)
            e = np.exp(sel - sel.max(-1, keepdims=True))
            w = (e / e.sum(-1, keepdims=True)).astype(F32)
        N = h2.shape[0]
        y = np.zeros((N, a.hidden), ACC())
        cache = {"idx": idx, "w": w, "logits": logits, "eo": {}}
        Wg, Wu, Wd = P[p + "experts.gate_proj"], P[p + "experts.up_proj"], P[p + "experts.down_proj"]
        for e in range(a.experts):
            rows, slots = np.nonzero(idx == e)
            if rows.size == 0:
                continue
            xe = h2[rows]
            g = self.mm(xe, Wg[e])
            u = self.mm(xe, Wu[e])
            act = silu(g) * u
            out = self.mm(act, Wd[e])
            cache["eo"][e] = (rows, slots, g, u, act, out)
            np.add.at(y, rows, out.astype(ACC(), copy=False) * w[rows, slots][:, None])
        return y.astype(F32), cache

    def moe_bwd(self, l, h2, cache, dy, G):
        a, P = self.a, self.P
        p = f"model.layers.{l}.mlp."
        N = h2.shape[0]
        Wg, Wu, Wd = P[p + "experts.gate_proj"], P[p + "experts.up_proj"], P[p + "experts.down_proj"]
        dWg = np.zeros(Wg.shape, F32)
        dWu = np.zeros(Wu.shape, F32)
        dWd = np.zeros(Wd.shape, F32)
        dh = np.zeros((N, a.hidden), ACC())
        dw = np.zeros((N, a.top_k), ACC())
        w = cache["w"]
        for e, (rows, slots, g, u, act, out) in cache["eo"].items():
            dout = (dy[rows] * w[rows, slots][:, None]).astype(F32)
            dw[rows, slots] = (dy[rows].astype(ACC(), copy=False) * out.astype(ACC(), copy=False)).sum(-1)
            dWd[e] = self.wgrad(dout, act)
            dact = self.r(self.dgrad(dout, Wd[e]))
            g, u = self.r(g), self.r(u)
            sg = 1.0 / (1.0 + np.exp(-g))
            du = dact * g * sg
            dg = dact * u * sg * (1.0 + g * (1.0 - sg))
            dWg[e] = self.wgrad(dg, h2[rows])
            dWu[e] = self.wgrad(du, h2[rows])
            dxe = self.dgrad(dg, Wg[e]) + self.dgrad(du, Wu[e])
            np.add.at(dh, rows, dxe.astype(ACC(), copy=False))
        # renormalised softmax over the selected logits
        dsel = w * (dw - (w * dw).sum(-1, keepdims=True))
        dlog = np.zeros((N, a.experts), F32)
        np.put_along_axis(dlog, cache["idx"], dsel.astype(F32), -1)
        G[p + "gate.weight"] = self.wgrad(dlog, h2)
        dh += self.dgrad(dlog, P[p + "gate.weight"])
        G[p + "experts.gate_proj"] = dWg
        G[p + "experts.up_proj"] = dWu
        G[p + "experts.down_proj"] = dWd
        return dh.astype(F32)


def adamw(params, grads, state, step, lr=1e-4, betas=(0.9, 0.95), eps=1e-8, wd=0.1):
    """torch.optim.AdamW semantics (decoupled decay), fp32."""
    b1, b2 = betas
    bc1 = 1 - b1 ** step
    bc2 = 1 - b2 ** step
    out = {}
    for k, p in params.items():
        g = grads[k].astype(F32)
        m, v = state.get(k, (np.zeros_like(p), np.zeros_like(p)))
        p = (p * F32(1 - lr * wd)).astype(F32)
        m = (m + (g - m) * F32(1 - b1)).astype(F32)
        v = (v * F32(b2) + F32(1 - b2) * g * g).astype(F32)
        denom = np.sqrt(v) / F32(math.sqrt(bc2)) + F32(eps)
        p = (p - F32(lr / bc1) * m / denom).astype(F32)
        state[k] = (m, v)
        out[k] = p
    return out


# ----------------------------------------------------------------------------
# simulated ranks (FSDP x SP x DP) for one step
# ----------------------------------------------------------------------------
def simulate_ranks(a: Arch, params: dict, batch, plan: dict, forced_routes=None, flips=None,
                   encoder=None, round_operands=True):
    """Runs the step the way the mesh partitions the batch: dp index r
    (= dp_replicate_idx*dp_shard + dp_shard_idx) owns rows
    [r*k*micro_batch, (r+1)*k*micro_batch), k = rows/(dp*micro_batch) the
    gradient-accumulation steps (step_graph.cpp:57), and runs them as k
    micro-batches of micro_batch consecutive rows.  Inside an SP group the Ulysses
    exchange is a pure relayout and every token-local op is row-independent,
    so the SP ranks of one group are evaluated jointly on their gathered rows.
    Parameter gradients of the dp ranks are summed in rank order (the FSDP
    reduce-scatter / HSDP all-reduce) and the loss is normalised by the global
    supervised-token count.  encoder = (EncArch, encoder params) runs the
    frozen encoder over batch["img"] (oracle/encoder.py).  round_operands=False
    skips the bf16 rounding of matmul operands (pure fp32/fp64 arithmetic: the
    reference point for the bf16 sensitivity floor the width-parity tests
    report).  Returns (loss_mean, grads)."""
    rows_per_dp = plan["micro_batch"]
    dp = plan["dp_replicate"] * plan["dp_shard"]
    ids, labels, pos, cus = batch["ids"], batch["labels"], batch["pos"], batch["cu_rows"]
    n_valid = int((labels >= 0).sum())
    total = None
    loss = 0.0
    assert ids.shape[0] % (dp * rows_per_dp) == 0, "rows must be a multiple of dp*micro_batch"
    for r in range(ids.shape[0] // rows_per_dp):  # micro-batches in (dp rank, micro) order
        sl = slice(r * rows_per_dp, (r + 1) * rows_per_dp)
        rid, rlab, rpos = ids[sl].reshape(-1), labels[sl].reshape(-1), pos[sl].reshape(-1)
        S = ids.shape[1]
        cu = [0]
        for i, c in enumerate(cus[sl]):
            cu += [i * S + x for x in c[1:]]
        fr = None
        if forced_routes:
            fr = {l: v[sl].reshape(-1, v.shape[-1]) for l, v in forced_routes.items()}
        inj = None
        if encoder is not None and "img" in batch:
            from oracle.encoder import inject_for_rows

            inj = inject_for_rows(encoder[0], encoder[1], batch["img"],
                                  range(r * rows_per_dp, (r + 1) * rows_per_dp), S)
        st = Step(a, params, round_operands=round_operands, forced_routes=fr)
        ls, g = st.run(rid, rlab, rpos, np.array(cu), n_valid, inject=inj)
        if flips is not None:
            for l, f in st.flips.items():
                flips.setdefault(l, []).append(f)
        loss += ls
        if total is None:
            total = {k: v.astype(np.float64) for k, v in g.items()}
        else:
            for k in total:
                total[k] += g[k]
    return loss / n_valid, {k: v.astype(F32) for k, v in total.items()}
