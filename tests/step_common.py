"""Shared configs and the GPU-vs-oracle comparison for full training steps."""
import numpy as np

from oracle import model as om

CLUSTER1 = {"num_nodes": 1, "gpus_per_node": 1, "gpu": {"peak_flops": 2.25e15, "hbm_bytes": 180e9},
            "link": {"intra_node_bw": 9e11, "inter_node_bw": 5e10, "intra_latency": 5e-6,
                     "inter_latency": 2e-5}}


def cluster(n):
    c = dict(CLUSTER1)
    c["gpus_per_node"] = n
    return c


def tiny_moe(layers=2, hidden=256, heads=2, kv=2, ffn=768, vocab=2048, experts=64, top_k=4,
             expert_ffn=256, stride=1):
    m = tiny_dense(layers, hidden, heads, kv, ffn, vocab)
    m["modules"][0]["arch"]["moe"] = {"num_experts": experts, "top_k": top_k,
                                      "expert_ffn_dim": expert_ffn, "moe_layer_stride": stride}
    return m


def gpu_param_names(arch):
    """Physical tensor names the executor exposes (gate|up stored interleaved)."""
    out = []
    for name, shape, _ in om.param_specs(arch):
        if name.endswith("mlp.gate_proj.weight"):
            out.append(name.replace("gate_proj", "gate_up_proj"))
        elif name.endswith("mlp.experts.gate_proj"):
            out.append(name.replace("gate_proj", "gate_up_proj"))
        elif name.endswith("mlp.up_proj.weight") or name.endswith("mlp.experts.up_proj"):
            continue
        else:
            out.append(name)
    return out


def tiny_dense(layers=2, hidden=256, heads=2, kv=2, ffn=768, vocab=2048):
    return {"param_dtype_bytes": 2, "modules": [{"name": "core", "kind": "foundation", "trainable": True,
            "arch": {"layers": layers, "hidden": hidden, "heads": heads, "kv_heads": kv,
                     "head_dim": hidden // heads, "ffn_dim": ffn, "vocab": vocab}}]}


def free_port() -> int:
    """A TCP port nothing listens on right now (the OS picks it)."""
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


EXEC = {"seed": 2508, "lr": 1e-4, "betas": [0.9, 0.95], "eps": 1e-8, "weight_decay": 0.1}

TOL_LOSS = 1e-3   # relative, north_star
TOL_GRAD = 2e-2   # max-abs-err / max-abs-ref, north_star
TOL_COS = 0.999


def gather_full(sessions, kind, name):
    """Reassemble a flattened tensor from every rank's slice (FSDP shards)."""
    parts = {}
    n = None
    for s in sessions:
        v, n, b, e = s.get(f"{kind}:{name}")
        if e > b:
            parts[b] = v
    out = np.zeros(n, np.float32)
    for b, v in parts.items():
        out[b:b + len(v)] = v
    return out


def global_routes(sessions, arch, plan, S):
    """Assemble every rank's forward top-k indices into [rows, S, k] per MoE layer
    (rank = (dp row block, SP token slice), runtime.local_slice layout)."""
    from paper_2508_02317_b200.runtime import rank_coords

    m, sp = plan["micro_batch"], plan["sp"]
    dpw = plan.get("dp_replicate", 1) * plan["dp_shard"]
    m *= sessions[0].accum  # rows per dp rank (all its micro-batches)
    rows = dpw * m
    Sl = S // sp
    out = {}
    for l in range(arch.layers):
        if not arch.is_moe(l):
            continue
        g = np.zeros((rows, S, arch.top_k), np.int32)
        for rank, s in enumerate(sessions):
            rep, sh, spi = rank_coords(rank, plan)
            dp = rep * plan["dp_shard"] + sh
            r = s.routes(l, m * Sl, arch.top_k).reshape(m, Sl, arch.top_k)
            g[dp * m:(dp + 1) * m, spi * Sl:(spi + 1) * Sl] = r
        out[l] = g
    return out


MAX_FLIP_RATE = 0.05  # fraction of tokens whose expert set differs from the oracle's own top-k (reported)


def tiny_encoder(layers=2, hidden=640, heads=8, head_dim=80, ffn=512, patch_dim=96, tokens_per_item=16,
                 window_merge=2):
    """Frozen Qwen2.5-VL-shaped encoder module (oracle/encoder.py); arch.vocab =
    patch width; window_merge 2 on the 8x8-patch items gives 4 windows, and the
    default full-attention block is the last one."""
    return {"name": "vision", "kind": "encoder", "trainable": False, "tokens_per_item": tokens_per_item,
            "arch": {"layers": layers, "hidden": hidden, "heads": heads, "kv_heads": heads,
                     "head_dim": head_dim, "ffn_dim": ffn, "vocab": patch_dim,
                     "window_merge": window_merge}}


BF16_FLOOR_FACTOR = 1.5


def _err_cos(x, ref):
    err = np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-30)
    cos = float(np.dot(x.ravel().astype(np.float64), ref.ravel()) /
                max(np.linalg.norm(x) * np.linalg.norm(ref), 1e-30))
    return float(err), cos


def compare_step(sessions, model, batch, plan, step_loss, check_params=True, bf16_floor=False):
    """Runs the oracle on the same batch/weights and compares loss, every
    gradient and the AdamW-updated master weights.  For MoE models the oracle
    is routed with the GPU's top-k choices (bf16 activations can flip near-tied
    experts) and the flip rate against the oracle's own routing is checked
    separately.

    bf16_floor=True (the BASELINE-width tests) also runs the oracle without
    bf16 operand rounding.  The distance between the two oracles is the
    sensitivity of each gradient to bf16 rounding of intermediates alone
    (at C1 width: up to 3.3 % max-err, cos 0.9996, on the attention-side
    gradients), so a gradient passes if it is within the flat north_star
    tolerance OR within BF16_FLOOR_FACTOR x that floor.  Returns a report dict."""
    arch = om.Arch.from_model_json(model)
    P0 = om.init_params(arch, EXEC["seed"])
    routes = global_routes(sessions, arch, plan, batch["ids"].shape[1]) if arch.experts else None
    flips = {}
    enc = None
    if "img" in batch:
        from oracle import encoder as oe

        ea = oe.EncArch.from_model_json(model)
        enc = (ea, oe.init_encoder(ea, EXEC["seed"]))
    loss_ref, G = om.simulate_ranks(arch, P0, batch, plan, forced_routes=routes, flips=flips, encoder=enc)
    floor = {}
    if bf16_floor:
        _, G32 = om.simulate_ranks(arch, P0, batch, plan, forced_routes=routes, encoder=enc,
                                   round_operands=False)
        floor = {k: _err_cos(G[k], v) for k, v in G32.items()}
        del G32
    rep = {"loss": step_loss, "loss_ref": loss_ref, "grads": {},
           "flip_rate": {l: float(np.mean(v)) for l, v in flips.items()}}
    for l, f in rep["flip_rate"].items():
        assert f <= MAX_FLIP_RATE, ("routing flip rate", l, f)
    assert abs(step_loss - loss_ref) / abs(loss_ref) < TOL_LOSS, (step_loss, loss_ref)
    F, H = arch.ffn, arch.hidden
    names = {}
    for name, shape, _ in om.param_specs(arch):
        names[name] = shape
    got = {}
    for l in range(arch.layers):
        p = f"model.layers.{l}.mlp."
        if arch.is_moe(l):
            Fe, E = arch.expert_ffn, arch.experts
            gu = gather_full(sessions, "grad", p + "experts.gate_up_proj").reshape(E, Fe // 128, 2, 128, H)
            got[p + "experts.gate_proj"] = gu[:, :, 0].reshape(E, Fe, H)
            got[p + "experts.up_proj"] = gu[:, :, 1].reshape(E, Fe, H)
            continue
        gu = gather_full(sessions, "grad", p + "gate_up_proj.weight")
        g, u = om_deint(gu, F, H)
        got[p + "gate_proj.weight"] = g
        got[p + "up_proj.weight"] = u
    for name in names:
        if name not in got:
            got[name] = gather_full(sessions, "grad", name).reshape(names[name])
    rep["floor"] = floor
    for name, ref in G.items():
        x = got[name].reshape(ref.shape)
        err, cos = _err_cos(x, ref)
        rep["grads"][name] = (err, cos)
        tol_e, tol_c = TOL_GRAD, TOL_COS
        if name in floor:
            fe, fc = floor[name]
            tol_e = max(tol_e, BF16_FLOOR_FACTOR * fe)
            tol_c = min(tol_c, 1.0 - BF16_FLOOR_FACTOR * (1.0 - fc))
        assert err < tol_e and cos > tol_c, (name, err, cos, floor.get(name))
    if check_params:
        P1 = om.adamw(P0, G, {}, 1, lr=EXEC["lr"], betas=tuple(EXEC["betas"]), eps=EXEC["eps"],
                      wd=EXEC["weight_decay"])
        masters = _gpu_masters(sessions, arch, P1)
        for name, ref in P1.items():
            x = masters[name].reshape(ref.shape)
            d = np.abs(x - ref)
            # step 1 AdamW moves each element by ~lr*sign(g): a near-zero
            # gradient whose sign differs between bf16 and fp64 costs 2*lr
            assert d.max() <= 2.05 * EXEC["lr"], (name, d.max())
            assert d.mean() <= 0.02 * EXEC["lr"], (name, d.mean())
        rep["masters_checked"] = len(P1)
    return rep


def _gpu_masters(sessions, arch, names):
    """Every master weight in HF naming; the interleaved gate|up matrices
    (dense and expert) are split back into gate_proj / up_proj."""
    out = {}
    H = arch.hidden
    for name in names:
        if name in out:
            continue
        if name.endswith(("mlp.gate_proj.weight", "mlp.up_proj.weight")):
            p = name.rsplit("mlp.", 1)[0] + "mlp."
            g, u = om_deint(gather_full(sessions, "master", p + "gate_up_proj.weight"), arch.ffn, H)
            out[p + "gate_proj.weight"], out[p + "up_proj.weight"] = g, u
        elif name.endswith(("experts.gate_proj", "experts.up_proj")):
            p = name.rsplit("experts.", 1)[0] + "experts."
            E, Fe = arch.experts, arch.expert_ffn
            gu = gather_full(sessions, "master", p + "gate_up_proj").reshape(E, Fe // 128, 2, 128, H)
            out[p + "gate_proj"] = gu[:, :, 0].reshape(E, Fe, H)
            out[p + "up_proj"] = gu[:, :, 1].reshape(E, Fe, H)
        else:
            out[name] = gather_full(sessions, "master", name)
    return out


def om_deint(flat, F, H):
    v = flat.reshape(F // 128, 2, 128, H)
    return v[:, 0].reshape(F, H), v[:, 1].reshape(F, H)
