"""Planner calibration from measured step traces.

The reference's simulator prices every compute node at one
``compute_efficiency`` times the GPU peak (simulator.cpp:25,41-44) and every
collective with an alpha-beta link model (comm.cpp:37-46).  opx measures the
same step with the same node names (``opx_step_trace``), so the two can be
joined: this module restates the reference's per-node costs
(step_graph.cpp:206-375: qkv/attn/out/mlp/router/experts FLOPs, the Ulysses
and EP all-to-all payloads, the backward ``rest`` node at twice the forward
cost), sums the measured device time of the nodes that realise each of them,
and returns the efficiency and link bandwidth that make the reference's model
reproduce the measurement.  ``calibrated_cluster`` writes them back into a
cluster JSON the reference CLI accepts, so ``omniplan plan`` ranks B200
recipes with measured rather than guessed constants; the backward Ulysses
exchanges and the recompute the reference's graph does not model are
reported as the residual it leaves unexplained.
"""
from __future__ import annotations

import re

_LAYER = re.compile(r"^(fwd|bwd)\.layer(\d+)\.m0\.(.+)$")


def _arch(model: dict) -> dict:
    for m in model["modules"]:
        if m.get("kind", "foundation") == "foundation":
            return m["arch"]
    raise ValueError("model has no foundation module")


def layer_shape(arch: dict, layer: int) -> dict:
    """specs.cpp:36-50 layer_shape: q/k/v + pre-attention norm, out, and the
    dense MLP + pre-MLP norm (just the norm on MoE layers, which add the router
    and the top-k experts' share)."""
    H = arch["hidden"]
    kv = arch["kv_heads"] * arch["head_dim"]
    moe = arch.get("moe")
    stride = moe.get("moe_layer_stride", 1) if moe else 1
    is_moe = bool(moe) and (layer + 1) % stride == 0
    s = {"qkv": H * H + 2 * H * kv + H, "out": H * H, "is_moe": is_moe}
    if is_moe:
        s["router"] = H * moe["num_experts"]
        s["mlp"] = H
        s["expert_active"] = 3 * H * moe["expert_ffn_dim"] * moe["top_k"]
    else:
        s["router"] = 0
        s["mlp"] = 3 * H * arch["ffn_dim"] + H
        s["expert_active"] = 0
    return s


def node_costs(plan: dict, model: dict, workload: dict, dtype_bytes: int = 2) -> dict:
    """Reference node name -> (kind, flops or bytes) for one micro-batch, the
    layer and MoE nodes of step_graph.cpp:206-375."""
    arch = _arch(model)
    T = plan.get("micro_batch", 1) * workload["seq_len"] / plan.get("sp", 1)
    H, S = arch["hidden"], workload["seq_len"]
    kvw = arch["kv_heads"] * arch["head_dim"]
    out = {}
    for l in range(arch["layers"]):
        sh = layer_shape(arch, l)
        f = f"fwd.layer{l}.m0"
        out[f + ".qkv_proj"] = ("compute", 2.0 * sh["qkv"] * T)
        out[f + ".attn_core"] = ("compute", 2.0 * H * S * T)
        out[f + ".out_proj"] = ("compute", 2.0 * sh["out"] * T)
        if plan.get("sp", 1) > 1:
            out[f + ".a2a_q"] = ("collective", T * H * dtype_bytes)
            out[f + ".a2a_k"] = ("collective", T * kvw * dtype_bytes)
            out[f + ".a2a_v"] = ("collective", T * kvw * dtype_bytes)
            out[f + ".a2a_out"] = ("collective", T * H * dtype_bytes)
        rest = 2.0 * (sh["qkv"] + sh["out"] + (0 if sh["is_moe"] else sh["mlp"])) * T
        b = f"bwd.layer{l}.m0"
        out[b + ".rest"] = ("compute", 2.0 * (rest + 2.0 * H * S * T))
        if not sh["is_moe"]:
            out[f + ".mlp"] = ("compute", 2.0 * sh["mlp"] * T)
            continue
        moe = arch["moe"]
        a2a = T * moe["top_k"] * H * dtype_bytes * plan.get("moe_imbalance", 1.0)
        for d, (pre, bf) in enumerate(((f, 1.0), (b, 2.0))):
            out[pre + ".router"] = ("compute", bf * 2.0 * (sh["router"] + sh["mlp"]) * T)
            out[pre + ".experts"] = ("compute", bf * 2.0 * sh["expert_active"] * T)
            if plan.get("ep", 1) > 1:
                out[pre + (".a2a_combine_grad" if d else ".a2a_dispatch")] = ("collective", a2a)
                out[pre + (".a2a_dispatch_grad" if d else ".a2a_combine")] = ("collective", a2a)
    return out


# measured trace node (suffix after ".m0.") -> reference node (suffix) it realises
_MEASURED_TO_REF = {
    "fwd": {"qkv_proj": "qkv_proj", "attn_core": "attn_core", "out_proj": "out_proj", "mlp": "mlp",
            "router": "router", "experts": "experts", "experts_b": "experts", "unpermute": "experts",
            "a2a_qkv": "a2a_q", "a2a_out": "a2a_out", "a2a_counts": "a2a_dispatch",
            "a2a_dispatch": "a2a_dispatch", "a2a_combine": "a2a_combine"},
    "bwd": {"router": "router", "experts": "experts", "experts_b": "experts", "gate_up_recompute": "experts",
            "a2a_combine_grad": "a2a_combine_grad", "a2a_dispatch_grad": "a2a_dispatch_grad",
            "a2a_redispatch_wait": "a2a_combine_grad", "combine_bwd": "experts"},
}


def calibrate(trace: dict, plan: dict, model: dict, workload: dict, cluster: dict,
              step_time_s: float | None = None) -> dict:
    """Efficiency and link bandwidth that make the reference's cost model
    reproduce a measured trace (tid 0 = compute stream, as opx records it)."""
    costs = node_costs(plan, model, workload)
    peak = cluster["gpu"]["peak_flops"]
    sp, ep = plan.get("sp", 1), plan.get("ep", 1)
    comp_flops = comp_s = 0.0
    coll_vol = coll_s = 0.0
    per_kind: dict[str, list[float]] = {}
    unexplained = 0.0
    seen = set()
    for e in trace["traceEvents"]:
        if e.get("tid", 0) != 0:
            continue
        dur = e["dur"] * 1e-6
        m = _LAYER.match(e["name"])
        if not m:
            if e["name"] in ("optimizer",) or e["name"].startswith("fwd_bwd.head"):
                unexplained += dur
            continue
        d, l, sub = m.group(1), int(m.group(2)), m.group(3)
        if sub == "moe":  # parent span of the MoE sub-nodes
            continue
        if d == "bwd" and sub not in _MEASURED_TO_REF["bwd"] and not sub.startswith("a2a"):
            ref = f"bwd.layer{l}.m0.rest"        # everything else of the layer backward
        elif sub in _MEASURED_TO_REF[d]:
            ref = f"{d}.layer{l}.m0.{_MEASURED_TO_REF[d][sub]}"
        else:
            unexplained += dur                   # e.g. a2a_wait, bwd a2a_dqkv (not modelled)
            continue
        if ref not in costs:
            unexplained += dur
            continue
        kind, amount = costs[ref]
        key = ref.split(".m0.")[-1]
        if kind == "compute":
            if ref not in seen:
                comp_flops += amount
                per_kind.setdefault(key, [0.0, 0.0])[0] += amount
                seen.add(ref)
            comp_s += dur
            per_kind.setdefault(key, [0.0, 0.0])[1] += dur
        else:
            if ref not in seen:
                group = sp if key.startswith("a2a_q") or key == "a2a_out" else ep
                coll_vol += amount * (group - 1) / group       # all_to_all volume (comm.cpp:8-22)
                if key == "a2a_q":  # the fused q/k/v exchange realises three reference nodes
                    base = ref[: -len("a2a_q")]
                    for kk in ("a2a_k", "a2a_v"):
                        if base + kk in costs:
                            coll_vol += costs[base + kk][1] * (group - 1) / group
                seen.add(ref)
            coll_s += dur
    eff = comp_flops / (comp_s * peak) if comp_s > 0 else None
    bw = coll_vol / coll_s if coll_s > 0 else None
    return {
        "compute_efficiency": eff,
        "intra_node_bw": bw,
        "per_kind_efficiency": {k: v[0] / (v[1] * peak) for k, v in per_kind.items() if v[1] > 0},
        "modelled_compute_s": comp_s,
        "modelled_collective_s": coll_s,
        "unmodelled_s": unexplained,
        "step_time_s": step_time_s,
    }


def calibrated_cluster(cluster: dict, cal: dict) -> dict:
    """The cluster JSON with the measured intra-node bandwidth; the efficiency
    is a simulate() option (SimOptions::compute_efficiency), returned alongside."""
    c = {**cluster, "link": dict(cluster.get("link", {}))}
    if cal.get("intra_node_bw"):
        c["link"]["intra_node_bw"] = cal["intra_node_bw"]
    return c
