"""Planner calibration: the restated per-node costs equal the
reference step graph's (compiled from /root/reference into oracle/_ref), and a
calibration from a trace fed back into the reference's simulate reproduces the
traced compute time.  CPU only."""
import ctypes
import json
import os

import pytest

from paper_2508_02317_b200 import calibrate as cal

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libomniplan_ref.so")

CLUSTER = {"num_nodes": 1, "gpus_per_node": 4, "gpu": {"peak_flops": 2.25e15, "hbm_bytes": 180e9},
           "link": {"intra_node_bw": 9e11, "inter_node_bw": 5e10, "intra_latency": 5e-6,
                    "inter_latency": 2e-5}}
DENSE = {"modules": [{"name": "core", "kind": "foundation", "trainable": True,
                      "arch": {"layers": 3, "hidden": 1024, "heads": 8, "kv_heads": 2, "head_dim": 128,
                               "ffn_dim": 2816, "vocab": 4096}}], "param_dtype_bytes": 2}
MOE = {"modules": [{"name": "core", "kind": "foundation", "trainable": True,
                    "arch": {"layers": 2, "hidden": 1024, "heads": 8, "kv_heads": 2, "head_dim": 128,
                             "ffn_dim": 2816, "vocab": 4096,
                             "moe": {"num_experts": 16, "top_k": 2, "expert_ffn_dim": 512,
                                     "moe_layer_stride": 1}}}], "param_dtype_bytes": 2}


def _ref_graph(model, plan, S):
    ref = ctypes.CDLL(REF_SO)
    ref.ref_simulate.argtypes = [ctypes.c_char_p] * 4 + [ctypes.c_char_p, ctypes.c_size_t]
    buf = ctypes.create_string_buffer(1 << 22)
    wl = {"seq_len": S, "micro_batch": plan["micro_batch"],
          "global_batch": plan["micro_batch"] * plan["dp_shard"] * plan.get("dp_replicate", 1)}
    rc = ref.ref_simulate(json.dumps(CLUSTER).encode(), json.dumps(model).encode(), json.dumps(wl).encode(),
                          json.dumps(plan).encode(), buf, len(buf))
    assert rc == 0, buf.value
    return json.loads(buf.value.decode()), wl


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (reference absent)")
@pytest.mark.parametrize("model,plan", [
    (DENSE, {"dp_replicate": 1, "dp_shard": 1, "sp": 4, "ep": 1, "micro_batch": 1}),
    (DENSE, {"dp_replicate": 1, "dp_shard": 4, "sp": 1, "ep": 1, "micro_batch": 2}),
    (MOE, {"dp_replicate": 1, "dp_shard": 4, "sp": 1, "ep": 4, "micro_batch": 1}),
    (MOE, {"dp_replicate": 1, "dp_shard": 2, "sp": 2, "ep": 2, "micro_batch": 1}),
])
def test_node_costs_match_reference_graph(model, plan):
    r, wl = _ref_graph(model, plan, 4096)
    mine = cal.node_costs(plan, model, wl)
    checked = 0
    for n in r["nodes"]:
        name = n["name"]
        if name in mine:
            kind, amount = mine[name]
            assert kind == n["kind"], name
            ref_amount = n["flops"] if kind == "compute" else n["bytes"]
            assert amount == pytest.approx(ref_amount, rel=1e-12), name
            checked += 1
        else:  # only head/optimizer/FSDP nodes are not restated
            assert any(k in name for k in ("head", "optimizer", ".ag.", ".rs.", ".ar.")), name
    assert checked >= 6 * model["modules"][0]["arch"]["layers"] - 4


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (reference absent)")
def test_calibration_round_trip_through_reference_simulate():
    """A synthetic trace at 55 % efficiency and 600 GB/s a2a calibrates back to
    those constants, and the reference simulate with them reproduces the
    traced compute + exchange time of the layers."""
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 4, "ep": 1, "micro_batch": 1}
    wl = {"seq_len": 4096, "micro_batch": 1, "global_batch": 1}
    costs = cal.node_costs(plan, DENSE, wl)
    eff, bw = 0.55, 6e11
    ev = []
    for name, (kind, amount) in costs.items():
        if name.endswith((".a2a_k", ".a2a_v")):
            continue
        if kind == "compute":
            dur = amount / (CLUSTER["gpu"]["peak_flops"] * eff)
        else:
            vol = amount * 3 / 4
            if name.endswith(".a2a_q"):
                vol += 2 * costs[name[:-1] + "k"][1] * 3 / 4
            dur = vol / bw
        short = name.replace(".a2a_q", ".a2a_qkv")
        ev.append({"name": short, "ph": "X", "tid": 0, "ts": 0, "dur": dur * 1e6, "args": {}})
    c = cal.calibrate({"traceEvents": ev}, plan, DENSE, wl, CLUSTER)
    assert c["compute_efficiency"] == pytest.approx(eff, rel=1e-6)
    assert c["intra_node_bw"] == pytest.approx(bw, rel=1e-6)
    r, _ = _ref_graph(DENSE, dict(plan, compute_efficiency=c["compute_efficiency"]), 4096)
    assert r["step_time_s"] > c["modelled_compute_s"]  # plus head/optimizer and the a2a latencies
