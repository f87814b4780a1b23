"""Plan layer (the drop-in API half of the boundary) on CPU:
  * the reference's own golden values (proj/tests/test_specs.cpp, test_comm.cpp,
    test_mesh.cpp, test_plan.cpp) through the opx C ABI;
  * a differential test against the compiled reference planner
    (oracle/_ref/libomniplan_ref.so) on random instances shaped like the
    reference's random_instance (tests/test_util.hpp:195-296)."""
import ctypes
import json
import os
import random

import pytest

from paper_2508_02317_b200 import OpxError, lib
from paper_2508_02317_b200.plan import resolve, validate

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libomniplan_ref.so")


def cluster(nodes=1, gpn=8):
    return {"num_nodes": nodes, "gpus_per_node": gpn, "gpu": {"peak_flops": 1e12, "hbm_bytes": 8e10},
            "link": {"intra_node_bw": 1e11, "inter_node_bw": 2e10, "intra_latency": 5e-6,
                     "inter_latency": 2e-5}}


def model(arch, extra=()):
    return {"param_dtype_bytes": 2, "modules": [{"name": "core", "kind": "foundation", "trainable": True,
                                                 "arch": arch}] + list(extra)}


TOY = {"layers": 2, "hidden": 4, "heads": 2, "kv_heads": 2, "head_dim": 2, "ffn_dim": 8, "vocab": 10}
TOY_MOE = dict(TOY, moe={"num_experts": 4, "top_k": 2, "expert_ffn_dim": 8, "moe_layer_stride": 1})


def _params(r):
    return r["module_plans"][0]["params"], r["module_plans"][0]["active_params"]


def test_golden_param_counts():
    wl = {"seq_len": 8, "micro_batch": 1, "global_batch": 1}
    c1 = cluster(1, 1)
    z = dict(TOY, layers=0)
    assert _params(resolve(c1, model(z), wl, {}))[0] == 84          # test_specs.cpp:50-54
    assert _params(resolve(c1, model(TOY), wl, {}))[0] == 420       # :56-61
    tot, act = _params(resolve(c1, model(TOY_MOE), wl, {}))
    assert tot == 84 + 2 * (64 + 8 + 16 + 384) == 1028               # :63-69
    assert act == 84 + 2 * (64 + 8 + 16 + 192) == 644                # :84-89


def test_golden_flops_per_token():
    wl = {"seq_len": 8, "micro_batch": 1, "global_batch": 1}
    assert resolve(cluster(1, 1), model(TOY), wl, {})["flops_per_token"] == 2904.0  # :136-140


def test_golden_volumes():
    wl = {"seq_len": 8, "micro_batch": 1, "global_batch": 1}
    r = resolve(cluster(1, 2), model(TOY), wl, {"sp": 2, "dp_shard": 1})
    assert r["volumes"]["ulysses_per_layer"] == 64.0                 # test_comm.cpp:100-116
    moe = dict(TOY, moe={"num_experts": 4, "top_k": 2, "expert_ffn_dim": 8, "moe_layer_stride": 1})
    wl16 = {"seq_len": 16, "micro_batch": 1, "global_batch": 4}
    r = resolve(cluster(1, 4), model(moe), wl16, {"dp_shard": 4, "ep": 4})
    assert r["volumes"]["ep_dispatch_per_moe_layer"] == 384.0       # test_comm.cpp:173-188


def test_golden_groups_and_labels():
    wl = {"seq_len": 8, "micro_batch": 1, "global_batch": 4}
    r = resolve(cluster(1, 8), model(dict(TOY, heads=2, kv_heads=2)), wl, {"sp": 2, "dp_replicate": 2})
    assert r["groups"]["sp"] == [[0, 1], [2, 3], [4, 5], [6, 7]]     # test_mesh.cpp:70-88
    assert r["groups"]["replicate"] == [[0, 4], [1, 5], [2, 6], [3, 7]]
    assert r["groups"]["shard"] == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert r["label"] == "HSDP2+SP2"
    moe = dict(TOY, moe={"num_experts": 4, "top_k": 2, "expert_ffn_dim": 8})
    r = resolve(cluster(1, 8), model(moe), {"seq_len": 8, "micro_batch": 1, "global_batch": 8},
                {"ep": 4})
    assert r["groups"]["ep"] == [[0, 1, 2, 3], [4, 5, 6, 7]]        # test_plan.cpp:269-281
    assert r["label"] == "FSDP+SP1+EP4"
    assert r["expert_sharding"] == {"experts_per_rank": 1, "per_expert_fsdp_degree": 2}


def test_violation_codes():
    wl = {"seq_len": 10, "micro_batch": 1, "global_batch": 3}
    v = validate(cluster(1, 8), model(dict(TOY, heads=2, kv_heads=1)), wl,
                 {"sp": 4, "dp_shard": 1, "tp": 2, "micro_batch": 2})
    codes = [c for c, _ in v]
    assert codes == ["tp_pp_unsupported", "world_product", "head_divisibility",
                     "kv_head_divisibility", "seq_divisibility", "batch_divisibility"]
    assert [c for c, _ in validate(cluster(1, 8), model(TOY), wl, {"sp": 0})] == ["size_positive"]


def test_config_errors_are_code_2():
    with pytest.raises(OpxError) as e:
        validate(cluster(1, 8), {"modules": []}, {"seq_len": 8, "micro_batch": 1, "global_batch": 1}, {})
    assert e.value.code == 2 and "foundation" in e.value.msg
    bad = dict(TOY, heads=3)
    with pytest.raises(OpxError) as e:
        validate(cluster(1, 8), model(bad), {"seq_len": 8, "micro_batch": 1, "global_batch": 1}, {})
    assert e.value.code == 2 and "heads * head_dim" in e.value.msg


# ---------------------------------------------------------------- differential vs the reference
def _random_instance(rng: random.Random):
    """Python restatement of the reference's random_instance (test_util.hpp:195-296)."""
    pick = lambda xs: xs[rng.randrange(len(xs))]  # noqa: E731
    nodes, gpn = pick([1, 2]), pick([1, 2, 4])
    c = cluster(nodes, gpn)
    hd, heads = pick([2, 4]), pick([2, 4, 8])
    arch = {"layers": pick([1, 2, 3, 4]), "head_dim": hd, "heads": heads, "hidden": heads * hd,
            "kv_heads": heads // pick([1, 2]), "vocab": pick([64, 128, 512])}
    arch["ffn_dim"] = arch["hidden"] * pick([2, 3])
    if rng.random() < 0.5:
        e = pick([2, 4, 8])
        arch["moe"] = {"num_experts": e, "top_k": 1 + rng.randrange(e), "expert_ffn_dim": arch["hidden"] * 2,
                       "moe_layer_stride": pick([1, 2])}
    extra, mix, text = [], {}, 1.0
    for i in range(rng.randrange(3)):
        m = {"name": f"enc{i}", "kind": "encoder" if i % 2 == 0 else "decoder",
             "raw_param_count": 1000 + rng.randrange(9000), "trainable": rng.random() < 0.25,
             "tokens_per_item": pick([0, 4, 16])}
        f = 0.1 + 0.2 * rng.randrange(2)
        if text - f > 0.05:
            mix[m["name"]] = f
            text -= f
        extra.append(m)
    if mix:
        mix["text"] = text
    world = nodes * gpn
    # half the instances are valid factorisations, half perturbed to hit codes
    sp = pick([s for s in range(1, world + 1) if world % s == 0])
    rest = world // sp
    rep = pick([r for r in range(1, rest + 1) if rest % r == 0])
    shard = rest // rep
    ep = 1
    if "moe" in arch:
        ep = pick([x for x in range(1, shard * sp + 1) if (shard * sp) % x == 0])
    mb = pick([1, 2])
    seq = sp * pick([4, 8, 16])
    gb = rep * shard * mb * pick([1, 2])
    if rng.random() < 0.3:
        seq += pick([0, 1])
        gb += pick([0, 1])
        ep = pick([ep, 3])
    plan = {"dp_replicate": rep, "dp_shard": shard, "sp": sp, "ep": ep, "micro_batch": mb,
            "fsdp_prefetch_depth": pick([0, 1, 2])}
    wl = {"seq_len": seq, "micro_batch": mb, "global_batch": gb}
    if mix:
        wl["modality_mix"] = mix
    return c, model(arch, extra), wl, plan


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (reference absent)")
def test_differential_against_compiled_reference():
    ref = ctypes.CDLL(REF_SO)
    ref.ref_resolve.argtypes = [ctypes.c_char_p] * 4 + [ctypes.c_char_p, ctypes.c_size_t]
    rng = random.Random(20260)
    checked_valid = 0
    for _ in range(400):
        c, m, w, p = _random_instance(rng)
        buf = ctypes.create_string_buffer(1 << 20)
        rc = ref.ref_resolve(*(json.dumps(x).encode() for x in (c, m, w, p)), buf, len(buf))
        assert rc == 0, buf.value
        r = json.loads(buf.value.decode())
        mine = [code for code, _ in validate(c, m, w, p)]
        assert mine == r["violations"], (c, m, w, p)
        if mine:
            continue
        checked_valid += 1
        o = resolve(c, m, w, p)
        assert o["flops_per_token"] == pytest.approx(r["flops_per_token"], rel=1e-12)
        for key in ("label", "groups", "head_params", "layers"):
            assert o[key] == r[key], key
        if "expert_sharding" in r:
            assert o["expert_sharding"] == r["expert_sharding"]
        for k, v in r["volumes"].items():
            assert o["volumes"][k] == pytest.approx(v, rel=1e-12), k
        for a, b in zip(o["module_plans"], r["module_plans"]):
            for k in ("module_name", "fsdp", "participates_in_sp", "expert_placement"):
                assert a[k] == b[k]
    assert checked_valid > 100


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (reference absent)")
def test_reference_step_graph_names_match_executor_phases():
    """The executor's trace names follow step_graph.cpp; check the reference's
    node naming for one dense SP layer matches the names opx emits."""
    ref = ctypes.CDLL(REF_SO)
    ref.ref_simulate.argtypes = [ctypes.c_char_p] * 4 + [ctypes.c_char_p, ctypes.c_size_t]
    buf = ctypes.create_string_buffer(1 << 22)
    c = cluster(1, 2)
    m = model(dict(TOY, layers=1))
    w = {"seq_len": 8, "micro_batch": 1, "global_batch": 1}
    p = {"sp": 2, "dp_shard": 1}
    assert ref.ref_simulate(*(json.dumps(x).encode() for x in (c, m, w, p)), buf, len(buf)) == 0
    r = json.loads(buf.value.decode())
    names = set(r["node_names"])
    for n in ("fwd.layer0.m0.qkv_proj", "fwd.layer0.m0.attn_core", "fwd.layer0.m0.out_proj",
              "fwd.layer0.m0.mlp", "optimizer"):
        assert n in names
    assert r["all_to_all"] == 4  # q, k, v, out (the reference models no backward a2a)
