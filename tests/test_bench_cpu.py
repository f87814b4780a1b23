"""bench.py's trace accounting on synthetic traces (no GPU): the NVLink rates
of the exchange kernels use the kernels' own spans, not the flag-barrier
waits traced after them (Ulysses row)."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _ev(name, dur_us):
    return {"name": name, "ph": "X", "tid": 0, "ts": 0, "dur": dur_us, "args": {}}


def test_ulysses_rates_exclude_barrier_wait(bench):
    arch = {"hidden": 3584, "kv_heads": 4, "head_dim": 128}
    plan = {"sp": 4, "micro_batch": 1}
    S = 32768
    T = S // 4
    qkv = T * (3584 + 2 * 512) * 2 * 3 / 4          # bytes that leave the rank
    out = T * 3584 * 2 * 3 / 4
    ev = []
    for l in range(3):
        ev += [_ev(f"fwd.layer{l}.m0.a2a_qkv", qkv / 500e9 * 1e6),
               _ev(f"fwd.layer{l}.m0.a2a_wait", 5000.0),   # rank skew: must not count
               _ev(f"fwd.layer{l}.m0.a2a_out", out / 400e9 * 1e6),
               _ev(f"bwd.layer{l}.m0.a2a_dqkv", qkv / 450e9 * 1e6),
               _ev(f"bwd.layer{l}.m0.a2a_wait", 7000.0)]
    r = bench.nvlink_rates({"traceEvents": ev}, plan, arch, S)
    assert r["fwd_a2a_qkv_GBps"] == pytest.approx(500.0, abs=0.1)
    assert r["fwd_a2a_out_GBps"] == pytest.approx(400.0, abs=0.1)
    assert r["bwd_a2a_dqkv_GBps"] == pytest.approx(450.0, abs=0.1)
    assert not any("wait" in k for k in r)


def test_no_exchange_rates_without_sp(bench):
    arch = {"hidden": 256, "kv_heads": 2, "head_dim": 64}
    r = bench.nvlink_rates({"traceEvents": [_ev("fwd.layer0.m0.a2a_qkv", 10.0)]},
                           {"sp": 1, "micro_batch": 1}, arch, 1024)
    assert r == {"peak_GBps_per_direction": 900.0}


def test_moe_overlap_rates_count_both_halves_in_dispatch_nodes(bench):
    """With moe_overlap the dispatch-direction nodes span both expert halves'
    kernels (full payload), the combine-direction nodes half A's only."""
    arch = {"hidden": 2048, "kv_heads": 4, "head_dim": 128, "moe": {"top_k": 8}}
    plan = {"sp": 1, "ep": 4, "micro_batch": 1, "moe_overlap": True}
    S = 8192
    b = S * 8 * 2048 * 2 * 3 / 4
    ev = [_ev("fwd.layer0.m0.a2a_dispatch", b / 600e9 * 1e6),
          _ev("fwd.layer0.m0.a2a_combine", b / 2 / 600e9 * 1e6),
          _ev("bwd.layer0.m0.a2a_combine_grad", b / 400e9 * 1e6),
          _ev("bwd.layer0.m0.a2a_dispatch_grad", b / 2 / 650e9 * 1e6)]
    r = bench.nvlink_rates({"traceEvents": ev}, plan, arch, S)
    assert r["fwd_a2a_dispatch_GBps"] == pytest.approx(600.0, abs=0.1)
    assert r["fwd_a2a_combine_GBps"] == pytest.approx(600.0, abs=0.1)
    assert r["bwd_a2a_combine_grad_GBps"] == pytest.approx(400.0, abs=0.1)
    assert r["bwd_a2a_dispatch_grad_GBps"] == pytest.approx(650.0, abs=0.1)


def test_node_keys_merge_layers_and_micro_batches():
    import bench

    assert bench.node_key("fwd.layer3.m0.qkv_proj") == "fwd.qkv_proj"
    assert bench.node_key("bwd.layer12.m1.mlp.dgrad_gu") == "bwd.mlp.dgrad_gu"
    assert bench.node_key("bwd.head.m1") == "bwd.head"
    assert bench.node_key("encoder.vision.m0") == "encoder.vision"
    assert bench.node_key("optimizer") == "optimizer"


@pytest.mark.parametrize("cfg", ["c0", "c1", "c2", "c3", "c4"])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_bench_plans_validate_at_every_gpu_count(bench, cfg, n):
    """The plan bench.py runs for each config at 1/2/4/8 GPUs (the driver's
    scaling sweep) passes the reference's validation (plan.cpp:19-83, through
    libopx's differential-tested validator) and resolves to world n."""
    from paper_2508_02317_b200 import plan as P

    pl, m, S = bench.plan_for(cfg, n), bench.model_for(cfg, n), bench.seq_for(cfg)
    rows = pl["dp_replicate"] * pl["dp_shard"] * pl["micro_batch"]
    wl = {"seq_len": S, "micro_batch": pl["micro_batch"], "global_batch": rows}
    if cfg == "c3":
        wl["modality_mix"] = {"vision": bench.C3_IMAGE_MIX, "text": 1.0 - bench.C3_IMAGE_MIX}
    assert P.validate(bench.cluster_for(n), m, wl, pl) == []
    assert P.resolve(bench.cluster_for(n), m, wl, pl)["world"] == n
