"""The measured StepReport (simulator.hpp:43-50 / report.cpp:117-128) and
gradient accumulation (step_graph.cpp:57,75-87,351-364) on one B200, through
the C ABI, against the reference's formulas and the CPU oracle."""
import numpy as np
import pytest

from tests.step_common import CLUSTER1, EXEC, cluster, compare_step, tiny_dense, tiny_moe

gpu = pytest.mark.gpu

REPORT_KEYS = {"step_time_s", "throughput_tokens_per_s_per_gpu", "mfu", "exposed_comm_fraction",
               "model_flops_per_token", "phase_breakdown"}


def _session(model, S, micro, gb, recompute="full"):
    from paper_2508_02317_b200.runtime import Session, synthetic_batch

    arch = model["modules"][0]["arch"]
    wl = {"seq_len": S, "micro_batch": micro, "global_batch": gb}
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": micro,
            "recompute": recompute}
    s = Session(cluster(1), model, wl, plan, EXEC, rank=0, device=0)
    s.init_weights(EXEC["seed"])
    batch = synthetic_batch(arch["vocab"], S, gb, seed=2508)
    s.load(batch)
    return s, batch, plan, wl


@gpu
def test_step_report_matches_reference_formulas():
    from paper_2508_02317_b200 import plan as pl

    model = tiny_dense(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048)
    s, batch, plan, wl = _session(model, 1024, 2, 2)
    r = s.run()
    # simulator.cpp:113-117
    assert r.throughput == pytest.approx(2 * 1024 / r.step_time_s, rel=1e-9)
    fpt = pl.resolve(cluster(1), model, wl, plan)["flops_per_token"]
    assert r.model_flops_per_token == pytest.approx(fpt, rel=1e-12)
    assert r.mfu == pytest.approx(r.throughput * fpt / CLUSTER1["gpu"]["peak_flops"], rel=1e-9)
    assert r.accum_steps == 1
    # one GPU: no collectives, nothing exposed
    assert r.comm_s == 0 and r.exposed_comm == 0 and r.comm_wait_s == 0
    j = s.report_json()
    assert set(j) == REPORT_KEYS
    assert j["step_time_s"] == pytest.approx(r.step_time_s)
    ph = j["phase_breakdown"]
    for p in ("fwd.layer0", "fwd.layer1", "bwd.layer0", "bwd.layer1", "fwd.head", "bwd.head",
              "optimizer"):
        assert p in ph and ph[p]["compute_s"] > 0, (p, ph)
    # the busy intervals of the compute stream fit inside the step
    cs = sum(v["compute_s"] for k, v in ph.items() if k != "optimizer")
    assert cs <= r.step_time_s * 1.001
    s.close()


@gpu
@pytest.mark.parametrize("recompute", ["full", "none"])
def test_grad_accumulation_two_micro_batches_matches_oracle(recompute):
    """global_batch = 2 x micro_batch on one GPU: two forward/backward passes
    summed into one fp32 gradient, AdamW once; the oracle runs both
    micro-batches' rows."""
    model = tiny_dense(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048)
    s, batch, plan, wl = _session(model, 1024, 1, 2, recompute)
    r = s.run()
    assert r.accum_steps == 2 and s.accum == 2
    assert r.tokens == 2 * 1024
    compare_step([s], model, batch, plan, r.loss)
    # a second step keeps training
    r2 = s.run()
    assert np.isfinite(r2.loss) and r2.loss < r.loss
    ph = s.report_json()["phase_breakdown"]
    assert "fwd.layer0" in ph
    names = {e["name"] for e in s.trace()["traceEvents"]}
    assert "fwd.layer0.m0.qkv_proj" in names and "fwd.layer0.m1.qkv_proj" in names
    s.close()


@gpu
def test_grad_accumulation_moe_matches_oracle():
    model = tiny_moe(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048, experts=64, top_k=4,
                     expert_ffn=256)
    s, batch, plan, wl = _session(model, 512, 1, 3)
    r = s.run()
    assert r.accum_steps == 3
    compare_step([s], model, batch, plan, r.loss)
    s.close()
