"""Full fwd+bwd+AdamW step on one B200 through the C ABI, against the CPU oracle."""
import numpy as np
import pytest
import torch

from tests.step_common import EXEC, cluster, compare_step, tiny_dense

gpu = pytest.mark.gpu


def _run(model, S, rows, single=False, trace=False, recompute="full", selective=True):
    from paper_2508_02317_b200.runtime import Session, synthetic_batch

    arch = model["modules"][0]["arch"]
    wl = {"seq_len": S, "micro_batch": rows, "global_batch": rows}
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": rows, "recompute": recompute}
    ex = dict(EXEC)
    ex["trace"] = trace
    ex["selective_recompute"] = selective
    s = Session(cluster(1), model, wl, plan, ex, rank=0, device=0)
    s.init_weights(EXEC["seed"])
    batch = synthetic_batch(arch["vocab"], S, rows, seed=2508, single_sample=single)
    s.load(batch)
    r = s.run()
    return s, batch, plan, r


@gpu
@pytest.mark.parametrize("single", [False, True])
def test_step_tiny_dense_matches_oracle(single):
    model = tiny_dense()
    s, batch, plan, r = _run(model, 1024, 2, single)
    assert r.kept_layers == model["modules"][0]["arch"]["layers"]  # attention-kept (selective)
    rep = compare_step([s], model, batch, plan, r.loss)
    assert r.launches > 0
    s.close()


@gpu
def test_step_pure_full_recompute_matches_oracle():
    """recompute=full with selective keeping off: every layer recomputed."""
    model = tiny_dense()
    s, batch, plan, r = _run(model, 1024, 2, selective=False)
    assert r.kept_layers == 0
    compare_step([s], model, batch, plan, r.loss)
    s.close()


@gpu
def test_step_recompute_none_matches_oracle():
    model = tiny_dense()
    s, batch, plan, r = _run(model, 1024, 2, recompute="none")
    compare_step([s], model, batch, plan, r.loss)
    r2 = s.run()  # second step reuses the per-layer activation buffers
    assert np.isfinite(r2.loss) and r2.loss < r.loss
    s.close()


@gpu
def test_step_gqa_matches_oracle():
    model = tiny_dense(layers=2, hidden=512, heads=4, kv=1, ffn=1024, vocab=4096)
    s, batch, plan, r = _run(model, 768, 1)
    compare_step([s], model, batch, plan, r.loss)
    s.close()


@gpu
def test_step_trace_schema():
    model = tiny_dense(layers=1)
    s, batch, plan, r = _run(model, 512, 1, trace=True)
    tr = s.trace()
    names = {e["name"] for e in tr["traceEvents"]}
    assert "fwd.layer0.m0.qkv_proj" in names and "optimizer" in names
    for e in tr["traceEvents"]:
        assert e["ph"] == "X" and e["dur"] >= 0 and "phase" in e["args"]
    s.close()


@gpu
def test_step_deterministic_loss_and_second_step():
    model = tiny_dense(layers=1)
    s, batch, plan, r1 = _run(model, 512, 1)
    r2 = s.run()  # second step on updated weights: loss must drop on the same batch
    assert np.isfinite(r2.loss) and r2.loss < r1.loss
    s2, _, _, r1b = _run(model, 512, 1)
    assert r1b.loss == r1.loss
    s.close()
    s2.close()


@gpu
def test_step_ffd_packed_batch_with_padding():
    """f1: a batch produced by the first-fit-decreasing packer (short rows get
    a trailing padding segment with ignored labels) through the full step."""
    from paper_2508_02317_b200 import packing as pk
    from paper_2508_02317_b200.runtime import Session

    model = tiny_dense()
    arch = model["modules"][0]["arch"]
    rng = np.random.default_rng(5)
    samples = [rng.integers(0, arch["vocab"], n) for n in (700, 250, 600, 180, 90, 77)]
    batch, rep = pk.packed_batch(samples, 1024, rows=2)
    assert rep["padding_ratio"] > 0
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": 2, "recompute": "full"}
    wl = {"seq_len": 1024, "micro_batch": 2, "global_batch": 2}
    s = Session(cluster(1), model, wl, plan, EXEC, rank=0, device=0)
    s.init_weights(EXEC["seed"])
    s.load(batch)
    r = s.run()
    compare_step([s], model, batch, plan, r.loss)
    s.close()


@gpu
@pytest.mark.parametrize("hidden,heads,kv", [(256, 4, 2), (640, 8, 2)])
def test_step_head_dim_below_128(hidden, heads, kv):
    """head_dim 64 (the SURVEY C0 shape: H=256, 4 heads, 2 kv heads) and 80
    (the omni-modal ViT's): attention runs on zero-padded 128-wide head vectors
    with the 1/sqrt(d) scale; RoPE rotates over d."""
    model = tiny_dense(layers=2, hidden=hidden, heads=heads, kv=kv, ffn=768, vocab=2048)
    s, batch, plan, r = _run(model, 1024, 2)
    compare_step([s], model, batch, plan, r.loss)
    s.close()


@gpu
def test_step_async_ulysses_fused_epilogue_matches_kernel_path():
    """async_ulysses (step_graph.cpp:217-241): the seq->head exchange rides in
    the QKV GEMM epilogue (GEMM_EPI_SEQ2HEAD) instead of a separate kernel.
    Same bf16 rounding point and RoPE arithmetic, so the step must agree with
    the kernel path (and with the oracle)."""
    from paper_2508_02317_b200.runtime import Session, synthetic_batch
    from tests.step_common import gather_full, gpu_param_names
    from oracle import model as om

    model = tiny_dense(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048)
    arch = model["modules"][0]["arch"]
    wl = {"seq_len": 1024, "micro_batch": 2, "global_batch": 2}
    batch = synthetic_batch(arch["vocab"], 1024, 2, seed=2508)
    out = {}
    for asy in (False, True):
        plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": 2,
                "async_ulysses": asy}
        s = Session(cluster(1), model, wl, plan, EXEC, rank=0, device=0)
        s.init_weights(EXEC["seed"])
        s.load(batch)
        r = s.run()
        names = gpu_param_names(om.Arch.from_model_json(model))
        out[asy] = (r.loss, {n: gather_full([s], "grad", n) for n in names})
        if asy:
            tr = s.trace()["traceEvents"]
            assert not any(e["name"].endswith(".a2a_qkv") for e in tr)
            assert any(e["args"].get("fused", "").startswith("qkv_proj,a2a_q") for e in tr)
            compare_step([s], model, batch, plan, r.loss)
        s.close()
    assert abs(out[True][0] - out[False][0]) <= 1e-6 * abs(out[False][0])
    for n, g in out[False][1].items():
        d = np.abs(out[True][1][n] - g).max() / max(np.abs(g).max(), 1e-30)
        assert d < 1e-3, (n, d)


def _batch_from_lengths(vocab, rows_lengths, seed=11):
    """Global batch from explicit per-row sample lengths (each row sums to S)."""
    rng = np.random.default_rng(seed)
    S = sum(rows_lengths[0])
    R = len(rows_lengths)
    ids = rng.integers(0, vocab, size=(R, S)).astype(np.int32)
    labels = np.full((R, S), -100, np.int32)
    pos = np.zeros((R, S), np.int32)
    cu_rows = []
    for r, lens in enumerate(rows_lengths):
        assert sum(lens) == S
        cu = [0]
        for l in lens:
            a = cu[-1]
            pos[r, a:a + l] = np.arange(l)
            labels[r, a:a + l - 1] = ids[r, a + 1:a + l]
            cu.append(a + l)
        cu_rows.append(cu)
    return {"ids": ids, "labels": labels, "pos": pos, "cu_rows": cu_rows}


@gpu
def test_step_extreme_varlen_packing():
    """cu_seqlens edge cases (packing.hpp:20-31): 1-token samples (no
    supervised token), samples straddling the 64-query / 128-key tile edges,
    a row that is one full-length sample, and a row of many tiny samples."""
    from paper_2508_02317_b200.runtime import Session

    model = tiny_dense(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048)
    lens = [[1, 1, 2, 63, 64, 65, 127, 128, 129, 1, 443],
            [1024],
            [3] * 300 + [124]]
    batch = _batch_from_lengths(2048, lens)
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": 3, "recompute": "none"}
    wl = {"seq_len": 1024, "micro_batch": 3, "global_batch": 3}
    s = Session(cluster(1), model, wl, plan, EXEC, rank=0, device=0)
    s.init_weights(EXEC["seed"])
    s.load(batch)
    r = s.run()
    compare_step([s], model, batch, plan, r.loss)
    s.close()


@gpu
def test_step_rejects_bad_cu_seqlens():
    """The ABI refuses malformed cu_seqlens with the argument error code."""
    from paper_2508_02317_b200 import OpxError
    from paper_2508_02317_b200.runtime import Session

    model = tiny_dense(layers=1)
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": 1}
    wl = {"seq_len": 512, "micro_batch": 1, "global_batch": 1}
    s = Session(cluster(1), model, wl, plan, EXEC, rank=0, device=0)
    good = _batch_from_lengths(2048, [[200, 312]])
    for cu in ([0, 300, 300, 512], [0, 200, 511]):
        bad = dict(good)
        bad["cu_rows"] = [cu]
        with pytest.raises(OpxError) as ei:
            s.load(bad)
        assert ei.value.code == 9
    # straight through the C ABI: cu_seqlens must start at 0
    import ctypes

    from paper_2508_02317_b200 import lib

    ids = np.zeros(512, np.int32)
    cu = np.array([1, 200, 512], np.int32)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    assert lib().opx_step_load_batch(s.h, vp(ids), vp(ids), vp(ids), vp(cu), 3, 10) == 9
    s.close()


@gpu
@pytest.mark.parametrize("sp_world", [1])
def test_step_zero_layer_foundation_trains_its_head(sp_world):
    """test_simulator.cpp:265-283: a zero-layer foundation still trains its
    head (embedding -> final norm -> LM head -> CE, AdamW)."""
    model = tiny_dense(layers=0, hidden=256, heads=2, kv=2, ffn=768, vocab=2048)
    s, batch, plan, r = _run(model, 512, 2, trace=True)
    assert r.step_time_s > 0 and r.launches > 0
    compare_step([s], model, batch, plan, r.loss)
    ph = s.report_json()["phase_breakdown"]
    assert "optimizer" in ph and not any(k.startswith("fwd.layer") for k in ph)
    s.close()
