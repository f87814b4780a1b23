"""Multi-GPU step parity: FSDP / Ulysses-SP / HSDP plans on 2 or 4 B200s (one
process per GPU, NCCL + CUDA-IPC peer memory inside libopx) against the CPU
oracle's simulated ranks.  Skipped when fewer GPUs are visible."""
import multiprocessing as mp
import random

import numpy as np
import pytest
import torch

from tests.step_common import compare_step, free_port, tiny_dense

gpu = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


class _Remote:
    """Adapter so compare_step can read per-rank slices returned by workers."""

    def __init__(self, out):
        self.out = out
        self.accum = int(out[("report_struct", 0)]["accum_steps"])

    def get(self, name):
        kind, n = name.split(":", 1)
        return self.out[(kind, n)]

    def routes(self, layer, T, k):
        return self.out[("route", layer)]


def _collect(q, ps, world, timeout=600):
    """Gather every worker's result; fail fast if a worker dies without one
    (a dead rank would otherwise leave its peers waiting in a collective)."""
    import queue
    import time

    res, t0 = {}, time.time()
    while len(res) < world:
        try:
            rank, loss, out, err = q.get(timeout=5)
        except queue.Empty:
            dead = [p.exitcode for p in ps if p.exitcode not in (None, 0)]
            if dead:
                for p in ps:
                    if p.is_alive():
                        p.kill()
                raise AssertionError(f"worker exited with {dead} before reporting")
            assert time.time() - t0 < timeout, "workers timed out"
            continue
        assert err is None, err
        res[rank] = (loss, out)
    for p in ps:
        p.join(60)
    return res


def _run(world, model, plan, S, rows):
    from oracle import model as om

    arch = om.Arch.from_model_json(model)
    from tests.step_common import gpu_param_names

    names = gpu_param_names(arch)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    from tests.dist_worker import step_worker

    ps = [ctx.Process(target=step_worker, args=(r, world, port, model, plan, S, rows, q, names))
          for r in range(world)]
    for p in ps:
        p.start()
    res = _collect(q, ps, world)
    losses = {round(v[0], 6) for v in res.values()}
    assert len(losses) == 1, losses  # every rank reports the same global loss
    return res[0][0], [_Remote(res[r][1]) for r in range(world)]


PLANS = [
    (2, {"dp_replicate": 1, "dp_shard": 1, "sp": 2, "ep": 1, "micro_batch": 1}, 1),
    (2, {"dp_replicate": 1, "dp_shard": 1, "sp": 2, "ep": 1, "micro_batch": 1, "recompute": "none"}, 1),
    (2, {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 1, "micro_batch": 1}, 2),
    (4, {"dp_replicate": 1, "dp_shard": 2, "sp": 2, "ep": 1, "micro_batch": 1}, 2),
    (4, {"dp_replicate": 2, "dp_shard": 1, "sp": 2, "ep": 1, "micro_batch": 1}, 2),
    (4, {"dp_replicate": 1, "dp_shard": 1, "sp": 4, "ep": 1, "micro_batch": 1}, 1),
    # gradient accumulation (step_graph.cpp:57,75-87,351-364): 2 micro-batches
    # per dp rank, per-micro reduce-scatter, HSDP all-reduce on the last one
    (2, {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 1, "micro_batch": 1}, 4),
    (4, {"dp_replicate": 2, "dp_shard": 1, "sp": 2, "ep": 1, "micro_batch": 1}, 4),
    # async_ulysses: the seq->head exchanges (q/k/v forward, dO backward) are
    # peer stores from the producing GEMM's epilogue
    (2, {"dp_replicate": 1, "dp_shard": 1, "sp": 2, "ep": 1, "micro_batch": 1, "async_ulysses": True}, 1),
    (4, {"dp_replicate": 1, "dp_shard": 2, "sp": 2, "ep": 1, "micro_batch": 1, "async_ulysses": True,
         "recompute": "none"}, 2),
]


MOE_PLANS = [
    (2, {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1}, 2),
    (4, {"dp_replicate": 1, "dp_shard": 4, "sp": 1, "ep": 4, "micro_batch": 1}, 4),
    (4, {"dp_replicate": 1, "dp_shard": 4, "sp": 1, "ep": 2, "micro_batch": 1}, 4),
    (4, {"dp_replicate": 1, "dp_shard": 2, "sp": 2, "ep": 4, "micro_batch": 1}, 2),
    (2, {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1, "recompute": "none"}, 2),
    (4, {"dp_replicate": 1, "dp_shard": 2, "sp": 2, "ep": 4, "micro_batch": 1, "recompute": "none"}, 2),
    (4, {"dp_replicate": 1, "dp_shard": 4, "sp": 1, "ep": 4, "micro_batch": 1, "recompute": "none",
         "moe_overlap": True}, 4),
    (2, {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1, "moe_overlap": True}, 2),
    (4, {"dp_replicate": 2, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1}, 4),  # HSDP x EP
    (2, {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1}, 4),  # 2 micro-batches
]


@gpu
@pytest.mark.parametrize("world,plan,rows", MOE_PLANS)
def test_dist_moe_step_matches_oracle(world, plan, rows):
    if NGPU < world:
        pytest.skip(f"needs {world} GPUs")
    from tests.step_common import tiny_moe

    model = tiny_moe(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048, experts=64, top_k=4,
                     expert_ffn=256)
    S = 512
    loss, sessions = _run(world, model, plan, S, rows)
    from paper_2508_02317_b200.runtime import synthetic_batch

    batch = synthetic_batch(2048, S, rows, seed=2508)
    compare_step(sessions, model, batch, plan, loss)


@gpu
def test_dist_moe_redispatch_path(monkeypatch):
    """recompute=none with no HBM headroom for per-layer dispatch buffers:
    the backward re-sends the tokens on the side stream (moe_redispatch)."""
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    from tests.step_common import tiny_moe

    monkeypatch.setenv("OPX_MOE_KEEP_X_MARGIN_GB", "100000")
    model = tiny_moe(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048, experts=64, top_k=4,
                     expert_ffn=256)
    plan = {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1, "recompute": "none"}
    loss, sessions = _run(2, model, plan, 512, 2)
    from paper_2508_02317_b200.runtime import synthetic_batch

    compare_step(sessions, model, synthetic_batch(2048, 512, 2, seed=2508), plan, loss)


@gpu
@pytest.mark.parametrize("env", [{"OPX_MOE_KEEP_X_MAX": "1"},
                                 {"OPX_MOE_KEEP_GU_MARGIN_GB": "100000"}],
                         ids=["mixed_kept_and_resent", "kept_x_gate_up_recomputed"])
@pytest.mark.parametrize("overlap", [False, True])
def test_dist_moe_partial_keep_paths(monkeypatch, env, overlap):
    """recompute=none under memory pressure: only the top MoE layer keeps its
    dispatch buffer (the lower one re-sends its tokens into the shared
    buffer), or layers keep their tokens but recompute gate|up."""
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    from tests.step_common import tiny_moe

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    model = tiny_moe(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048, experts=64, top_k=4,
                     expert_ffn=256)
    plan = {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1, "recompute": "none",
            "moe_overlap": overlap}
    loss, sessions = _run(2, model, plan, 512, 2)
    from paper_2508_02317_b200.runtime import synthetic_batch

    compare_step(sessions, model, synthetic_batch(2048, 512, 2, seed=2508), plan, loss)


@gpu
@pytest.mark.parametrize("fused_dy", ["0", "1"])
def test_dist_moe_dy_dispatch_modes(monkeypatch, fused_dy):
    """The backward's dY rows reach the expert ranks either through a
    dispatch pass after the combine backward (OPX_MOE_FUSED_DY=0) or peer-
    stored by the combine backward itself (=1), under moe_overlap (whose
    default is the per-half dispatch)."""
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    from tests.step_common import tiny_moe

    monkeypatch.setenv("OPX_MOE_FUSED_DY", fused_dy)
    model = tiny_moe(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048, experts=64, top_k=4,
                     expert_ffn=256)
    plan = {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1, "recompute": "none",
            "moe_overlap": True}
    loss, sessions = _run(2, model, plan, 512, 2)
    from paper_2508_02317_b200.runtime import synthetic_batch

    compare_step(sessions, model, synthetic_batch(2048, 512, 2, seed=2508), plan, loss)
    for s in sessions:
        names = _comm_nodes(s.out[("trace", 0)])
        assert sum(x.endswith(".a2a_combine_grad") for x in names) >= 2, names


@gpu
def test_dist_c0_fsdp2_sp2_head_dim_64():
    """BASELINE C0 as specified: 2 layers, H=256, 4 heads of 64 (2 kv),
    ffn 768, V=2048, S=1024, FSDP2 x SP2 on 4 GPUs, global batch 2."""
    if NGPU < 4:
        pytest.skip("needs 4 GPUs")
    model = tiny_dense(layers=2, hidden=256, heads=4, kv=2, ffn=768, vocab=2048)
    plan = {"dp_replicate": 1, "dp_shard": 2, "sp": 2, "ep": 1, "micro_batch": 1}
    loss, sessions = _run(4, model, plan, 1024, 2)
    from paper_2508_02317_b200.runtime import synthetic_batch

    batch = synthetic_batch(2048, 1024, 2, seed=2508)
    compare_step(sessions, model, batch, plan, loss)


@gpu
@pytest.mark.parametrize("world,plan,rows", PLANS)
def test_dist_step_matches_oracle(world, plan, rows):
    if NGPU < world:
        pytest.skip(f"needs {world} GPUs")
    model = tiny_dense(layers=2, hidden=512, heads=4, kv=4 if plan["sp"] == 4 else 2, ffn=768, vocab=2048)
    S = 1024
    loss, sessions = _run(world, model, plan, S, rows)
    from paper_2508_02317_b200.runtime import synthetic_batch

    batch = synthetic_batch(2048, S, rows, seed=2508)
    compare_step(sessions, model, batch, plan, loss)


@gpu
def test_checkpoint_reshard_fsdp2_to_1(tmp_path):
    """f3: save FSDP2 shards after one step, reshard 2 -> 1 with the reference's
    copy plan, load on one GPU: masters are bit-identical and the next step's
    loss matches the FSDP2 run's."""
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    from oracle import model as om
    from paper_2508_02317_b200 import checkpoint
    from paper_2508_02317_b200.runtime import Session, synthetic_batch
    from tests.dist_worker import ckpt_worker
    from tests.step_common import EXEC, cluster, gpu_param_names

    model = tiny_dense(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048)
    arch = om.Arch.from_model_json(model)
    names = gpu_param_names(arch)
    S, rows = 512, 2
    plan2 = {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 1, "micro_batch": 1}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    a = str(tmp_path / "fsdp2")
    ps = [ctx.Process(target=ckpt_worker, args=(r, 2, port, model, plan2, S, rows, q, names, a))
          for r in range(2)]
    for p in ps:
        p.start()
    res = _collect(q, ps, 2)
    b = str(tmp_path / "fsdp1")
    checkpoint.reshard(a, b, dp_shard=1, sp=1)

    plan1 = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": rows}
    wl = {"seq_len": S, "micro_batch": rows, "global_batch": rows}
    s = Session(cluster(1), model, wl, plan1, EXEC, rank=0, device=0)
    s.load_checkpoint(b)
    for n in names:
        full, numel, b0, e0 = s.get(f"master:{n}")
        parts = sorted((res[r][1][n] for r in range(2)), key=lambda t: t[2])
        cat = np.concatenate([p[0] for p in parts if p[3] > p[2]])
        assert cat.size == numel and full.size == numel
        assert np.array_equal(full, cat), n
    s.load(synthetic_batch(2048, S, rows, seed=2508))
    r2 = s.run()
    assert abs(r2.loss - res[0][0]) <= 1e-3 * abs(res[0][0]), (r2.loss, res[0][0])
    s.close()


# ---------------------------------------------------------------------------
# the reference's step-graph structure pins (test_simulator.cpp:183-263)
# replayed on MEASURED traces.  A fused exchange node carries the reference
# node names it stands for in args.fused ("a2a_q,a2a_k,a2a_v").
# ---------------------------------------------------------------------------
def _comm_nodes(trace):
    """Collective node names of a measured trace; a fused node (an exchange
    carried by a kernel's epilogue) contributes every name it stands for."""
    out = []
    for e in trace["traceEvents"]:
        if e["name"].endswith(".a2a_wait"):
            continue
        fused = e["args"].get("fused")
        base = e["name"].rsplit(".", 1)[0]
        if fused:
            out += [base + "." + f for f in fused.split(",") if ".a2a_" in "." + f]
        elif e["cat"] == "comm":
            out.append(e["name"])
    return out


@gpu
def test_measured_trace_sp2_dense_layer_structure():
    """test_simulator.cpp:183-208 (sp=2, one dense layer): four forward
    attention exchanges (q, k, v, out); the executor adds the four backward
    ones the model omits (dO, dq, dk, dv).  No FSDP
    gathers / reduce-scatters: dp_shard*sp = 2 shards, so one per unit."""
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    model = tiny_dense(layers=1, hidden=512, heads=4, kv=2, ffn=768, vocab=2048)
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 2, "ep": 1, "micro_batch": 1}
    loss, sessions = _run(2, model, plan, 1024, 1)
    for s in sessions:
        names = _comm_nodes(s.out[("trace", 0)])
        fwd = sorted(n.rsplit(".", 1)[1] for n in names if n.startswith("fwd.layer0.m0.a2a_"))
        bwd = sorted(n.rsplit(".", 1)[1] for n in names if n.startswith("bwd.layer0.m0.a2a_"))
        assert fwd == ["a2a_k", "a2a_out", "a2a_q", "a2a_v"], fwd
        assert bwd == ["a2a_dk", "a2a_do", "a2a_dq", "a2a_dv"], bwd
        assert sum(n.startswith("bwd.rs.layer0.m0") for n in names) == 1
        rep = s.out[("report", 0)]
        assert set(rep) == {"step_time_s", "throughput_tokens_per_s_per_gpu", "mfu",
                            "exposed_comm_fraction", "model_flops_per_token", "phase_breakdown"}
        assert rep["phase_breakdown"]["fwd.layer0"]["comm_s"] > 0
        assert 0 <= rep["exposed_comm_fraction"] <= 1


@gpu
def test_measured_trace_ep2_moe_routing_nodes():
    """test_simulator.cpp:210-229: an ep=2 MoE layer has one dispatch, one
    combine, one dispatch_grad and one combine_grad node."""
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    from tests.step_common import tiny_moe

    model = tiny_moe(layers=1, hidden=512, heads=4, kv=2, ffn=768, vocab=2048, experts=64, top_k=4,
                     expert_ffn=256)
    plan = {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "ep": 2, "micro_batch": 1}
    loss, sessions = _run(2, model, plan, 512, 2)
    for s in sessions:
        names = _comm_nodes(s.out[("trace", 0)])
        for suf in (".a2a_dispatch", ".a2a_combine", ".a2a_dispatch_grad", ".a2a_combine_grad"):
            n = sum(x.endswith(suf) and ".recompute" not in x for x in names)
            assert n >= 1, (suf, names)


@gpu
def test_measured_trace_hsdp_accum_all_reduce_on_last_micro():
    """test_simulator.cpp:231-251: with two micro-batches the replicate
    all-reduce happens once per unit, on the last micro-batch (.m1), while
    reduce-scatters run per micro-batch."""
    if NGPU < 4:
        pytest.skip("needs 4 GPUs")
    model = tiny_dense(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048)
    plan = {"dp_replicate": 2, "dp_shard": 2, "sp": 1, "ep": 1, "micro_batch": 1}
    loss, sessions = _run(4, model, plan, 512, 8)
    from paper_2508_02317_b200.runtime import synthetic_batch

    compare_step(sessions, model, synthetic_batch(2048, 512, 8, seed=2508), plan, loss)
    for s in sessions:
        names = _comm_nodes(s.out[("trace", 0)])
        ar = [n for n in names if n.startswith("bwd.ar.")]
        assert len(ar) == 3 and all(n.endswith(".m1") for n in ar), ar  # 2 layers + head
        for l in range(2):
            assert sum(n.startswith(f"bwd.rs.layer{l}.") for n in names) == 2
        assert s.accum == 2
