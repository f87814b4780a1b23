"""Multi-rank host logic on CPU (gloo, world_size 2): the rendezvous used for
NCCL ids / IPC handles, the per-rank batch partition (dp rows x SP token
slices), rank coordinates vs the C++ mesh, and gradient reduction semantics of
the oracle's simulated ranks."""
import multiprocessing as mp
import os
import random

from tests.step_common import free_port

import numpy as np

from paper_2508_02317_b200.plan import resolve
from paper_2508_02317_b200.runtime import local_slice, rank_coords, synthetic_batch


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as td

    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1) rendezvous primitives used by Session (bytes only)
        obj = [b"id-from-rank0" if rank == 0 else None]
        td.broadcast_object_list(obj, src=0)
        handles = [None] * world
        td.all_gather_object(handles, f"ipc-{rank}".encode())
        # 2) batch partition for an SP2 plan and an FSDP2 plan
        b = synthetic_batch(997, 512, 2, seed=11)
        sp_plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 2, "micro_batch": 2}
        dp_plan = {"dp_replicate": 1, "dp_shard": 2, "sp": 1, "micro_batch": 1}
        parts = {}
        for name, plan in (("sp", sp_plan), ("dp", dp_plan)):
            ids, labels, pos, cu, nv = local_slice(b, rank, plan)
            got = [None] * world
            td.all_gather_object(got, (ids.tolist(), labels.tolist(), pos.tolist(), cu.tolist(), nv))
            parts[name] = got
        # 3) gradient reduction of simulated dp ranks (gloo all-reduce == FSDP RS + AG)
        from oracle import model as om

        a = om.Arch(layers=1, hidden=128, heads=1, kv_heads=1, head_dim=128, ffn=256, vocab=256)
        P = om.init_params(a, 5)
        bb = synthetic_batch(a.vocab, 128, 2, seed=3)
        mine = {k: v[rank:rank + 1] if k != "cu_rows" else v[rank:rank + 1] for k, v in bb.items()}
        n_valid = int((bb["labels"] >= 0).sum())
        st = om.Step(a, P)
        cu = np.array(mine["cu_rows"][0])
        loss, G = st.run(mine["ids"][0], mine["labels"][0], mine["pos"][0], cu, n_valid)
        t = torch.tensor(np.concatenate([g.ravel() for g in G.values()]).astype(np.float64))
        td.all_reduce(t)
        lt = torch.tensor([loss], dtype=torch.float64)
        td.all_reduce(lt)
        q.put((rank, obj[0], handles, parts, t.numpy(), float(lt[0]) / n_valid, None))
    except Exception:
        import traceback

        q.put((rank, None, None, None, None, None, traceback.format_exc()))
    finally:
        td.destroy_process_group()


def test_gloo_world2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        assert r[-1] is None, r[-1]
        res[r[0]] = r
    for p in ps:
        p.join(30)
    assert res[1][1] == b"id-from-rank0"
    assert res[0][2] == [b"ipc-0", b"ipc-1"]
    b = synthetic_batch(997, 512, 2, seed=11)
    # SP2: each rank holds half of every row's tokens; positions/cu cover whole rows
    sp = res[0][3]["sp"]
    ids = np.concatenate([np.array(sp[0][0]).reshape(2, 256), np.array(sp[1][0]).reshape(2, 256)], 1)
    assert np.array_equal(ids, b["ids"])
    assert sp[0][2] == sp[1][2] and sp[0][3] == sp[1][3]
    assert sp[0][3][-1] == 1024 and sp[0][4] == int((b["labels"] >= 0).sum())
    # FSDP2: each rank holds one full row
    dp = res[0][3]["dp"]
    assert np.array_equal(np.array(dp[0][0]), b["ids"][0]) and np.array_equal(np.array(dp[1][0]), b["ids"][1])
    # reduced gradients == single-process gradients on the whole batch
    from oracle import model as om

    a = om.Arch(layers=1, hidden=128, heads=1, kv_heads=1, head_dim=128, ffn=256, vocab=256)
    P = om.init_params(a, 5)
    bb = synthetic_batch(a.vocab, 128, 2, seed=3)
    loss, G = om.simulate_ranks(a, P, bb, {"micro_batch": 2, "dp_replicate": 1, "dp_shard": 1, "sp": 1})
    ref = np.concatenate([g.ravel() for g in G.values()])
    got = res[0][4]
    assert np.allclose(got, ref, rtol=1e-4, atol=1e-8)
    assert abs(res[0][5] - loss) < 1e-6 * abs(loss)


def test_rank_coords_match_cpp_mesh():
    cl = {"num_nodes": 1, "gpus_per_node": 8, "gpu": {"peak_flops": 1e15, "hbm_bytes": 1e11},
          "link": {"intra_node_bw": 9e11, "inter_node_bw": 5e10, "intra_latency": 5e-6, "inter_latency": 2e-5}}
    m = {"modules": [{"name": "core", "kind": "foundation", "trainable": True,
                      "arch": {"layers": 1, "hidden": 512, "heads": 4, "kv_heads": 4, "head_dim": 128,
                               "ffn_dim": 512, "vocab": 64}}]}
    for rep, sh, sp in ((1, 8, 1), (1, 2, 4), (2, 2, 2), (2, 1, 4), (4, 2, 1)):
        plan = {"dp_replicate": rep, "dp_shard": sh, "sp": sp}
        wl = {"seq_len": 64, "micro_batch": 1, "global_batch": rep * sh}
        g = resolve(cl, m, wl, plan)["groups"]
        for r in range(8):
            ri, si, pi = rank_coords(r, plan)
            assert [x for x in g["sp"] if r in x][0][pi] == r
            assert [x for x in g["replicate"] if r in x][0][ri] == r
            assert [x for x in g["shard"] if r in x][0][si * sp + pi] == r


def test_accumulation_partition_covers_the_batch():
    """global_batch = k * dp_width * micro_batch (step_graph.cpp:57): dp rank r
    feeds rows [r*k*m, (r+1)*k*m) as k micro-batches, SP ranks split tokens;
    together the ranks cover every token once, and the oracle's simulated
    micro-batches walk the same rows in the same order."""
    from paper_2508_02317_b200.runtime import accum_steps

    b = synthetic_batch(997, 256, 8, seed=4)
    plan = {"dp_replicate": 2, "dp_shard": 1, "sp": 2, "micro_batch": 2}
    assert accum_steps(b, plan) == 2
    seen = np.zeros((8, 256), int)
    for r in range(4):
        ids, labels, pos, cu, nv = local_slice(b, r, plan)
        rep, sh, spi = rank_coords(r, plan)
        dp = rep * plan["dp_shard"] + sh
        rows = slice(dp * 4, (dp + 1) * 4)
        assert np.array_equal(ids.reshape(4, 128), b["ids"][rows, spi * 128:(spi + 1) * 128])
        assert cu[-1] == 4 * 256 and len(pos) == 4 * 256  # all k*m rows' positions / boundaries
        seen[rows, spi * 128:(spi + 1) * 128] += 1
    assert (seen == 1).all()
    try:
        accum_steps(synthetic_batch(997, 256, 6, seed=4), plan)
        raise AssertionError("6 rows with dp_width*m = 4 must be rejected")
    except ValueError:
        pass
