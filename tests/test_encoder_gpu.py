"""Frozen omni-modal encoder path on B200 against the CPU
oracle (oracle/encoder.py): the bidirectional tcgen05 attention kernel, the
encoder features each rank receives through the SP scatter, and the full
training step with those features injected (loss, gradients, AdamW)."""
import ctypes
import math
import multiprocessing as mp

import numpy as np
import pytest
import torch

from tests.step_common import EXEC, cluster, compare_step, free_port, tiny_dense, tiny_encoder

gpu = pytest.mark.gpu
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
TOL_FEAT = 2e-2  # max-abs-err / max-abs-ref on the bf16 feature rows


def _P(t):
    return ctypes.c_void_p(t.data_ptr())


@gpu
@pytest.mark.parametrize("hq,hk", [(4, 4), (4, 2)])
def test_attn_bidir_matches_torch(hq, hk):
    from paper_2508_02317_b200 import check, lib

    torch.manual_seed(0)
    bounds = [0, 64, 300, 301, 555, 700]  # ragged items, one of a single token
    N = bounds[-1]
    st = torch.empty(N, dtype=torch.int32)
    en = torch.empty(N, dtype=torch.int32)
    for a, b in zip(bounds[:-1], bounds[1:]):
        st[a:b], en[a:b] = a, b
    st, en = st.cuda(), en.cuda()
    q = torch.randn(N, hq, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(N, hk, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(N, hk, 128, device="cuda", dtype=torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty(hq, N, device="cuda")
    sc = 1 / math.sqrt(128)
    check(lib().opx_attn_fwd_bidir_tc(_P(q), _P(k), _P(v), _P(o), _P(lse), hq * 128, hk * 128, hk * 128,
                                      hq * 128, _P(st), _P(en), N, hq, hk, ctypes.c_float(sc),
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref = torch.empty(N, hq, 128)
    G = hq // hk
    for a, b in zip(bounds[:-1], bounds[1:]):
        qs = q[a:b].float().cpu().transpose(0, 1)
        ks = k[a:b].float().cpu().repeat_interleave(G, 1).transpose(0, 1)
        vs = v[a:b].float().cpu().repeat_interleave(G, 1).transpose(0, 1)
        p = torch.softmax(qs @ ks.transpose(1, 2) * sc, -1)
        ref[a:b] = (p @ vs).transpose(0, 1)
    err = (o.float().cpu() - ref).abs().max() / ref.abs().max()
    assert err < 2e-2, float(err)


def _model():
    m = tiny_dense(layers=2, hidden=512, heads=4, kv=2, ffn=768, vocab=2048)
    m["modules"].append(tiny_encoder())
    return m


IMAGES = {"tokens_per_item": 16, "patch_dim": 96, "items_per_row": 3}


def _oracle_features(model, batch, plan, rank):
    """Oracle features at this rank's local placeholder positions ([T, H], mask)."""
    from oracle import encoder as oe
    from paper_2508_02317_b200.runtime import rank_coords

    ea = oe.EncArch.from_model_json(model)
    P = oe.init_encoder(ea, EXEC["seed"])
    S = batch["ids"].shape[1]
    m, sp = plan["micro_batch"], plan["sp"]
    rep, sh, spi = rank_coords(rank, plan)
    dp = rep * plan["dp_shard"] + sh
    mask, feats = oe.inject_for_rows(ea, P, batch["img"], range(dp * m, (dp + 1) * m), S)
    full = np.zeros((m * S, ea.out_hidden), np.float32)
    full[mask] = feats
    Sl = S // sp
    loc = full.reshape(m, S, -1)[:, spi * Sl:(spi + 1) * Sl].reshape(m * Sl, -1)
    lm = mask.reshape(m, S)[:, spi * Sl:(spi + 1) * Sl].reshape(-1)
    return loc, lm


def _check_features(got, ref, mask):
    assert mask.any()
    err = np.abs(got[mask] - ref[mask]).max() / np.abs(ref[mask]).max()
    assert err < TOL_FEAT, err


@gpu
def test_step_with_frozen_encoder_one_gpu():
    from paper_2508_02317_b200.runtime import Session, synthetic_batch, synthetic_images

    model = _model()
    S, rows = 1024, 2
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": rows}
    wl = {"seq_len": S, "micro_batch": rows, "global_batch": rows}
    s = Session(cluster(1), model, wl, plan, EXEC, rank=0, device=0)
    s.init_weights(EXEC["seed"])
    batch = synthetic_images(synthetic_batch(2048, S, rows, seed=2508), **IMAGES)
    assert len(batch["img"]["row"]) >= 4
    s.load(batch)
    r = s.run()
    ref, mask = _oracle_features(model, batch, plan, 0)
    _check_features(s.features(rows * S, 512), ref, mask)
    compare_step([s], model, batch, plan, r.loss)
    s.close()


def _run_dist(world, model, plan, S, rows):
    from oracle import model as om
    from tests.dist_worker import step_worker
    from tests.step_common import gpu_param_names
    from tests.test_step_dist_gpu import _collect, _Remote

    names = gpu_param_names(om.Arch.from_model_json(model))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=step_worker, args=(r, world, port, model, plan, S, rows, q, names, IMAGES))
          for r in range(world)]
    for p in ps:
        p.start()
    res = _collect(q, ps, world)
    assert len({round(v[0], 6) for v in res.values()}) == 1
    return res[0][0], [_Remote(res[r][1]) for r in range(world)], res


@gpu
@pytest.mark.parametrize("world,plan,rows", [
    (2, {"dp_replicate": 1, "dp_shard": 1, "sp": 2, "ep": 1, "micro_batch": 2}, 2),
    (4, {"dp_replicate": 1, "dp_shard": 2, "sp": 2, "ep": 1, "micro_batch": 1}, 2),
])
def test_step_with_frozen_encoder_sp(world, plan, rows):
    """Items dealt round-robin to the SP ranks; features reach the ranks that
    own the placeholder positions through the peer-store scatter."""
    if NGPU < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2508_02317_b200.runtime import synthetic_batch, synthetic_images

    model = _model()
    S = 1024
    loss, sessions, res = _run_dist(world, model, plan, S, rows)
    batch = synthetic_images(synthetic_batch(2048, S, rows, seed=2508), **IMAGES)
    for rank in range(world):
        ref, mask = _oracle_features(model, batch, plan, rank)
        if mask.any():
            _check_features(res[rank][1][("features", 0)], ref, mask)
    compare_step(sessions, model, batch, plan, loss)
