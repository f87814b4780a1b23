"""__graft_entry__.smoke(): one tiny fwd+bwd+AdamW step of the flagship path on
cuda:0 through libopx's C ABI, checked against the CPU oracle."""


def run_smoke():
    import torch

    from paper_2508_02317_b200.runtime import Session, synthetic_batch
    from tests.step_common import EXEC, cluster, compare_step, tiny_dense

    assert torch.cuda.is_available(), "smoke() needs a GPU"
    model = tiny_dense(layers=2, hidden=256, heads=2, kv=2, ffn=768, vocab=2048)
    S, rows = 1024, 2
    wl = {"seq_len": S, "micro_batch": rows, "global_batch": rows}
    plan = {"dp_replicate": 1, "dp_shard": 1, "sp": 1, "ep": 1, "micro_batch": rows}
    s = Session(cluster(1), model, wl, plan, EXEC, rank=0, device=0)
    s.init_weights(EXEC["seed"])
    batch = synthetic_batch(2048, S, rows, seed=2508)
    s.load(batch)
    r = s.run()
    assert r.launches > 0
    rep = compare_step([s], model, batch, plan, r.loss)
    s.close()
    worst = max(v[0] for v in rep["grads"].values())
    print(f"smoke ok: loss {r.loss:.6f} (oracle {rep['loss_ref']:.6f}), worst grad err {worst:.2e}, "
          f"{r.launches} kernel launches, step {r.step_time_s * 1e3:.2f} ms")
