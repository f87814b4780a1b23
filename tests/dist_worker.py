"""Worker for multi-rank step tests: one process per GPU (or per CPU rank for
the gloo host-logic tests).  Returns this rank's loss and tensor slices."""
import os


def step_worker(rank, world, port, model, plan, S, rows, q, names, images=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as td

    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_02317_b200.runtime import Session, synthetic_batch
        from tests.step_common import EXEC, cluster

        wl = {"seq_len": S, "micro_batch": plan["micro_batch"], "global_batch": rows}
        s = Session(cluster(world), model, wl, plan, EXEC, rank=rank, device=rank, dist=td)
        s.init_weights(EXEC["seed"])
        batch = synthetic_batch(model["modules"][0]["arch"]["vocab"], S, rows, seed=2508)
        if images:
            from paper_2508_02317_b200.runtime import synthetic_images

            synthetic_images(batch, **images)
        s.load(batch)
        r = s.run()
        out = {}
        if images:
            H = model["modules"][0]["arch"]["hidden"]
            out[("features", 0)] = s.features(plan["micro_batch"] * S // plan["sp"], H)
        for kind in ("grad", "master"):
            for n in names:
                v, numel, b, e = s.get(f"{kind}:{n}")
                out[(kind, n)] = (v, numel, b, e)
        out[("trace", 0)] = s.trace()
        out[("report", 0)] = s.report_json()
        out[("report_struct", 0)] = {f[0]: getattr(r, f[0]) for f in r._fields_}
        arch = model["modules"][0]["arch"]
        if "moe" in arch:
            T = s.accum * plan["micro_batch"] * S // plan["sp"]
            k = arch["moe"]["top_k"]
            stride = arch["moe"].get("moe_layer_stride", 1)
            for l in range(arch["layers"]):
                if (l + 1) % stride == 0:
                    out[("route", l)] = s.routes(l, T, k)
        q.put((rank, r.loss, out, None))
        s.close()
    except Exception as ex:  # report instead of hanging the parent
        import traceback

        q.put((rank, None, None, traceback.format_exc()))
    finally:
        td.destroy_process_group()


def ckpt_worker(rank, world, port, model, plan, S, rows, q, names, path):
    """One step, save a checkpoint, then a second step; returns the masters at
    the checkpoint and the second step's loss."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as td

    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2508_02317_b200.runtime import Session, synthetic_batch
        from tests.step_common import EXEC, cluster

        wl = {"seq_len": S, "micro_batch": plan["micro_batch"], "global_batch": rows}
        s = Session(cluster(world), model, wl, plan, EXEC, rank=rank, device=rank, dist=td)
        s.init_weights(EXEC["seed"])
        batch = synthetic_batch(model["modules"][0]["arch"]["vocab"], S, rows, seed=2508)
        s.load(batch)
        s.run()
        s.save(path)
        out = {n: s.get(f"master:{n}") for n in names}
        r2 = s.run()
        q.put((rank, r2.loss, out, None))
        s.close()
    except Exception:
        import traceback

        q.put((rank, None, None, traceback.format_exc()))
    finally:
        td.destroy_process_group()
