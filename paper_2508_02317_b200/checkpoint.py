"""Reshard an opx FSDP checkpoint to another world size.

The reference moves flat FSDP shards between world sizes with an
interval-intersection copy plan (``omniplan reshard``: reshard.cpp:20-56
``make_plan``, :112-137 ``apply_plan``, driven by cli.cpp:422-496).  The opx
checkpoint (``opx_step_save``) stores, per unit, the chunked interval each
shard owns of the logical flat parameter; this tool asks libopx for the same
copy plan (``opx_reshard_plan``) and moves the fp32 master / exp_avg /
exp_avg_sq bytes accordingly.  Expert units keep their EP position in their
name, so the EP degree must not change; dense and expert FSDP degrees may.

    python -m paper_2508_02317_b200.checkpoint SRC DST --dp-shard 1 --sp 1 [--ep 1]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os

import numpy as np

from . import check, lib


def reshard_plan(numel: int, src_parts: int, dst_parts: int, src_align: int = 64,
                 dst_align: int = 64) -> dict:
    """Copy ops [[src_rank, src_off, dst_rank, dst_off, len], ...] (libopx)."""
    cap = 256 + 96 * (src_parts + dst_parts) * 2
    buf = ctypes.create_string_buffer(cap)
    check(lib().opx_reshard_plan(numel, src_parts, src_align, dst_parts, dst_align, buf, cap))
    return json.loads(buf.value.decode())


def _chunk_len(numel: int, chunk: int, r: int) -> int:
    return max(0, min((r + 1) * chunk, numel) - min(r * chunk, numel))


def reshard(src: str, dst: str, dp_shard: int, sp: int, ep: int | None = None,
            dp_replicate: int = 1) -> dict:
    """Writes a checkpoint for a plan with shard degree dp_shard*sp (experts:
    dp_shard*sp/ep) and returns its manifest."""
    with open(os.path.join(src, "manifest.json")) as f:
        man = json.load(f)
    old_ep = int(man["plan"]["ep"])
    ep = old_ep if ep is None else ep
    if ep != old_ep:
        raise ValueError(f"EP degree {old_ep} -> {ep}: expert placement changes, not a reshard")
    align = int(man.get("align", 64))
    shard_deg = dp_shard * sp
    if shard_deg % ep:
        raise ValueError("dp_shard*sp must be a multiple of ep")
    out_units = []
    for u in man["units"]:
        name, numel, sp_, sc = u["name"], int(u["numel"]), int(u["parts"]), int(u["chunk"])
        dp_ = shard_deg // ep if ".experts." in name else shard_deg
        plan = reshard_plan(numel, sp_, dp_, align, align)
        if plan["src_chunk"] != sc:
            raise ValueError(f"{name}: manifest chunk {sc} != layout chunk {plan['src_chunk']}")
        dc = plan["dst_chunk"]
        srcs = []
        for r in range(sp_):
            n = _chunk_len(numel, sc, r)
            a = np.fromfile(os.path.join(src, name, f"shard{r}.bin"), dtype=np.float32)
            if a.size != 3 * n:
                raise ValueError(f"{name}/shard{r}.bin: {a.size} floats, expected {3 * n}")
            srcs.append(a.reshape(3, n))
        dsts = [np.zeros((3, _chunk_len(numel, dc, d)), np.float32) for d in range(dp_)]
        for s_rank, s_off, d_rank, d_off, ln in plan["ops"]:
            dsts[d_rank][:, d_off:d_off + ln] = srcs[s_rank][:, s_off:s_off + ln]
        os.makedirs(os.path.join(dst, name), exist_ok=True)
        for d, a in enumerate(dsts):
            a.tofile(os.path.join(dst, name, f"shard{d}.bin"))
        out_units.append({"name": name, "numel": numel, "parts": dp_, "chunk": dc})
    new = dict(man)
    new["units"] = out_units
    new["plan"] = {"dp_replicate": dp_replicate, "dp_shard": dp_shard, "sp": sp, "ep": ep}
    with open(os.path.join(dst, "manifest.json"), "w") as f:
        json.dump(new, f, indent=1)
    return new


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("src")
    ap.add_argument("dst")
    ap.add_argument("--dp-shard", type=int, required=True)
    ap.add_argument("--sp", type=int, default=1)
    ap.add_argument("--ep", type=int, default=None)
    ap.add_argument("--dp-replicate", type=int, default=1)
    a = ap.parse_args(argv)
    m = reshard(a.src, a.dst, a.dp_shard, a.sp, a.ep, a.dp_replicate)
    print(f"resharded {len(m['units'])} units to dp_shard={a.dp_shard} sp={a.sp}")


if __name__ == "__main__":
    main()
