"""Python mirror of the reference's ParallelPlan API (proj/include/omniplan/plan.hpp:26-46).

Validation, mesh/group derivation and accounting run in libopx (C++); these
helpers only marshal JSON across the C ABI.
"""
from __future__ import annotations

import ctypes
import dataclasses
import json


@dataclasses.dataclass
class ParallelPlan:
    dp_replicate: int = 1
    dp_shard: int = -1  # derived as world / (dp_replicate * sp) when < 0 (cli.cpp:46-65)
    sp: int = 1
    ep: int = 1
    micro_batch: int = 1
    recompute: str = "full"
    offload_optimizer: bool = False
    offload_activations: bool = False
    async_ulysses: bool = False
    moe_overlap: bool = False
    fsdp_prefetch_depth: int = 1
    moe_imbalance: float = 1.0
    tp: int = 1
    pp: int = 1

    def to_json(self) -> str:
        return json.dumps(dataclasses.asdict(self))


def _s(x) -> bytes:
    if isinstance(x, (dict, list)):
        x = json.dumps(x)
    if isinstance(x, ParallelPlan):
        x = x.to_json()
    return x.encode()


def validate(cluster, model, workload, plan) -> list[tuple[str, str]]:
    """Returns [(code, message)], empty when the plan is valid (plan.cpp:19-83)."""
    from . import OpxError, lib

    buf = ctypes.create_string_buffer(1 << 16)
    rc = lib().opx_plan_validate(_s(cluster), _s(model), _s(workload), _s(plan), buf, len(buf))
    if rc not in (0, 3):
        raise OpxError(rc, lib().opx_last_error().decode())
    out = []
    for line in buf.value.decode().splitlines():
        code, _, msg = line.partition("\t")
        out.append((code, msg))
    return out


def resolve(cluster, model, workload, plan) -> dict:
    """Label, mesh, groups, expert sharding, accounting and volumes for a valid plan."""
    from . import OpxError, lib

    buf = ctypes.create_string_buffer(1 << 22)
    rc = lib().opx_plan_resolve(_s(cluster), _s(model), _s(workload), _s(plan), buf, len(buf))
    if rc != 0:
        raise OpxError(rc, lib().opx_last_error().decode() + " " + buf.value.decode())
    return json.loads(buf.value.decode())
