"""Host-side session around the opx step executor (C ABI ``opx_step_*``).

Mirrors the reference's driver flow (cli.cpp:239-289 cmd_simulate:
load configs -> validate plan -> build the step -> run -> StepReport), with
the simulation replaced by execution on the local GPU.  torch.distributed is
used only as the out-of-band rendezvous for the NCCL unique id and the CUDA
IPC handles of the peer-memory arenas.
"""
from __future__ import annotations

import ctypes
import json
import math
import os

import numpy as np

from . import OpxError, check, lib


class StepReport(ctypes.Structure):
    _fields_ = [("step_time_s", ctypes.c_double), ("fwd_s", ctypes.c_double),
                ("bwd_s", ctypes.c_double), ("opt_s", ctypes.c_double),
                ("comm_wait_s", ctypes.c_double), ("loss", ctypes.c_double),
                ("tokens", ctypes.c_double), ("n_valid", ctypes.c_double),
                ("launches", ctypes.c_int64), ("enqueue_s", ctypes.c_double),
                ("kept_layers", ctypes.c_int64),
                # StepReport (simulator.hpp:43-50) on the measured step
                ("throughput", ctypes.c_double), ("mfu", ctypes.c_double),
                ("exposed_comm", ctypes.c_double), ("model_flops_per_token", ctypes.c_double),
                ("comm_s", ctypes.c_double), ("accum_steps", ctypes.c_int64)]


def _s(x) -> bytes:
    return (json.dumps(x) if not isinstance(x, str) else x).encode()


# ---------------------------------------------------------------------------
# synthetic packed batches
# ---------------------------------------------------------------------------
def pack_row_lengths(S: int, rng: np.random.Generator, min_len: int = 64) -> list[int]:
    """One row of exactly S tokens cut into samples with
    l ~ clamp(round(LogNormal(ln(S/8), 1)), min_len, S); the last sample takes
    the remainder (padding ratio 0, packing.cpp:53-64)."""
    out, used = [], 0
    while used < S:
        l = int(np.clip(round(rng.lognormal(math.log(S / 8), 1.0)), min(min_len, S), S))
        l = min(l, S - used)
        out.append(l)
        used += l
    return out


def synthetic_batch(vocab: int, seq_len: int, rows: int, seed: int = 2508, single_sample: bool = False):
    """Global batch: ids/labels/pos [rows, S] int32, cu_rows: per-row cumulative
    boundaries (PackedBatch.boundaries convention, packing.hpp:28)."""
    rng = np.random.default_rng(seed)
    ids = rng.integers(0, vocab, size=(rows, seq_len), dtype=np.int64).astype(np.int32)
    labels = np.full((rows, seq_len), -100, np.int32)
    pos = np.zeros((rows, seq_len), np.int32)
    cu_rows = []
    for r in range(rows):
        lens = [seq_len] if single_sample else pack_row_lengths(seq_len, rng)
        cu = [0]
        for l in lens:
            a = cu[-1]
            pos[r, a:a + l] = np.arange(l)
            labels[r, a:a + l - 1] = ids[r, a + 1:a + l]
            cu.append(a + l)
        cu_rows.append(cu)
    return {"ids": ids, "labels": labels, "pos": pos, "cu_rows": cu_rows}


def synthetic_images(batch, tokens_per_item: int, patch_dim: int, items_per_row: int = 2,
                     placeholder: int | None = None, seed: int = 2508):
    """Places up to ``items_per_row`` image items in every row of ``batch`` (in
    place) for a frozen encoder module: an item occupies
    ``tokens_per_item`` placeholder tokens inside one sample (from its second
    token, 8 text tokens between consecutive images); those positions, and the
    one predicting the first of them, are unsupervised.  Adds batch["img"] = {"row", "pos",
    "pixels" [n, 4*tokens_per_item, patch_dim] float32} sorted by (row, pos)."""
    rng = np.random.default_rng(seed + 1)
    ids, labels = batch["ids"], batch["labels"]
    vocab_ph = int(ids.max()) if placeholder is None else placeholder
    rows, pos = [], []
    for r, cu in enumerate(batch["cu_rows"]):
        placed = 0
        for a, b in zip(cu[:-1], cu[1:]):
            p0 = a + 1  # images back to back (8 text tokens apart) from the sample's 2nd token
            while placed < items_per_row and p0 + tokens_per_item + 1 <= b:
                ids[r, p0:p0 + tokens_per_item] = vocab_ph
                labels[r, p0 - 1:p0 + tokens_per_item] = -100
                rows.append(r)
                pos.append(p0)
                placed += 1
                p0 += tokens_per_item + 8
    n = len(rows)
    pix = rng.standard_normal((n, 4 * tokens_per_item, patch_dim)).astype(np.float32)
    batch["img"] = {"row": np.array(rows, np.int32), "pos": np.array(pos, np.int32), "pixels": pix}
    return batch


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def rank_coords(rank: int, plan: dict):
    sp, sh = plan["sp"], plan["dp_shard"]
    return rank // (sp * sh), (rank // sp) % sh, rank % sp  # rep, shard, sp


def accum_steps(batch, plan: dict) -> int:
    """Gradient-accumulation steps of a global batch: rows/(dp_width*micro_batch)
    (step_graph.cpp:57)."""
    unit = plan["dp_replicate"] * plan["dp_shard"] * plan["micro_batch"]
    rows = batch["ids"].shape[0]
    if rows % unit:
        raise ValueError(f"batch rows {rows} not divisible by dp_width*micro_batch = {unit}")
    return rows // unit


def local_slice(batch, rank: int, plan: dict):
    """What rank `rank` feeds its executor: its dp rows (k micro-batches of
    micro_batch consecutive rows, k = accum_steps), its SP token slice."""
    rep, sh, spi = rank_coords(rank, plan)
    m, sp = plan["micro_batch"] * accum_steps(batch, plan), plan["sp"]
    dp = rep * plan["dp_shard"] + sh
    rows = slice(dp * m, (dp + 1) * m)
    S = batch["ids"].shape[1]
    Sl = S // sp
    tok = slice(spi * Sl, (spi + 1) * Sl)
    ids = np.ascontiguousarray(batch["ids"][rows, tok]).reshape(-1)
    labels = np.ascontiguousarray(batch["labels"][rows, tok]).reshape(-1)
    pos = np.ascontiguousarray(batch["pos"][rows]).reshape(-1)
    cu = [0]
    for i, c in enumerate(batch["cu_rows"][rows]):
        cu += [i * S + x for x in c[1:]]
    n_valid = int((batch["labels"] >= 0).sum())
    return ids, labels, pos, np.array(cu, np.int32), n_valid


# ---------------------------------------------------------------------------
# session
# ---------------------------------------------------------------------------
class Session:
    """One rank's executor.  ``dist`` (optional) is an initialised
    torch.distributed default group used for rendezvous only."""

    def __init__(self, cluster, model, workload, plan, exec_cfg=None, rank=0, device=0, dist=None):
        L = lib()
        self.cluster, self.model, self.workload = cluster, model, workload
        self.plan = dict(plan)
        world = cluster["num_nodes"] * cluster["gpus_per_node"]
        if self.plan.get("dp_shard", -1) in (-1, None):
            self.plan["dp_shard"] = world // (self.plan.get("dp_replicate", 1) * self.plan.get("sp", 1))
        for k, v in (("dp_replicate", 1), ("sp", 1), ("ep", 1), ("micro_batch", 1)):
            self.plan.setdefault(k, v)
        self.rank, self.world, self.dist = rank, world, dist
        dpw = self.plan["dp_replicate"] * self.plan["dp_shard"]
        self.accum = max(1, workload["global_batch"] // (dpw * self.plan["micro_batch"]))
        nid = ctypes.create_string_buffer(128)
        if world > 1:
            if rank == 0:
                check(L.opx_nccl_unique_id(nid))
            nid = ctypes.create_string_buffer(self._bcast(bytes(nid.raw)), 128)
        self.h = ctypes.c_void_p()
        rc = L.opx_step_create(_s(cluster), _s(model), _s(workload), _s(self.plan),
                               _s(exec_cfg or {}), rank, device, nid, ctypes.byref(self.h))
        if rc:
            raise OpxError(rc, L.opx_last_error().decode())
        buf = ctypes.create_string_buffer(256)
        n = ctypes.c_size_t()
        check(L.opx_step_ipc_export(self.h, buf, 256, ctypes.byref(n)))
        mine = bytes(buf.raw[:n.value])
        allh = self._allgather(mine) if world > 1 else [mine]
        blob = b"".join(allh)
        check(L.opx_step_ipc_import(self.h, blob, n.value))

    # -- rendezvous helpers (bytes only; never tensors of the step)
    def _bcast(self, b: bytes) -> bytes:
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def _allgather(self, b: bytes):
        out = [None] * self.world
        self.dist.all_gather_object(out, b)
        return out

    def init_weights(self, seed: int = 2508):
        check(lib().opx_step_init_weights(self.h, seed))

    def load(self, batch):
        ids, labels, pos, cu, n_valid = local_slice(batch, self.rank, self.plan)
        i32 = ctypes.POINTER(ctypes.c_int32)
        check(lib().opx_step_load_batch(self.h, ids.ctypes.data_as(ctypes.c_void_p),
                                        labels.ctypes.data_as(ctypes.c_void_p),
                                        pos.ctypes.data_as(ctypes.c_void_p),
                                        cu.ctypes.data_as(ctypes.c_void_p), len(cu), n_valid))
        if "img" in batch:  # frozen encoder inputs of this rank's dp rows
            rep, sh, _ = rank_coords(self.rank, self.plan)
            m = self.plan["micro_batch"]
            dp = rep * self.plan["dp_shard"] + sh
            img = batch["img"]
            sel = np.nonzero((img["row"] >= dp * m) & (img["row"] < (dp + 1) * m))[0]
            rows = np.ascontiguousarray(img["row"][sel] - dp * m, np.int32)
            posi = np.ascontiguousarray(img["pos"][sel], np.int32)
            if "_bf16" not in img:  # converted once per batch
                img["_bf16"] = _bf16_bits(img["pixels"])
            # items are sorted by row: this rank's rows are one contiguous (view) range
            pix = img["_bf16"][sel[0]:sel[-1] + 1] if len(sel) else np.zeros(1, np.uint16)
            check(lib().opx_step_load_images(self.h, pix.ctypes.data_as(ctypes.c_void_p), len(sel),
                                             rows.ctypes.data_as(ctypes.c_void_p),
                                             posi.ctypes.data_as(ctypes.c_void_p)))
        return n_valid

    def run(self) -> StepReport:
        r = StepReport()
        check(lib().opx_step_run(self.h, ctypes.byref(r)))
        return r

    def info(self, name):
        n, b, e = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib().opx_step_tensor_info(self.h, name.encode(), ctypes.byref(n), ctypes.byref(b), ctypes.byref(e)))
        return n.value, b.value, e.value

    def get(self, name):
        """This rank's [begin, end) slice of a flattened tensor (fp32, or bf16 bits as uint16 for param:)."""
        n, b, e = self.info(name)
        dt = np.uint16 if name.startswith("param:") else np.float32
        out = np.empty(e - b, dt)
        check(lib().opx_step_get(self.h, name.encode(), out.ctypes.data_as(ctypes.c_void_p), out.nbytes))
        return out, n, b, e

    def routes(self, layer: int, T: int, k: int):
        """Forward top-k expert indices of MoE layer `layer` for this rank's T
        tokens (T = every micro-batch's local tokens under accumulation)."""
        out = np.empty((T, k), np.int32)
        check(lib().opx_step_get(self.h, f"route:{layer}".encode(), out.ctypes.data_as(ctypes.c_void_p),
                                 out.nbytes))
        return out

    def features(self, T, H):
        """[T, H] encoder feature rows this rank received (meaningful at its
        placeholder positions only)."""
        out = np.empty((T, H), np.float32)
        check(lib().opx_step_get(self.h, b"features", out.ctypes.data_as(ctypes.c_void_p), out.nbytes))
        return out

    def loss_rows(self, T):
        out = np.empty(T, np.float32)
        check(lib().opx_step_get(self.h, b"loss_rows", out.ctypes.data_as(ctypes.c_void_p), out.nbytes))
        return out

    def save(self, path: str):
        """FSDP flat-shard checkpoint (opx_step_save); every rank calls it."""
        if self.dist is not None and self.world > 1:
            self.dist.barrier()
        check(lib().opx_step_save(self.h, os.fspath(path).encode()))
        if self.dist is not None and self.world > 1:
            self.dist.barrier()

    def load_checkpoint(self, path: str):
        """Loads a checkpoint with this plan's shard counts (see checkpoint.reshard)."""
        if self.dist is not None and self.world > 1:
            self.dist.barrier()
        check(lib().opx_step_load(self.h, os.fspath(path).encode()))

    def report_json(self) -> dict:
        """The last step as to_json(StepReport) (report.cpp:117-128)."""
        cap = 1 << 20
        buf = ctypes.create_string_buffer(cap)
        n = ctypes.c_size_t()
        check(lib().opx_step_report_json(self.h, buf, cap, ctypes.byref(n)))
        return json.loads(buf.value.decode())

    def trace(self) -> dict:
        cap = 1 << 24
        buf = ctypes.create_string_buffer(cap)
        n = ctypes.c_size_t()
        check(lib().opx_step_trace(self.h, buf, cap, ctypes.byref(n)))
        return json.loads(buf.value.decode())

    def close(self):
        if self.h:
            lib().opx_step_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def deinterleave_gate_up(flat: np.ndarray, F: int, H: int):
    """[2F, H] 128-row interleaved gate|up -> (gate [F,H], up [F,H])."""
    v = flat.reshape(F // 128, 2, 128, H)
    return v[:, 0].reshape(F, H), v[:, 1].reshape(F, H)


def bf16_bits_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)
