#!/usr/bin/env python
"""Benchmark of the fwd+bwd+AdamW training step (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3|c4|c0] [--impl opx|reference]

N > 1 is launched by the driver under torchrun (one rank per GPU).  Rank 0
prints ONE JSON line.  `value` is whole-job tokens/s from device time (CUDA
events inside the executor, max over ranks); `e2e` is the same metric through
the public C ABI with host input buffers (H2D of ids/labels/positions and the
D2H loss read inside the timed region); `--impl reference` times the CPU
reference path (the numpy oracle; the reference itself computes no tensors).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train tokens/sec/GPU and MFU (fwd+bwd+opt step) at 1/2/4/8 B200 vs CPU ref"

QWEN2_7B = {"layers": 28, "hidden": 3584, "heads": 28, "kv_heads": 4, "head_dim": 128,
            "ffn_dim": 18944, "vocab": 152064}
# C4: Qwen2-72B-shaped 8-layer slice, the long-context HBM-sizing stress
QWEN2_72B_SLICE = {"layers": 8, "hidden": 8192, "heads": 64, "kv_heads": 8, "head_dim": 128,
                   "ffn_dim": 29568, "vocab": 152064}
QWEN3_30B_A3B = {"layers": 48, "hidden": 2048, "heads": 16, "kv_heads": 4, "head_dim": 128,
                 "ffn_dim": 6144, "vocab": 151936,
                 "moe": {"num_experts": 128, "top_k": 8, "expert_ffn_dim": 768, "moe_layer_stride": 1}}
# C3: Qwen2.5-VL-7B-shaped = the Qwen2-7B backbone + a frozen ViT (32 x 1280, 16
# heads of 80; ffn 3420 rounded up to 3456 for the 128-wide tiles; 14x14x3x2
# patches = 1176 wide; 2x2 merger -> 256 tokens per 448x448 image)
QWEN25_VL_VIT = {"layers": 32, "hidden": 1280, "heads": 16, "kv_heads": 16, "head_dim": 80,
                 "ffn_dim": 3456, "vocab": 1176}
C3_TOKENS_PER_IMAGE = 256
C3_IMAGE_MIX = 0.25  # workload modality_mix: 16K of the 64K tokens are image tokens
# C0: 2 layers, H=256, 4 heads of 64, 2 kv heads, ffn 768, V=2048, S=1024
TINY = {"layers": 2, "hidden": 256, "heads": 4, "kv_heads": 2, "head_dim": 64, "ffn_dim": 768,
        "vocab": 2048}


def plan_for(cfg: str, n: int) -> dict:
    """Parallel plan per GPU count: C1 FSDP1 -> SP2 -> SP4 -> FSDP2xSP4."""
    if cfg == "c1":
        sp = min(n, 4)
        # 1 GPU holds 7.6B params x 18 B (137 GB) + the 32K-token working set only
        # with full recompute (the paper's setting); from 2 GPUs the per-layer
        # activations fit and recompute=none removes the extra forward.
        return {"dp_replicate": 1, "dp_shard": n // sp, "sp": sp, "ep": 1, "micro_batch": 1,
                "recompute": "full" if n == 1 else "none", "fsdp_prefetch_depth": 1}
    if cfg == "c3":  # FSDP + SP like C1 at 64K tokens per row: recompute below SP4
        sp = min(n, 4)
        return {"dp_replicate": 1, "dp_shard": n // sp, "sp": sp, "ep": 1, "micro_batch": 1,
                "recompute": "full" if sp < 4 else "none", "fsdp_prefetch_depth": 1}
    if cfg == "c4":  # SP over all GPUs (SP8, shard 1); 128K tokens, one row
        # per-layer activations at 128K/sp tokens (~10 GB at SP4, ~5 GB at SP8):
        # keep them from 8 GPUs, recompute below
        return {"dp_replicate": 1, "dp_shard": 1, "sp": n, "ep": 1, "micro_batch": 1,
                "recompute": "none" if n >= 8 else "full", "fsdp_prefetch_depth": 1}
    if cfg == "c2":  # FSDP + EP over all GPUs (FSDP8+EP8)
        # recompute=none keeps attention activations, routing and combined expert
        # outputs (~0.6 GB/layer at 8K tokens); the backward re-sends tokens and
        # redoes gate|up only
        return {"dp_replicate": 1, "dp_shard": n, "sp": 1, "ep": n, "micro_batch": 1,
                "recompute": "none", "fsdp_prefetch_depth": 1,
                "moe_overlap": os.environ.get("OPX_BENCH_MOE_OVERLAP", "1") == "1"}
    sp = 2 if n % 2 == 0 else 1  # C0: FSDP2 x SP2 at 4 GPUs
    return {"dp_replicate": 1, "dp_shard": n // sp, "sp": sp, "ep": 1, "micro_batch": 1,
            "recompute": "full", "fsdp_prefetch_depth": 1}


def model_for(cfg: str, n: int = 8) -> dict:
    arch = dict({"c1": QWEN2_7B, "c0": TINY, "c2": QWEN3_30B_A3B, "c3": QWEN2_7B,
                 "c4": QWEN2_72B_SLICE}[cfg])
    if cfg == "c2" and n < 8:
        # 30B does not fit below 8 GPUs (reference memory model: 235/455 GiB at
        # EP2/EP1); scale the layer count with the GPU count (a layer slice)
        arch["layers"] = 48 * n // 8
    mods = [{"name": "core", "kind": "foundation", "trainable": True, "arch": arch}]
    if cfg == "c3":
        mods.append({"name": "vision", "kind": "encoder", "trainable": False,
                     "tokens_per_item": C3_TOKENS_PER_IMAGE, "arch": dict(QWEN25_VL_VIT)})
    return {"param_dtype_bytes": 2, "modules": mods}


def seq_for(cfg: str) -> int:
    return {"c1": 32768, "c0": 1024, "c2": 8192, "c3": 65536, "c4": 131072}[cfg]


def cluster_for(n: int) -> dict:
    return {"num_nodes": 1, "gpus_per_node": n, "gpu": {"peak_flops": 2.25e15, "hbm_bytes": 180e9},
            "link": {"intra_node_bw": 9e11, "inter_node_bw": 5e10, "intra_latency": 5e-6,
                     "inter_latency": 2e-5}}


def mlp_traffic(cfg: str, T_loc: int):
    """DRAM bytes of one forward MLP node (gate|up + down GEMM) from the committed
    ncu capture at 32768 tokens, scaled linearly to this rank's tokens; None when
    there is no capture for this config."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None
    if cfg != "c1":
        return None
    return t["mlp_node_dram_bytes"] * T_loc / t["tokens"]


def node_key(name: str) -> str:
    """Trace node name -> its kind summed over layers and micro-batches:
    fwd.layer3.m0.qkv_proj -> fwd.qkv_proj, bwd.head.m1 -> bwd.head."""
    import re

    n = re.sub(r"\.m\d+(?=\.|$)", "", name)
    return re.sub(r"^(fwd|bwd)\.layer\d+\.", r"\1.", n)


def nvlink_rates(trace, plan, arch, S):
    """Achieved per-GPU NVLink bytes/s of the all-to-all kernels (bytes that
    leave the rank, (P-1)/P of the payload, comm.cpp:8-22) over their traced
    device time, against 900 GB/s per direction."""
    T = plan["micro_batch"] * S // plan["sp"]
    H, kvw = arch["hidden"], arch["kv_heads"] * arch["head_dim"]
    out = {"peak_GBps_per_direction": 900.0}
    nodes = {}
    for e in trace["traceEvents"]:
        if e.get("tid", 0) != 0 or ".m0." not in e["name"]:
            continue
        key = e["name"].split(".", 1)[0] + "." + e["name"].split(".m0.")[-1]
        nodes.setdefault(key, []).append(e["dur"] * 1e-6)
    sp, ep = plan["sp"], plan.get("ep", 1)
    if sp > 1:
        frac = (sp - 1) / sp
        qkv = T * (H + 2 * kvw) * 2 * frac
        # kernel-only spans: the flag barrier after each exchange is its own
        # node (a2a_wait, rank skew), not counted here
        for key, b in (("fwd.a2a_qkv", qkv), ("fwd.a2a_out", T * H * 2 * frac),
                       ("bwd.a2a_dqkv", qkv)):
            if key in nodes:
                out[key.replace(".", "_") + "_GBps"] = round(b * len(nodes[key]) / sum(nodes[key]) / 1e9, 1)
    if ep > 1 and "moe" in arch:
        frac = (ep - 1) / ep
        b = T * arch["moe"]["top_k"] * H * 2 * frac
        for key in ("fwd.a2a_dispatch", "fwd.a2a_combine", "bwd.a2a_combine_grad", "bwd.a2a_dispatch_grad"):
            if key in nodes:
                # moe_overlap: the dispatch-direction nodes (fwd dispatch, bwd dY
                # dispatch = a2a_combine_grad) span BOTH halves' kernels (half B's
                # is launched first on the side stream and fills the GPU, half A's
                # ends the node); the combine-direction nodes carry half A only
                # (half B's combine runs after its GEMMs)
                dispatch_dir = key in ("fwd.a2a_dispatch", "bwd.a2a_combine_grad")
                bk = b / 2 if plan.get("moe_overlap") and not dispatch_dir else b
                out[key.replace(".", "_") + "_GBps"] = round(bk * len(nodes[key]) / sum(nodes[key]) / 1e9, 1)
    return out


def calibration(trace, plan, model, wl, n, step_s):
    """the reference simulator's constants (compute_efficiency,
    intra-node bandwidth) fitted to this run's trace (paper_2508_02317_b200.calibrate)."""
    try:
        from paper_2508_02317_b200 import calibrate as cal

        c = cal.calibrate(trace, plan, model, wl, cluster_for(n), step_s)
        keep = ("compute_efficiency", "intra_node_bw", "unmodelled_s", "modelled_compute_s")
        out = {k: c[k] for k in keep}
        out["per_kind_efficiency"] = {k: round(v, 3) for k, v in c["per_kind_efficiency"].items()}
        return out
    except Exception as e:  # reporting only
        return {"error": str(e)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"] * 1e12, p.get("bf16_tflops_sustained", p["bf16_tflops"]) * 1e12, \
            p["hbm_gbs"], "measured"
    except Exception:
        return 1.59e15, 1.4e15, 6650.0, "fallback"


def active_layer_params(arch: dict) -> float:
    H, F = arch["hidden"], arch["ffn_dim"]
    kvw = arch["kv_heads"] * arch["head_dim"]
    attn = H * (H + 2 * kvw) + H + H * H + H
    if "moe" in arch:
        m = arch["moe"]
        return attn + H * m["num_experts"] + 3 * H * m["expert_ffn_dim"] * m["top_k"]
    return attn + 3 * H * F


def exact_flops_per_step(arch: dict, batch, T_total: int) -> float:
    """6*N_active,strict per token + exact causal attention 6*L*H*sum(l_i^2)
    (SURVEY.md §8d); N_active,strict excludes the embedding gather."""
    H, L, V = arch["hidden"], arch["layers"], arch["vocab"]
    n_strict = L * active_layer_params(arch) + V * H + H
    sq = 0
    for cu in batch["cu_rows"]:
        for a, b in zip(cu[:-1], cu[1:]):
            sq += (b - a) ** 2
    return 6.0 * n_strict * T_total + 6.0 * L * H * sq


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, dev: int):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a few hundred ms to start: wait for its first row
            # so a short timed region (C2 on 1 GPU: ~0.35 s) still gets samples;
            # rows seen before the region are kept apart
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        self.n0 = len(self.rows)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows[self.n0:] or self.rows
        sm = [float(r[0]) for r in rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower().startswith("active"):
                    reasons.add(n)
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU reference arm / baseline (SURVEY §8d "CPU timing beside it"): the numpy
# oracle switched to fp32 accumulation (all-core BLAS), on
#   (1) the full C0 step (2 layers, H=256, S=1024, FSDP2 x SP2 simulated ranks,
#       global batch 2) -- measured tokens/s;
#   (2) one transformer block (fwd+bwd) of the benched config at its true
#       widths (MoE keeps E and top-k) with S = 2048 packed tokens -- its
#       FLOP rate, extrapolated to the config's exact step FLOPs.
# ---------------------------------------------------------------------------
CPU_BLOCK_SEQ = 2048


def _cpu_setup():
    import numpy as np

    from oracle import model as om

    om.set_accumulate(np.float32)
    return np, om


def cpu_c0_step() -> dict:
    np, om = _cpu_setup()
    from paper_2508_02317_b200.runtime import synthetic_batch

    m = model_for("c0")
    a = om.Arch.from_model_json(m)
    P = om.init_params(a, 2508)
    b = synthetic_batch(a.vocab, seq_for("c0"), 2, seed=2508)
    plan = {"dp_replicate": 1, "dp_shard": 2, "sp": 2, "micro_batch": 1}
    t0 = time.perf_counter()
    _, G = om.simulate_ranks(a, P, b, plan, round_operands=False)
    om.adamw(P, G, {}, 1)
    dt = time.perf_counter() - t0
    return {"tokens_per_s": 2 * seq_for("c0") / dt, "seconds": dt}


class CpuBlock:
    """One block of `cfg` at its true widths on CPU_BLOCK_SEQ packed tokens."""

    def __init__(self, cfg: str):
        np, om = _cpu_setup()
        from paper_2508_02317_b200.runtime import synthetic_batch

        self.np, self.om, self.cfg = np, om, cfg
        full = dict(model_for(cfg)["modules"][0]["arch"])
        blk = dict(full, layers=1, vocab=512)  # the head is a small V=512 one
        self.arch = om.Arch.from_model_json({"modules": [{"kind": "foundation", "arch": blk}]})
        self.P = om.init_params(self.arch, 2508)
        self.b = synthetic_batch(512, CPU_BLOCK_SEQ, 1, seed=2508)
        self.flops = exact_flops_per_step(blk, self.b, CPU_BLOCK_SEQ)
        self.full = full

    def run(self) -> float:
        """Seconds for one fwd+bwd of the block sample."""
        b = self.b
        t0 = time.perf_counter()
        st = self.om.Step(self.arch, self.P, round_operands=False)
        st.run(b["ids"][0], b["labels"][0], b["pos"][0], self.np.array(b["cu_rows"][0]), CPU_BLOCK_SEQ)
        return time.perf_counter() - t0

    def tokens_per_s(self, dt: float, step_flops: float, step_tokens: int) -> float:
        """The config's step on this host at the block's FLOP rate (extrapolated)."""
        return step_tokens / (step_flops / (self.flops / dt))


def cpu_full_step(cfg: str, n: int = 1):
    """Exact FLOPs and tokens of the benched step (the GPU arm's batch)."""
    from paper_2508_02317_b200.runtime import synthetic_batch

    plan = plan_for(cfg, n)
    arch = model_for(cfg, n)["modules"][0]["arch"]
    rows = plan["dp_replicate"] * plan["dp_shard"] * plan["micro_batch"]
    S = seq_for(cfg)
    batch = synthetic_batch(arch["vocab"], S, rows, seed=2508)
    return exact_flops_per_step(arch, batch, rows * S), rows * S


def cpu_reference(cfg: str, n: int = 1) -> dict:
    """The cpu_baseline object: C0 step + one timed block of `cfg`."""
    c0 = cpu_c0_step()
    blk = CpuBlock(cfg)
    dt = blk.run()
    step_flops, step_tokens = cpu_full_step(cfg, n)
    v = blk.tokens_per_s(dt, step_flops, step_tokens)
    H, F = blk.full["hidden"], blk.full["ffn_dim"]
    return {"value": v, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"numpy oracle, fp32 accumulation, {os.cpu_count()} host threads (BLAS): "
                      f"(1) full C0 step (FSDP2xSP2 simulated, 2x1024 tokens) {c0['seconds']:.2f} s = "
                      f"{c0['tokens_per_s']:.0f} tokens/s measured; (2) one {cfg} block (H={H}, "
                      f"ffn={F}) fwd+bwd on {CPU_BLOCK_SEQ} packed tokens in {dt:.2f} s = "
                      f"{blk.flops / dt / 1e9:.1f} GFLOP/s, extrapolated to the {cfg} step's exact "
                      f"{step_flops:.3e} FLOP ({step_tokens} tokens)",
            "gflops": blk.flops / dt / 1e9, "c0_step_tokens_per_s": c0["tokens_per_s"],
            "extrapolated": True}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c1")
    ap.add_argument("--impl", default="opx", choices=["opx", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # also a single-sample row (l = S), where the exact FLOPs equal
    # the reference formula's full causal S (diagnostic line, not the default)
    ap.add_argument("--single-sample", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.gpus
    if world != n and world != 1:
        n = world
    cfg = args.config

    if args.impl == "reference":
        if rank != 0:
            return
        # one timed block sample per step (each its own measurement), after
        # one untimed warm-up sample; value = median extrapolated tokens/s
        c0 = cpu_c0_step()
        blk = CpuBlock(cfg)
        step_flops, step_tokens = cpu_full_step(cfg, n)
        warm = min(args.warmup, 1)
        for _ in range(warm):
            blk.run()
        vals, secs = [], []
        for _ in range(max(args.steps, 1)):
            dt = blk.run()
            secs.append(dt)
            vals.append(blk.tokens_per_s(dt, step_flops, step_tokens))
        v = statistics.median(vals)
        sample = (f"numpy oracle, fp32 accumulation, {os.cpu_count()} host threads (BLAS); per step one "
                  f"{cfg} block fwd+bwd at true widths on {CPU_BLOCK_SEQ} packed tokens "
                  f"(median {statistics.median(secs):.2f} s, {blk.flops / statistics.median(secs) / 1e9:.1f} "
                  f"GFLOP/s) extrapolated to the {cfg} step's exact {step_flops:.3e} FLOP; full C0 step "
                  f"measured at {c0['tokens_per_s']:.0f} tokens/s")
        line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": n, "steps": len(vals),
                "warmup": warm, "ms_per_step": statistics.median(secs) * 1e3,
                "higher_is_better": True, "impl": "reference",
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": cfg, "model": "qwen2-7b-shaped" if cfg == "c1" else cfg,
                           "seq_len": seq_for(cfg)},
                "step_values": vals,
                "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                                 "sample": sample, "c0_step_tokens_per_s": c0["tokens_per_s"],
                                 "extrapolated": True},
                "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import numpy as np
    import torch

    dist = None
    if world > 1:
        import torch.distributed as td

        td.init_process_group("gloo")
        dist = td
    from paper_2508_02317_b200.runtime import Session, local_slice, synthetic_batch

    plan = plan_for(cfg, n)
    model = model_for(cfg, n)
    arch = model["modules"][0]["arch"]
    S = seq_for(cfg)
    # diagnostics only (profiling a rank-sized slice on one GPU); the driver's
    # bench lines never set these
    if os.environ.get("OPX_BENCH_SEQ"):
        S = int(os.environ["OPX_BENCH_SEQ"])
    if os.environ.get("OPX_BENCH_RECOMPUTE"):
        plan["recompute"] = os.environ["OPX_BENCH_RECOMPUTE"]
    if os.environ.get("OPX_BENCH_ASYNC"):  # async_ulysses: exchanges fused into the GEMM epilogues
        plan["async_ulysses"] = os.environ["OPX_BENCH_ASYNC"] == "1"
    rows = plan["dp_replicate"] * plan["dp_shard"] * plan["micro_batch"]
    wl = {"seq_len": S, "micro_batch": plan["micro_batch"], "global_batch": rows}
    if cfg == "c3":  # WorkloadSpec.modality_mix (config_io.cpp:144-147)
        wl["modality_mix"] = {"vision": C3_IMAGE_MIX, "text": 1.0 - C3_IMAGE_MIX}
    ex = {"seed": 2508, "lr": 1e-4, "betas": [0.9, 0.95], "eps": 1e-8, "weight_decay": 0.1,
          "trace": True}
    sess = Session(cluster_for(n), model, wl, plan, ex, rank=rank, device=local, dist=dist)
    sess.init_weights(2508)
    batch = synthetic_batch(arch["vocab"], S, rows, seed=2508, single_sample=args.single_sample)
    enc = next((m for m in model["modules"] if m["kind"] == "encoder"), None)
    if enc:
        from paper_2508_02317_b200.runtime import rank_coords, synthetic_images

        # images per row from the mix: mix_fraction * tokens (step_graph.cpp:147)
        per_row = int(round(wl["modality_mix"][enc["name"]] * S / enc["tokens_per_item"]))
        synthetic_images(batch, enc["tokens_per_item"], enc["arch"]["vocab"], per_row,
                         placeholder=arch["vocab"] - 1)
    ids, labels, pos, cu, n_valid = local_slice(batch, rank, plan)
    # opx_step_load_batch uploads ids, labels, positions and, per token, the
    # start / end of its sample (computed on the host from cu_seqlens)
    h2d = ids.nbytes + labels.nbytes + 3 * pos.nbytes
    n_img = n_patch_local = 0
    if enc:  # this rank's dp rows' items; it uploads the patches of items j % sp == its SP index
        rep_i, sh_i, sp_i = rank_coords(rank, plan)
        dp_i = rep_i * plan["dp_shard"] + sh_i
        img = batch["img"]
        mine = np.nonzero((img["row"] >= dp_i * plan["micro_batch"]) &
                          (img["row"] < (dp_i + 1) * plan["micro_batch"]))[0]
        n_img = len(mine)
        n_patch_local = len(mine[sp_i::plan["sp"]]) * 4 * enc["tokens_per_item"]
        h2d += n_patch_local * enc["arch"]["vocab"] * 2 + n_img * 8 + n_img
    sess.load(batch)
    for _ in range(args.warmup):
        sess.run()
    times, walls, launches, losses, enq = [], [], 0, [], []
    kept = 0
    with Clocks(local) as clk:
        if dist:  # after every rank's clock sampler is up
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            sess.load(batch)          # H2D of this step's inputs (host buffers)
            r = sess.run()            # device-timed step + D2H of the loss
            walls.append(time.perf_counter() - t0)
            times.append(r.step_time_s)
            launches += r.launches
            enq.append(r.enqueue_s)
            kept = int(r.kept_layers)
            losses.append(r.loss)
    trace = sess.trace()
    if os.environ.get("OPX_TRACE_DIR"):  # diagnostics: every rank's compute-stream node totals
        tot_r = {}
        for e in trace["traceEvents"]:
            if e.get("tid", 0) == 0:
                k = e["name"].split(".m0.")[-1] if ".m0." in e["name"] else e["name"]
                k = e["name"].split(".", 1)[0] + "." + k
                tot_r[k] = round(tot_r.get(k, 0.0) + e["dur"] * 1e-3, 3)
        with open(os.path.join(os.environ["OPX_TRACE_DIR"], f"nodes_rank{rank}.json"), "w") as f:
            json.dump(tot_r, f, indent=0, sort_keys=True)
    if dist:
        import torch.distributed as td

        t = torch.tensor([max(times), statistics.mean(times), statistics.mean(walls)], dtype=torch.float64)
        td.all_reduce(t, op=td.ReduceOp.MAX)
        t_max, t_mean, w_mean = t.tolist()
    else:
        t_max, t_mean, w_mean = max(times), statistics.mean(times), statistics.mean(walls)
    if rank != 0:
        sess.close()
        return

    tokens_step = rows * S
    value = tokens_step / t_mean
    peak, peak_sus, hbm, peak_kind = peaks()
    fpt_ref = 6.0 * (arch["layers"] * active_layer_params(arch) + 2 * arch["vocab"] * arch["hidden"]
                     + arch["hidden"]) + 6.0 * arch["layers"] * arch["hidden"] * S
    exact = exact_flops_per_step(arch, batch, tokens_step)
    enc_line = None
    if enc:  # frozen encoder forward: 2 * params per patch + bidirectional attention
        ea = enc["arch"]
        He, Fe, nb = ea["hidden"], ea["ffn_dim"], ea["layers"]
        Wq = ea["heads"] * ea["head_dim"]
        P_item = 4 * enc["tokens_per_item"]
        blk = He * 3 * Wq + Wq * He + 3 * He * Fe
        per_patch = 2.0 * (nb * blk + ea["vocab"] * He + 4 * He * He + He * arch["hidden"])
        n_items_all = len(batch["img"]["row"])
        enc_flops = n_items_all * P_item * (per_patch + nb * 4.0 * Wq * P_item)
        exact += enc_flops
        fpt_ref += enc_flops / tokens_step
        en = [e["dur"] for e in trace["traceEvents"] if e["name"] == f"encoder.{enc['name']}.m0"]
        sc = [e["dur"] for e in trace["traceEvents"] if e["name"] == f"scatter.{enc['name']}.m0"]
        enc_line = {"items_per_step": n_items_all, "patches_per_item": P_item,
                    "image_token_fraction": n_items_all * enc["tokens_per_item"] / tokens_step,
                    "encoder_ms": statistics.mean(en) / 1e3 if en else None,
                    "scatter_ms": statistics.mean(sc) / 1e3 if sc else None,
                    "encoder_tflops_per_gpu": (enc_flops / n) / (statistics.mean(en) * 1e-6) / 1e12 if en else None,
                    "model": "qwen2.5-vl-7b-shaped ViT, frozen (fwd only; 2-D RoPE, 112 px windows, "
                             "full attention in blocks 7/15/23/31)"}
    per_gpu = value / n
    # roofline: dominant kernel = the forward MLP block (gate|up GEMM + SwiGLU
    # epilogue + down GEMM), 6*T*H*F algorithmic FLOPs per layer-call
    T_loc = S // plan["sp"] * plan["micro_batch"]
    mlp = [e["dur"] for e in trace["traceEvents"] if e["name"].startswith("fwd.layer") and e["name"].endswith(".mlp")]
    node_s = statistics.mean(mlp) * 1e-6 if mlp else float("nan")
    mlp_flops = 6.0 * T_loc * arch["hidden"] * arch["ffn_dim"]
    if "moe" in arch:  # MoE block node: router + dispatch + experts + combine
        mlp = [e["dur"] for e in trace["traceEvents"] if e["name"].startswith("fwd.layer") and e["name"].endswith(".moe")]
        node_s = statistics.mean(mlp) * 1e-6 if mlp else float("nan")
        m = arch["moe"]
        mlp_flops = 6.0 * T_loc * arch["hidden"] * m["expert_ffn_dim"] * m["top_k"]
    achieved = mlp_flops / node_s
    # attention kernels (the kernels VERDICT r1 named furthest below roofline):
    # exact causal varlen FLOPs of one layer's core on this rank's heads
    # (4 d h sum(l^2)/2 forward, 2.5x that backward) / mean node time
    sq_all = sum((b - a) ** 2 for cu in batch["cu_rows"][:plan["micro_batch"]] for a, b in zip(cu[:-1], cu[1:]))
    hq_loc = arch["heads"] // plan["sp"]
    attn_fwd_flops = 4.0 * arch["head_dim"] * hq_loc * sq_all / 2.0
    attn = {}
    for d_, mult in (("fwd", 1.0), ("bwd", 2.5)):
        ts = [e["dur"] for e in trace["traceEvents"]
              if e["name"].startswith(d_ + ".layer") and e["name"].endswith(".attn_core")]
        if ts:
            ach = attn_fwd_flops * mult / (statistics.mean(ts) * 1e-6)
            attn[d_] = {"achieved": ach / 1e12, "peak": peak_sus / 1e12, "unit": "TFLOP/s",
                        "frac": ach / peak_sus, "frac_of_burst": ach / peak,
                        "launch_ms": statistics.mean(ts) * 1e-3, "flops_per_launch": attn_fwd_flops * mult}
    share = {}
    for e in trace["traceEvents"]:
        if e["tid"] != 0 or node_key(e["name"]) in ("fwd.moe", "bwd.moe"):  # parent span of the MoE sub-nodes
            continue
        key = node_key(e["name"])
        share[key] = share.get(key, 0.0) + e["dur"] * 1e-6
    tot = sum(share.values()) or 1.0
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_mean * 1e3, "ms_per_step_max": t_max * 1e3,
        "higher_is_better": True, "scaling": "strong" if n <= 4 else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "tokens_per_s_per_gpu": per_gpu,
        "mfu_ref": per_gpu * fpt_ref / peak, "mfu_ref_datasheet": per_gpu * fpt_ref / 2.25e15,
        "mfu_exact": exact / t_mean / n / peak, "model_flops_per_token_ref": fpt_ref,
        "config": {"workload": cfg, "model": {"c1": "qwen2-7b-shaped (random init)",
                                              "c2": f"qwen3-30b-a3b-shaped, {arch['layers']} layers (random init)",
                                              "c3": "qwen2.5-vl-7b-shaped: qwen2-7b backbone + frozen ViT (random init)",
                                              "c4": "qwen2-72b-shaped 8-layer slice (random init)"}.get(cfg, cfg),
                   "global_batch": rows, "seq_len": S, "tokens_per_step": tokens_step,
                   "parallelism": f"fsdp{plan['dp_shard']}xsp{plan['sp']}",
                   "recompute": plan["recompute"], "kept_layers": kept,
                   "async_ulysses": bool(plan.get("async_ulysses", False)),
                   "packing": "one sample per row" if args.single_sample else "lognormal varlen, 0 padding",
                   "l2": "inputs+weights >> 126 MB L2 (no flush needed)",
                   "peak_kind": peak_kind},
        "loss": losses[-1],
        "e2e": {"value": tokens_step / w_mean, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 4},
        "gpu_launches": launches,
        # the node is timed inside a long step -> the sustained measured peak
        "roofline": {"bound": "tensor", "kernel": "fwd MLP block (tcgen05 gate|up GEMM+SwiGLU, down GEMM)",
                     "achieved": achieved / 1e12, "peak": peak_sus / 1e12, "unit": "TFLOP/s",
                     "frac": achieved / peak_sus, "peak_kind": f"{peak_kind} sustained",
                     "traffic": mlp_traffic(cfg, T_loc),
                     "traffic_unit": "bytes per node (ncu dram__bytes_read+write, profiles/ncu_traffic.json)",
                     "flops_per_launch": mlp_flops, "launch_ms": node_s * 1e3,
                     "frac_of_burst": achieved / peak,
                     "note": "peak = the driver's sustained figure (cuBLAS bf16 8192^3 back to back under "
                             "the power cap); the node's tcgen05 GEMMs can exceed it (frac > 1), "
                             "frac_of_burst is against the burst figure"},
        "roofline_attention": attn,
        "phase_share": {k: round(v / tot, 4) for k, v in sorted(share.items(), key=lambda kv: -kv[1])[:16]},
        "node_ms": {k: round(v * 1e3, 2) for k, v in sorted(share.items(), key=lambda kv: -kv[1])[:24]},
        "clocks": clk.summary(),
        "calibration": calibration(trace, plan, model, wl, n, t_mean),
        "nvlink": nvlink_rates(trace, plan, arch, S),
        "host_enqueue_ms": statistics.mean(enq) * 1e3, "host_cpus": os.cpu_count(),
        "hbm_free_gb": torch.cuda.mem_get_info(local)[0] / 1e9,
    }
    if enc_line:
        line["encoder"] = enc_line
    if not args.no_cpu_baseline and n == 1:
        ref = cpu_reference(cfg, n)
        line["cpu_baseline"] = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                     "c0_step_tokens_per_s", "extrapolated")}
    print(json.dumps(line), flush=True)
    sess.close()


if __name__ == "__main__":
    main()
