"""INTEGRATION.md section 1 compiled and run: tools/integration/omniplan_run.cpp
is built (oracle/Makefile) against the reference's own headers and the
reference library compiled from its sources, linked with libopx.so.  On CPU the
plan path runs (both validators must agree, the reference simulates); on a GPU
the same binary executes the step through the C ABI and serialises the
measured report with the reference's to_json(StepReport)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "omniplan_run")
REF = "/root/reference/proj/configs"
REPORT_KEYS = {"step_time_s", "throughput_tokens_per_s_per_gpu", "mfu", "exposed_comm_fraction",
               "model_flops_per_token", "phase_breakdown"}


def _run(args):
    p = subprocess.run([BIN] + args, capture_output=True, text=True, timeout=600)
    return p.returncode, (json.loads(p.stdout) if p.stdout.strip() else None), p.stderr


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference configs absent")
def test_cmd_run_plan_path_against_reference():
    subprocess.check_call(["make", "-s"], cwd=os.path.join(ROOT, "oracle"))
    c8, m7, moe, w8 = (os.path.join(REF, f) for f in
                       ("cluster-8x80g.json", "dense-7b.json", "moe-30b.json", "workload-8k.json"))
    rc, out, err = _run([c8, m7, w8, "--sp", "4", "--plan-only"])
    assert rc == 0, err
    assert out["validate"]["reference"] == out["validate"]["opx"] == []
    assert set(out["simulated"]) == REPORT_KEYS
    # invalid plans: same codes from both validators, exit 3 (cli.hpp kExitPlanInvalid)
    rc, out, err = _run([c8, m7, w8, "--sp", "8", "--plan-only"])
    assert rc == 3 and out["validate"]["reference"] == out["validate"]["opx"]
    assert "kv_head_divisibility" in out["validate"]["opx"]
    rc, out, err = _run([c8, moe, w8, "--ep", "8", "--plan-only"])
    assert rc == 0, err
    rc, out, err = _run([c8, moe, w8, "--ep", "3", "--plan-only"])
    assert rc == 3 and out["validate"]["reference"] == out["validate"]["opx"]


def _tiny(tmp):
    cluster = {"num_nodes": 1, "gpus_per_node": 1, "gpu": {"peak_flops": 2.25e15, "hbm_bytes": 180e9},
               "link": {"intra_node_bw": 9e11, "inter_node_bw": 5e10, "intra_latency": 5e-6,
                        "inter_latency": 2e-5}}
    model = {"param_dtype_bytes": 2, "modules": [{"name": "core", "kind": "foundation", "trainable": True,
             "arch": {"layers": 2, "hidden": 512, "heads": 4, "kv_heads": 2, "head_dim": 128,
                      "ffn_dim": 1024, "vocab": 2048}}]}
    workload = {"seq_len": 1024, "micro_batch": 1, "global_batch": 2}
    paths = []
    for name, obj in (("cluster", cluster), ("model", model), ("workload", workload)):
        p = os.path.join(tmp, name + ".json")
        with open(p, "w") as f:
            json.dump(obj, f)
        paths.append(p)
    return paths


@pytest.mark.gpu
def test_cmd_run_executes_and_reports_through_reference_to_json(tmp_path):
    if not os.path.exists(BIN):
        pytest.skip("omniplan_run not built (needs the reference sources at build time)")
    rc, out, err = _run(_tiny(str(tmp_path)) + ["--steps", "2"])
    assert rc == 0, err
    m = out["measured"]
    assert set(m) == REPORT_KEYS
    assert m["step_time_s"] > 0 and 0 < m["mfu"] < 1
    # global_batch 2 = 2 micro-batches of 1 row: gradient accumulation path
    assert m["throughput_tokens_per_s_per_gpu"] == pytest.approx(2 * 1024 / m["step_time_s"], rel=1e-6)
    assert {"fwd.layer0", "bwd.layer1", "fwd.head", "bwd.head", "optimizer"} <= set(m["phase_breakdown"])
    assert out["loss"] == out["loss"] and out["loss"] > 0
