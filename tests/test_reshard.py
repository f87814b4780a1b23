"""Checkpoint resharding: libopx's copy plan against the
reference's make_plan (compiled from /root/reference into oracle/_ref) and its
own known answers (test_reshard.cpp:81-94), plus round trips of opx checkpoint
directories through paper_2508_02317_b200.checkpoint.  CPU only."""
import ctypes
import json
import os
import random

import numpy as np
import pytest

from paper_2508_02317_b200 import checkpoint

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libomniplan_ref.so")


def test_known_answer_10_elements_2_to_4():
    # test_reshard.cpp:81-94
    p = checkpoint.reshard_plan(10, 2, 4, 0, 0)
    assert p["ops"] == [[0, 0, 0, 0, 3], [0, 3, 1, 0, 2], [1, 0, 1, 2, 1], [1, 1, 2, 0, 3],
                        [1, 4, 3, 0, 1]]


def test_identity_and_padded_layout():
    assert checkpoint.reshard_plan(10, 1, 1, 0, 0)["ops"] == [[0, 0, 0, 0, 10]]
    # executor layout: 1000 elements over 3 shards padded to 64*3 -> chunk 384
    p = checkpoint.reshard_plan(1000, 3, 2, 64, 64)
    assert p["src_chunk"] == 384 and p["dst_chunk"] == 512
    assert sum(op[4] for op in p["ops"]) == 1000


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (reference absent)")
def test_plan_matches_compiled_reference():
    ref = ctypes.CDLL(REF_SO)
    ref.ref_reshard_plan.argtypes = [ctypes.c_longlong] * 3 + [ctypes.c_char_p, ctypes.c_size_t]
    rng = random.Random(11)
    buf = ctypes.create_string_buffer(1 << 16)
    for _ in range(300):
        n = rng.randrange(0, 5000)
        a, b = rng.randrange(1, 17), rng.randrange(1, 17)
        assert ref.ref_reshard_plan(n, a, b, buf, len(buf)) == 0
        r = json.loads(buf.value.decode())
        if n == 0:
            continue
        mine = checkpoint.reshard_plan(n, a, b, 0, 0)
        assert mine["ops"] == r["ops"], (n, a, b)
        assert r["violations"] == []


def _fake_ckpt(path, units, parts, seed=0):
    rng = np.random.default_rng(seed)
    man = {"format": "opx-fsdp-shards-1", "step": 3, "align": 64, "plan": {"dp_replicate": 1,
           "dp_shard": parts, "sp": 1, "ep": 1}, "units": []}
    flats = {}
    for name, numel in units:
        flat = rng.standard_normal((3, numel)).astype(np.float32)
        flats[name] = flat
        c = checkpoint.reshard_plan(numel, parts, parts)["src_chunk"]
        os.makedirs(os.path.join(path, name))
        for r in range(parts):
            b, e = min(r * c, numel), min((r + 1) * c, numel)
            np.ascontiguousarray(flat[:, b:e]).tofile(os.path.join(path, name, f"shard{r}.bin"))
        man["units"].append({"name": name, "numel": numel, "parts": parts, "chunk": c})
    with open(os.path.join(path, "manifest.json"), "w") as f:
        json.dump(man, f)
    return flats


def _assemble(path):
    man = json.load(open(os.path.join(path, "manifest.json")))
    out = {}
    for u in man["units"]:
        parts = [np.fromfile(os.path.join(path, u["name"], f"shard{r}.bin"), np.float32).reshape(3, -1)
                 for r in range(u["parts"])]
        out[u["name"]] = np.concatenate(parts, axis=1)
    return out, man


@pytest.mark.parametrize("a,b", [(3, 5), (4, 1), (1, 8), (8, 6)])
def test_checkpoint_round_trip(tmp_path, a, b):
    units = [("head", 4099), ("layer0", 70001), ("layer1", 64)]
    flats = _fake_ckpt(tmp_path / "a", units, a)
    checkpoint.reshard(str(tmp_path / "a"), str(tmp_path / "b"), dp_shard=b, sp=1)
    got, man = _assemble(tmp_path / "b")
    assert all(u["parts"] == b for u in man["units"])
    for name, _ in units:
        assert np.array_equal(got[name], flats[name])
    checkpoint.reshard(str(tmp_path / "b"), str(tmp_path / "c"), dp_shard=a, sp=1)
    for name, _ in units:
        for r in range(a):
            x = np.fromfile(tmp_path / "a" / name / f"shard{r}.bin", np.float32)
            y = np.fromfile(tmp_path / "c" / name / f"shard{r}.bin", np.float32)
            assert np.array_equal(x, y)
