"""Sequence packing: libopx's packer against the reference's
known answers (test_packing.cpp:37-153) and against the reference packer
itself (compiled into oracle/_ref) on random corpora; the executor batch
built from a packing.  CPU only."""
import ctypes
import json
import os
import random

import numpy as np
import pytest

from paper_2508_02317_b200 import OpxError
from paper_2508_02317_b200 import packing as pk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libomniplan_ref.so")


def lens_of(row):
    return [e[2] for e in row["entries"]]


def test_known_answers():
    r = pk.pack([5, 4, 3, 2], 8)
    assert [lens_of(x) for x in r["rows"]] == [[5, 3], [4, 2]]
    assert r["padding_ratio"] == pytest.approx(0.125)
    assert pk.pack([], 8) == {"rows": [], "padding_ratio": 0.0}
    assert pk.pack([8], 8)["padding_ratio"] == 0.0
    assert pk.pack([1], 8, pk.ARRIVAL)["padding_ratio"] == pytest.approx(0.875)
    a = pk.pack([2, 7, 3], 8, pk.ARRIVAL)["rows"]
    assert [e[0] for e in a[0]["entries"]] == [0, 2] and a[1]["entries"][0][0] == 1
    t = pk.pack([4, 4, 4], 8)["rows"]
    assert [e[0] for e in t[0]["entries"]] == [0, 1] and t[1]["entries"][0][0] == 2
    for row in pk.pack([5, 4, 3, 2, 1], 8)["rows"]:
        b = row["boundaries"]
        assert b[0] == 0 and all(b[i + 1] - b[i] == e[2] and e[1] == b[i] for i, e in enumerate(row["entries"]))
    with pytest.raises(OpxError, match="length 9 > target 8"):
        pk.pack([3, 9, 2], 8)


def test_streaming_packer():
    p = pk.StreamingPacker(8, pk.FFD, buffer_factor=2)
    assert p.push(0, 5) == [] and p.push(1, 5) == []
    assert p.push(2, 6) and p.buffered_tokens == 0 and p.flush() == []
    assert p.push(3, 3) == []
    rest = p.flush()
    assert len(rest) == 1 and rest[0]["entries"][0][0] == 3


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (reference absent)")
@pytest.mark.parametrize("policy", [pk.FFD, pk.ARRIVAL])
def test_matches_compiled_reference(policy):
    ref = ctypes.CDLL(REF_SO)
    ref.ref_pack.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_int,
                             ctypes.c_char_p, ctypes.c_size_t]
    rng = random.Random(7 + policy)
    buf = ctypes.create_string_buffer(1 << 20)
    for _ in range(300):
        target = rng.randrange(16, 65)
        lens = [rng.randrange(1, target + 1) for _ in range(rng.randrange(1, 120))]
        arr = np.array(lens, np.int64)
        assert ref.ref_pack(arr.ctypes.data, len(lens), target, policy, buf, len(buf)) == 0
        assert pk.pack(lens, target, policy) == json.loads(buf.value.decode())


def test_packed_batch_layout():
    rng = np.random.default_rng(0)
    samples = [rng.integers(0, 100, n) for n in (500, 300, 700, 120, 64, 900)]
    batch, rep = pk.packed_batch(samples, 1024, rows=3)
    assert batch["ids"].shape == (3, 1024)
    for r, cu in enumerate(batch["cu_rows"]):
        assert cu[0] == 0 and cu[-1] == 1024 and all(b > a for a, b in zip(cu, cu[1:]))
        for a, b in zip(cu, cu[1:]):
            assert np.array_equal(batch["pos"][r, a:b], np.arange(b - a))
            assert batch["labels"][r, b - 1] == pk.IGNORE
    n_valid = sum(len(s) - 1 for s in samples)
    assert int((batch["labels"] >= 0).sum()) == n_valid
    with pytest.raises(ValueError):
        pk.packed_batch(samples, 1024, rows=2)
