"""StepReport's exposed-comm figure on CPU: libopx's
opx_exposed_comm_seconds -- the function the step applies to its measured node
intervals -- against the reference's report() (simulator.cpp:71-130, compiled
from /root/reference into oracle/_ref) on random timelines, and against known
answers.  No GPU."""
import ctypes
import os
import random

import numpy as np
import pytest

from paper_2508_02317_b200 import lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libomniplan_ref.so")


def _arr(xs):
    return (ctypes.c_double * max(1, len(xs)))(*xs)


def exposed(compute, comm):
    cs, ce = [a for a, _ in compute], [b for _, b in compute]
    ms, me = [a for a, _ in comm], [b for _, b in comm]
    return lib().opx_exposed_comm_seconds(_arr(cs), _arr(ce), len(cs), _arr(ms), _arr(me), len(ms))


def test_known_answers():
    assert exposed([], []) == 0.0
    assert exposed([], [(1.0, 4.0)]) == pytest.approx(3.0)
    assert exposed([(0.0, 10.0)], [(2.0, 5.0)]) == 0.0                  # fully hidden
    assert exposed([(2.0, 5.0)], [(0.0, 10.0)]) == pytest.approx(7.0)   # compute inside comm
    assert exposed([(0.0, 3.0), (6.0, 8.0)], [(1.0, 7.0)]) == pytest.approx(3.0)
    # a compute interval nested in an earlier one (two streams) changes nothing
    assert exposed([(0.0, 5.0), (1.0, 2.0)], [(1.5, 7.0)]) == pytest.approx(2.0)
    # overlapping comm intervals are each charged (the reference sums per interval)
    assert exposed([], [(0.0, 2.0), (1.0, 3.0)]) == pytest.approx(4.0)


def _timeline(rng, n):
    ivs = []
    for _ in range(n):
        a = rng.uniform(0, 100)
        ivs.append((a, a + rng.expovariate(0.2), rng.random() < 0.4))
    return ivs


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built (reference absent)")
def test_matches_compiled_reference_report():
    ref = ctypes.CDLL(REF_SO)
    ref.ref_exposed_comm.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p]
    rng = random.Random(7)
    for trial in range(400):
        ivs = _timeline(rng, rng.randrange(0, 40))
        n = len(ivs)
        st = np.array([a for a, _, _ in ivs] or [0.0])
        en = np.array([b for _, b, _ in ivs] or [0.0])
        ch = np.array([int(c) for _, _, c in ivs] or [0], dtype=np.int32)
        makespan = float(max(en.max(), 1.0))
        out = ctypes.c_double()
        assert ref.ref_exposed_comm(st.ctypes.data, en.ctypes.data, ch.ctypes.data, n, makespan,
                                    ctypes.byref(out)) == 0
        mine = exposed([(a, b) for a, b, c in ivs if not c], [(a, b) for a, b, c in ivs if c])
        assert mine == pytest.approx(out.value, rel=1e-12, abs=1e-9), (trial, ivs)
