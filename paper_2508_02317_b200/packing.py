"""Sequence packing -> the step's packed varlen batch.

``pack`` binds ``opx_pack`` (libopx, restating the reference's first-fit
packer, packing.cpp:10-83); ``StreamingPacker`` mirrors packing.hpp:58-75;
``packed_batch`` turns token lists into the executor's input (ids, labels
shifted within each sample, positions reset per sample, per-row cu_seqlens
boundaries).  A row that FFD leaves short gets one trailing padding segment
(pad token 0, labels ignored) so every row is exactly S tokens and the
boundaries end at S, as ``opx_step_load_batch`` requires.
"""
from __future__ import annotations

import ctypes
import json

import numpy as np

from . import check, lib

FFD, ARRIVAL = 0, 1
IGNORE = -100


def pack(lengths, target: int, policy: int = FFD, ids=None) -> dict:
    """{"rows": [{"capacity", "entries": [[id, offset, length]...], "boundaries"}],
    "padding_ratio"} for samples of the given lengths."""
    n = len(lengths)
    L = np.ascontiguousarray(np.asarray(lengths, dtype=np.int64))
    I = None if ids is None else np.ascontiguousarray(np.asarray(ids, dtype=np.int64))
    cap = 4096 + 64 * n
    buf = ctypes.create_string_buffer(cap)
    check(lib().opx_pack(None if I is None else I.ctypes.data_as(ctypes.c_void_p),
                         L.ctypes.data_as(ctypes.c_void_p), n, int(target), int(policy), buf, cap))
    return json.loads(buf.value.decode())


class StreamingPacker:
    """Buffers samples and packs once buffer_factor * target tokens are held
    (packing.hpp:58-75)."""

    def __init__(self, target: int, policy: int = FFD, buffer_factor: int = 4):
        self.target, self.policy, self.factor = target, policy, buffer_factor
        self._ids, self._lens, self.buffered_tokens = [], [], 0

    def push(self, sample_id: int, length: int):
        self._ids.append(sample_id)
        self._lens.append(length)
        self.buffered_tokens += length
        return self.flush() if self.buffered_tokens >= self.factor * self.target else []

    def flush(self):
        if not self._ids:
            return []
        rows = pack(self._lens, self.target, self.policy, self._ids)["rows"]
        self._ids, self._lens, self.buffered_tokens = [], [], 0
        return rows


def packed_batch(samples, S: int, policy: int = FFD, rows: int | None = None):
    """samples: list of int token arrays.  Returns the executor batch dict
    (ids/labels/pos [rows, S] int32, cu_rows) plus the packing report.  With
    ``rows`` set, the packing must fit in that many rows (empty rows become one
    padding segment each)."""
    res = pack([len(s) for s in samples], S, policy)
    prow = res["rows"]
    nrows = len(prow) if rows is None else rows
    if len(prow) > nrows:
        raise ValueError(f"{len(samples)} samples need {len(prow)} rows of {S}, only {nrows} given")
    ids = np.zeros((nrows, S), np.int32)
    labels = np.full((nrows, S), IGNORE, np.int32)
    pos = np.zeros((nrows, S), np.int32)
    cu_rows = []
    for r in range(nrows):
        cu = [0]
        for sid, off, ln in (prow[r]["entries"] if r < len(prow) else []):
            tok = np.asarray(samples[sid], np.int32)
            ids[r, off:off + ln] = tok
            labels[r, off:off + ln - 1] = tok[1:]
            pos[r, off:off + ln] = np.arange(ln)
            cu.append(off + ln)
        if cu[-1] < S:  # padding segment: its own attention span, no loss
            pos[r, cu[-1]:] = np.arange(S - cu[-1])
            cu.append(S)
        cu_rows.append(cu)
    return {"ids": ids, "labels": labels, "pos": pos, "cu_rows": cu_rows}, res
