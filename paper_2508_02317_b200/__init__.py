"""opx: B200-native FSDP + Ulysses-SP + EP training step (VeOmni hot path).

The product is ``libopx.so`` (C++ host + sm_100a CUDA kernels) behind the C ABI
declared in ``include/opx.h``.  This package only binds that ABI with ctypes and
mirrors the reference planner's Python-visible names; it contains no compute
path of its own and raises if the native library is missing.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# OPX_LIB_PATH: diagnostics only (tools/ profiling builds of the same sources)
LIB_PATH = os.environ.get("OPX_LIB_PATH") or os.path.join(_HERE, "libopx.so")
_lib = None


class OpxError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"opx error {code}: {msg}")
        self.code = code
        self.msg = msg


def lib() -> ctypes.CDLL:
    """Load libopx.so (fails loudly: there is no fallback implementation)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OpxError(6, f"native library not built: {LIB_PATH} (run __graft_entry__.build())")
        _lib = ctypes.CDLL(LIB_PATH)
        from . import _abi

        _abi.declare(_lib)
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        raise OpxError(rc, lib().opx_last_error().decode())


from .plan import ParallelPlan, validate, resolve  # noqa: E402,F401
