"""The drop-in boundary on CPU: libopx.so loads without a GPU and exports
every function include/opx.h declares (no compute calls are made here)."""
import ctypes

from paper_2508_02317_b200 import _abi, lib


def test_every_declared_symbol_is_exported():
    decl = _abi.parse_header()
    assert len(decl) >= 30
    L = lib()
    missing = [n for n in decl if not hasattr(L, n)]
    assert not missing, missing


def test_version_and_error_plumbing():
    L = lib()
    assert L.opx_version().startswith(b"opx")
    buf = ctypes.create_string_buffer(256)
    rc = L.opx_plan_validate(b"{", b"{}", b"{}", b"{}", buf, 256)
    assert rc == 2 and b"cluster" in L.opx_last_error()


def test_no_torch_types_in_header():
    text = open(_abi.HEADER).read()
    for bad in ("torch", "at::", "Tensor", "std::"):
        assert bad not in text
