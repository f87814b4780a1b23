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


def test_step_report_struct_matches_header():
    """runtime.StepReport (ctypes) has exactly the fields, order and types of
    the opx_step_report typedef in include/opx.h."""
    import re

    from paper_2508_02317_b200.runtime import StepReport

    text = open(_abi.HEADER).read()
    body = text[text.index("typedef struct {"):text.index("} opx_step_report;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.replace("typedef struct {", "").strip()
        if not decl:
            continue
        typ, names = decl.split(None, 1)
        for n in names.split(","):
            fields.append((n.strip(), typ))
    want = {"double": ctypes.c_double, "int64_t": ctypes.c_int64}
    assert [(n, want[t]) for n, t in fields] == [(n, t) for n, t in StepReport._fields_]


def test_missing_native_library_fails_loudly():
    """No fallback: with libopx.so absent every entry point raises."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("from paper_2508_02317_b200 import lib, OpxError\n"
            "try:\n    lib()\nexcept OpxError as e:\n    print('raised', e.code)\n")
    env = dict(os.environ, OPX_LIB_PATH="/nonexistent/libopx.so")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=120)
    assert out.stdout.strip() == "raised 6", out.stdout + out.stderr
