"""ctypes signatures for every function declared in include/opx.h.

The header is the single source of truth: it is parsed here so the binding and
the export test (tests/test_abi.py) can never drift from the declared ABI.
"""
from __future__ import annotations

import ctypes
import os
import re

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "opx.h")

_SCALARS = {
    "int": ctypes.c_int,
    "int64_t": ctypes.c_int64,
    "uint64_t": ctypes.c_uint64,
    "size_t": ctypes.c_size_t,
    "float": ctypes.c_float,
    "double": ctypes.c_double,
    "void": None,
}


def _ctype(decl: str):
    decl = decl.strip()
    if decl.endswith("*") or "*" in decl:
        base = decl.replace("const", "").replace("*", "").strip()
        if base == "char" and decl.count("*") == 1:
            return ctypes.c_char_p
        return ctypes.c_void_p
    base = decl.replace("const", "").strip()
    return _SCALARS[base]


def parse_header(path: str = HEADER):
    """Returns {name: (restype, [argtypes])} for every opx_* function."""
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    out = {}
    for m in re.finditer(r"([A-Za-z_][\w\s\*]*?)\b(opx_\w+)\s*\(([^)]*)\)\s*;", text):
        ret, name, args = m.group(1).strip().split("\n")[-1], m.group(2), m.group(3)
        if "typedef" in ret:
            continue
        argtypes = []
        args = args.strip()
        if args and args != "void":
            for a in args.split(","):
                a = a.strip()
                # drop the parameter name
                mm = re.match(r"(.*?)([A-Za-z_]\w*)\s*$", a)
                typ = mm.group(1) if mm and mm.group(1).strip() else a
                argtypes.append(_ctype(typ))
        out[name] = (_ctype(ret), argtypes)
    return out


def declare(lib: ctypes.CDLL) -> None:
    for name, (res, args) in parse_header().items():
        fn = getattr(lib, name, None)
        if fn is None:  # reported by tests/test_abi.py
            continue
        fn.restype = res
        fn.argtypes = args
