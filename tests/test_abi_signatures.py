"""The C ABI as three documents must agree: every
prototype in include/sparseconv_b200.h, the ctypes binding the engine uses
(_native._SIGS), and every ctypes argtypes list INTEGRATION.md shows a
reference maintainer.  CPU only: parses text, loads nothing on the GPU."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _prototypes():
    """name -> (return type, [param types]) from the header."""
    text = (ROOT / "include" / "sparseconv_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", " ", text, flags=re.S)
    text = re.sub(r"//[^\n]*", " ", text)
    out = {}
    for m in re.finditer(r"([A-Za-z_][A-Za-z0-9_ ]*?\**)\s*\b(scb_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;",
                         text):
        ret, name, params = m.group(1).strip(), m.group(2), m.group(3).strip()
        ps = [] if params in ("", "void") else [p.strip() for p in params.split(",")]
        out[name] = (ret, ps)
    return out


def _param_type(decl: str) -> str:
    """Strip the parameter name: 'const int32_t* hits' -> 'const int32_t*'."""
    decl = re.sub(r"\s+", " ", decl)
    m = re.match(r"(.*?[\s\*])([A-Za-z_][A-Za-z0-9_]*)$", decl)
    return (m.group(1) if m else decl).replace(" *", "*").strip()


def _compatible(ctype_decl: str, ct) -> bool:
    t = ctype_decl.replace("const ", "").strip()
    if t.endswith("*"):
        base = t[:-1].strip()
        if base == "scb_grid_t":
            from paper_2204_10319_b200._native import GridT
            return ct is ctypes.POINTER(GridT)
        if base == "scb_segment_t":
            from paper_2204_10319_b200._native import SegmentT
            return ct is ctypes.POINTER(SegmentT)
        if base == "char":
            return ct is ctypes.c_char_p
        return ct is ctypes.c_void_p or (hasattr(ct, "_type_") and ct.__name__.startswith("LP_"))
    return {"int32_t": ct is ctypes.c_int32, "int64_t": ct is ctypes.c_int64,
            "uint32_t": ct is ctypes.c_uint32, "double": ct is ctypes.c_double,
            "scb_stream_t": ct is ctypes.c_void_p}.get(t, False)


def test_header_prototypes_match_the_ctypes_binding():
    from paper_2204_10319_b200._native import _SIGS
    protos = _prototypes()
    assert set(protos) == set(_SIGS), set(protos) ^ set(_SIGS)
    for name, (ret, params) in protos.items():
        res, args = _SIGS[name]
        assert _compatible(ret, res), (name, ret, res)
        assert len(params) == len(args), (name, len(params), len(args))
        for i, (p, a) in enumerate(zip(params, args)):
            assert _compatible(_param_type(p), a), (name, i, p, a)


_CT = {"c_int32": ctypes.c_int32, "c_int64": ctypes.c_int64, "c_void_p": ctypes.c_void_p,
       "c_double": ctypes.c_double, "c_char_p": ctypes.c_char_p}


def test_integration_bindings_match_the_abi():
    """Each `_lib.scb_X.argtypes = [...]` block in INTEGRATION.md has the
    header's arity and types (the r1 scb_gather stub passed 10 of 11)."""
    from paper_2204_10319_b200._native import _SIGS
    text = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"_lib\.(scb_[a-z0-9_]+)\.argtypes\s*=\s*\[(.*?)\]", text, flags=re.S)
    assert blocks, "INTEGRATION.md shows no ctypes binding"
    for name, body in blocks:
        names = re.findall(r"ctypes\.(c_[a-z0-9_]+)", body)
        want = _SIGS[name][1]
        assert len(names) == len(want), (name, len(names), len(want))
        for i, (n, w) in enumerate(zip(names, want)):
            got = _CT[n]
            assert got is w or (got is ctypes.c_void_p and w.__name__.startswith("LP_")), (name, i)
    # every call in the stubs passes as many arguments as the entry point takes
    for name, args in re.findall(r"_lib\.(scb_[a-z0-9_]+)\(([^()]*(?:\([^()]*\)[^()]*)*)\)", text):
        n = len([a for a in re.split(r",(?![^()]*\))", args) if a.strip()])
        assert n == len(_SIGS[name][1]), (name, n, len(_SIGS[name][1]))


def test_integration_table_lists_every_entry_point():
    from paper_2204_10319_b200._native import _SIGS
    text = (ROOT / "INTEGRATION.md").read_text()
    listed = set(re.findall(r"`(scb_[a-z0-9_]+)`", text))
    helpers = {"scb_last_error", "scb_abi_version", "scb_device_sm_count", "scb_launch_count"}
    missing = set(_SIGS) - listed - helpers
    assert not missing, sorted(missing)
    stale = listed - set(_SIGS)
    assert not stale, sorted(stale)
