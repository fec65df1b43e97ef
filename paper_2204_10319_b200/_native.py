"""ctypes binding of the C ABI in ``include/sparseconv_b200.h``.

This is exactly the binding a maintainer of the (pure-Python) reference would
add to call the B200 engine.  There is deliberately no
fallback: if ``libsparseconv_b200.so`` is missing or no CUDA device is
present, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / os.environ.get("SCB_LIB_NAME", "libsparseconv_b200.so")

SCB_F32, SCB_F16 = 0, 1
SCB_INDEX_HASH, SCB_INDEX_GRID = 0, 1
TILE_ROWS = 128
MAX_SEGMENTS = 128


class NativeError(RuntimeError):
    """A CUDA-side failure reported by the C ABI."""


class GridT(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("_pad", ctypes.c_int32),
                ("batch_size", ctypes.c_int64), ("extent", ctypes.c_int64 * 4)]


class SegmentT(ctypes.Structure):
    _fields_ = [("a_row", ctypes.c_int64), ("c_row", ctypes.c_int64), ("rows", ctypes.c_int32),
                ("b_index", ctypes.c_int32), ("a_src", ctypes.c_int32), ("_pad", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_GP = ctypes.POINTER(GridT)

# name -> (restype, argtypes)
_SIGS = {
    "scb_last_error": (ctypes.c_char_p, []),
    "scb_abi_version": (_I32, []),
    "scb_device_sm_count": (_I32, []),
    "scb_launch_count": (_I64, []),
    "scb_hash_slots": (_I64, [_I64]),
    "scb_hits_ld": (_I64, [_I64]),
    "scb_index_build": (_I32, [_I32, _P, _I64, _GP, _P, _P, _I64, _P, _P]),
    "scb_index_query": (_I32, [_I32, _P, _I64, _GP, _P, _P, _I64, _P, _P]),
    "scb_output_coords_capacity": (_I64, [_I64, _I32, _I32, _I32]),
    "scb_output_coords_workspace": (_I64, [_I64, _I32, _I32, _I32]),
    "scb_output_coords": (_I32, [_P, _I64, _GP, _I32, _I32, _I32, _P, _I64, _P, _P, _P]),
    "scb_output_keys_next": (_I32, [_P, _P, _I64, _GP, _GP, _I32, _I32, _I32, _P, _I64, _P, _P,
                                    _P]),
    "scb_unflatten": (_I32, [_P, _I64, _GP, _P, _P]),
    "scb_voxelize_workspace": (_I64, [_I64, _I32]),
    "scb_voxelize": (_I32, [_P, _I64, _I32, _I32, ctypes.c_double, _I32, _P, _I64, _P, _P, _P, _P]),
    "scb_voxelize_batch": (_I32, [_P, _P, _I32, _I64, _I32, _I32, ctypes.c_double, _I32, _P, _I64,
                                  _P, _P, _P, _P]),
    "scb_map_search": (_I32, [_I32, _P, _I64, _GP, _I32, _I32, _I32, _I32, _P, _P, _I64, _P, _P]),
    "scb_map_search_dilated": (_I32, [_I32, _P, _I64, _GP, _I32, _I32, _I32, _I32, _I32, _P, _P,
                                      _I64, _P, _P]),
    "scb_map_workspace": (_I64, [_I32, _I64]),
    "scb_map_count": (_I32, [_P, _I32, _I64, _P, _P, _P]),
    "scb_map_compact": (_I32, [_P, _I32, _I64, _P, _P, _P, _P, _P]),
    "scb_map_transpose": (_I32, [_P, _P, _P, _I32, _I64, _I64, _P, _P]),
    "scb_hits_transpose": (_I32, [_P, _I32, _I64, _I64, _P, _P]),
    "scb_plan_build": (_I32, [_P, _P, _P, _I32, _I64, _I64, _I32, _I32, _P, _I64, _P, _P, _P]),
    "scb_gather": (_I32, [_I32, _P, _I64, _I32, _I64, _P, _I64, _P, _I64, _P, _P]),
    "scb_plan_rows_cap": (_I64, [_I32, _I64, _I32]),
    "scb_segtable_bytes": (_I64, []),
    "scb_plan_from_hits": (_I32, [_P, _I32, _I64, _I32, _I32, _I64, _I32, _I32, _I32, _I64, _P,
                                  _P, _P, _P, _P, _P]),
    "scb_grouped_gemm_table": (_I32, [_I32, _P, _I64, _I64, _P, _I64, _I64, _I32, _P, _I32, _I32,
                                      _P, _I64, _I64, _P, _P]),
    "scb_gemm_tile_geometry": (_I32, [_I32, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "scb_scatter": (_I32, [_P, _I64, _P, _I32, _I64, _I32, _I64, _I32, _P, _I64, _P, _P, _P,
                           _P, _I32, _P]),
    "scb_scatter_csr": (_I32, [_I32, _P, _I64, _P, _P, _I64, _I32, _I32, _P, _I64, _P]),
    "scb_store_to_host": (_I32, [_P, _P, _I64, _P]),
    "scb_pointwise": (_I32, [_I32, _P, _I64, _I32, _I32, _P, _P, _P]),
    "scb_add": (_I32, [_I32, _P, _P, _P, _I64, _I32, _P]),
    "scb_quantize_f16": (_I32, [_P, _P, _I64, _P, _P]),
    "scb_pack_weights_f16": (_I32, [_P, _I32, _I32, _I32, _P, _I32, _I32, _P]),
    "scb_grouped_gemm": (_I32, [_I32, _P, _I64, _I64, _P, _I64, _I64, _I32, _P, _I32, _I32, _P,
                                _I64, _I64, ctypes.POINTER(SegmentT), _I32, _P]),
    "scb_conv_implicit": (_I32, [_P, _I64, _I32, _I64, _P, _I32, _I64, _P, _I32, _P, _P, _P, _P,
                                 _P, _I32, _P]),
    "scb_conv_implicit_cat": (_I32, [_P, _I64, _I32, _P, _I64, _I64, _I32, _P, _I32, _I64, _P,
                                     _P, _I32, _P, _I64, _P, _P, _P, _P, _I32, _P]),
    "scb_conv_implicit_tuned": (_I32, [_P, _I64, _I32, _P, _I64, _I64, _I32, _P, _I32, _I64, _P,
                                       _P, _I32, _P, _I64, _P, _P, _P, _P, _I32, _I32, _I32, _P]),
    "scb_conv_implicit_rows": (_I32, [_P, _I64, _I32, _P, _I64, _I64, _I32, _P, _I32, _I64, _P,
                                      _P, _P, _I32, _P, _I64, _P, _P, _P, _P, _I32, _I32, _I32,
                                      _P]),
    "scb_onehot_order_workspace": (_I64, [_I64]),
    "scb_onehot_order": (_I32, [_P, _I32, _I64, _P, _I64, _P, _P, _P, _P]),
    "scb_tile_masks": (_I32, [_P, _I32, _I64, _P, _P]),
    "scb_conv_transposed_scatter": (_I32, [_P, _I64, _I64, _I32, _P, _I32, _P, _I32, _P, _I64,
                                            _I64, _P, _P, _P, _I32, _P]),
    "scb_conv_pointwise": (_I32, [_P, _I64, _I32, _P, _I64, _I64, _I32, _P, _I32, _P, _I64, _P,
                                   _P, _P, _I32, _P]),
    "scb_presence_masks": (_I32, [_I32, _P, _I64, _GP, _I32, _I32, _P, _P, _I64, _P, _P, _P]),
    "scb_map_search_masked": (_I32, [_I32, _P, _I64, _GP, _I32, _I32, _P, _P, _I64, _P, _P, _P, _P]),
    "scb_mask_sort_workspace": (_I64, [_I64]),
    "scb_mask_sort": (_I32, [_P, _P, _P, _I32, _I64, _I32, _I64, _P, _I64, _P, _P]),
    "scb_permute_rows": (_I32, [_P, _I64, _P, _I64, _I32, _P, _I64, _I32, _P]),
    "scb_apply_order": (_I32, [_P, _I64, _P, _I32, _P, _P, _P]),
    "scb_index_relabel": (_I32, [_I32, _P, _P, _I64, _P, _P, _P]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load the engine library (once).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH.name} not built — run `make` (or __graft_entry__.build()); "
                "the B200 engine has no CPU fallback")
        lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 sparse-conv engine needs a CUDA device; there is no CPU path")


_raw_stream = torch._C._cuda_getCurrentRawStream
_cur_device = torch._C._cuda_getDevice


def stream_handle() -> int:
    """cudaStream_t of the current torch stream (two C calls; the Python
    torch.cuda.current_stream() path costs ~3 us per call)."""
    return _raw_stream(_cur_device())


def ptr(t) -> int | None:
    """Raw device address of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


_FN: dict = {}
_NO_STATUS = ("scb_abi_version", "scb_device_sm_count")


def call(name: str, *args) -> int:
    """Invoke an ABI function, raising NativeError with the library's
    message on a non-zero status."""
    fn = _FN.get(name)
    if fn is None:
        fn = getattr(load(), name)
        _FN[name] = fn
    status = fn(*args)
    if status and fn.restype is _I32 and name not in _NO_STATUS:
        lib = load()
        msg = lib.scb_last_error().decode(errors="replace")
        if status == 1:
            raise ValueError(msg)
        raise NativeError(f"{name} failed ({status}): {msg}")
    return status


def make_grid(boundary, batch_size) -> GridT:
    g = GridT()
    g.dim = len(boundary)
    g.batch_size = int(batch_size)
    for d in range(4):
        g.extent[d] = int(boundary[d]) if d < len(boundary) else 1
    return g


def dtype_code(dtype) -> int:
    if dtype == torch.float16:
        return SCB_F16
    if dtype == torch.float32:
        return SCB_F32
    raise ValueError(f"unsupported feature dtype {dtype}")
