"""ctypes binding of the in-tree C-ABI library `libivfpq_b200.so`.

The declarations mirror include/ivfpq_b200.h one for one.  There is no
fallback: if the library is missing the import fails loudly, and calls that
need a GPU raise when no CUDA device is visible.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# IVFPQ_LIB: alternative build of the same library (kernel experiments only)
LIB_PATH = os.environ.get("IVFPQ_LIB") or os.path.join(HERE, "libivfpq_b200.so")

OK, EINVAL, ECUDA, EUNSUPPORTED = 0, 1, 2, 3
LUT_CODES = {"f32": 0, "f16": 1, "e5m3": 2, "e4m4": 3}

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int

# name -> argtypes (restype is int status unless listed in _RESTYPES)
SIGNATURES = {
    "ivfpq_last_error": [],
    "ivfpq_version": [],
    "ivfpq_device_count": [_P],
    "ivfpq_max_k": [],
    "ivfpq_launch_count": [_P],
    "ivfpq_set_scan_kernel": [_I32],
    "ivfpq_set_select_kernel": [_I32],
    "ivfpq_debug_select_flagged": [_P, _P],
    "ivfpq_index_create": [_I32, _P, _I64, _I64, _P, _I64, _I64, _P, _P, _P, _P, _I64, _P],
    "ivfpq_index_destroy": [_P],
    "ivfpq_index_bytes": [_P, _P],
    "ivfpq_search": [_P, _P, _I64, _I64, _I64, _I32, _P, _P, _P],
    "ivfpq_search_device": [_P, _P, _I64, _I64, _I64, _I32, _P, _P, _P, _P],
    "ivfpq_select_device": [_P, _P, _I64, _I64, _P, _P],
    "ivfpq_merge_keys_device": [_P, _I64, _I64, _I64, _I64, _P, _P],
    "ivfpq_scan_device": [_P, _P, _I64, _P, _I64, _I64, _I32, _P, _P, _P],
    "ivfpq_finalize_device": [_P, _P, _I64, _I64, _P, _P, _P, _P],
    "ivfpq_fp8_encode": [_P, _I64, _I32, _P],
    "ivfpq_fp8_decode": [_P, _I64, _I32, _P],
    "ivfpq_f16_encode": [_P, _I64, _P],
    "ivfpq_f16_decode": [_P, _I64, _P],
    "ivfpq_build_lut": [_P, _I64, _I64, _I64, _P, _I32, _P],
    "ivfpq_scan_list": [_P, _I64, _I64, _I64, _P, _I32, _P],
    "ivfpq_select_clusters": [_P, _P, _I64, _I64, _P],
    "ivfpq_top_k": [_P, _P, _I64, _I64, _P, _P],
    "ivfpq_pq_encode_device": [_P, _I64, _I64, _P, _P, _P, _I64, _I64, _P, _P],
    "ivfpq_pq_encode": [_P, _I64, _I64, _P, _I64, _I64, _P],
    "ivfpq_assign_device": [_P, _I64, _I64, _P, _I64, _P, _P, _P],
    "ivfpq_assign": [_P, _I64, _I64, _P, _I64, _P, _P],
    "ivfpq_compute_residuals": [_P, _I64, _I64, _P, _I64, _P, _P],
    "ivfpq_reconstruct": [_P, _I64, _P, _I64, _I64, _I64, _P],
    "ivfpq_squared_l2_to_all": [_P, _I64, _I64, _P, _P],
    "ivfpq_knn_create": [_I32, _P, _I64, _I64, _P],
    "ivfpq_brute_force_knn": [_P, _I64, _I64, _P, _I64, _I64, _P, _P],
}
_RESTYPES = {"ivfpq_last_error": ctypes.c_char_p}


class IvfpqError(RuntimeError):
    """A CUDA-side failure reported by the library."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, ctypes.c_int)
    return lib


lib = _load()


def last_error() -> str:
    return lib.ivfpq_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = last_error()
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == EUNSUPPORTED:
        raise ValueError(f"unsupported on the device path: {msg}")
    raise IvfpqError(msg)


def device_count() -> int:
    n = ctypes.c_int(0)
    check(lib.ivfpq_device_count(ctypes.byref(n)))
    return n.value


def require_gpu() -> None:
    if device_count() < 1:
        raise RuntimeError("paper_2301_06672_b200 needs a CUDA device (B200); no CPU fallback exists")


def max_k() -> int:
    return int(lib.ivfpq_max_k())


def launch_count() -> int:
    n = ctypes.c_int64(0)
    check(lib.ivfpq_launch_count(ctypes.byref(n)))
    return n.value


def ptr(a) -> int:
    """Data pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()
