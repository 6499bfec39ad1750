"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/ivfpq_oracle.c.

Bit-exact C restatement of the reference search path (see the .c header).
Index arrays use the reference layout: CSR `list_off` int64[nlist+1],
`ids` int64[N] and row-major `codes` uint8[N, s], concatenated over lists.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle.so")
PREC_CODE = {"f32": 0, "f16": 1, "e5m3": 2, "e4m4": 3}

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int, ctypes.c_int64
        L.orc_search_batch.restype = i64
        L.orc_search_batch.argtypes = [P, i32, i32, P, i32, i32, P, P, P, P, i32, i32, i32, i32, P, P, i32]
        L.orc_select.argtypes = [P, i32, i32, P, i32, P]
        L.orc_build_lut.argtypes = [P, i32, i32, i32, P, i32, P]
        L.orc_scan.argtypes = [P, i64, i32, i32, P, i32, P]
        L.orc_brute_force_knn.argtypes = [P, i64, i32, P, i32, i32, P, P, i32]
        L.orc_pq_encode.argtypes = [P, i64, i32, P, i32, i32, P]
        L.orc_fp8_encode.restype = ctypes.c_uint8
        L.orc_fp8_encode.argtypes = [ctypes.c_float, i32]
        L.orc_f16_encode.restype = ctypes.c_uint16
        L.orc_f16_encode.argtypes = [ctypes.c_float]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def flatten_lists(list_ids, list_codes, s):
    """Reference per-list arrays -> CSR (list_off, ids, row-major codes)."""
    lens = np.array([x.shape[0] for x in list_ids], dtype=np.int64)
    off = np.zeros(len(list_ids) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    ids = np.ascontiguousarray(np.concatenate(list_ids).astype(np.int64)) if len(list_ids) else np.zeros(0, np.int64)
    codes = np.ascontiguousarray(np.concatenate([c.reshape(-1, s) for c in list_codes]).astype(np.uint8))
    return off, ids, codes


def search_batch(coarse, centers, list_off, ids, codes, queries, k, nprobe, prec, threads=None):
    coarse = np.ascontiguousarray(coarse, np.float32)
    centers = np.ascontiguousarray(centers, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    nlist, d = coarse.shape
    s, n_codes, _ = centers.shape
    p = int(n_codes).bit_length() - 1
    nq = queries.shape[0]
    out_ids = np.empty((nq, k), np.int64)
    out_d = np.empty((nq, k), np.float32)
    n_short = lib().orc_search_batch(
        _p(coarse), nlist, d, _p(centers), s, p, _p(list_off), _p(ids), _p(codes),
        _p(queries), nq, k, nprobe, PREC_CODE[prec], _p(out_ids), _p(out_d),
        threads or os.cpu_count() or 1)
    return out_ids, out_d, int(n_short)


def select(coarse, q, nprobe):
    coarse = np.ascontiguousarray(coarse, np.float32)
    q = np.ascontiguousarray(q, np.float32)
    out = np.empty(nprobe, np.int64)
    lib().orc_select(_p(coarse), coarse.shape[0], coarse.shape[1], _p(q), nprobe, _p(out))
    return out


def build_lut(centers, rq, prec):
    centers = np.ascontiguousarray(centers, np.float32)
    rq = np.ascontiguousarray(rq, np.float32)
    s, n_codes, sub_d = centers.shape
    dt = {"f32": np.float32, "f16": np.uint16}.get(prec, np.uint8)
    out = np.empty((s, n_codes), dt)
    lib().orc_build_lut(_p(centers), s, n_codes, sub_d, _p(rq), PREC_CODE[prec], _p(out))
    return out


def scan(codes, entries, prec):
    codes = np.ascontiguousarray(codes, np.uint8)
    entries = np.ascontiguousarray(entries)
    L, s = codes.shape
    out = np.empty(L, np.float32)
    lib().orc_scan(_p(codes), L, s, entries.shape[1], _p(entries), PREC_CODE[prec], _p(out))
    return out


def brute_force_knn(base, queries, k, threads=None):
    base = np.ascontiguousarray(base, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    nq = queries.shape[0]
    out_ids = np.empty((nq, k), np.int64)
    out_d = np.empty((nq, k), np.float32)
    lib().orc_brute_force_knn(_p(base), base.shape[0], base.shape[1], _p(queries), nq, k,
                              _p(out_ids), _p(out_d), threads or os.cpu_count() or 1)
    return out_ids, out_d


def pq_encode(residuals: np.ndarray, centers: np.ndarray) -> np.ndarray:
    """pq.py:92-110 restated (sub_d <= 4): codes uint8[n, s]."""
    X = np.ascontiguousarray(residuals, dtype=np.float32)
    C = np.ascontiguousarray(centers, dtype=np.float32)
    s, n_codes, sub = C.shape
    out = np.empty((X.shape[0], s), dtype=np.uint8)
    rc = lib().orc_pq_encode(_p(X), X.shape[0], X.shape[1], _p(C), s, n_codes, _p(out))
    if rc != 0:
        raise ValueError("oracle pq_encode supports sub_d <= 4 only")
    return out
