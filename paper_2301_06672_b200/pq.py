"""The reference's `pq` module surface (pq.py:20-127) on the B200 path:
`PQCodebook` (index.py), `pq_encode` (ingest.py, bit-exact device encoder),
and the two helpers below, whose arithmetic runs on the device (ingest.cuh)
through the C ABI.  PQ training is out of scope."""

from __future__ import annotations

import numpy as np

from . import _lib
from .index import PQCodebook
from .ingest import pq_encode
from .validation import check_matrix

__all__ = ["PQCodebook", "compute_residuals", "pq_encode", "reconstruct"]


def compute_residuals(data, centroids, assignments) -> np.ndarray:
    """Row i minus its assigned centroid, exact float32 subtraction
    (pq.py:54-63; same validation and messages)."""
    data = check_matrix(data, "data")
    centroids = check_matrix(centroids, "centroids")
    assignments = np.ascontiguousarray(assignments, dtype=np.int64)
    if assignments.shape != (data.shape[0],):
        raise ValueError("assignments must have one entry per data row")
    if assignments.size and (assignments.min() < 0 or assignments.max() >= centroids.shape[0]):
        raise ValueError("assignment index out of range")
    if data.shape[1] != centroids.shape[1]:
        raise ValueError(f"dimension mismatch: data d={data.shape[1]}, centroids d={centroids.shape[1]}")
    _lib.require_gpu()
    out = np.empty_like(data)
    _lib.check(_lib.lib.ivfpq_compute_residuals(_lib.ptr(data), data.shape[0], data.shape[1], _lib.ptr(centroids),
                                                centroids.shape[0], _lib.ptr(assignments), _lib.ptr(out)))
    return out


def reconstruct(codes, cb: PQCodebook) -> np.ndarray:
    """Concatenate the sub-centroids named by each code (pq.py:113-127);
    one code row (s,) -> (d,), a batch (n, s) -> (n, d)."""
    arr = np.asarray(codes, dtype=np.uint8)
    single = arr.ndim == 1
    if single:
        arr = arr[None, :]
    if arr.ndim != 2 or arr.shape[1] != cb.s:
        raise ValueError(f"codes must have {cb.s} bytes per vector")
    if arr.size and arr.max() >= cb.n_codes:
        raise ValueError(f"code byte out of range for p={cb.p}")
    arr = np.ascontiguousarray(arr)
    centers = np.ascontiguousarray(cb.centers, dtype=np.float32)
    _lib.require_gpu()
    out = np.empty((arr.shape[0], cb.d), dtype=np.float32)
    _lib.check(_lib.lib.ivfpq_reconstruct(_lib.ptr(arr), arr.shape[0], _lib.ptr(centers), cb.s, cb.p, cb.sub_d,
                                          _lib.ptr(out)))
    return out[0] if single else out
