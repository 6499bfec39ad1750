"""The .fvecs / .bvecs / .ivecs record containers the reference CLI reads and
writes (datasets.py:60-138): every record is an int32 dimension followed by
that many elements (float32 / uint8 / int32, little endian)."""

from __future__ import annotations

import numpy as np

from .datasets import NeighborLists


def _records(path, elem) -> np.ndarray:
    raw = np.fromfile(path, dtype=np.uint8)
    if raw.size == 0:
        return np.empty((0, 0), dtype=elem)
    if raw.size < 4:
        raise ValueError(f"{path}: truncated file (no leading dimension)")
    d = int(raw[:4].view("<i4")[0])
    if d <= 0:
        raise ValueError(f"{path}: invalid leading dimension {d}")
    width = 4 + d * np.dtype(elem).itemsize
    if raw.size % width:
        raise ValueError(f"{path}: truncated file (not a multiple of record size)")
    rec = raw.reshape(-1, width)
    dims = np.ascontiguousarray(rec[:, :4]).view("<i4").ravel()
    bad = np.flatnonzero(dims != d)
    if bad.size:
        raise ValueError(f"{path}: record {int(bad[0])} has dimension {int(dims[bad[0]])}, expected {d}")
    return np.ascontiguousarray(rec[:, 4:]).view(elem)


def read_vectors(path) -> np.ndarray:
    """.fvecs -> float32 rows; .bvecs -> uint8 rows widened to float32 (exact)."""
    name = str(path).lower()
    if name.endswith(".fvecs"):
        return np.ascontiguousarray(_records(path, "<f4"), dtype=np.float32)
    if name.endswith(".bvecs"):
        return _records(path, np.uint8).astype(np.float32)
    raise ValueError(f"{path}: unknown vector container (expected .fvecs or .bvecs)")


def read_ivecs(path) -> NeighborLists:
    return NeighborLists(ids=_records(path, "<i4").astype(np.int64))


def write_ivecs(path, lists: NeighborLists) -> None:
    ids = lists.ids
    if ids.size and (ids.max() > np.iinfo(np.int32).max or ids.min() < np.iinfo(np.int32).min):
        raise ValueError("ids exceed the int32 range of the ivecs container")
    out = np.empty((ids.shape[0], ids.shape[1] + 1), dtype="<i4")
    out[:, 0] = ids.shape[1]
    out[:, 1:] = ids
    out.tofile(path)


def write_fvecs(path, X) -> None:
    X = np.ascontiguousarray(X, dtype=np.float32)
    out = np.empty((X.shape[0], X.shape[1] + 1), dtype="<f4")
    out.view("<i4")[:, 0] = X.shape[1]
    out[:, 1:] = X
    out.tofile(path)
