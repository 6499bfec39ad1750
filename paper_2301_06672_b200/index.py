"""Index types (reference index.py:27-70, pq.py:20-51), the IVFPQ001 file
format (index.py:1-8, 100-161) and the device-resident handle.

`IvfPqIndex` keeps the reference's fields -- coarse, cb, list_ids[c],
list_codes[c] -- so reference-built indexes can be handed over unchanged.
Internally it also carries the CSR form (list_off, ids, codes) that the C ABI
uploads; `from_csr` builds an index whose per-list arrays are views into it.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib

__all__ = ["PQCodebook", "IvfPqIndex", "DeviceIndex", "device_index", "save_index", "load_index"]

MAGIC = b"IVFPQ001"
_HEADER = struct.Struct("<8s5IQ")


@dataclass
class PQCodebook:
    """pq.py:20-51: centers (s, 2^p, sub_d); subspace j = dims [j*sub_d, (j+1)*sub_d)."""

    centers: np.ndarray
    p: int

    def __post_init__(self):
        self.centers = np.ascontiguousarray(self.centers, dtype=np.float32)
        if self.centers.ndim != 3:
            raise ValueError("centers must have shape (s, n_codes, sub_d)")
        if self.centers.shape[1] != 1 << self.p:
            raise ValueError(f"expected {1 << self.p} codes per subspace, got {self.centers.shape[1]}")

    @property
    def s(self) -> int:
        return self.centers.shape[0]

    @property
    def n_codes(self) -> int:
        return self.centers.shape[1]

    @property
    def sub_d(self) -> int:
        return self.centers.shape[2]

    @property
    def d(self) -> int:
        return self.s * self.sub_d


@dataclass(eq=False)
class IvfPqIndex:
    """index.py:27-70.  Immutable after construction (the device handle is
    cached on the object)."""

    coarse: np.ndarray
    cb: PQCodebook
    list_ids: list
    list_codes: list
    _csr: tuple | None = field(default=None, repr=False)
    _device: dict = field(default_factory=dict, repr=False)

    @property
    def d(self) -> int:
        return self.coarse.shape[1]

    @property
    def nlist(self) -> int:
        return self.coarse.shape[0]

    @property
    def n_total(self) -> int:
        return sum(ids.shape[0] for ids in self.list_ids)

    @classmethod
    def from_csr(cls, coarse, cb: PQCodebook, list_off, ids, codes) -> "IvfPqIndex":
        coarse = np.ascontiguousarray(coarse, dtype=np.float32)
        list_off = np.ascontiguousarray(list_off, dtype=np.int64)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        codes = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1, cb.s)
        list_ids = [ids[list_off[c]:list_off[c + 1]] for c in range(coarse.shape[0])]
        list_codes = [codes[list_off[c]:list_off[c + 1]] for c in range(coarse.shape[0])]
        return cls(coarse=coarse, cb=cb, list_ids=list_ids, list_codes=list_codes, _csr=(list_off, ids, codes))

    def csr(self):
        """(list_off int64[nlist+1], ids int64[N], codes uint8[N, s]) in list order."""
        if self._csr is None:
            lens = np.array([x.shape[0] for x in self.list_ids], dtype=np.int64)
            off = np.zeros(self.nlist + 1, dtype=np.int64)
            np.cumsum(lens, out=off[1:])
            ids = (np.concatenate([np.asarray(x, dtype=np.int64) for x in self.list_ids])
                   if self.nlist else np.zeros(0, np.int64))
            codes = (np.concatenate([np.asarray(c, dtype=np.uint8).reshape(-1, self.cb.s) for c in self.list_codes])
                     if self.nlist else np.zeros((0, self.cb.s), np.uint8))
            self._csr = (off, np.ascontiguousarray(ids), np.ascontiguousarray(codes))
        return self._csr

    def validate(self) -> None:
        """index.py:52-70 structural invariants."""
        if self.cb.d != self.d:
            raise ValueError(f"codebook covers {self.cb.d} dims, index has {self.d}")
        if len(self.list_ids) != self.nlist or len(self.list_codes) != self.nlist:
            raise ValueError("one inverted list required per coarse centroid")
        for c, (ids, codes) in enumerate(zip(self.list_ids, self.list_codes)):
            if codes.shape != (ids.shape[0], self.cb.s):
                raise ValueError(f"list {c}: ids/codes shape mismatch")
            if ids.size and np.any(np.diff(ids) <= 0):
                raise ValueError(f"list {c}: ids not strictly ascending")
            if codes.size and codes.max() >= self.cb.n_codes:
                raise ValueError(f"list {c}: code byte out of range for p={self.cb.p}")
        _, ids, _ = self.csr()
        if ids.size and not np.array_equal(np.sort(ids), np.arange(ids.size)):
            raise ValueError("inverted lists do not partition ids 0..N-1")


class DeviceIndex:
    """Owner of one `ivfpq_index*` handle (device copies of coarse, codebook,
    ids and interleaved codes).  `owned` selects a list shard."""

    def __init__(self, idx: IvfPqIndex, device: int = 0, owned=None):
        _lib.require_gpu()
        off, ids, codes = idx.csr()
        coarse = np.ascontiguousarray(idx.coarse, dtype=np.float32)
        centers = np.ascontiguousarray(idx.cb.centers, dtype=np.float32)
        own = None if owned is None else np.ascontiguousarray(owned, dtype=np.int32)
        h = _lib.ctypes.c_void_p()
        _lib.check(_lib.lib.ivfpq_index_create(
            device, coarse.ctypes.data, idx.nlist, idx.d, centers.ctypes.data, idx.cb.s, idx.cb.p,
            off.ctypes.data, ids.ctypes.data, codes.ctypes.data,
            None if own is None else own.ctypes.data, 0 if own is None else own.size, _lib.ctypes.byref(h)))
        self.handle = h
        self.device = device
        self.nlist, self.d, self.s, self.p = idx.nlist, idx.d, idx.cb.s, idx.cb.p
        self.owned = own
        self.list_len = np.diff(off)

    @property
    def nbytes(self) -> int:
        b = _lib.ctypes.c_int64()
        _lib.check(_lib.lib.ivfpq_index_bytes(self.handle, _lib.ctypes.byref(b)))
        return b.value

    def close(self):
        if getattr(self, "handle", None):
            _lib.lib.ivfpq_index_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_index(idx: IvfPqIndex, device: int = 0) -> DeviceIndex:
    """Cached full-index upload for `idx` on `device`."""
    h = idx._device.get(device)
    if h is None:
        h = DeviceIndex(idx, device)
        idx._device[device] = h
    return h


def save_index(idx: IvfPqIndex, path) -> None:
    """index.py:100-112: canonical little-endian IVFPQ001 bytes."""
    off, ids, codes = idx.csr()
    with open(path, "wb") as f:
        f.write(_HEADER.pack(MAGIC, idx.d, idx.nlist, idx.cb.s, idx.cb.p, idx.cb.sub_d, int(off[-1])))
        f.write(np.ascontiguousarray(idx.coarse, dtype="<f4").tobytes())
        f.write(np.ascontiguousarray(idx.cb.centers, dtype="<f4").tobytes())
        for c in range(idx.nlist):
            lo, hi = off[c], off[c + 1]
            f.write(struct.pack("<Q", int(hi - lo)))
            f.write(ids[lo:hi].astype("<u8").tobytes())
            f.write(codes[lo:hi].tobytes())


def load_index(path) -> IvfPqIndex:
    """index.py:115-161: read + validate; returns a CSR-backed index."""
    with open(path, "rb") as f:
        blob = f.read()
    if len(blob) < _HEADER.size:
        raise ValueError(f"{path}: truncated header")
    magic, d, nlist, s, p, sub_d, n_total = _HEADER.unpack_from(blob, 0)
    if magic != MAGIC:
        raise ValueError(f"{path}: not an index file (bad magic {magic!r})")
    if d <= 0 or nlist <= 0 or s <= 0 or sub_d <= 0 or not 1 <= p <= 8:
        raise ValueError(f"{path}: invalid header fields")
    if s * sub_d != d:
        raise ValueError(f"{path}: s*sub_d = {s * sub_d} does not match d = {d}")
    pos = _HEADER.size
    n_codes = 1 << p

    def take(nbytes):
        nonlocal pos
        if pos + nbytes > len(blob):
            raise ValueError(f"{path}: truncated file")
        out = memoryview(blob)[pos:pos + nbytes]
        pos += nbytes
        return out

    coarse = np.frombuffer(take(nlist * d * 4), dtype="<f4").reshape(nlist, d).astype(np.float32)
    centers = np.frombuffer(take(s * n_codes * sub_d * 4), dtype="<f4").reshape(s, n_codes, sub_d).astype(np.float32)
    off = np.zeros(nlist + 1, dtype=np.int64)
    spans = []
    for c in range(nlist):
        (length,) = struct.unpack("<Q", take(8))
        ids_at = pos
        take(length * 8)
        codes_at = pos
        take(length * s)
        spans.append((ids_at, codes_at, length))
        off[c + 1] = off[c] + length
    if pos != len(blob):
        raise ValueError(f"{path}: {len(blob) - pos} trailing bytes")
    if off[-1] != n_total:
        raise ValueError(f"{path}: header claims {n_total} vectors, lists hold {off[-1]}")
    ids = np.empty(off[-1], dtype=np.int64)
    codes = np.empty((off[-1], s), dtype=np.uint8)
    buf = np.frombuffer(blob, dtype=np.uint8)
    for c, (ia, ca, L) in enumerate(spans):
        ids[off[c]:off[c + 1]] = buf[ia:ia + 8 * L].view("<u8")
        codes[off[c]:off[c + 1]] = buf[ca:ca + s * L].reshape(L, s)
    idx = IvfPqIndex.from_csr(coarse, PQCodebook(centers=centers, p=p), off, ids, codes)
    idx.validate()
    return idx
