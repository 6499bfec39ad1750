"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference search path.

Each function cites the reference function it restates (paths relative to
`/root/reference/pkg/src/ivfpq8/`).  Arithmetic is IEEE binary32 with one
rounding per numpy ufunc, exactly as the reference computes it; the loop
structure (Python loop over queries, then over probed lists) is kept so that
timing this module is timing the reference algorithm (`kind: "port"`).

The index is passed as plain arrays so that this module has no dependency on
the product package:  coarse f32[nlist,d], centers f32[s,2^p,sub_d],
list_ids list[int64[L_c]], list_codes list[uint8[L_c,s]].
"""

from __future__ import annotations

import numpy as np

PRECISIONS = ("f32", "f16", "e5m3", "e4m4")

# (exponent_bits, mantissa_bits, bias) -- minifloat.py:87-88
SPECS = {"e5m3": (5, 3, 15), "e4m4": (4, 4, 7)}


# ---------------------------------------------------------------- codec ----
def fp8_encode(x: np.ndarray, prec: str) -> np.ndarray:
    """minifloat.py:91-116 (`encode_array`): exponent rebase by bias-127,
    mantissa truncated to m bits, flush below min_normal, clamp to 0xFF."""
    e_bits, m_bits, bias = SPECS[prec]
    bits = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    exp = (bits >> np.uint32(23)).astype(np.int64) - 127 + bias
    mant = (bits & np.uint32(0x7FFFFF)) >> np.uint32(23 - m_bits)
    code = (exp << m_bits) | mant.astype(np.int64)
    code = np.where(exp < 1, 0, code)
    code = np.where(exp > (1 << e_bits) - 1, 0xFF, code)
    return code.astype(np.uint8)


def fp8_decode(codes: np.ndarray, prec: str) -> np.ndarray:
    """minifloat.py:119-133 (`decode_array`): exact; zero exponent -> 0.0."""
    _, m_bits, bias = SPECS[prec]
    c = np.asarray(codes, dtype=np.uint8).astype(np.uint32)
    exp = c >> np.uint32(m_bits)
    mant = c & np.uint32((1 << m_bits) - 1)
    bits = ((exp + np.uint32(127 - bias)) << np.uint32(23)) | (mant << np.uint32(23 - m_bits))
    return np.where(exp == 0, np.float32(0.0), bits.view(np.float32))


def f16_encode(x: np.ndarray) -> np.ndarray:
    """minifloat.py:151-164: clamp at 65504 then binary16 round-to-nearest-even."""
    return np.minimum(np.asarray(x, dtype=np.float32), np.float32(65504.0)).astype(np.float16).view(np.uint16)


def f16_decode(bits: np.ndarray) -> np.ndarray:
    """minifloat.py:167-169."""
    return np.asarray(bits, dtype=np.uint16).view(np.float16).astype(np.float32)


def lut_encode(raw: np.ndarray, prec: str) -> np.ndarray:
    """search.py:123-127 storage step."""
    if prec == "f32":
        return raw
    if prec == "f16":
        return f16_encode(raw)
    return fp8_encode(raw, prec)


def lut_decode(entries: np.ndarray, prec: str) -> np.ndarray:
    """search.py:76-82 (`Lut.decoded`)."""
    if prec == "f32":
        return entries
    if prec == "f16":
        return f16_decode(entries)
    return fp8_decode(entries, prec)


# --------------------------------------------------------------- search ----
def squared_l2_to_all(base: np.ndarray, q: np.ndarray) -> np.ndarray:
    """datasets.py:166-176: acc += diff*diff sequentially over dims, fp32."""
    diff = base - q
    acc = np.zeros(base.shape[0], dtype=np.float32)
    for t in range(base.shape[1]):
        acc += diff[:, t] * diff[:, t]
    return acc


def select_clusters(coarse: np.ndarray, q: np.ndarray, nprobe: int) -> np.ndarray:
    """search.py:91-97: ascending squared L2, ties to the lower cluster id."""
    if not 1 <= nprobe <= coarse.shape[0]:
        raise ValueError(f"nprobe={nprobe} out of range 1..{coarse.shape[0]}")
    return np.argsort(squared_l2_to_all(coarse, q), kind="stable")[:nprobe]


def raw_table(centers: np.ndarray, rq: np.ndarray) -> np.ndarray:
    """search.py:100-111: T[j][m] = sum_t (centers[j][m][t] - rq[j*sub_d+t])^2,
    sequential in t, fp32, no fused multiply-add."""
    s, n_codes, sub_d = centers.shape
    diff = centers - rq.reshape(s, 1, sub_d)
    acc = np.zeros((s, n_codes), dtype=np.float32)
    for t in range(sub_d):
        acc += diff[:, :, t] * diff[:, :, t]
    return acc


def build_lut(centers: np.ndarray, rq: np.ndarray, prec: str) -> np.ndarray:
    """search.py:114-127: returns the stored entries (f32 / u16 bits / u8 codes)."""
    return lut_encode(raw_table(centers, np.asarray(rq, dtype=np.float32)), prec)


def scan_list(codes: np.ndarray, entries: np.ndarray, prec: str) -> np.ndarray:
    """search.py:130-142: R = sum_j decode(T[j][code_j]), fp32, sequential j."""
    table = lut_decode(entries, prec)
    s = table.shape[0]
    if codes.size and codes.max() >= table.shape[1]:
        raise ValueError("code byte out of range for the table")
    acc = np.zeros(codes.shape[0], dtype=np.float32)
    for j in range(s):
        acc += table[j, codes[:, j]]
    return acc


def top_k(ids: np.ndarray, dists: np.ndarray, k: int):
    """search.py:145-155: lexicographic (distance, id), first k; short flag."""
    order = np.lexsort((ids, dists))[:k]
    return ids[order], dists[order], ids.shape[0] < k


def search_one(coarse, centers, list_ids, list_codes, q, k, nprobe, prec):
    """search.py:158-184 for one query."""
    clusters = select_clusters(coarse, q, nprobe)
    id_parts, d_parts = [], []
    for c in clusters:
        ids = list_ids[c]
        if ids.shape[0] == 0:
            continue
        rq = q - coarse[c]
        lut = build_lut(centers, rq, prec)
        id_parts.append(ids)
        d_parts.append(scan_list(list_codes[c], lut, prec))
    if not id_parts:
        return np.empty(0, np.int64), np.empty(0, np.float32), True
    return top_k(np.concatenate(id_parts), np.concatenate(d_parts), k)


def search_batch(coarse, centers, list_ids, list_codes, queries, k, nprobe, prec):
    """search.py:187-203: rows padded with id -1 / +inf; returns (ids, dists, n_short)."""
    queries = np.ascontiguousarray(queries, dtype=np.float32)
    nq = queries.shape[0]
    out_ids = np.full((nq, k), -1, dtype=np.int64)
    out_d = np.full((nq, k), np.inf, dtype=np.float32)
    n_short = 0
    for i in range(nq):
        ids, dists, short = search_one(coarse, centers, list_ids, list_codes, queries[i], k, nprobe, prec)
        out_ids[i, : ids.shape[0]] = ids
        out_d[i, : dists.shape[0]] = dists
        n_short += int(short)
    return out_ids, out_d, n_short


def recall(res_ids: np.ndarray, gt_ids: np.ndarray) -> tuple[np.ndarray, float]:
    """search.py:206-221: |ids ∩ gt| / gt.k per query; -1 never matches."""
    hits = (res_ids[:, :, None] == gt_ids[:, None, :]) & (res_ids[:, :, None] >= 0)
    per = hits.any(axis=2).sum(axis=1) / gt_ids.shape[1]
    return per, float(per.mean())


def brute_force_knn(base: np.ndarray, queries: np.ndarray, k: int):
    """datasets.py:179-201: exact k-NN with the sequential fp32 distance,
    ties to the lower id."""
    ids = np.empty((queries.shape[0], k), dtype=np.int64)
    dists = np.empty((queries.shape[0], k), dtype=np.float32)
    for i in range(queries.shape[0]):
        d2 = squared_l2_to_all(base, queries[i])
        order = np.argsort(d2, kind="stable")[:k]
        ids[i] = order
        dists[i] = d2[order]
    return ids, dists
