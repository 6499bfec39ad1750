"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything written here is an output of reference code paths
(`ivfpq8.index.build_index`, `ivfpq8.search.*`, `ivfpq8.minifloat.*`), so the
fixtures pin both the oracle restatement (tests/test_oracle_golden.py) and the
CUDA path (tests/test_gpu_parity.py).  The GPU box never runs this script.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from ivfpq8 import minifloat  # noqa: E402
from ivfpq8.datasets import brute_force_knn, synth_gaussian_mixture  # noqa: E402
from ivfpq8.index import build_index, save_index  # noqa: E402
from ivfpq8.kmeans import assign_to_centroids  # noqa: E402
from ivfpq8.pq import PQCodebook, compute_residuals, pq_encode, train_pq  # noqa: E402
from ivfpq8.search import SearchParams, build_lut, scan_list, search_batch, select_clusters  # noqa: E402

PRECS = ["f32", "f16", "e5m3", "e4m4"]


def flat(idx):
    lens = np.array([x.shape[0] for x in idx.list_ids], dtype=np.int64)
    off = np.zeros(idx.nlist + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    ids = np.concatenate(idx.list_ids).astype(np.int64)
    codes = np.concatenate([c.reshape(-1, idx.cb.s) for c in idx.list_codes]).astype(np.uint8)
    return off, ids, codes


def dump_case(name, idx, queries, runs, lut_pairs=4, save_file=False):
    """runs: list of (k, nprobe) -- each run is done for every precision."""
    off, ids, codes = flat(idx)
    out = dict(coarse=idx.coarse, centers=idx.cb.centers, p=np.int64(idx.cb.p),
               list_off=off, ids=ids, codes=codes, queries=queries)
    out["runs"] = np.array(runs, dtype=np.int64)
    for (k, nprobe) in runs:
        for prec in PRECS:
            lists, n_short = search_batch(idx, queries, SearchParams(k=k, nprobe=nprobe, precision=prec))
            out[f"ids_{prec}_k{k}_p{nprobe}"] = lists.ids
            out[f"d_{prec}_k{k}_p{nprobe}"] = lists.distances
            out[f"short_{prec}_k{k}_p{nprobe}"] = np.int64(n_short)
    # coarse selection for every query at the largest nprobe of the runs
    pmax = max(p for _, p in runs)
    out["select"] = np.stack([select_clusters(idx, q, pmax) for q in queries])
    # LUTs + scans for a few (query, probed list) pairs
    pairs = []
    for qi in range(min(lut_pairs, queries.shape[0])):
        cl = select_clusters(idx, queries[qi], min(3, idx.nlist))
        for c in cl:
            if idx.list_ids[c].shape[0]:
                pairs.append((qi, int(c)))
                break
    out["lut_pairs"] = np.array(pairs, dtype=np.int64)
    for n, (qi, c) in enumerate(pairs):
        rq = queries[qi] - idx.coarse[c]
        for prec in PRECS:
            lut = build_lut(idx.cb, rq, prec)
            out[f"lut_{prec}_{n}"] = lut.entries
            _, r = scan_list(idx.list_ids[c], idx.list_codes[c], lut)
            out[f"scan_{prec}_{n}"] = r
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    if save_file:
        save_index(idx, os.path.join(HERE, f"{name}.ivfpq"))
    print(name, "lists", idx.nlist, "N", ids.shape[0], "pairs", len(pairs))


def codec():
    rng = np.random.default_rng(2024)
    xs = [np.float32([0.0, 1.0, 1.3, 2.0 ** 20, 65504.0, 65520.0, 1e9, 122880.0, 496.0,
                      2.0 ** -14, 2.0 ** -6, 1e-30, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11])]
    xs.append(np.nextafter(np.float32([122880.0, 496.0]), np.float32(np.inf)))
    xs.append(np.nextafter(np.float32([2.0 ** -14, 2.0 ** -6]), np.float32(0.0)))
    xs.append(np.exp2(rng.uniform(-30, 24, 20000)).astype(np.float32))
    xs.append(rng.random(5000).astype(np.float32))
    xs.append(np.arange(0x0001, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float32))  # all f16 finite > 0
    xs.append(rng.integers(0, 0x7F800000, 20000, dtype=np.uint32).view(np.float32))  # random finite bit patterns
    x = np.concatenate(xs).astype(np.float32)
    out = dict(x=x, f16=minifloat.encode_f16_array(x))
    for name, spec in (("e5m3", minifloat.E5M3), ("e4m4", minifloat.E4M4)):
        out[name] = minifloat.encode_array(x, spec)
        out[f"table_{name}"] = minifloat.decode_table(spec)
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **out)
    print("codec", x.shape[0])


def pq_encode_golden():
    """pq_encode (pq.py:92-110) on inputs that stress its rounding: residual
    sub-vectors at exact codewords (dist clipped at 0), one ulp off them, at
    midpoints of codeword pairs, duplicated codewords (ties -> lower code),
    plus random rows.  `exact64` counts rows where a float64 argmin would
    disagree -- proof the fixture discriminates the fp32 recipe."""
    rng = np.random.default_rng(77)
    out = {}
    for sub, p in [(1, 8), (2, 8), (3, 8), (4, 8), (4, 5), (2, 6)]:
        s, n_codes = 12, 1 << p
        C = (rng.standard_normal((s, n_codes, sub)) * 0.3).astype(np.float32)
        C[:, n_codes - 1] = C[:, 3]          # duplicated codeword
        C[:, 7] = C[:, 2] * np.float32(1.0000001)
        rows = []
        n = 500
        X = (rng.standard_normal((n, s * sub)) * 0.3).astype(np.float32)
        rows.append(X)
        pick = rng.integers(0, n_codes, (n, s))
        Xc = np.stack([C[j, pick[:, j]] for j in range(s)], 1).reshape(n, -1)
        rows.append(Xc)                                                  # exact codewords
        rows.append(np.nextafter(Xc, np.float32(np.inf)))                # one ulp off
        pick2 = rng.integers(0, n_codes, (n, s))
        Xm = np.stack([(C[j, pick[:, j]] + C[j, pick2[:, j]]) * np.float32(0.5) for j in range(s)], 1).reshape(n, -1)
        rows.append(Xm.astype(np.float32))                               # midpoints
        X = np.ascontiguousarray(np.concatenate(rows).astype(np.float32))
        codes = pq_encode(X, PQCodebook(centers=C, p=p))
        # float64 argmin (direct form) for the discrimination count
        d64 = ((X.reshape(X.shape[0], s, 1, sub).astype(np.float64) - C[None].astype(np.float64)) ** 2).sum(3)
        exact64 = int((d64.argmin(2) != codes).sum())
        key = f"sub{sub}_p{p}"
        out[f"{key}_x"], out[f"{key}_centers"], out[f"{key}_codes"] = X, C, codes
        out[f"{key}_exact64"] = np.int64(exact64)
        print("pq_encode", key, X.shape, "rows differing from a float64 argmin:", exact64)
    # fused residual path: data - coarse[assign] (compute_residuals, pq.py:54-63)
    data = synth_gaussian_mixture(3000, 24, 8, 0.3, seed=15)
    coarse = data[rng.choice(3000, 16, replace=False)].copy()
    assign, d2 = assign_to_centroids(data, coarse)
    res = compute_residuals(data, coarse, assign)
    C = (rng.standard_normal((8, 256, 3)) * 0.2).astype(np.float32)
    out.update(res_data=data, res_coarse=coarse, res_assign=assign, res_d2=d2, res_centers=C,
               res_codes=pq_encode(res, PQCodebook(centers=C, p=8)))
    np.savez_compressed(os.path.join(HERE, "pq_encode.npz"), **out)


def main():
    if sys.argv[1:] == ["--only", "pq_encode"]:
        pq_encode_golden()
        return
    codec()
    pq_encode_golden()

    # test_search.py:23-26 small_index + queries of test_search.py:202
    data = synth_gaussian_mixture(2000, 16, 8, 0.05, seed=21)
    idx = build_index(data, nlist=16, s=8, p=8, seed=3)
    q = synth_gaussian_mixture(20, 16, 8, 0.05, seed=22)
    dump_case("small", idx, q, [(10, 1), (10, 4), (10, 16), (2000, 16)], save_file=True)

    # p=6 codebook (test_search.py:29-33), random rq LUTs only
    rng = np.random.default_rng(31)
    cb = train_pq(rng.standard_normal((2000, 16)).astype(np.float32), s=8, p=6, seed=4)
    rqs = np.random.default_rng(2).standard_normal((4, 16)).astype(np.float32)
    rqs[3] = np.concatenate([cb.centers[j, 5] for j in range(cb.s)])  # exact codeword row
    out = dict(centers=cb.centers, rq=rqs)
    for i in range(rqs.shape[0]):
        for prec in PRECS:
            out[f"lut_{prec}_{i}"] = build_lut(cb, rqs[i], prec).entries
    np.savez_compressed(os.path.join(HERE, "codebook_p6.npz"), **out)

    # test_search.py:232-244: two far-apart blobs, short rows
    rng = np.random.default_rng(9)
    blobs = np.vstack([rng.normal(0, 0.01, (16, 4)), rng.normal(100, 0.01, (16, 4))]).astype(np.float32)
    idx = build_index(blobs, nlist=2, s=2, p=4, seed=0)
    dump_case("blobs", idx, np.zeros((2, 4), np.float32) + np.float32([[0], [100]]), [(20, 1), (40, 2)])

    # sub_d = 3 and p = 5 shapes (cfg5 / cfg3-p5 style), desk scale
    data = synth_gaussian_mixture(3000, 24, 8, 0.3, seed=5)
    idx = build_index(data, nlist=16, s=8, p=5, seed=1)
    q = synth_gaussian_mixture(30, 24, 8, 0.3, seed=6)
    dump_case("sub3_p5", idx, q, [(10, 3), (100, 8)])

    # SIFT-shaped (d=128, s=64, p=8) at desk scale, base/queries from one draw
    x = synth_gaussian_mixture(20_300, 128, 16, 0.3, seed=1)
    idx = build_index(x[:20_000], nlist=64, s=64, p=8, seed=0)
    dump_case("sift_mini", idx, x[20_000:20_100], [(10, 8), (100, 4)])
    gt = brute_force_knn(x[:20_000], x[20_000:20_100], 10)
    np.savez_compressed(os.path.join(HERE, "sift_mini_gt.npz"), ids=gt.ids, d=gt.distances)


if __name__ == "__main__":
    main()
