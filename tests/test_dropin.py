"""Drop-in surface: the reference package's public names exist here with the
same behaviour, and the helpers outside the hot path
(record containers, squared_l2_to_all, compute_residuals, reconstruct,
IVFPQ001 load -> search) match the reference / oracle on the same inputs."""

import os
import warnings

import numpy as np
import pytest

from conftest import GOLDEN, PRECS, load_case

# reference __init__.py:1-86 minus the out-of-scope training / bank-model names
# (k-means / PQ training and the analytical bank model are not on
# the search path)
REFERENCE_NAMES = [
    "E4M4", "E5M3", "IvfPq", "IvfPqIndex", "LUT_PRECISIONS", "Lut", "MiniFloatSpec", "NeighborLists", "PQCodebook",
    "SearchParams", "brute_force_knn", "build_index", "build_lut", "compute_residuals", "decode", "decode_table",
    "encode", "load_index", "pq_encode", "read_bvecs", "read_fvecs", "read_ivecs", "recall", "reconstruct",
    "save_index", "scan_list", "search", "search_batch", "select_clusters", "synth_gaussian_mixture", "top_k",
    "write_fvecs", "write_ivecs",
]
DATASETS_NAMES = ["NeighborLists", "read_fvecs", "read_bvecs", "read_ivecs", "write_ivecs", "write_fvecs",
                  "read_vectors", "synth_gaussian_mixture", "squared_l2_to_all", "brute_force_knn"]


def test_reference_names_exported():
    import paper_2301_06672_b200 as pkg
    from paper_2301_06672_b200 import datasets, pq
    missing = [n for n in REFERENCE_NAMES if not hasattr(pkg, n)]
    assert not missing, missing
    assert [n for n in DATASETS_NAMES if not hasattr(datasets, n)] == []
    assert all(hasattr(pq, n) for n in ("PQCodebook", "compute_residuals", "pq_encode", "reconstruct"))


def test_record_containers_roundtrip_and_errors(tmp_path):
    from paper_2301_06672_b200 import datasets as D
    X = np.random.default_rng(0).random((7, 5)).astype(np.float32)
    D.write_fvecs(tmp_path / "x.fvecs", X)
    assert np.array_equal(D.read_fvecs(tmp_path / "x.fvecs"), X)
    assert np.array_equal(D.read_vectors(tmp_path / "x.fvecs"), X)
    ids = np.arange(12, dtype=np.int64).reshape(3, 4)
    D.write_ivecs(tmp_path / "r.ivecs", D.NeighborLists(ids=ids))
    assert np.array_equal(D.read_ivecs(tmp_path / "r.ivecs").ids, ids)
    rec = np.array([3, 0, 0, 0, 1, 2, 255], dtype=np.uint8)
    rec.tofile(tmp_path / "b.bvecs")
    b = D.read_bvecs(tmp_path / "b.bvecs")
    assert b.dtype == np.float32 and b.tolist() == [[1.0, 2.0, 255.0]]
    (tmp_path / "e.fvecs").write_bytes(b"")
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        e = D.read_fvecs(tmp_path / "e.fvecs")
    assert e.shape == (0, 0) and any("empty file" in str(x.message) for x in w)
    (tmp_path / "t.fvecs").write_bytes(np.int32(4).tobytes() + b"\0" * 9)
    with pytest.raises(ValueError, match="truncated"):
        D.read_fvecs(tmp_path / "t.fvecs")
    with pytest.raises(ValueError, match="int32 range"):
        D.write_ivecs(tmp_path / "big.ivecs", D.NeighborLists(ids=np.array([[2 ** 40]])))
    with pytest.raises(ValueError, match="unknown vector container"):
        D.read_vectors(tmp_path / "x.txt")


@pytest.mark.gpu
def test_squared_l2_to_all_bit_exact():
    from paper_2301_06672_b200.datasets import squared_l2_to_all
    rng = np.random.default_rng(5)
    base = rng.standard_normal((3001, 37)).astype(np.float32)
    q = rng.standard_normal(37).astype(np.float32)
    diff = base - q                                  # datasets.py:172-176, sequential over dimensions
    acc = np.zeros(base.shape[0], dtype=np.float32)
    for j in range(base.shape[1]):
        acc += diff[:, j] * diff[:, j]
    assert np.array_equal(squared_l2_to_all(base, q), acc)


@pytest.mark.gpu
def test_compute_residuals_and_reconstruct():
    import paper_2301_06672_b200 as pkg
    rng = np.random.default_rng(9)
    X = rng.standard_normal((500, 12)).astype(np.float32)
    C = rng.standard_normal((7, 12)).astype(np.float32)
    a = rng.integers(0, 7, 500)
    assert np.array_equal(pkg.compute_residuals(X, C, a), X - C[a])
    with pytest.raises(ValueError, match="out of range"):
        pkg.compute_residuals(X, C, np.full(500, 7))
    with pytest.raises(ValueError, match="one entry per data row"):
        pkg.compute_residuals(X, C, a[:10])
    cb = pkg.PQCodebook(centers=rng.standard_normal((4, 32, 3)).astype(np.float32), p=5)
    codes = rng.integers(0, 32, (50, 4)).astype(np.uint8)
    ref = np.concatenate([cb.centers[j, codes[:, j]] for j in range(4)], axis=1)
    assert np.array_equal(pkg.reconstruct(codes, cb), ref)
    assert np.array_equal(pkg.reconstruct(codes[3], cb), ref[3])
    with pytest.raises(ValueError, match="out of range"):
        pkg.reconstruct(np.full((1, 4), 40, np.uint8), cb)


@pytest.mark.gpu
def test_reference_written_index_file_search():
    """A reference-written IVFPQ001 file (tests/golden/small.ivfpq, made by
    tests/golden/make_golden.py) loads and searches to the reference's golden
    ids and distances."""
    import paper_2301_06672_b200 as pkg
    c = load_case("small")
    idx = pkg.load_index(os.path.join(GOLDEN, "small.ivfpq"))
    for prec in PRECS:
        for P in (1, 4, 16):
            lists, n_short = pkg.search_batch(idx, c["queries"], pkg.SearchParams(k=10, nprobe=P, precision=prec))
            assert np.array_equal(lists.ids, c[f"ids_{prec}_k10_p{P}"]), (prec, P)
            assert np.array_equal(lists.distances, c[f"d_{prec}_k10_p{P}"]), (prec, P)
