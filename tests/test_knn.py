"""K7 exact k-NN ground truth (datasets.py:179-201) on the GPU: ids and
distances bit-identical to the reference (golden) and to the C oracle,
including ties (duplicate rows -> lower id)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import c_oracle


@pytest.fixture(scope="module")
def pkg():
    import paper_2301_06672_b200 as pkg
    pkg._lib.require_gpu()
    return pkg


def test_knn_validation():
    import paper_2301_06672_b200 as pkg
    with pytest.raises(ValueError, match="exceeds base size"):
        pkg.brute_force_knn(np.zeros((3, 4), np.float32), np.zeros((1, 4), np.float32), 5)
    with pytest.raises(ValueError, match="dimension mismatch"):
        pkg.brute_force_knn(np.zeros((3, 4), np.float32), np.zeros((1, 5), np.float32), 1)


@pytest.mark.gpu
def test_knn_matches_reference_golden(pkg):
    gt = np.load(os.path.join(GOLDEN, "sift_mini_gt.npz"))
    x = pkg.synth_gaussian_mixture(20_300, 128, 16, 0.3, seed=1)
    res = pkg.brute_force_knn(x[:20_000], x[20_000:20_100], 10)
    assert np.array_equal(res.ids, gt["ids"])
    assert np.array_equal(res.distances, gt["d"])


@pytest.mark.gpu
@pytest.mark.parametrize("n,d,k", [(50_000, 96, 100), (3_000, 24, 7), (70_000, 128, 10)])
def test_knn_vs_oracle_with_ties(pkg, n, d, k):
    rng = np.random.default_rng(n + d)
    base = rng.random((n, d), dtype=np.float32)
    base[n // 2: n // 2 + 50] = base[10]             # exact duplicates: ties -> lower id
    q = rng.random((200, d), dtype=np.float32)
    q[0] = base[10]                                  # zero-distance ties
    res = pkg.brute_force_knn(base, q, k)
    ids, dists = c_oracle.brute_force_knn(base, q, k)
    assert np.array_equal(res.ids, ids)
    assert np.array_equal(res.distances, dists)
