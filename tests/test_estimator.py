"""IvfPq facade (reference estimator.py) and GPU build_index (index.py:73):
same API and validation; the facade's kneighbors equals search_batch on its
own index; recall against exact ground truth is in the reference's range."""

import numpy as np
import pytest


@pytest.fixture(scope="module")
def data():
    import paper_2301_06672_b200 as pkg
    X = pkg.synth_gaussian_mixture(2000, 16, 8, 0.05, seed=11)
    Q = pkg.synth_gaussian_mixture(50, 16, 8, 0.05, seed=12)
    return X, Q


def test_estimator_params_and_unfitted(data):
    from sklearn.exceptions import NotFittedError
    import paper_2301_06672_b200 as pkg
    est = pkg.IvfPq(nlist=4, pq_dims=4, random_state=0)
    assert est.get_params()["nlist"] == 4
    with pytest.raises(NotFittedError):
        est.kneighbors(data[1])
    with pytest.raises(ValueError, match="2-dimensional"):
        est.fit(np.zeros(5, np.float32))


def test_build_index_validation():
    import paper_2301_06672_b200 as pkg
    with pytest.raises(ValueError, match="need at least"):
        pkg.build_index(np.zeros((10, 8), np.float32), nlist=16, s=4, p=8, seed=0)
    with pytest.raises(ValueError, match="not divisible"):
        pkg.build_index(np.zeros((300, 10), np.float32), nlist=4, s=4, p=4, seed=0)


@pytest.mark.gpu
def test_estimator_matches_search_batch_and_recall(data):
    import paper_2301_06672_b200 as pkg
    X, Q = data
    est = pkg.IvfPq(nlist=16, pq_dims=8, pq_bits=8, nprobe=4, lut_precision="e5m3", random_state=5)
    dist, ids = est.fit(X).kneighbors(Q, n_neighbors=7)
    lists, _ = pkg.search_batch(est.index_, Q, pkg.SearchParams(k=7, nprobe=4, precision="e5m3"))
    assert np.array_equal(ids, lists.ids) and np.array_equal(dist, lists.distances)
    assert est.n_features_in_ == 16
    assert np.all(np.diff(dist, axis=1) >= 0)
    est.index_.validate()
    gt = pkg.brute_force_knn(X, Q, 10)
    est2 = pkg.IvfPq(nlist=8, pq_dims=8, nprobe=8, random_state=2).fit(X)
    assert 0.5 < est2.score(Q, gt.ids) <= 1.0
