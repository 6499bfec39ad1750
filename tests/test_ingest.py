"""Ingest path: pq_encode bit-exact vs the reference's
own outputs (tests/golden/pq_encode.npz, made by tests/golden/make_golden.py
with the reference package), coarse assignment at decision level, and the
device list builder against a reference-built index."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, load_case
from oracle import c_oracle

KEYS = ["sub1_p8", "sub2_p8", "sub3_p8", "sub4_p8", "sub4_p5", "sub2_p6"]


@pytest.fixture(scope="module")
def enc():
    z = np.load(os.path.join(GOLDEN, "pq_encode.npz"))
    return {k: z[k] for k in z.files}


# ---------------------------------------------------------------- CPU: oracle
@pytest.mark.parametrize("key", KEYS)
def test_oracle_pq_encode_matches_reference(enc, key):
    got = c_oracle.pq_encode(enc[f"{key}_x"], enc[f"{key}_centers"])
    assert np.array_equal(got, enc[f"{key}_codes"])


def test_fixture_discriminates_rounding(enc):
    """The fixture is full of near-ties: a float64 argmin disagrees with the
    reference's fp32 recipe on many rows, so bit-exact agreement is a real test."""
    assert all(int(enc[f"{k}_exact64"]) > 50 for k in KEYS)


def test_oracle_residual_path(enc):
    res = enc["res_data"] - enc["res_coarse"][enc["res_assign"]]
    assert np.array_equal(c_oracle.pq_encode(res, enc["res_centers"]), enc["res_codes"])


def test_pq_encode_validation():
    import paper_2301_06672_b200 as pkg
    cb = pkg.PQCodebook(centers=np.zeros((4, 16, 2), np.float32), p=4)
    with pytest.raises(ValueError, match="dimensions"):
        pkg.pq_encode(np.zeros((3, 9), np.float32), cb)


# ---------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def pkg():
    import paper_2301_06672_b200 as pkg
    pkg._lib.require_gpu()
    return pkg


@pytest.mark.gpu
@pytest.mark.parametrize("key", KEYS)
def test_pq_encode_bit_exact(pkg, enc, key):
    C = enc[f"{key}_centers"]
    cb = pkg.PQCodebook(centers=C, p=int(np.log2(C.shape[1])))
    got = pkg.pq_encode(enc[f"{key}_x"], cb)
    assert np.array_equal(got, enc[f"{key}_codes"])
    one = pkg.pq_encode(enc[f"{key}_x"][5], cb)
    assert one.shape == (C.shape[0],) and np.array_equal(one, enc[f"{key}_codes"][5])


@pytest.mark.gpu
def test_fused_residual_encode_and_assign(pkg, enc):
    import torch
    x = torch.from_numpy(enc["res_data"]).cuda()
    coarse = torch.from_numpy(enc["res_coarse"]).cuda()
    a, d2 = pkg.ingest.assign_device(x, coarse)
    a = a.cpu().numpy()
    # decision-level parity (einsum's norm order at d=24 is not modelled)
    assert (a != enc["res_assign"]).mean() < 1e-3
    # expanded-form distances cancel near 0: absolute tolerance
    np.testing.assert_allclose(d2.cpu().numpy(), enc["res_d2"], rtol=1e-5, atol=1e-5)
    codes = pkg.ingest.pq_encode_device(x, torch.from_numpy(enc["res_centers"]).cuda(), 8, coarse,
                                        torch.from_numpy(enc["res_assign"]).cuda())
    assert np.array_equal(codes.cpu().numpy(), enc["res_codes"])
    a2, d22 = pkg.assign_to_centroids(enc["res_data"], enc["res_coarse"])
    assert np.array_equal(a2, a)


@pytest.mark.gpu
def test_populate_lists_matches_reference_build(pkg):
    """sift_mini was built by the reference's build_index (coarse + PQ trained
    by the reference); re-populating its lists from the same base rows on the
    GPU gives the same lists and bit-identical codes."""
    c = load_case("sift_mini")
    x = pkg.synth_gaussian_mixture(20_300, 128, 16, 0.3, seed=1)[:20_000]
    cb = pkg.PQCodebook(centers=c["centers"], p=int(c["p"]))
    idx = pkg.ingest.populate_lists(x, c["coarse"], cb)
    off, ids, codes = idx.csr()
    ref_list = np.empty(20_000, np.int64)
    ref_code = np.empty((20_000, cb.s), np.uint8)
    for l in range(c["list_off"].size - 1):
        sl = slice(c["list_off"][l], c["list_off"][l + 1])
        ref_list[c["ids"][sl]] = l
        ref_code[c["ids"][sl]] = c["codes"][sl].reshape(-1, cb.s)
    my_list = np.empty(20_000, np.int64)
    my_code = np.empty((20_000, cb.s), np.uint8)
    for l in range(off.size - 1):
        sl = slice(off[l], off[l + 1])
        my_list[ids[sl]] = l
        my_code[ids[sl]] = codes[sl].reshape(-1, cb.s)
        assert np.all(np.diff(ids[sl]) > 0)
    same = my_list == ref_list
    assert same.mean() > 0.999
    assert np.array_equal(my_code[same], ref_code[same])
