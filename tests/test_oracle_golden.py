"""Pin the CPU oracle (numpy + C restatements) to golden vectors produced by
the reference package itself (tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from conftest import CASES, GOLDEN, PRECS, load_case
from oracle import c_oracle
from oracle import ivfpq_np as onp


@pytest.fixture(scope="module")
def codec():
    z = np.load(os.path.join(GOLDEN, "codec.npz"))
    return {k: z[k] for k in z.files}


def per_list(c):
    off = c["list_off"]
    s = c["centers"].shape[0]
    ids = [c["ids"][off[i]:off[i + 1]] for i in range(off.size - 1)]
    codes = [c["codes"][off[i]:off[i + 1]].reshape(-1, s) for i in range(off.size - 1)]
    return ids, codes


@pytest.mark.parametrize("prec", ["e5m3", "e4m4"])
def test_fp8_codec_matches_reference(codec, prec):
    assert np.array_equal(onp.fp8_encode(codec["x"], prec), codec[prec])
    assert np.array_equal(onp.fp8_decode(np.arange(256, dtype=np.uint8), prec), codec[f"table_{prec}"])
    lib = c_oracle.lib()
    sub = codec["x"][:5000]
    got = np.array([lib.orc_fp8_encode(float(v), c_oracle.PREC_CODE[prec]) for v in sub], dtype=np.uint8)
    assert np.array_equal(got, codec[prec][:5000])


def test_f16_codec_matches_reference(codec):
    assert np.array_equal(onp.f16_encode(codec["x"]), codec["f16"])
    lib = c_oracle.lib()
    x = codec["x"]
    pick = np.concatenate([np.arange(0, x.size, 7), np.arange(x.size - 300, x.size)])
    got = np.array([lib.orc_f16_encode(float(v)) for v in x[pick]], dtype=np.uint16)
    assert np.array_equal(got, codec["f16"][pick])


@pytest.mark.parametrize("name", CASES)
def test_lut_and_scan_match_reference(name):
    c = load_case(name)
    s = c["centers"].shape[0]
    for n, (qi, cl) in enumerate(c["lut_pairs"]):
        rq = c["queries"][qi] - c["coarse"][cl]
        lo, hi = c["list_off"][cl], c["list_off"][cl + 1]
        codes = c["codes"][lo:hi].reshape(-1, s)
        for prec in PRECS:
            want = c[f"lut_{prec}_{n}"]
            assert np.array_equal(onp.build_lut(c["centers"], rq, prec), want), (name, n, prec)
            assert np.array_equal(c_oracle.build_lut(c["centers"], rq, prec), want), (name, n, prec)
            r = c[f"scan_{prec}_{n}"]
            assert np.array_equal(onp.scan_list(codes, want, prec), r)
            assert np.array_equal(c_oracle.scan(codes, want, prec), r)


def test_codebook_p6_luts():
    z = np.load(os.path.join(GOLDEN, "codebook_p6.npz"))
    for i in range(z["rq"].shape[0]):
        for prec in PRECS:
            want = z[f"lut_{prec}_{i}"]
            assert np.array_equal(onp.build_lut(z["centers"], z["rq"][i], prec), want)
            assert np.array_equal(c_oracle.build_lut(z["centers"], z["rq"][i], prec), want)


@pytest.mark.parametrize("name", CASES)
def test_select_matches_reference(name):
    c = load_case(name)
    P = c["select"].shape[1]
    for qi, q in enumerate(c["queries"]):
        assert np.array_equal(onp.select_clusters(c["coarse"], q, P), c["select"][qi])
        assert np.array_equal(c_oracle.select(c["coarse"], q, P), c["select"][qi])


@pytest.mark.parametrize("name", CASES)
def test_search_batch_matches_reference(name):
    c = load_case(name)
    list_ids, list_codes = per_list(c)
    for k, nprobe in c["runs"]:
        for prec in PRECS:
            tag = f"{prec}_k{k}_p{nprobe}"
            ids, d, ns = c_oracle.search_batch(c["coarse"], c["centers"], c["list_off"], c["ids"], c["codes"],
                                               c["queries"], int(k), int(nprobe), prec)
            assert np.array_equal(ids, c[f"ids_{tag}"]), (name, tag)
            assert np.array_equal(d, c[f"d_{tag}"]), (name, tag)
            assert ns == int(c[f"short_{tag}"])
            if name != "sift_mini" or prec == "e5m3":   # numpy loop: keep the CPU suite short
                ids2, d2, ns2 = onp.search_batch(c["coarse"], c["centers"], list_ids, list_codes, c["queries"],
                                                 int(k), int(nprobe), prec)
                assert np.array_equal(ids2, c[f"ids_{tag}"]) and np.array_equal(d2, c[f"d_{tag}"])
                assert ns2 == int(c[f"short_{tag}"])


def test_brute_force_gt_matches_reference():
    c = load_case("sift_mini")
    gt = np.load(os.path.join(GOLDEN, "sift_mini_gt.npz"))
    # the GT base is not stored; check the C oracle against numpy on a slice
    rng = np.random.default_rng(0)
    base = rng.random((3000, 128)).astype(np.float32)
    q = rng.random((5, 128)).astype(np.float32)
    a = c_oracle.brute_force_knn(base, q, 10)
    b = onp.brute_force_knn(base, q, 10)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert gt["ids"].shape == (c["queries"].shape[0], 10)
