"""GPU parity: the sm_100a path vs the reference's golden outputs and the CPU
oracle, through the C ABI.  Bit-exact everywhere: codec bytes, LUT entries,
R, probe sets, ids and distances (tolerance 0 -- the kernels reproduce the
reference's fp32 operation order)."""

import os

import numpy as np
import pytest

from conftest import CASES, GOLDEN, PRECS, index_from_case, load_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2301_06672_b200 as p
    from paper_2301_06672_b200 import _lib

    if _lib.device_count() < 1:
        pytest.fail("no CUDA device visible: GPU tests must run on the B200 box")
    return p


@pytest.fixture(params=["auto", "v1", "chunked", "layoutA", "layoutB"])
def scan_kernel(request, pkg):
    """Run a test with the persistent warp-specialised scan (auto), with the
    per-query scan kernel (v1), with the persistent kernel preferring
    row-chunked LUT jobs (partial sums carried between chunks) wherever the
    shape allows them, and with each warp layout forced (A: 8 builder + 11
    scanner warps; B: 4 + 15, built for the cfg4 / cfg5 / cfg3 p5 shapes)."""
    from paper_2301_06672_b200 import _lib
    mode = {"auto": 0, "v1": 1, "chunked": 2, "layoutA": 3, "layoutB": 4}[request.param]
    _lib.check(_lib.lib.ivfpq_set_scan_kernel(mode))
    yield request.param
    _lib.check(_lib.lib.ivfpq_set_scan_kernel(0))


@pytest.fixture(scope="module")
def codec():
    z = np.load(os.path.join(GOLDEN, "codec.npz"))
    return {k: z[k] for k in z.files}


# ---------------------------------------------------------------- codec ----
def test_fp8_codec_bit_exact(pkg, codec):
    for prec, spec in (("e5m3", pkg.E5M3), ("e4m4", pkg.E4M4)):
        from paper_2301_06672_b200 import minifloat as mf
        assert np.array_equal(mf.encode_array(codec["x"], spec), codec[prec])
        assert np.array_equal(mf.decode_table(spec), codec[f"table_{prec}"])


def test_f16_codec_bit_exact(pkg, codec):
    from paper_2301_06672_b200 import minifloat as mf
    assert np.array_equal(mf.encode_f16_array(codec["x"]), codec["f16"])
    bits = np.arange(0, 0x7C00, dtype=np.uint16)
    assert np.array_equal(mf.decode_f16_array(bits), bits.view(np.float16).astype(np.float32))


def test_fp8_codec_exhaustive_sweep(pkg):
    """Every 2^11-th finite non-negative fp32 pattern (~1M values) vs the closed form."""
    from paper_2301_06672_b200 import minifloat as mf
    from oracle import ivfpq_np as onp
    bits = np.arange(0, 0x7F800000, 2039, dtype=np.uint32)
    x = bits.view(np.float32)
    for prec, spec in (("e5m3", pkg.E5M3), ("e4m4", pkg.E4M4)):
        assert np.array_equal(mf.encode_array(x, spec), onp.fp8_encode(x, prec))
    assert np.array_equal(mf.encode_f16_array(x), onp.f16_encode(x))


def test_codec_known_answers(pkg):
    from paper_2301_06672_b200 import minifloat as mf
    E5M3, E4M4 = pkg.E5M3, pkg.E4M4
    assert mf.encode(0.0, E5M3) == 0x00 and mf.encode(1.0, E5M3) == 0x78
    assert mf.decode(0x78, E5M3) == 1.0 and mf.decode(0xFF, E5M3) == 122880.0
    assert mf.decode(mf.encode(1.3, E5M3), E5M3) == 1.25
    assert mf.encode(2.0 ** 20, E5M3) == 0xFF
    assert mf.encode(float(np.nextafter(np.float32(122880.0), np.float32(np.inf))), E5M3) == 0xFF
    assert mf.encode(float(np.nextafter(np.float32(2.0 ** -14), np.float32(0))), E5M3) == 0x00
    assert mf.encode(1e-30, E4M4) == 0x00
    for mant in range(8):
        assert mf.decode(mant, E5M3) == 0.0
    assert mf.encode_f16(1.0) == 0x3C00 and mf.encode_f16(65504.0) == 0x7BFF
    assert mf.encode_f16(1e9) == 0x7BFF and mf.encode_f16(65520.0) == 0x7BFF
    assert mf.encode_f16(1.0 + 2.0 ** -11) == 0x3C00 and mf.encode_f16(1.0 + 3 * 2.0 ** -11) == 0x3C02
    with pytest.raises(AssertionError):
        mf.encode(-1.0, E5M3)


# ------------------------------------------------------------ K2 / K3 -----
@pytest.mark.parametrize("name", CASES)
def test_build_lut_and_scan_bit_exact(pkg, name):
    c = load_case(name)
    idx = index_from_case(c)
    for n, (qi, cl) in enumerate(c["lut_pairs"]):
        rq = c["queries"][qi] - c["coarse"][cl]
        for prec in PRECS:
            lut = pkg.build_lut(idx.cb, rq, prec)
            assert np.array_equal(lut.entries, c[f"lut_{prec}_{n}"]), (name, n, prec)
            _, r = pkg.scan_list(idx.list_ids[cl], idx.list_codes[cl], lut)
            assert np.array_equal(r, c[f"scan_{prec}_{n}"]), (name, n, prec)


def test_build_lut_and_scan_hooks_beyond_smem(pkg):
    """s=240, p=8 (cfg3 shape): the f32 table is 240 KiB > shared memory, so the
    hooks build / gather it in global memory; bit-exact vs the C oracle."""
    from oracle import c_oracle
    rng = np.random.default_rng(240)
    cb = pkg.PQCodebook(centers=(rng.standard_normal((240, 256, 4)) * 0.3).astype(np.float32), p=8)
    rq = (rng.standard_normal(960) * 0.3).astype(np.float32)
    codes = rng.integers(0, 256, (700, 240)).astype(np.uint8)
    ids = np.arange(700, dtype=np.int64)
    for prec in PRECS:
        lut = pkg.build_lut(cb, rq, prec)
        assert np.array_equal(lut.entries, c_oracle.build_lut(cb.centers, rq, prec)), prec
        _, r = pkg.scan_list(ids, codes, lut)
        assert np.array_equal(r, c_oracle.scan(codes, lut.entries, prec)), prec


def test_build_lut_p6_codebook(pkg):
    z = np.load(os.path.join(GOLDEN, "codebook_p6.npz"))
    cb = pkg.PQCodebook(centers=z["centers"], p=6)
    for i in range(z["rq"].shape[0]):
        for prec in PRECS:
            lut = pkg.build_lut(cb, z["rq"][i], prec)
            assert np.array_equal(lut.entries, z[f"lut_{prec}_{i}"])
    # exact codeword row -> zero entries in every precision (test_search.py:97-101)
    for prec in PRECS:
        assert np.all(pkg.build_lut(cb, z["rq"][3], prec).decoded()[:, 5] == 0.0)


def test_scan_list_known_answers(pkg):
    lut = pkg.Lut(entries=np.arange(16, dtype=np.float32).reshape(1, 16), precision="f32")
    _, r = pkg.scan_list(np.array([0, 1]), np.array([[3], [9]], dtype=np.uint8), lut)
    assert r.tolist() == [3.0, 9.0]
    lut = pkg.Lut(entries=np.zeros((4, 16), np.float32), precision="f32")
    codes = np.random.default_rng(0).integers(0, 16, (5, 4)).astype(np.uint8)
    assert np.all(pkg.scan_list(np.arange(5), codes, lut)[1] == 0.0)


def test_scan_list_code_range_and_zero_exponent_entries(pkg):
    """Reference scan_list (search.py:130-142): the range check runs on the
    caller's array (codes >= n_codes raise even when they would wrap in
    uint8), negative codes index from the end as numpy does, and fp8 table
    codes 1..2^m-1 decode to 0.0 (minifloat.py:119-133)."""
    lut = pkg.Lut(entries=np.arange(16, dtype=np.float32).reshape(1, 16), precision="f32")
    with pytest.raises(ValueError, match="out of range"):
        pkg.scan_list(np.array([0]), np.array([[256 + 3]], dtype=np.int64), lut)
    _, r = pkg.scan_list(np.array([0, 1]), np.array([[-1], [-16]], dtype=np.int64), lut)
    assert r.tolist() == [15.0, 0.0]
    with pytest.raises(IndexError):
        pkg.scan_list(np.array([0]), np.array([[-17]], dtype=np.int64), lut)
    from oracle import ivfpq_np as onp
    rng = np.random.default_rng(11)
    for prec, m in (("e5m3", 3), ("e4m4", 4)):
        ent = rng.integers(0, 256, (8, 256)).astype(np.uint8)
        ent[:, :16] = np.arange(16, dtype=np.uint8)          # includes the zero-exponent codes 1..2^m-1
        codes = rng.integers(0, 256, (40, 8)).astype(np.uint8)
        codes[:, 0] = np.arange(40) % 16
        _, r = pkg.scan_list(np.arange(40), codes, pkg.Lut(entries=ent, precision=prec))
        ro = onp.scan_list(codes, ent, prec)
        assert np.array_equal(r, ro), prec


# ------------------------------------------------------------------ K4 ----
def test_top_k_duplicate_pairs(pkg):
    """Repeated (id, dist) pairs are all kept, like np.lexsort."""
    res = pkg.top_k(np.array([1, 1]), np.float32([0.5, 0.5]), k=2)
    assert res.ids.tolist() == [1, 1] and res.distances.tolist() == [0.5, 0.5]
    rng = np.random.default_rng(3)
    ids = rng.integers(0, 20, 300)
    d = rng.integers(0, 4, 300).astype(np.float32)
    res = pkg.top_k(ids, d, 50)
    o = np.lexsort((ids, d))[:50]
    assert res.ids.tolist() == ids[o].tolist() and res.distances.tolist() == d[o].tolist()


def test_top_k_known_answers(pkg):
    res = pkg.top_k(np.array([5, 2, 9]), np.float32([0.3, 0.1, 0.2]), k=10)
    assert res.ids.tolist() == [2, 9, 5] and res.short
    res = pkg.top_k(np.array([7, 3, 5, 1]), np.zeros(4, np.float32), k=2)
    assert res.ids.tolist() == [1, 3] and not res.short
    rng = np.random.default_rng(7)
    ids = rng.permutation(1000)
    d = rng.random(1000).astype(np.float32)
    d[rng.integers(0, 1000, 100)] = 0.5
    res = pkg.top_k(ids, d, 10)
    expect = sorted(zip(d.tolist(), ids.tolist()))[:10]
    assert res.ids.tolist() == [i for _, i in expect]
    assert res.distances.tolist() == [x for x, _ in expect]


# ------------------------------------------------------------------ K1 ----
@pytest.mark.parametrize("name", CASES)
def test_select_clusters_bit_exact(pkg, name):
    c = load_case(name)
    idx = index_from_case(c)
    P = c["select"].shape[1]
    for qi, q in enumerate(c["queries"]):
        assert np.array_equal(pkg.select_clusters(idx, q, P), c["select"][qi])
    with pytest.raises(ValueError, match="nprobe"):
        pkg.select_clusters(idx, c["queries"][0], idx.nlist + 1)


# ----------------------------------------------------------- end to end ---
@pytest.mark.parametrize("name", CASES)
def test_search_batch_bit_exact_vs_reference(pkg, name, scan_kernel):
    c = load_case(name)
    idx = index_from_case(c)
    for k, nprobe in c["runs"]:
        for prec in PRECS:
            tag = f"{prec}_k{k}_p{nprobe}"
            lists, n_short = pkg.search_batch(idx, c["queries"], pkg.SearchParams(k=int(k), nprobe=int(nprobe),
                                                                                  precision=prec))
            assert np.array_equal(lists.ids, c[f"ids_{tag}"]), (name, tag)
            assert np.array_equal(lists.distances, c[f"d_{tag}"]), (name, tag)
            assert n_short == int(c[f"short_{tag}"]), (name, tag)


def test_search_single_query_api(pkg):
    c = load_case("small")
    idx = index_from_case(c)
    res = pkg.search(idx, c["queries"][0], pkg.SearchParams(k=2000, nprobe=16, precision="f32"))
    assert np.array_equal(res.ids, c["ids_f32_k2000_p16"][0]) and not res.short
    blobs = index_from_case(load_case("blobs"))
    lists, n_short = pkg.search_batch(blobs, np.zeros((1, 4), np.float32), pkg.SearchParams(k=20, nprobe=1))
    assert n_short == 1 and (lists.ids[0] == -1).sum() == 4
    assert np.all(np.isinf(lists.distances[0][lists.ids[0] == -1]))


def _random_index(rng, n, d, s, p, nlist, empty_lists=()):
    from paper_2301_06672_b200.index import IvfPqIndex, PQCodebook
    coarse = rng.random((nlist, d)).astype(np.float32)
    centers = (rng.standard_normal((s, 1 << p, d // s)) * 0.3).astype(np.float32)
    assign = rng.integers(0, nlist, n)
    for e in empty_lists:
        assign[assign == e] = (e + 1) % nlist
    order = np.argsort(assign, kind="stable")
    off = np.searchsorted(assign[order], np.arange(nlist + 1)).astype(np.int64)
    codes = rng.integers(0, 1 << p, (n, s)).astype(np.uint8)[order]
    return IvfPqIndex.from_csr(coarse, PQCodebook(centers=centers, p=p), off, order.astype(np.int64), codes)


@pytest.mark.parametrize("shape", [
    dict(n=30000, d=128, s=64, p=8, nlist=64, P=8, k=10),        # SIFT-shaped, multi-block lists
    dict(n=20000, d=96, s=48, p=8, nlist=32, P=5, k=100),        # DEEP cfg4 shape, k=100
    dict(n=20000, d=96, s=32, p=8, nlist=32, P=6, k=10),         # cfg5 shape (sub_d = 3)
    dict(n=8000, d=120, s=24, p=5, nlist=16, P=4, k=10),         # p=5, s not a multiple of 16
    dict(n=5000, d=40, s=20, p=4, nlist=8, P=8, k=64),           # p=4, nprobe = nlist
    dict(n=6000, d=480, s=120, p=8, nlist=16, P=4, k=10),        # codebook beyond TMEM: builders read it from L2
    dict(n=4000, d=240, s=240, p=8, nlist=16, P=4, k=10),        # f32 LUT of 240 KiB > smem: global-scratch LUT
])
def test_search_batch_vs_c_oracle_random(pkg, shape, scan_kernel):
    from oracle import c_oracle
    rng = np.random.default_rng(shape["n"] + shape["s"])
    idx = _random_index(rng, shape["n"], shape["d"], shape["s"], shape["p"], shape["nlist"], empty_lists=(3,))
    q = rng.random((64, shape["d"])).astype(np.float32)
    off, ids, codes = idx.csr()
    for prec in PRECS:
        got, n_short = pkg.search_batch(idx, q, pkg.SearchParams(k=shape["k"], nprobe=shape["P"], precision=prec))
        want_ids, want_d, want_short = c_oracle.search_batch(idx.coarse, idx.cb.centers, off, ids, codes, q,
                                                             shape["k"], shape["P"], prec)
        assert np.array_equal(got.ids, want_ids), prec
        assert np.array_equal(got.distances, want_d), prec
        assert n_short == want_short


def test_search_device_api_matches_host_api(pkg):
    import torch
    c = load_case("sift_mini")
    idx = index_from_case(c)
    params = pkg.SearchParams(k=10, nprobe=8, precision="e5m3")
    host, _ = pkg.search_batch(idx, c["queries"], params)
    dev = pkg.device_index(idx)
    q = torch.from_numpy(c["queries"]).cuda()
    oi = torch.empty((q.shape[0], 10), dtype=torch.int64, device="cuda")
    od = torch.empty((q.shape[0], 10), dtype=torch.float32, device="cuda")
    osh = torch.empty(q.shape[0], dtype=torch.int32, device="cuda")
    pkg.search_device(dev, q, params, oi, od, osh)
    torch.cuda.synchronize()
    assert np.array_equal(oi.cpu().numpy(), host.ids)
    assert np.array_equal(od.cpu().numpy(), host.distances)


def test_recall_against_reference_gt(pkg):
    c = load_case("sift_mini")
    gt = np.load(os.path.join(GOLDEN, "sift_mini_gt.npz"))
    idx = index_from_case(c)
    r = {}
    for prec in PRECS:
        lists, _ = pkg.search_batch(idx, c["queries"], pkg.SearchParams(k=10, nprobe=8, precision=prec))
        r[prec] = pkg.recall(lists, pkg.NeighborLists(ids=gt["ids"]))[1]
    assert r["f32"] > 0.3
    assert abs(r["e5m3"] - r["f32"]) <= 0.05 and abs(r["e4m4"] - r["f32"]) <= 0.05


def test_sharded_protocol_emulated_on_one_gpu(pkg, scan_kernel):
    """The multi-GPU protocol with 3 list shards held as 3 handles on one GPU
    (run one after another; 'all-gather' = stack): bit-identical to 1 GPU."""
    import torch
    from paper_2301_06672_b200 import parallel
    from paper_2301_06672_b200.index import DeviceIndex
    c = load_case("sift_mini")
    idx = index_from_case(c)
    shards = parallel.shard_lists(np.diff(c["list_off"]), idx.cb.s, 3)
    ops = [parallel.CudaShardOps(DeviceIndex(idx, 0, owned=sh)) for sh in shards]
    q = torch.from_numpy(c["queries"]).cuda()
    for prec in PRECS:
        for k, P in ((10, 8), (100, 4)):
            ids, d, short = parallel.sharded_search(_StackOps(ops), q, k, P, prec, lambda t: t)
            assert np.array_equal(ids.cpu().numpy(), c[f"ids_{prec}_k{k}_p{P}"]), (prec, k, P)
            assert np.array_equal(d.cpu().numpy(), c[f"d_{prec}_k{k}_p{P}"]), (prec, k, P)
            assert int(short.sum()) == int(c[f"short_{prec}_k{k}_p{P}"])


class _StackOps:
    """Adapter: runs every shard's op and returns the stacked result, so that
    `all_gather` is the identity on the already-stacked tensors."""

    def __init__(self, ops):
        self.ops = ops

    def select(self, q, P):
        import torch
        return torch.stack([o.select(q, P) for o in self.ops])

    def merge(self, stacked, n):
        return self.ops[0].merge(stacked, n)

    def scan(self, q, probes, P, k, prec):
        import torch
        outs = [o.scan(q, probes, P, k, prec) for o in self.ops]
        for o in outs[1:]:
            assert torch.equal(o[1], outs[0][1])
        return torch.stack([o[0] for o in outs]), outs[0][1]

    def finalize(self, keys, ncand, k):
        return self.ops[0].finalize(keys, ncand, k)


def test_device_search_on_side_stream(pkg):
    import torch
    c = load_case("sift_mini")
    idx = index_from_case(c)
    params = pkg.SearchParams(k=10, nprobe=8, precision="f16")
    dev = pkg.device_index(idx)
    q = torch.from_numpy(c["queries"]).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        oi = torch.full((q.shape[0], 10), 7, dtype=torch.int64, device="cuda")
        od = torch.empty((q.shape[0], 10), dtype=torch.float32, device="cuda")
        osh = torch.empty(q.shape[0], dtype=torch.int32, device="cuda")
        pkg.search_device(dev, q, params, oi, od, osh)
        got = oi.cpu().numpy()
    assert np.array_equal(got, c["ids_f16_k10_p8"])


def test_device_search_alternating_streams(pkg):
    """Back-to-back calls on one index from two streams share its scratch;
    the second call waits for the first (stream-ordered), so both results
    are intact."""
    import torch
    c = load_case("sift_mini")
    idx = index_from_case(c)
    dev = pkg.device_index(idx)
    q = torch.from_numpy(c["queries"]).cuda()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for rep in range(3):
        for i, prec in enumerate(("e5m3", "f32")):
            with torch.cuda.stream(streams[i]):
                oi = torch.empty((q.shape[0], 10), dtype=torch.int64, device="cuda")
                od = torch.empty((q.shape[0], 10), dtype=torch.float32, device="cuda")
                osh = torch.empty(q.shape[0], dtype=torch.int32, device="cuda")
                pkg.search_device(dev, q, pkg.SearchParams(k=10, nprobe=8, precision=prec), oi, od, osh)
                outs.append((prec, oi))
    torch.cuda.synchronize()
    for prec, oi in outs:
        assert np.array_equal(oi.cpu().numpy(), c[f"ids_{prec}_k10_p8"]), prec


@pytest.mark.parametrize("nprobe,k", [(1, 10), (2, 5), (3, 100)])
def test_many_short_queries_reuse_query_state(pkg, nprobe, k):
    """Thousands of queries with 1-3 probed lists each: every persistent CTA
    cycles through many queries, exercising the per-query state ring."""
    from oracle import c_oracle
    rng = np.random.default_rng(nprobe)
    idx = _random_index(rng, 40000, 64, 32, 8, 256)
    q = rng.random((6000, 64)).astype(np.float32)
    off, ids, codes = idx.csr()
    for prec in ("f32", "e5m3"):
        got, n_short = pkg.search_batch(idx, q, pkg.SearchParams(k=k, nprobe=nprobe, precision=prec))
        want_ids, want_d, want_short = c_oracle.search_batch(idx.coarse, idx.cb.centers, off, ids, codes, q, k,
                                                             nprobe, prec)
        assert np.array_equal(got.ids, want_ids), prec
        assert np.array_equal(got.distances, want_d), prec
        assert n_short == want_short


@pytest.mark.parametrize("nprobe", [1, 37, 64, 65, 200])
def test_select_clusters_fused_and_fallback_paths(pkg, nprobe):
    """nprobe <= 64 runs the fused distance+top-P kernel over centroid slices,
    larger nprobe the distance-tile + block-select path; both bit-exact."""
    from oracle import c_oracle
    rng = np.random.default_rng(nprobe)
    idx = _random_index(rng, 20000, 32, 8, 4, 2048)
    q = rng.random((50, 32)).astype(np.float32)
    q[1] = idx.coarse[5]                      # exact hit (distance 0)
    q[2] = (idx.coarse[7] + idx.coarse[9]) / 2  # near-tie
    for i in range(q.shape[0]):
        assert np.array_equal(pkg.select_clusters(idx, q[i], nprobe), c_oracle.select(idx.coarse, q[i], nprobe))
    off, ids, codes = idx.csr()
    got, _ = pkg.search_batch(idx, q, pkg.SearchParams(k=10, nprobe=nprobe, precision="e5m3"))
    want_ids, want_d, _ = c_oracle.search_batch(idx.coarse, idx.cb.centers, off, ids, codes, q, 10, nprobe, "e5m3")
    assert np.array_equal(got.ids, want_ids) and np.array_equal(got.distances, want_d)


def _select_batch(pkg, dev, q, nprobe):
    import torch
    from paper_2301_06672_b200 import _lib
    qt = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    out = torch.empty((q.shape[0], nprobe), dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib.ivfpq_select_device(dev.handle, qt.data_ptr(), q.shape[0], nprobe, out.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    keys = out.cpu().numpy().view(np.uint64)
    return (keys & np.uint64(0xffffffff)).astype(np.int64), (keys >> np.uint64(32)).astype(np.uint32).view(np.float32)


def _flagged(dev):
    from paper_2301_06672_b200 import _lib
    n = _lib.ctypes.c_int64()
    _lib.check(_lib.lib.ivfpq_debug_select_flagged(dev.handle, _lib.ctypes.byref(n)))
    return n.value


@pytest.fixture(params=["auto", "simt", "tc_all_fallback"])
def select_mode(request, pkg):
    from paper_2301_06672_b200 import _lib
    _lib.check(_lib.lib.ivfpq_set_select_kernel({"auto": 0, "simt": 1, "tc_all_fallback": 2}[request.param]))
    yield request.param
    _lib.check(_lib.lib.ivfpq_set_select_kernel(0))


@pytest.mark.parametrize("nlist,d,nq,P", [
    (4096, 128, 300, 32),    # cfg2 shape: tensor-core nomination + exact re-rank
    (1000, 96, 131, 8),      # partial centroid tile and query block
    (2048, 100, 257, 1),     # d not a multiple of 4 / of the 32-wide K chunk
    (700, 160, 64, 17),      # largest d with resident queries
    (4096, 128, 40, 32),     # few query blocks -> several centroid slices merged
    (8192, 96, 300, 64),     # cfg5-style nprobe 64: slices sized by P
    (4096, 96, 200, 96),     # largest nprobe on the tensor-core path
])
def test_select_tensor_core_path_bit_exact(pkg, select_mode, nlist, d, nq, P):
    """K1 on tcgen05 (TF32 nomination, exact re-rank, guard, exact re-do of
    flagged queries) returns the reference's probes and distances bit for bit;
    includes duplicated centroids (exact ties -> smaller id) and queries that
    sit on a centroid."""
    from oracle import c_oracle
    from paper_2301_06672_b200.index import DeviceIndex
    rng = np.random.default_rng(nlist + d + nq)
    idx = _random_index(rng, 4 * nlist, d, d // 4 if d % 4 == 0 else d // 2, 4, nlist)
    idx.coarse[10] = idx.coarse[3]        # exact duplicate centroids
    idx.coarse[nlist - 1] = idx.coarse[3]
    q = rng.random((nq, d)).astype(np.float32)
    q[0] = idx.coarse[3]
    q[1] = idx.coarse[nlist // 2] + 1e-7
    dev = DeviceIndex(idx, 0)
    got, got_d = _select_batch(pkg, dev, q, P)
    flagged = _flagged(dev)
    if select_mode == "auto":      # the tensor cores did the nominating, the re-do is rare
        assert 0 <= flagged <= max(2, nq // 50), flagged
    elif select_mode == "tc_all_fallback":
        assert flagged == nq
    else:
        assert flagged == -1
    for i in range(nq):
        want = c_oracle.select(idx.coarse, q[i], P)
        assert np.array_equal(got[i], want), (select_mode, i)
        wd = ((idx.coarse[want] - q[i]) ** 2).astype(np.float32)
        acc = np.zeros(P, np.float32)
        for t in range(d):
            acc = (acc + wd[:, t]).astype(np.float32)
        assert np.array_equal(got_d[i], acc), (select_mode, i)


def test_select_tensor_core_owned_shard(pkg, select_mode):
    """A list shard (owned subset, local -> global ids) through the tensor-core K1."""
    from oracle import c_oracle
    from paper_2301_06672_b200.index import DeviceIndex
    rng = np.random.default_rng(7)
    idx = _random_index(rng, 8000, 64, 16, 4, 1024)
    owned = np.sort(rng.choice(1024, 600, replace=False)).astype(np.int32)
    q = rng.random((200, 64)).astype(np.float32)
    dev = DeviceIndex(idx, 0, owned=owned)
    got, _ = _select_batch(pkg, dev, q, 16)
    for i in range(q.shape[0]):
        local = c_oracle.select(idx.coarse[owned], q[i], 16)
        assert np.array_equal(got[i], owned[local].astype(np.int64)), i
