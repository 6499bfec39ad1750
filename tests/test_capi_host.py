"""CPU-side checks: the C-ABI library loads and exports every symbol the header
declares; host validation raises the reference's ValueErrors before any
device work; IVFPQ001 persistence is byte-compatible with the reference."""

import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, index_from_case, load_case

import paper_2301_06672_b200 as pkg
from paper_2301_06672_b200 import _lib
from paper_2301_06672_b200.search import SearchParams, search_batch, select_clusters, build_lut, scan_list, Lut
from paper_2301_06672_b200.validation import check_matrix, check_vector


def header_functions():
    text = open(os.path.join(ROOT, "include", "ivfpq_b200.h")).read()
    return sorted(set(re.findall(r"\b(ivfpq_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported_and_bound():
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(_lib.lib, n), n
        assert n in _lib.SIGNATURES, n
    assert set(_lib.SIGNATURES) == set(names)


def test_library_is_sm100a_build():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_device_count_and_limits():
    assert _lib.device_count() >= 0
    assert _lib.max_k() >= 1024
    assert _lib.lib.ivfpq_version() >= 1


def test_search_params_validation():
    with pytest.raises(ValueError):
        SearchParams(k=0)
    with pytest.raises(ValueError):
        SearchParams(nprobe=0)
    with pytest.raises(ValueError, match="unknown LUT precision"):
        SearchParams(precision="f64")


def test_validation_messages():
    with pytest.raises(ValueError, match="2-dimensional"):
        check_matrix(np.zeros(3))
    with pytest.raises(ValueError, match="at least one row"):
        check_matrix(np.zeros((0, 3)))
    with pytest.raises(ValueError, match="non-finite"):
        check_matrix(np.array([[np.nan, 1.0]]))
    with pytest.raises(ValueError, match="length"):
        check_vector(np.zeros(3), 4)


def test_search_rejects_bad_arguments_before_device_work():
    idx = index_from_case(load_case("small"))
    q = np.zeros((2, idx.d + 1), np.float32)
    with pytest.raises(ValueError, match="queries have d="):
        search_batch(idx, q, SearchParams(k=3, nprobe=2))
    with pytest.raises(ValueError, match="nprobe"):
        search_batch(idx, np.zeros((2, idx.d), np.float32), SearchParams(k=3, nprobe=idx.nlist + 1))
    with pytest.raises(ValueError, match="nprobe"):
        select_clusters(idx, np.zeros(idx.d, np.float32), idx.nlist + 1)
    with pytest.raises(ValueError, match="length"):
        build_lut(idx.cb, np.zeros(idx.d - 1, np.float32), "f32")
    with pytest.raises(ValueError, match="unknown LUT precision"):
        build_lut(idx.cb, np.zeros(idx.d, np.float32), "f64")
    with pytest.raises(ValueError, match="out of range"):
        scan_list(np.array([0]), np.array([[8, 0]], dtype=np.uint8), Lut(np.zeros((2, 8), np.float32), "f32"))


def test_ivfpq001_roundtrip_is_byte_identical(tmp_path):
    ref_path = os.path.join(GOLDEN, "small.ivfpq")
    idx = pkg.load_index(ref_path)
    c = load_case("small")
    assert np.array_equal(idx.coarse, c["coarse"]) and np.array_equal(idx.cb.centers, c["centers"])
    off, ids, codes = idx.csr()
    assert np.array_equal(off, c["list_off"]) and np.array_equal(ids, c["ids"]) and np.array_equal(codes, c["codes"])
    out = tmp_path / "again.ivfpq"
    pkg.save_index(idx, out)
    assert open(ref_path, "rb").read() == open(out, "rb").read()


def test_load_index_rejects_corruption(tmp_path):
    blob = open(os.path.join(GOLDEN, "small.ivfpq"), "rb").read()
    bad = tmp_path / "bad.ivfpq"
    bad.write_bytes(b"XXXXXXXX" + blob[8:])
    with pytest.raises(ValueError, match="magic"):
        pkg.load_index(bad)
    bad.write_bytes(blob[:-3])
    with pytest.raises(ValueError, match="truncated"):
        pkg.load_index(bad)
    bad.write_bytes(blob + b"\0")
    with pytest.raises(ValueError, match="trailing"):
        pkg.load_index(bad)


def test_index_validate():
    idx = index_from_case(load_case("small"))
    idx.validate()
    c = load_case("small")
    ids = c["ids"].copy()
    ids[0] = ids[1]
    bad = type(idx).from_csr(c["coarse"], idx.cb, c["list_off"], ids, c["codes"])
    with pytest.raises(ValueError):
        bad.validate()


def test_product_package_does_not_import_oracle():
    pkgdir = os.path.join(ROOT, "paper_2301_06672_b200")
    for dirpath, _, files in os.walk(pkgdir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).replace("oracle/", ""), f


def test_no_fma_contraction_in_device_code():
    """Bit-exactness needs every fp32 op rounded on its own (the reference runs
    one numpy ufunc per op): no FFMA/FFMA2 may appear in the shipped SASS."""
    import subprocess
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "FADD" in sass and "LDS" in sass
    # per function: only the ingest kernels may hold FMAs -- there the FMA is
    # the reference's own arithmetic (OpenBLAS sgemm, csrc/ingest.cuh)
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    assert len(funcs) > 10
    allowed = ("pq_encode_kernel", "assign_kernel")
    for f in funcs:
        name = f.split("\n", 1)[0]
        if not any(a in name for a in allowed):
            assert "FFMA" not in f, name
