"""CLI (reference cli.py) and the vector containers: container round trips
and error exits on CPU; build -> gt -> search -> eval -> bench and
codec-dump on the GPU."""

import os

import numpy as np
import pytest

from conftest import GOLDEN


def test_vecio_roundtrip_and_errors(tmp_path):
    from paper_2301_06672_b200.datasets import NeighborLists
    from paper_2301_06672_b200 import vecio
    X = np.random.default_rng(0).random((7, 5), dtype=np.float32)
    vecio.write_fvecs(tmp_path / "x.fvecs", X)
    assert np.array_equal(vecio.read_vectors(tmp_path / "x.fvecs"), X)
    ids = np.arange(12).reshape(3, 4)
    vecio.write_ivecs(tmp_path / "r.ivecs", NeighborLists(ids=ids))
    assert np.array_equal(vecio.read_ivecs(tmp_path / "r.ivecs").ids, ids)
    (tmp_path / "b.bvecs").write_bytes(np.array([3], "<i4").tobytes() + bytes([1, 2, 255]))
    assert np.array_equal(vecio.read_vectors(tmp_path / "b.bvecs"), np.float32([[1, 2, 255]]))
    (tmp_path / "t.fvecs").write_bytes(np.array([4], "<i4").tobytes() + b"\0" * 7)
    with pytest.raises(ValueError, match="truncated"):
        vecio.read_vectors(tmp_path / "t.fvecs")
    with pytest.raises(ValueError, match="unknown vector container"):
        vecio.read_vectors(tmp_path / "x.txt")


def test_cli_errors_exit_1(tmp_path, capsys):
    from paper_2301_06672_b200 import cli
    rc = cli.main(["search", "--index", str(tmp_path / "missing.ivfpq"), "--queries", str(tmp_path / "q.fvecs"),
                   "--k", "5", "--nprobe", "2", "--out", str(tmp_path / "o.ivecs")])
    assert rc == 1 and "error:" in capsys.readouterr().err


@pytest.mark.gpu
def test_cli_codec_dump_matches_reference_table(capsys):
    from paper_2301_06672_b200 import cli
    z = np.load(os.path.join(GOLDEN, "codec.npz"))
    for fmt in ("e5m3", "e4m4"):
        assert cli.main(["codec-dump", "--format", fmt]) == 0
        lines = capsys.readouterr().out.strip().split("\n")
        assert lines[0] == "code,value" and len(lines) == 257
        vals = np.float32([float(l.split(",")[1]) for l in lines[1:]])
        assert np.array_equal(vals, z[f"table_{fmt}"])


@pytest.mark.gpu
def test_cli_build_gt_search_eval_bench(tmp_path, capsys):
    import paper_2301_06672_b200 as pkg
    from paper_2301_06672_b200 import cli, vecio
    X = pkg.synth_gaussian_mixture(3000, 16, 8, 0.05, seed=21)
    vecio.write_fvecs(tmp_path / "base.fvecs", X[:2900])
    vecio.write_fvecs(tmp_path / "q.fvecs", X[2900:])
    d = str(tmp_path)
    assert cli.main(["build", "--dataset", f"{d}/base.fvecs", "--nlist", "16", "--pq-dims", "8", "--out",
                     f"{d}/idx.ivfpq"]) == 0
    assert cli.main(["gt", "--dataset", f"{d}/base.fvecs", "--queries", f"{d}/q.fvecs", "--k", "10", "--out",
                     f"{d}/gt.ivecs"]) == 0
    assert cli.main(["search", "--index", f"{d}/idx.ivfpq", "--queries", f"{d}/q.fvecs", "--k", "10", "--nprobe",
                     "8", "--lut-precision", "e5m3", "--out", f"{d}/r.ivecs", "--distances-out", f"{d}/r.fvecs"]) == 0
    capsys.readouterr()
    assert cli.main(["eval", "--results", f"{d}/r.ivecs", "--gt", f"{d}/gt.ivecs"]) == 0
    out = capsys.readouterr().out.strip().split("\n")
    assert out[0] == "query,recall" and out[-1].startswith("mean,") and float(out[-1].split(",")[1]) > 0.5
    assert cli.main(["bench", "--index", f"{d}/idx.ivfpq", "--queries", f"{d}/q.fvecs", "--gt", f"{d}/gt.ivecs",
                     "--k", "10", "--nprobe-list", "2,8", "--precisions", "f32,e5m3", "--out", f"{d}/b.csv"]) == 0
    rows = open(f"{d}/b.csv").read().strip().split("\n")
    assert rows[0] == "precision,nprobe,k,mean_recall,queries_per_second,wall_time_ms" and len(rows) == 5
