"""Benchmark CLI parity (reference cli.py:63-182, tests/test_cli.py).

The golden directory ``tests/golden/cli`` holds files written by the
reference's own CLI (tests/golden/gen_cli_golden.py): the workspace vectors,
its ground truth, two IVRQ1 indexes it built and its search results.  The GPU
tests run our CLI on those same files: ``gt`` and ``search`` over the
reference-written index must reproduce the reference's ivecs byte for byte.
"""

from __future__ import annotations

import csv
import json
import shutil

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2602_23999_b200.cli import CSV_HEADER, default_train_fraction, main, padded_ids, recall_at_k
from paper_2602_23999_b200.io import read_fvecs, read_ivecs, write_fvecs, write_ivecs

CLI = GOLDEN / "cli"


@pytest.fixture
def ws(tmp_path):
    for f in ("base.fvecs", "query.fvecs", "gt.ivecs", "toy.idx", "toy4.idx"):
        shutil.copy(CLI / f, tmp_path / f)
    return tmp_path


# ---------------------------------------------------------------- CPU


def test_recall_at_k_values():
    gt = np.arange(20).reshape(2, 10).astype(np.int32)
    assert recall_at_k(gt.copy(), gt, 10) == 1.0
    assert recall_at_k(gt + 100, gt, 10) == 0.0
    half = gt.copy()
    half[:, 5:] += 100
    assert recall_at_k(half, gt, 10) == 0.5
    pad = gt.copy()
    pad[:, 3:] = -1  # padded slots never match
    assert recall_at_k(pad, gt, 10) == 0.3
    dup = gt.copy()
    dup[:, 1] = dup[:, 0]  # a repeated id counts once
    assert recall_at_k(dup, gt, 10) == 0.9


def test_recall_rejects_mismatched_files():
    gt = np.zeros((3, 10), dtype=np.int32)
    with pytest.raises(ValueError):
        recall_at_k(np.zeros((2, 10), dtype=np.int32), gt, 10)
    with pytest.raises(ValueError):
        recall_at_k(np.zeros((3, 4), dtype=np.int32), gt, 10)


def test_helpers():
    assert default_train_fraction(2000, 12) == 200 / 2000
    assert default_train_fraction(2000, 50) == 500 / 2000
    assert default_train_fraction(100, 50) == 1.0
    res = [(np.array([4, 5, 6]), np.zeros(3)), (np.array([7]), np.zeros(1))]
    assert padded_ids(res, 2).tolist() == [[4, 5], [7, -1]]


def test_eval_reference_results_reproduce_reference_csv(ws):
    """eval over the reference's own result files gives the reference's CSV (qps column aside)."""
    for f in CLI.glob("res_lut*"):
        shutil.copy(f, ws / f.name)
    meta = json.loads((ws / "res_lut.meta.json").read_text())
    for s in meta["sweeps"]:
        s["results"] = str(ws / s["results"])
    (ws / "res_lut.meta.json").write_text(json.dumps(meta))
    assert main(["eval", "--results", str(ws / "res_lut"), "--gt", str(ws / "gt.ivecs"), "--k", "10",
                 "--csv", str(ws / "out.csv")]) == 0
    got = (ws / "out.csv").read_text().splitlines()
    want = (CLI / "out.csv").read_text().splitlines()
    assert got[0] == want[0] == CSV_HEADER
    for a, b in zip(got[1:], want[1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[:5] + fa[6:] == fb[:5] + fb[6:]


def test_eval_single_ivecs_file(ws):
    write_ivecs(str(ws / "copy.ivecs"), read_ivecs(str(ws / "gt.ivecs")))
    assert main(["eval", "--results", str(ws / "copy.ivecs"), "--gt", str(ws / "gt.ivecs"), "--k", "10",
                 "--csv", str(ws / "one.csv")]) == 0
    with open(ws / "one.csv") as f:
        rows = list(csv.DictReader(f))
    assert len(rows) == 1 and float(rows[0]["recall"]) == 1.0


def test_missing_file_is_an_error(tmp_path, capsys):
    assert main(["build", "--base", str(tmp_path / "missing.fvecs"), "--out", str(tmp_path / "x.idx")]) == 2
    assert capsys.readouterr().err.startswith("error:")


@pytest.mark.gpu
def test_bad_nprobe_list_is_an_error(ws):
    assert main(["search", "--index", str(ws / "toy.idx"), "--query", str(ws / "query.fvecs"), "--k", "5",
                 "--nprobe", ",", "--out", str(ws / "r")]) == 2


# ---------------------------------------------------------------- GPU


@pytest.mark.gpu
def test_gt_matches_reference_and_is_deterministic(ws):
    args = ["gt", "--base", str(ws / "base.fvecs"), "--query", str(ws / "query.fvecs"), "--k", "10",
            "--out-prefix", str(ws / "gt")]
    assert main(args) == 0
    first = (ws / "gt.ivecs").read_bytes()
    assert first == (CLI / "gt.ivecs").read_bytes()
    # distances: float64 GEMM sums differ from OpenBLAS's in the last bits, then round to float32
    np.testing.assert_allclose(read_fvecs(str(ws / "gt.fvecs")), read_fvecs(str(CLI / "gt.fvecs")), rtol=1e-6)
    assert main(args) == 0
    assert (ws / "gt.ivecs").read_bytes() == first


@pytest.mark.gpu
def test_gt_query_in_base(ws, tmp_path):
    base = read_fvecs(str(ws / "base.fvecs"))
    write_fvecs(str(tmp_path / "self.fvecs"), base[123][None, :])
    assert main(["gt", "--base", str(ws / "base.fvecs"), "--query", str(tmp_path / "self.fvecs"), "--k", "1",
                 "--out-prefix", str(tmp_path / "selfgt")]) == 0
    assert read_ivecs(str(tmp_path / "selfgt.ivecs"))[0, 0] == 123
    assert read_fvecs(str(tmp_path / "selfgt.fvecs"))[0, 0] == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("idx,mode,probes,tag", [
    ("toy.idx", "lut", "2,12", "res_lut"),
    ("toy.idx", "bitwise", "2,12", "res_bw"),
    ("toy4.idx", "bitwise", "2,9", "res4_bw"),
])
def test_search_on_reference_written_index_matches_reference(ws, idx, mode, probes, tag):
    """Our GPU search over an IVRQ1 file the reference wrote returns the reference's ivecs, byte for byte."""
    assert main(["search", "--index", str(ws / idx), "--query", str(ws / "query.fvecs"), "--k", "10",
                 "--nprobe", probes, "--mode", mode, "--out", str(ws / tag)]) == 0
    meta = json.loads((ws / f"{tag}.meta.json").read_text())
    ref = json.loads((CLI / f"{tag}.meta.json").read_text())
    assert {k: meta[k] for k in ("k", "bits", "index_bytes", "batch")} == \
        {k: ref[k] for k in ("k", "bits", "index_bytes", "batch")}
    for s, r in zip(meta["sweeps"], ref["sweeps"]):
        assert (s["sweep"], s["n_probe"], s["ip_mode"]) == (r["sweep"], r["n_probe"], r["ip_mode"])
        assert open(s["results"], "rb").read() == (CLI / r["results"]).read_bytes()


@pytest.mark.gpu
def test_loaded_reference_index_keeps_float32_eps_bound(ws):
    """A loaded file carries the float32-rounded eps_bound (reference tests/test_index.py:109)."""
    from paper_2602_23999_b200.index import load_index

    ix = load_index(str(ws / "toy.idx"))
    assert ix.eps_bound == float(np.float32(ix.eps_bound))
    assert ix.bits == 8 and ix.n_clusters == 12 and ix.size == 2000


@pytest.mark.gpu
def test_build_search_eval_pipeline(ws):
    """build -> gt -> search -> eval through our CLI (reference tests/test_cli.py:75-120); the
    index we build has the reference's list assignment and file size."""
    from paper_2602_23999_b200.index import load_index

    assert main(["build", "--base", str(ws / "base.fvecs"), "--out", str(ws / "mine.idx"), "--nk", "12",
                 "--bits", "8", "--seed", "3", "--iters", "8"]) == 0
    mine, ref = load_index(str(ws / "mine.idx")), load_index(str(ws / "toy.idx"))
    assert (ws / "mine.idx").stat().st_size == (ws / "toy.idx").stat().st_size
    assert np.array_equal(mine.offsets, ref.offsets) and np.array_equal(mine.pids, ref.pids)
    assert np.array_equal(mine.rotation, ref.rotation)
    assert main(["gt", "--base", str(ws / "base.fvecs"), "--query", str(ws / "query.fvecs"), "--k", "10",
                 "--out-prefix", str(ws / "gt")]) == 0
    assert main(["search", "--index", str(ws / "mine.idx"), "--query", str(ws / "query.fvecs"), "--k", "10",
                 "--nprobe", "2,12", "--mode", "lut", "--out", str(ws / "res")]) == 0
    meta = json.loads((ws / "res.meta.json").read_text())
    assert [s["n_probe"] for s in meta["sweeps"]] == [2, 12]
    assert meta["bits"] == 8 and meta["index_bytes"] > 0
    assert main(["eval", "--results", str(ws / "res"), "--gt", str(ws / "gt.ivecs"), "--k", "10",
                 "--csv", str(ws / "out.csv")]) == 0
    with open(ws / "out.csv") as f:
        rows = list(csv.DictReader(f))
    recalls = [float(r["recall"]) for r in rows]
    assert len(rows) == 2 and recalls[1] >= recalls[0] and recalls[1] >= 0.9
    assert rows[0]["ip_mode"] == "lut" and int(rows[0]["index_bytes"]) == meta["index_bytes"]
    # the reference's recall on its own index: within 0.002 (north star)
    want = [float(line.split(",")[4]) for line in (CLI / "out.csv").read_text().splitlines()[1:]]
    assert all(abs(a - b) <= 0.002 for a, b in zip(recalls, want))


@pytest.mark.gpu
def test_search_rerun_is_deterministic(ws, tmp_path):
    for out in ("runA", "runB"):
        assert main(["search", "--index", str(ws / "toy.idx"), "--query", str(ws / "query.fvecs"), "--k", "10",
                     "--nprobe", "3", "--out", str(tmp_path / out)]) == 0
    assert (tmp_path / "runA.np3.ivecs").read_bytes() == (tmp_path / "runB.np3.ivecs").read_bytes()


@pytest.mark.gpu
def test_search_dim_mismatch_is_an_error(ws, tmp_path):
    write_fvecs(str(tmp_path / "wrong.fvecs"), np.zeros((2, 9), dtype=np.float32))
    assert main(["search", "--index", str(ws / "toy.idx"), "--query", str(tmp_path / "wrong.fvecs"), "--k", "5",
                 "--nprobe", "2", "--out", str(tmp_path / "r")]) == 2
