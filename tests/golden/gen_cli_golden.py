"""Golden files for the benchmark CLI, written by running the reference's own CLI.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_cli_golden.py

Uses the reference test workspace recipe (reference tests/test_cli.py:11-20:
4 Gaussian centres, 2000 x 16 base, 40 queries) and the reference's
``ivfrabitq.cli.main`` for ``gt``, ``build`` and ``search`` (both modes,
two sweep points) and ``eval``.  The outputs land in tests/golden/cli/: the
reference-written IVRQ1 index ``toy.idx`` (searched by our GPU path in
tests/test_cli.py), the ground truth, the result ivecs and the CSV.
"""

from __future__ import annotations

import json
import shutil
import tempfile
from pathlib import Path

import numpy as np

from ivfrabitq.cli import main  # the reference
from ivfrabitq.io import write_fvecs

OUT = Path(__file__).resolve().parent / "cli"


def workspace(root: Path) -> None:
    rng = np.random.default_rng(0)
    centers = rng.normal(0, 2.0, (4, 16))
    base = np.vstack([rng.normal(c, 0.4, (500, 16)) for c in centers]).astype(np.float32)
    queries = np.vstack([rng.normal(c, 0.4, (10, 16)) for c in centers]).astype(np.float32)
    write_fvecs(str(root / "base.fvecs"), base)
    write_fvecs(str(root / "query.fvecs"), queries)


def run() -> None:
    OUT.mkdir(exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        t = Path(td)
        workspace(t)
        b, q = str(t / "base.fvecs"), str(t / "query.fvecs")
        assert main(["gt", "--base", b, "--query", q, "--k", "10", "--out-prefix", str(t / "gt")]) == 0
        assert main(["build", "--base", b, "--out", str(t / "toy.idx"), "--nk", "12", "--bits", "8",
                     "--seed", "3", "--iters", "8"]) == 0
        assert main(["build", "--base", b, "--out", str(t / "toy4.idx"), "--nk", "9", "--bits", "4",
                     "--seed", "1", "--iters", "5"]) == 0
        for idx, mode, probes, tag in (("toy.idx", "lut", "2,12", "res_lut"), ("toy.idx", "bitwise", "2,12", "res_bw"),
                                       ("toy4.idx", "bitwise", "2,9", "res4_bw")):
            assert main(["search", "--index", str(t / idx), "--query", q, "--k", "10", "--nprobe", probes,
                         "--mode", mode, "--out", str(t / tag)]) == 0
        assert main(["eval", "--results", str(t / "res_lut"), "--gt", str(t / "gt.ivecs"), "--k", "10",
                     "--csv", str(t / "out.csv")]) == 0
        for f in sorted(t.iterdir()):
            if f.suffix in (".fvecs", ".ivecs", ".idx", ".csv") or f.name.endswith(".meta.json"):
                shutil.copy(f, OUT / f.name)
    # result paths in the metadata are relative to the golden directory
    for m in OUT.glob("*.meta.json"):
        meta = json.loads(m.read_text())
        for s in meta["sweeps"]:
            s["results"] = Path(s["results"]).name
        m.write_text(json.dumps(meta, indent=2))


if __name__ == "__main__":
    run()
