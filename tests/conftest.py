"""Shared fixtures: golden vectors produced by the reference (tests/golden/gen_golden.py)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))

CASE_NAMES = ["b1_d32", "b4_d48", "b8_d128", "b3_d96", "b2_dup", "b6_d20", "b8_d768", "b4_d1536", "b4_d96_l512"]
# the headline-shape cases (D = 768 / 1536, nlist 512); slower on the CPU oracle
BIG_CASES = {"b8_d768", "b4_d1536", "b4_d96_l512"}

# must match SEARCHES in tests/golden/gen_golden.py
SEARCHES = [
    dict(k=10, n_probe=4, ip_mode="bitwise", query_bits=4, refine=True, prune=True),
    dict(k=10, n_probe=4, ip_mode="lut", query_bits=4, refine=True, prune=True),
    dict(k=5, n_probe=2, ip_mode="bitwise", query_bits=8, refine=True, prune=True),
    dict(k=7, n_probe=3, ip_mode="bitwise", query_bits=2, refine=False, prune=True),
    dict(k=10, n_probe=4, ip_mode="bitwise", query_bits=4, refine=True, prune=False),
    dict(k=40, n_probe=1, ip_mode="lut", query_bits=4, refine=True, prune=True),
    dict(k=10, n_probe=16, ip_mode="bitwise", query_bits=4, refine=True, prune=True),
    dict(k=10, n_probe=32, ip_mode="lut", query_bits=4, refine=True, prune=True),
]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


def load_case(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        g = {k: z[k] for k in z.files}
    if "x" not in g:  # seeded mixture, regenerated (tests/golden/datagen.py)
        sys.path.insert(0, str(GOLDEN))
        from datagen import mix_data

        kind, n, nq, dims, seed = (str(v) for v in g["gen"])
        assert kind == "mix"
        x, q = mix_data(int(n), int(nq), int(dims), int(seed))
        assert np.array_equal(q, g["queries"]), "regenerated queries differ from the stored ones"
        g["x"] = x
    return g


def case_params(g: dict) -> dict:
    nlist, bits, iters, seed = (int(v) for v in g["params"])
    return dict(nlist=nlist, bits=bits, iters=iters, seed=seed, train_fraction=float(g["train_fraction"]))


def golden_index_arrays(g: dict) -> dict:
    p = case_params(g)
    n, dims = g["x"].shape
    return dict(
        dims=dims, bits=p["bits"], n_clusters=p["nlist"], size=n, eps_bound=float(g["eps_bound"]),
        rotation=g["rotation"], centroids=g["centroids"], centroid_sqnorms=g["centroid_sqnorms"],
        offsets=g["offsets"], packed_msb=g["packed_msb"], excodes=g["excodes"],
        short_factors=g["short_factors"], long_factors=g["long_factors"], pids=g["pids"],
    )


def padded(results, k):
    ids = np.full((len(results), k), -1, dtype=np.int64)
    dists = np.full((len(results), k), np.inf)
    cnt = np.zeros(len(results), dtype=np.int32)
    for i, (a, b) in enumerate(results):
        ids[i, : len(a)] = a
        dists[i, : len(b)] = b
        cnt[i] = len(a)
    return ids, dists, cnt


@pytest.fixture(params=CASE_NAMES)
def golden(request):
    g = load_case(request.param)
    g["_name"] = request.param
    return g


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
