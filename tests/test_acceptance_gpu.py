"""The reference's acceptance workload and criteria on the GPU backend.

Workload: the reference's seeded mixture (reference tests/conftest.py:1-52: 50
anisotropic Gaussian blobs in 128 dims, 100K base vectors, 1000 queries, seed
20260810), restated below as test input; nlist 316, k-means 25 iterations,
train fraction 0.25, seed 1 (conftest.py:84-93).  Criteria follow
tests/test_acceptance.py:186-320 (5 space accuracy, 6 probe trade-off, 7
pruning safety, 8 LUT/bitwise parity, 9 schedule independence, 10 storage
formula, 11 save/load round trip, the recall-monotone invariant), and the GPU
search is compared id for id with the CPU oracle (oracle/ivrq_oracle.py) on
the same index.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import ivrq_oracle as orc

pytestmark = pytest.mark.gpu

import paper_2602_23999_b200 as iv  # noqa: E402

SEED = 20260810
N_BASE, N_QUERIES, DIMS, N_BLOBS, N_CLUSTERS, K = 100_000, 1_000, 128, 50, 316, 10


def make_dataset(n_base=N_BASE, n_queries=N_QUERIES, dims=DIMS, n_blobs=N_BLOBS, seed=SEED, tau=12.0):
    """The reference acceptance mixture: per-blob log-uniform sigma, random orientation, decaying axes."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, 1.0, (n_blobs, dims))
    sigmas = np.exp(rng.uniform(np.log(0.5), np.log(1.5), n_blobs))
    decay = np.exp(-np.arange(dims) / tau)
    weights = rng.dirichlet(np.full(n_blobs, 5.0))
    counts = rng.multinomial(n_base, weights)
    q_counts = rng.multinomial(n_queries, weights)
    parts, q_parts = [], []
    for j in range(n_blobs):
        basis, _ = np.linalg.qr(rng.standard_normal((dims, dims)))
        cov = basis * (sigmas[j] * decay)[np.newaxis, :]
        parts.append(centers[j] + rng.standard_normal((counts[j], dims)) @ cov.T)
        q_parts.append(centers[j] + rng.standard_normal((q_counts[j], dims)) @ cov.T)
    base = np.vstack(parts).astype(np.float32)
    rng.shuffle(base)
    queries = np.vstack(q_parts).astype(np.float32)
    rng.shuffle(queries)
    return base, queries


class Workload:
    def __init__(self):
        self.base, self.queries = make_dataset()
        self.gt = iv.exact_knn(self.base, self.queries, K)[0]
        self._ix, self._res = {}, {}

    def index(self, bits):
        if bits not in self._ix:
            p = iv.BuildParams(n_clusters=N_CLUSTERS, quant=iv.QuantizationParams(bits=bits), kmeans_iters=25,
                               train_fraction=0.25, seed=1)
            self._ix[bits] = iv.build_index(self.base, p)
        return self._ix[bits]

    def results(self, bits, mode="lut", n_probe=N_CLUSTERS, prune=True, workers=None):
        key = (bits, mode, n_probe, prune, workers)
        if key not in self._res:
            sp = iv.SearchParams(k=K, n_probe=n_probe, ip_mode=mode, prune=prune)
            self._res[key] = iv.search_batch(self.queries, self.index(bits), sp, workers=workers)
        return self._res[key]

    def recall(self, results):
        hits = sum(len(set(ids.tolist()) & set(t.tolist())) for (ids, _), t in zip(results, self.gt))
        return hits / (len(results) * K)


@pytest.fixture(scope="module")
def wl():
    return Workload()


def test_ground_truth_matches_oracle(wl):
    ids, _ = orc.exact_knn(wl.base, wl.queries[:40], K)
    np.testing.assert_array_equal(wl.gt[:40], ids)


def test_criterion_05_space_accuracy(wl):
    assert wl.recall(wl.results(bits=5)) >= 0.95
    assert wl.recall(wl.results(bits=7)) >= 0.99


def test_criterion_06_probe_tradeoff(wl):
    sweep = {p: wl.recall(wl.results(bits=8, n_probe=p)) for p in (8, 32, 64)}
    assert any(p < N_CLUSTERS // 4 and r >= 0.95 for p, r in sweep.items()), sweep


def test_criterion_07_pruning_safety(wl):
    pruned, unpruned = wl.results(bits=7), wl.results(bits=7, prune=False)
    diff = total = 0
    for (a, _), (b, _) in zip(pruned, unpruned):
        total += b.size
        diff += sum(1 for r in range(b.size) if r >= a.size or a[r] != b[r])
    assert diff / total <= 0.002


def test_criterion_08_backend_parity(wl):
    for p in (4, 16, 64, N_CLUSTERS):
        gap = abs(wl.recall(wl.results(bits=7, mode="lut", n_probe=p)) -
                  wl.recall(wl.results(bits=7, mode="bitwise", n_probe=p)))
        assert gap <= 0.005, (p, gap)


def test_criterion_09_schedule_independence(wl, monkeypatch):
    """Identical (ids, dists) across worker counts, host chunking of the batch and repeated runs."""
    ref = wl.results(bits=7, workers=1)
    others = [wl.results(bits=7, workers=w) for w in (4, 16)]
    monkeypatch.setenv("IVRQ_E2E_CHUNKS", "3")
    sp = iv.SearchParams(k=K, n_probe=N_CLUSTERS, ip_mode="lut")
    others.append(iv.search_batch(wl.queries, wl.index(7), sp))
    for other in others:
        for (ia, da), (ib, db) in zip(ref, other):
            assert np.array_equal(ia, ib) and np.array_equal(da, db)


def test_criterion_10_storage_formula(wl, tmp_path):
    for bits in (5, 7):
        ix = wl.index(bits)
        path = tmp_path / f"b{bits}.idx"
        iv.save_index(ix, str(path))
        formula = (ix.size * ix.dims * bits / 8 + 20 * ix.size + 8 * ix.size
                   + 4 * (ix.dims ** 2 + ix.n_clusters * ix.dims))
        assert abs(path.stat().st_size - formula) / formula <= 0.15


def test_criterion_11_serialization_round_trip(wl, tmp_path):
    ix = wl.index(7)
    path = tmp_path / "rt.idx"
    iv.save_index(ix, str(path))
    loaded = iv.load_index(str(path))
    sp = iv.SearchParams(k=K, n_probe=32)
    for (ia, da), (ib, db) in zip(iv.search_batch(wl.queries[:100], ix, sp),
                                  iv.search_batch(wl.queries[:100], loaded, sp)):
        assert np.array_equal(ia, ib) and np.array_equal(da, db)


def test_invariant_recall_monotone_in_probes(wl):
    recalls = [wl.recall(wl.results(bits=8, n_probe=p)) for p in (1, 2, 4, 8, 16, 32, 64, 128, 256, N_CLUSTERS)]
    assert all(b >= a for a, b in zip(recalls, recalls[1:])), recalls


def _arrays(ix):
    return {
        "dims": ix.dims, "bits": ix.bits, "n_clusters": ix.n_clusters, "size": ix.size, "eps_bound": ix.eps_bound,
        "rotation": ix.rotation, "centroids": ix.centroids.values, "centroid_sqnorms": ix.centroids.squared_norms,
        "offsets": ix.offsets, "packed_msb": ix.packed_msb, "excodes": ix.excodes,
        "short_factors": ix.short_factors, "long_factors": ix.long_factors, "pids": ix.pids,
    }


@pytest.mark.parametrize("bits,mode,n_probe", [(7, "lut", 32), (7, "bitwise", 32), (8, "bitwise", 16),
                                               (5, "lut", 64)])
def test_gpu_search_matches_oracle_id_for_id(wl, bits, mode, n_probe):
    """The acceptance index searched on the GPU and by the CPU oracle: same ids, same order."""
    ix = wl.index(bits)
    q = wl.queries[:60]
    got = iv.search_batch(q, ix, iv.SearchParams(k=K, n_probe=n_probe, ip_mode=mode))
    want = orc.search(q, _arrays(ix), K, n_probe, ip_mode=mode)
    for (a, b), (c, d) in zip(got, want):
        np.testing.assert_array_equal(a, c)
        np.testing.assert_allclose(b, d, rtol=1e-9)
