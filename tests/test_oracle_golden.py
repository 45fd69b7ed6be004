"""Pin the CPU oracle against the reference's own outputs (golden vectors).

These run without a GPU.  Integer/byte/index outputs must match exactly;
float outputs whose reference arithmetic is host independent (einsum-order
reductions, elementwise float64) must match exactly given identical inputs;
values that pass through an OpenBLAS GEMM in the reference are compared to
1e-12 relative (their last bits depend on the host's BLAS kernel).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import SEARCHES, case_params, golden_index_arrays, load_case, padded
from oracle import ivrq_oracle as orc


def test_reduction_orders_known_answers():
    with np.load("tests/golden/reductions.npz") as z:
        red = {k: z[k] for k in z.files}
    for d in (1, 7, 8, 13, 32, 96, 100, 128, 768, 1536):
        a, b = red[f"einsum_a_{d}"], red[f"einsum_b_{d}"]
        assert np.array_equal(orc.rowdot(a, b), red[f"einsum_ab_{d}"])
        assert np.array_equal(orc.rowdot(a, a), red[f"einsum_aa_{d}"])
        assert float(red[f"sum_v_{d}"].sum()) == float(red[f"sum_{d}"])


def test_oracle_kmeans_matches_reference(golden):
    p = case_params(golden)
    rows = golden["stage_train_rows"]
    xt = golden["x"][rows]
    pp = orc.seed_centres(xt.astype(np.float64), p["nlist"], np.random.default_rng(int(golden["stage_km_seed"])))
    np.testing.assert_array_equal(pp, golden["stage_pp_centers"])
    c = orc.kmeans(xt, p["nlist"], p["iters"], int(golden["stage_km_seed"]))
    np.testing.assert_allclose(c, golden["stage_centroids64"], rtol=1e-12, atol=1e-12)


def test_oracle_build_matches_reference(golden):
    p = case_params(golden)
    ix = orc.build(golden["x"], p["nlist"], p["bits"], p["iters"], p["train_fraction"], p["seed"])
    np.testing.assert_array_equal(ix["labels"], golden["stage_labels"])
    np.testing.assert_array_equal(ix["offsets"], golden["offsets"])
    np.testing.assert_array_equal(ix["pids"], golden["pids"])
    np.testing.assert_allclose(ix["rotation"], golden["rotation"], rtol=0, atol=1e-6)
    np.testing.assert_allclose(ix["centroids"], golden["centroids"], rtol=1e-6, atol=1e-6)


def test_oracle_encoder_given_reference_inputs(golden):
    """Codes, planes, ex-codes and factors are bit-exact given identical o_rot / centroids."""
    p = case_params(golden)
    inject = dict(
        centroids64=golden["stage_centroids64"],
        rotation=golden["rotation"],
        cent_rot=golden["centroids"],
        o_rot=golden["stage_o_rot"],
    )
    ix = orc.build(golden["x"], p["nlist"], p["bits"], p["iters"], p["train_fraction"], p["seed"], inject=inject)
    np.testing.assert_array_equal(ix["codes"], golden["stage_codes"])
    np.testing.assert_array_equal(ix["packed_msb"], golden["packed_msb"])
    np.testing.assert_array_equal(ix["excodes"], golden["excodes"])
    np.testing.assert_array_equal(ix["dist"], golden["stage_dist"])
    np.testing.assert_array_equal(ix["short_factors"], golden["short_factors"])
    np.testing.assert_array_equal(ix["long_factors"], golden["long_factors"])
    np.testing.assert_array_equal(ix["pids"], golden["pids"])


def test_oracle_quantizer_t(golden):
    p = case_params(golden)
    off = golden["offsets"].astype(np.int64)
    for c in range(p["nlist"]):
        lo, hi = off[c], off[c + 1]
        if hi == lo:
            continue
        u, t = orc.quantize(golden["stage_o_rot"][lo:hi], p["bits"])
        np.testing.assert_array_equal(u, golden["stage_codes"][lo:hi])
        np.testing.assert_array_equal(t.astype(np.float32), golden["stage_t"][lo:hi])


@pytest.mark.parametrize("si", range(len(SEARCHES)))
def test_oracle_search_matches_reference(golden, si):
    sp = SEARCHES[si]
    if f"s{si}_ids" not in golden:
        pytest.skip("n_probe exceeds n_clusters for this case")
    ix = golden_index_arrays(golden)
    res = orc.search(golden["queries"], ix, q_rot=golden["q_rot"], **sp)
    ids, dists, cnt = padded(res, sp["k"])
    np.testing.assert_array_equal(cnt, golden[f"s{si}_counts"])
    np.testing.assert_array_equal(ids, golden[f"s{si}_ids"])
    np.testing.assert_allclose(dists, golden[f"s{si}_dists"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("si", [0, 1, 2])
def test_oracle_query_state(golden, si):
    sp = SEARCHES[si]
    if f"s{si}_qstate" not in golden:
        pytest.skip("n_probe exceeds n_clusters for this case")
    for i in range(golden["q_rot"].shape[0]):
        st = orc.query_state(golden["q_rot"][i], sp["ip_mode"], sp["query_bits"], float(golden["eps_bound"]))
        want = golden[f"s{si}_qstate"][i]
        assert st["sum_q"] == want[0]
        assert st["delta"] == want[1]
        assert st["code_sum"] == want[2]
        assert st["ip_margin"] == want[3]
        if sp["ip_mode"] == "bitwise":
            np.testing.assert_array_equal(st["planes"], golden[f"s{si}_planes"][i])
        else:
            if i < len(golden[f"s{si}_luts"]):
                np.testing.assert_array_equal(st["luts"], golden[f"s{si}_luts"][i])


def test_oracle_probe(golden):
    for si in range(len(SEARCHES)):
        if f"s{si}_probe_ids" not in golden:
            continue
        sel, d2 = orc.probe(golden["q_rot"], golden["centroids"], golden["centroid_sqnorms"], SEARCHES[si]["n_probe"])
        np.testing.assert_array_equal(sel, golden[f"s{si}_probe_ids"])
        np.testing.assert_allclose(d2, golden[f"s{si}_probe_d2"], rtol=1e-12, atol=1e-12)


def test_oracle_exact_knn_small():
    base = np.array([[0.0, 0.0], [1.0, 0.0], [3.0, 0.0]])
    ids, d = orc.exact_knn(base, np.array([[0.9, 0.0]]), 2)
    assert ids.tolist() == [[1, 0]]
    tie = np.array([[1.0, 0.0], [-1.0, 0.0], [1.0, 0.0]])
    ids, _ = orc.exact_knn(tie, np.zeros((1, 2)), 3)
    assert ids.tolist() == [[0, 1, 2]]


def test_golden_cases_cover_edge_shapes():
    names = {n: load_case(n) for n in ("b2_dup", "b4_d48")}
    # duplicated points: some list is empty or tiny; 48 dims: ragged last 32-dim group
    off = names["b2_dup"]["offsets"].astype(np.int64)
    assert np.diff(off).min() <= 1
    assert names["b4_d48"]["x"].shape[1] % 32 != 0
