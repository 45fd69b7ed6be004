"""GPU parity: every CUDA stage against the reference's golden vectors and the oracle.

Bar (BASELINE.json north star): ids / labels / codes / planes bit-exact;
distances and factors within 1e-4 relative (we check much tighter where the
arithmetic allows); recall within 0.002.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import SEARCHES, case_params, golden_index_arrays, load_case, padded
from oracle import ivrq_oracle as orc

pytestmark = pytest.mark.gpu

import paper_2602_23999_b200 as iv  # noqa: E402
from paper_2602_23999_b200 import _device as dev  # noqa: E402
from paper_2602_23999_b200.clustering import Centroids, row_sqnorms, train_kmeans_device  # noqa: E402
from paper_2602_23999_b200.codec import encode_rows  # noqa: E402
from paper_2602_23999_b200.index import IvfRabitqIndex, build_index_device  # noqa: E402
from paper_2602_23999_b200.search import prepare_queries_device, search_device  # noqa: E402


def _index(g) -> IvfRabitqIndex:
    a = golden_index_arrays(g)
    return IvfRabitqIndex(
        dims=a["dims"], bits=a["bits"], n_clusters=a["n_clusters"], size=a["size"], eps_bound=a["eps_bound"],
        seed=int(g["params"][3]), rotation=a["rotation"], centroids=Centroids(a["centroids"]),
        offsets=a["offsets"], packed_msb=a["packed_msb"], excodes=a["excodes"],
        short_factors=a["short_factors"], long_factors=a["long_factors"], pids=a["pids"],
    )


def test_row_sqnorms_bit_exact_einsum_order():
    with np.load("tests/golden/reductions.npz") as z:
        red = {k: z[k] for k in z.files}
    for d in (1, 7, 8, 13, 32, 96, 100, 128, 768, 1536):
        a = red[f"einsum_a_{d}"]
        got = dev.to_host(row_sqnorms(dev.to_device(a)))
        np.testing.assert_array_equal(got, red[f"einsum_aa_{d}"])
        b32 = red[f"einsum_b_{d}"]
        got32 = dev.to_host(row_sqnorms(dev.to_device(b32)))
        np.testing.assert_array_equal(got32, np.einsum("ij,ij->i", b32, b32, dtype=np.float64))


def test_centroid_sqnorms_match_reference(golden):
    c = Centroids(golden["centroids"])
    np.testing.assert_array_equal(c.squared_norms, golden["centroid_sqnorms"])


def test_select_clusters_matches_reference(golden):
    c = Centroids(golden["centroids"])
    for si, sp in enumerate(SEARCHES):
        if f"s{si}_probe_ids" not in golden:
            continue
        ids, d2 = iv.select_clusters(golden["q_rot"], c, sp["n_probe"])
        np.testing.assert_array_equal(ids, golden[f"s{si}_probe_ids"])
        np.testing.assert_allclose(d2, golden[f"s{si}_probe_d2"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("si", [0, 1, 2, 3])
def test_query_state_matches_reference(golden, si):
    if f"s{si}_qstate" not in golden:
        pytest.skip("n_probe exceeds n_clusters")
    sp = iv.SearchParams(**SEARCHES[si])
    ix = _index(golden)
    scal, planes, luts, _ = prepare_queries_device(dev.to_device(golden["q_rot"]), ix, sp)
    scal = dev.to_host(scal)
    want = golden[f"s{si}_qstate"]
    np.testing.assert_array_equal(scal[:, 0], want[:, 0])  # sum_q (pairwise order)
    np.testing.assert_array_equal(scal[:, 1], want[:, 1])  # delta
    np.testing.assert_array_equal(scal[:, 2], want[:, 2])  # code_sum_q
    np.testing.assert_array_equal(scal[:, 3], want[:, 3])  # ip_margin
    if sp.ip_mode == "bitwise":
        np.testing.assert_array_equal(dev.to_host(planes).view(np.uint32), golden[f"s{si}_planes"])
    else:
        want_l = golden[f"s{si}_luts"]  # the fixture keeps the first 16 queries' tables
        np.testing.assert_array_equal(dev.to_host(luts)[: len(want_l)], want_l)


@pytest.mark.parametrize("si", range(len(SEARCHES)))
def test_scan_bit_exact_given_reference_q_rot(golden, si):
    """IDs bit-exact and distances to 1e-12 given the reference's rotated queries."""
    if f"s{si}_ids" not in golden:
        pytest.skip("n_probe exceeds n_clusters")
    sp = iv.SearchParams(**SEARCHES[si])
    ix = _index(golden)
    q_rot = dev.to_device(golden["q_rot"])
    res = search_device(None, ix, sp, q_rot=q_rot, with_stats=True)
    cnt = dev.to_host(res.counts)
    ids = dev.to_host(res.ids)
    dists = dev.to_host(res.dists)
    np.testing.assert_array_equal(cnt, golden[f"s{si}_counts"])
    np.testing.assert_array_equal(ids, golden[f"s{si}_ids"])
    np.testing.assert_allclose(dists, golden[f"s{si}_dists"], rtol=1e-12, atol=1e-12)
    # survivor counts agree with the oracle's stage-1 pruning
    stats = {}
    orc.search(golden["queries"], golden_index_arrays(golden), q_rot=golden["q_rot"], stats=stats, **SEARCHES[si])
    st = dev.to_host(res.stats)
    assert int(st[:, 0].sum()) == stats.get("probed", 0)
    assert int(st[:, 1].sum()) == stats.get("survivors", 0)


@pytest.mark.parametrize("si", [0, 1, 3])
def test_search_batch_end_to_end(golden, si):
    """Public API, GPU query rotation included: ids equal the reference's."""
    if f"s{si}_ids" not in golden:
        pytest.skip("n_probe exceeds n_clusters")
    sp = iv.SearchParams(**SEARCHES[si])
    res = iv.search_batch(golden["queries"], _index(golden), sp)
    ids, dists, cnt = padded(res, sp.k)
    np.testing.assert_array_equal(cnt, golden[f"s{si}_counts"])
    np.testing.assert_array_equal(ids, golden[f"s{si}_ids"])
    np.testing.assert_allclose(dists, golden[f"s{si}_dists"], rtol=1e-9, atol=1e-9)


def test_encoder_bit_exact_given_reference_inputs(golden):
    p = case_params(golden)
    o_rot = dev.to_device(golden["stage_o_rot"])
    dist = dev.to_device(golden["stage_dist"])
    cent_rot = dev.to_device(golden["centroids"])
    offsets = dev.to_device(golden["offsets"].astype(np.int64))
    out = encode_rows(o_rot, dist, cent_rot, offsets, iv.QuantizationParams(bits=p["bits"]), want_codes=True)
    np.testing.assert_array_equal(dev.to_host(out["codes"]), golden["stage_codes"])
    np.testing.assert_array_equal(dev.to_host(out["t"]).astype(np.float32), golden["stage_t"])
    np.testing.assert_array_equal(dev.to_host(out["packed_msb"]).view(np.uint32), golden["packed_msb"])
    sf = np.stack([dev.to_host(out[k]) for k in ("short_add", "short_scale", "short_err")], axis=1)
    np.testing.assert_array_equal(sf, golden["short_factors"])
    np.testing.assert_array_equal(dev.to_host(out["long_factors"]), golden["long_factors"])
    if p["bits"] > 1:
        from paper_2602_23999_b200.codec import codes_from_rcodes, excodes_from_rcodes

        rc = dev.to_host(out["rcodes"])
        np.testing.assert_array_equal(codes_from_rcodes(rc, golden["x"].shape[1], p["bits"]), golden["stage_codes"])
        np.testing.assert_array_equal(excodes_from_rcodes(rc, golden["x"].shape[1], p["bits"]), golden["excodes"])
    assert int(out["bad_rows"].item()) == 0


@pytest.mark.parametrize("bits", [1, 2, 3, 5, 8])
def test_quantize_batch_float64_rows_match_oracle(bits):
    rng = np.random.default_rng(bits)
    o = rng.standard_normal((300, 24))
    o /= np.linalg.norm(o, axis=1)[:, None]
    o[7] = 0.0
    u, t = iv.quantize_batch(o, iv.QuantizationParams(bits=bits))
    u_o, t_o = orc.quantize(o, bits)
    np.testing.assert_array_equal(u, u_o)
    np.testing.assert_array_equal(t, t_o)
    with pytest.raises(ValueError):
        iv.quantize_batch(np.ones((1, 4)), iv.QuantizationParams(bits=bits))


def test_kmeans_matches_reference(golden):
    p = case_params(golden)
    xt = golden["x"][golden["stage_train_rows"]]
    c = train_kmeans_device(dev.to_device(xt), p["nlist"], p["iters"], int(golden["stage_km_seed"]))
    np.testing.assert_allclose(dev.to_host(c), golden["stage_centroids64"], rtol=1e-12, atol=1e-12)


def test_assign_matches_reference(golden):
    c = Centroids(golden["stage_centroids64"], None)
    labels = iv.assign(golden["x"], c)
    np.testing.assert_array_equal(labels, golden["stage_labels"])


def test_build_bit_exact_given_reference_centroids_and_rotations(golden):
    p = case_params(golden)
    params = iv.BuildParams(
        n_clusters=p["nlist"], quant=iv.QuantizationParams(bits=p["bits"]), kmeans_iters=p["iters"],
        train_fraction=p["train_fraction"], seed=p["seed"],
    )
    inject = dict(
        centroids64=golden["stage_centroids64"], rotation=golden["rotation"], cent_rot=golden["centroids"],
        o_rot=golden["stage_o_rot"],
    )
    ix = build_index_device(dev.to_device(golden["x"]), params, inject=inject)
    for field in ("offsets", "pids", "packed_msb", "excodes", "short_factors", "long_factors"):
        np.testing.assert_array_equal(getattr(ix, field), golden[field], err_msg=field)


def test_build_full_pipeline_matches_reference(golden):
    """No injection: GPU k-means, assignment, rotation GEMMs and encoder."""
    p = case_params(golden)
    params = iv.BuildParams(
        n_clusters=p["nlist"], quant=iv.QuantizationParams(bits=p["bits"]), kmeans_iters=p["iters"],
        train_fraction=p["train_fraction"], seed=p["seed"],
    )
    keep: dict = {}
    ix = build_index_device(dev.to_device(golden["x"]), params, keep=keep)
    np.testing.assert_allclose(dev.to_host(keep["centers"]), golden["stage_centroids64"], rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(dev.to_host(keep["labels"]), golden["stage_labels"])
    np.testing.assert_array_equal(ix.pids, golden["pids"])
    np.testing.assert_array_equal(ix.offsets, golden["offsets"])
    # the rotation is the host's LAPACK QR (gen_rotation, linalg.py:25-40): the GPU box's
    # OpenBLAS may round a rare element of a large Q one ulp differently than the host that
    # generated the fixture (QR is parity-unpinned across machines)
    rot_ulp = np.abs(ix.rotation.view(np.int32).astype(np.int64) - golden["rotation"].view(np.int32).astype(np.int64))
    assert rot_ulp.max() <= 1 and (rot_ulp > 0).mean() < 1e-4
    # float64-accumulated rotations round to float32 like the reference's GEMMs
    # except for rare last-ulp cases; codes follow from o_rot
    o_rot = dev.to_host(keep["o_rot"])
    ulp = np.abs(o_rot.view(np.int32).astype(np.int64) - golden["stage_o_rot"].view(np.int32).astype(np.int64))
    if rot_ulp.max() == 0:
        assert ulp.max() <= 1
    else:  # a rotation element differs by one ulp on this host: o_rot moves by ~2^-24 absolute
        assert np.abs(o_rot - golden["stage_o_rot"]).max() <= 2.0**-22
    assert (ulp > 1).mean() < 1e-3
    # cent_rot: the reference's float32 sgemm (index.py:235) accumulates in float32, so it sits
    # ~sqrt(D) float32 ulps from the float64-accumulated value computed here
    d = golden["x"].shape[1]
    np.testing.assert_allclose(ix.centroids.values, golden["centroids"], rtol=1e-6, atol=1e-6 * np.sqrt(d))
    codes = dev.to_host(keep["codes"])
    code_mismatch = (codes != golden["stage_codes"]).mean()
    assert code_mismatch < 1e-3
    # factors follow the codes: rows whose code took a 1-ulp o_rot flip differently are excluded
    same = (codes == golden["stage_codes"]).all(axis=1)
    assert same.mean() > 0.99
    # (the additive factor also takes cent_rot, whose float32 sgemm the reference rounds differently;
    # bit-exact factors given the reference's cent_rot: test_build_bit_exact_given_reference_...)
    np.testing.assert_allclose(ix.short_factors[same], golden["short_factors"][same], rtol=1e-4, atol=1e-4)


def test_build_and_search_recall_parity_with_oracle():
    """Mid-size seeded workload: GPU build+search recall within 0.002 of the oracle's."""
    g = load_case("b8_d128")
    x = g["x"]
    q = g["queries"]
    params = iv.BuildParams(n_clusters=20, quant=iv.QuantizationParams(bits=8), kmeans_iters=5, seed=1)
    ix = iv.build_index(x, params)
    gt, _ = orc.exact_knn(x, q, 10)
    ref = orc.build(x, 20, 8, 5, 1.0, 1)
    for mode in ("bitwise", "lut"):
        sp = iv.SearchParams(k=10, n_probe=5, ip_mode=mode)
        r_gpu = orc.recall_at_k(iv.search_batch(q, ix, sp), gt, 10)
        r_ref = orc.recall_at_k(orc.search(q, ref, 10, 5, ip_mode=mode), gt, 10)
        assert abs(r_gpu - r_ref) <= 0.002, (mode, r_gpu, r_ref)


def test_exact_knn_matches_oracle():
    rng = np.random.default_rng(4)
    base = rng.standard_normal((1000, 16)).astype(np.float32)
    queries = rng.standard_normal((20, 16))
    ids, d = iv.exact_knn(base, queries, 10)
    ids_o, d_o = orc.exact_knn(base, queries, 10)
    np.testing.assert_array_equal(ids, ids_o)
    np.testing.assert_allclose(d, d_o, rtol=1e-12, atol=1e-12)


def test_rotate_matches_oracle():
    rot = iv.gen_rotation(24, 9)
    rng = np.random.default_rng(2)
    x = rng.standard_normal((30, 24))
    np.testing.assert_allclose(iv.rotate(rot, x), x @ rot.matrix.T, rtol=1e-12, atol=1e-12)


def test_edge_cases_empty_lists_and_small_k():
    g = load_case("b2_dup")
    ix = _index(g)
    sp = iv.SearchParams(k=50, n_probe=ix.n_clusters, ip_mode="bitwise")
    res = iv.search_batch(g["queries"], ix, sp)
    ref = orc.search(g["queries"], golden_index_arrays(g), 50, ix.n_clusters, ip_mode="bitwise", q_rot=g["q_rot"])
    for (a, b), (c, d) in zip(res, ref):
        np.testing.assert_array_equal(a, c)
        np.testing.assert_allclose(b, d, rtol=1e-9)
    assert iv.search_batch(np.zeros((0, ix.dims)), ix, sp) == []


@pytest.mark.parametrize("case,si", [("b8_d128", 0), ("b4_d48", 1), ("b3_d96", 2), ("b1_d32", 0)])
def test_sharded_scan_chain_and_merge_on_one_gpu(case, si):
    """The shard kernel path: two list ranges, the second continuing the first's pools."""
    from paper_2602_23999_b200.distributed import _merge_gpu, cluster_ranges, slice_lists
    from paper_2602_23999_b200.search import _probe_device, prepare_queries_device

    g = load_case(case)
    if f"s{si}_ids" not in g:
        pytest.skip("n_probe exceeds n_clusters")
    sp = iv.SearchParams(**SEARCHES[si])
    full = _index(g)
    counts = np.diff(g["offsets"].astype(np.int64))
    ranges = cluster_ranges(counts, 2)
    shards = [slice_lists(full, lo, hi, ranges) for lo, hi in ranges]
    q_rot = dev.to_device(g["q_rot"])
    t = full.device
    probe_ids, probe_d2 = _probe_device(q_rot, t["centroids"], t["centroid_sqnorms"], sp.n_probe, True)
    nq, k = q_rot.shape[0], sp.k

    def scan(sh, init):
        scal, planes, luts, qsl = prepare_queries_device(q_rot, sh.local, sp)
        ids = torch.empty((nq, k), dtype=torch.int64, device=q_rot.device)
        dd = torch.empty((nq, k), dtype=torch.float64, device=q_rot.device)
        cc = torch.empty(nq, dtype=torch.int32, device=q_rot.device)
        from paper_2602_23999_b200 import _lib

        _lib.call(
            "ivrq_search_scan_shard", sh.local.view(), sh.list_lo, sh.list_hi, None, dev.ptr(probe_ids),
            dev.ptr(probe_d2), dev.ptr(scal), dev.ptr(planes), dev.ptr(luts), dev.ptr(qsl), nq, sp.to_c(),
            dev.ptr(init[0]) if init else None, dev.ptr(init[1]) if init else None,
            dev.ptr(init[2]) if init else None, dev.ptr(ids), dev.ptr(dd), dev.ptr(cc), None, dev.stream_ptr(),
        )
        return ids, dd, cc

    p0 = scan(shards[0], None)
    chained = scan(shards[1], p0)
    np.testing.assert_array_equal(dev.to_host(chained[2]), g[f"s{si}_counts"])
    np.testing.assert_array_equal(dev.to_host(chained[0]), g[f"s{si}_ids"])
    np.testing.assert_allclose(dev.to_host(chained[1]), g[f"s{si}_dists"], rtol=1e-12, atol=1e-12)
    if case.startswith("b1"):  # order-independent: fresh shards + merge is exact too
        p1 = scan(shards[1], None)
        stacked = tuple(torch.stack([a, b]) for a, b in zip(p0, p1))
        mi, md, mc = _merge_gpu(stacked, 2, k)
        np.testing.assert_array_equal(dev.to_host(mi), g[f"s{si}_ids"])
        np.testing.assert_array_equal(dev.to_host(mc), g[f"s{si}_counts"])


def _synthetic_index(n, d, nlist, bits, seed):
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((16, d)) * 3.0
    x = (centers[rng.integers(0, 16, n)] + rng.standard_normal((n, d))).astype(np.float32)
    q = (centers[rng.integers(0, 16, 700)] + rng.standard_normal((700, d))).astype(np.float32)
    params = iv.BuildParams(n_clusters=nlist, quant=iv.QuantizationParams(bits=bits), kmeans_iters=3, seed=seed)
    return iv.build_index(x, params), q


@pytest.mark.parametrize(
    "n,d,nlist,bits,qbits,nprobe,k",
    [
        (20000, 96, 64, 4, 4, 8, 10),  # int16 inner products, first-list phase
        (12000, 300, 32, 8, 8, 6, 10),  # int32 inner products (300 * 128 > 2^15)
        (15000, 128, 48, 1, 4, 7, 10),  # 1-bit index: every probe on the tensor-core stage 1
        (15000, 70, 40, 3, 2, 40, 32),  # every list probed, ragged dims, k = 32
        (8000, 64, 16, 5, 4, 4, 1),
        (6000, 1000, 12, 4, 4, 5, 10),  # D = 1000: kpad 1024 (8 refine chunks), g = 32
    ],
)
def test_tensor_core_stage1_matches_popcount_path(monkeypatch, n, d, nlist, bits, qbits, nprobe, k):
    """Every list-major tensor-core path == the per-query AND+POPC scan: ids, dists, counts, survivor stats.

    Variants: the default policy; tcgen05 stage 1 and tcgen05 dense refine forced on (4-bit codes
    go through the producer-warp nibble unpack); mma.sync stage 1 with the in-warp survivor refine.
    """
    ix, q = _synthetic_index(n, d, nlist, bits, seed=d)
    sp = iv.SearchParams(k=k, n_probe=nprobe, ip_mode="bitwise", query_bits=qbits)
    qd = dev.to_device(q)
    variants = {
        "popcount": {"IVRQ_TC_STAGE1": "0"},
        "default": {},
        "tcgen05": {"IVRQ_TC_IP": "1", "IVRQ_TC_REFINE": "1"},
        "mma_sync": {"IVRQ_TC_IP": "0", "IVRQ_TC_REFINE": "0"},
    }
    out = {}
    for name, env in variants.items():
        for key in ("IVRQ_TC_STAGE1", "IVRQ_TC_IP", "IVRQ_TC_REFINE"):
            monkeypatch.delenv(key, raising=False)
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        r = search_device(qd, ix, sp, with_stats=True)
        out[name] = [dev.to_host(t) for t in (r.ids, r.dists, r.counts, r.stats)]
    for name in ("default", "tcgen05", "mma_sync"):
        for a, b in zip(out["popcount"], out[name]):
            np.testing.assert_array_equal(a, b, err_msg=name)


def test_search_batch_pipeline_chunks_identical(monkeypatch):
    """The chunked host pipeline of search_batch returns exactly the single-batch results."""
    ix, q = _synthetic_index(20000, 64, 40, 4, seed=3)
    q = np.concatenate([q] * 7)  # 4900 queries: two chunks by default
    sp = iv.SearchParams(k=10, n_probe=5, ip_mode="bitwise")
    r = search_device(dev.to_device(q), ix, sp)
    ids, dists, counts = dev.to_host(r.ids), dev.to_host(r.dists), dev.to_host(r.counts)
    for chunks in ("1", "2", "3", "5"):
        monkeypatch.setenv("IVRQ_E2E_CHUNKS", chunks)
        res = iv.search_batch(q, ix, sp)
        assert len(res) == len(q)
        for i in (0, 1, 2449, 2450, 4899):
            np.testing.assert_array_equal(res[i][0], ids[i, : counts[i]])
            np.testing.assert_array_equal(res[i][1], dists[i, : counts[i]])
        got = np.stack([a for a, _ in res])
        np.testing.assert_array_equal(got, ids)


@pytest.mark.parametrize("stream_wait", [True, False])
@pytest.mark.parametrize("pieces", ["1", "3", "8"])
def test_search_batch_published_pieces_identical(monkeypatch, stream_wait, pieces):
    """search_batch's single-batch pipeline (pieces staged by the host threads, published through a
    page-locked flag the stream waits on, or host waits when stream_wait is off; rotation, probe and
    query prep per piece) returns exactly the device search of the whole batch; two threads searching
    at once get their own results."""
    import threading

    from paper_2602_23999_b200 import search as S

    ix, q = _synthetic_index(20000, 64, 40, 4, seed=3)
    q = np.concatenate([q] * 7)  # 4900 queries: up to 4 pieces of >= 1024 rows
    sp = iv.SearchParams(k=10, n_probe=5, ip_mode="bitwise")
    r = search_device(dev.to_device(q), ix, sp)
    ids = dev.to_host(r.ids)
    monkeypatch.setenv("IVRQ_STAGE_PIECES", pieces)
    monkeypatch.setattr(S, "_WAIT_OK", None if stream_wait else False)
    res = iv.search_batch(q, ix, sp)
    if stream_wait:
        assert S._WAIT_OK is True  # the driver takes the stream wait on a B200
    np.testing.assert_array_equal(np.stack([a for a, _ in res]), ids)
    q2 = np.ascontiguousarray(q[::-1])
    out = {}

    def worker(name, qq):
        for _ in range(3):
            out[name] = iv.search_batch(qq, ix, sp)

    th = [threading.Thread(target=worker, args=("a", q)), threading.Thread(target=worker, args=("b", q2))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    np.testing.assert_array_equal(np.stack([a for a, _ in out["a"]]), ids)
    np.testing.assert_array_equal(np.stack([a for a, _ in out["b"]]), ids[::-1])


def test_kmeanspp_parallel_exact_matches_sequential_walk(monkeypatch):
    """k-means++ sampling decided by the double-double prefix + rounding band equals
    NumPy's sequential cumsum walk (searchsorted(cumsum(d2), r * total)) step for step."""
    from paper_2602_23999_b200.clustering import _kmeanspp_device

    rng = np.random.default_rng(12)
    x = (rng.standard_normal((40000, 24)) * rng.uniform(0.1, 10.0, (40000, 1))).astype(np.float32)
    xd = dev.to_device(x)
    out = {}
    for seq in ("0", "1"):
        monkeypatch.setenv("IVRQ_KPP_SEQUENTIAL", seq)
        out[seq] = dev.to_host(_kmeanspp_device(xd, 300, seed=5))
    np.testing.assert_array_equal(out["0"], out["1"])


@pytest.mark.parametrize(
    "nlist,nprobe,dup",
    [(1024, 8, 1), (8192, 64, 1), (16384, 128, 1), (20000, 16, 1), (8192, 32, 128), (16384, 64, 2048)],
)
def test_tensor_core_probe_matches_gemm_probe(monkeypatch, nlist, nprobe, dup):
    """The tcgen05 bounds probe (register or radix tau, candidate or full-row rescoring) selects the
    same clusters as the float64 GEMM probe, ties included (dup copies of every centroid)."""
    rng = np.random.default_rng(nlist + dup)
    d = 96
    q = rng.standard_normal((300, d))
    uniq = rng.standard_normal((nlist // dup, d)).astype(np.float32)
    cent = Centroids(np.repeat(uniq, dup, axis=0))
    out = {}
    for env in ("1", "0"):
        monkeypatch.setenv("IVRQ_TC_PROBE", env)
        out[env] = iv.select_clusters(q, cent, nprobe)
    np.testing.assert_array_equal(out["1"][0], out["0"][0])
    np.testing.assert_allclose(out["1"][1], out["0"][1], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("chunks", ["1", "2"])
def test_search_batch_short_rows(monkeypatch, chunks):
    """Queries whose probed lists hold fewer than k vectors come back trimmed to their count
    (row views made before the results land are re-cut afterwards)."""
    ix, q = _synthetic_index(600, 32, 40, 4, seed=11)
    sp = iv.SearchParams(k=40, n_probe=1, ip_mode="bitwise")
    r = search_device(dev.to_device(q), ix, sp)
    ids, dists, counts = dev.to_host(r.ids), dev.to_host(r.dists), dev.to_host(r.counts)
    assert counts.min() < 40 <= counts.max() or counts.max() < 40
    assert (counts < 40).any()
    monkeypatch.setenv("IVRQ_E2E_CHUNKS", chunks)
    res = iv.search_batch(q, ix, sp)
    assert len(res) == len(q)
    for i in range(len(q)):
        np.testing.assert_array_equal(res[i][0], ids[i, : counts[i]])
        np.testing.assert_array_equal(res[i][1], dists[i, : counts[i]])


@pytest.mark.parametrize("k,copies,bits,mode", [(10, 40, 8, "bitwise"), (30, 6, 8, "bitwise"), (10, 12, 4, "bitwise"),
                                                (10, 40, 8, "lut"), (30, 6, 8, "lut")])
def test_refine_intervals_near_duplicates(monkeypatch, k, copies, bits, mode):
    """Near-duplicate vectors (distances apart by ~1e-7 relative, well inside the approximate
    refine's radius) force every interval decision of scan_rda_kernel open: the exact threshold
    from the list-start queue, the final exact top k, and (k = 30: more than 32 - k near-ties)
    the exact rerun.  The dense tcgen05 refine must equal the exact per-query popcount path."""
    rng = np.random.default_rng(k * 100 + copies)
    d = 128
    base = (rng.standard_normal((300, d)) * 2.0).astype(np.float64)
    x = np.repeat(base, copies, axis=0)
    x = x * (1.0 + 1e-7 * rng.standard_normal(x.shape))
    x[::5] = np.repeat(base, copies, axis=0)[::5]  # some exact copies: ties broken by id
    x = x.astype(np.float32)
    q = (base[rng.integers(0, 300, 200)] + 0.05 * rng.standard_normal((200, d))).astype(np.float32)
    ix = iv.build_index(x, iv.BuildParams(n_clusters=8, quant=iv.QuantizationParams(bits=bits), kmeans_iters=3,
                                          seed=1))
    sp = iv.SearchParams(k=k, n_probe=4, ip_mode=mode, query_bits=4)
    qd = dev.to_device(q)
    out = {}
    for name, env in {"popcount": {"IVRQ_TC_STAGE1": "0"}, "tcgen05": {"IVRQ_TC_IP": "1", "IVRQ_TC_REFINE": "1"}}.items():
        for key in ("IVRQ_TC_STAGE1", "IVRQ_TC_IP", "IVRQ_TC_REFINE"):
            monkeypatch.delenv(key, raising=False)
        for key, val in env.items():
            monkeypatch.setenv(key, val)
        r = search_device(qd, ix, sp, with_stats=True)
        out[name] = [dev.to_host(t) for t in (r.ids, r.dists, r.counts, r.stats)]
    for a, b in zip(out["popcount"], out["tcgen05"]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("n,d,nlist,nprobe,k", [(12000, 300, 32, 6, 10), (8000, 768, 16, 5, 10), (6000, 128, 24, 24, 32)])
def test_lut_list_major_path_matches_per_query_lut_scan(monkeypatch, n, d, nlist, nprobe, k):
    """LUT mode (the reference's default ip_mode) on 8-bit indexes: the list-major path with the
    certified LUT estimate (tc_refine's digit rows read as signed bytes, exact table sums where the
    estimate leaves a test open) == the per-query LUT scan: ids, dists, counts and survivor stats."""
    ix, q = _synthetic_index(n, d, nlist, 8, seed=d + 1)
    sp = iv.SearchParams(k=k, n_probe=nprobe, ip_mode="lut")
    qd = dev.to_device(q)
    out = {}
    for name, val in (("per_query", "0"), ("list_major", "1")):
        monkeypatch.setenv("IVRQ_LUT_RD", val)
        r = search_device(qd, ix, sp, with_stats=True)
        out[name] = [dev.to_host(t) for t in (r.ids, r.dists, r.counts, r.stats)]
    for a, b in zip(out["per_query"], out["list_major"]):
        np.testing.assert_array_equal(a, b)
