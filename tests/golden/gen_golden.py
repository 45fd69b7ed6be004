"""Generate golden vectors by running the reference package itself.

Run in the container that has the read-only reference mounted:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

It imports ``ivfrabitq`` (the reference, pure NumPy), runs its build pipeline
stage by stage exactly as ``build_index`` does (reference index.py:190-281),
checks that the staged result equals ``build_index``'s own, and stores inputs,
intermediates and search outputs as compressed ``.npz`` fixtures next to this
script.  The fixtures travel with the repository; nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import importlib.util
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_TESTS = Path("/root/reference/pkg/tests")
sys.path.insert(0, str(HERE))

from datagen import mix_data  # noqa: E402

import ivfrabitq  # noqa: E402  (the reference)
from ivfrabitq import clustering as rc  # noqa: E402
from ivfrabitq import codec as rcodec  # noqa: E402
from ivfrabitq import index as rindex  # noqa: E402
from ivfrabitq import linalg as rlin  # noqa: E402
from ivfrabitq import search as rs  # noqa: E402


def _make_dataset():
    spec = importlib.util.spec_from_file_location("ref_conftest", REF_TESTS / "conftest.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.make_dataset


CASES = [
    # name, generator, n, nq, dims, nlist, bits, iters, train_fraction, seed, searches
    dict(name="b1_d32", gen="blobs", n=3000, nq=64, dims=32, nlist=16, bits=1, iters=8, tf=1.0, seed=0),
    dict(name="b4_d48", gen="gauss", n=2500, nq=64, dims=48, nlist=12, bits=4, iters=6, tf=1.0, seed=3),
    dict(name="b8_d128", gen="blobs", n=2000, nq=48, dims=128, nlist=20, bits=8, iters=5, tf=0.5, seed=1),
    dict(name="b3_d96", gen="blobs", n=1600, nq=48, dims=96, nlist=10, bits=3, iters=5, tf=1.0, seed=7),
    dict(name="b2_dup", gen="dup", n=40, nq=8, dims=8, nlist=3, bits=2, iters=3, tf=1.0, seed=0),
    dict(name="b6_d20", gen="gauss", n=900, nq=32, dims=20, nlist=7, bits=6, iters=4, tf=0.7, seed=11),
    # headline shapes (BASELINE.json C3 / C5 / C4), small n.  "mix" data is regenerated from its seed
    # at test time (tests/golden/datagen.py), so x is not stored.
    # D = 768, 8-bit: tcgen05 stage 1 (g = 24) and the 6-chunk tcgen05 dense refine, ~128 queries
    # per list (several refine groups per list, several 128-row tiles per list)
    dict(name="b8_d768", gen="mix", n=3000, nq=256, dims=768, nlist=8, bits=8, iters=4, tf=1.0, seed=21),
    # D = 1536, 4-bit: tcgen05 stage 1 (g = 48) + the warp-per-query survivor refine on nibble codes
    dict(name="b4_d1536", gen="mix", n=1500, nq=128, dims=1536, nlist=4, bits=4, iters=3, tf=1.0, seed=22),
    # D = 96, nlist 512: many short lists, the tensor-core probe at n_probe 16 / 32
    dict(name="b4_d96_l512", gen="mix", n=12000, nq=160, dims=96, nlist=512, bits=4, iters=3, tf=0.5, seed=23),
]

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


def _data(case, make_dataset):
    rng = np.random.default_rng(1000 + case["seed"])
    n, nq, d = case["n"], case["nq"], case["dims"]
    if case["gen"] == "mix":
        return mix_data(n, nq, d, case["seed"])
    if case["gen"] == "blobs":
        base, queries = make_dataset(n_base=n, n_queries=nq, dims=d, n_blobs=8, seed=20260810 + case["seed"])
        return base, queries.astype(np.float64)
    if case["gen"] == "gauss":
        return rng.standard_normal((n, d)).astype(np.float32), rng.standard_normal((nq, d))
    # duplicated points: forces empty clusters during training (test_clustering.py:98-105)
    x = np.zeros((n, d), dtype=np.float32)
    x[n // 2 :] = 1.0
    x[-1] = 5.0
    return x, rng.standard_normal((nq, d))


def _stage_build(x, params):
    """build_index, stage by stage, keeping every intermediate (index.py:190-281)."""
    n, dims = x.shape
    seeds = np.random.SeedSequence(params.seed).spawn(2)
    if params.train_fraction < 1.0:
        n_train = max(1, math.ceil(params.train_fraction * n))
        n_train = max(n_train, min(n, params.n_clusters))
        rows = np.sort(np.random.default_rng(seeds[0]).choice(n, size=n_train, replace=False))
        x_train = x[rows]
    else:
        rows = np.arange(n)
        x_train = x
    km_seed = int(seeds[1].generate_state(1)[0])
    xt64 = np.ascontiguousarray(x_train, dtype=np.float64)
    pp = rc._kmeans_pp_init(xt64, params.n_clusters, np.random.default_rng(km_seed))
    cents = rc.train_kmeans(x_train, params.n_clusters, params.kmeans_iters, km_seed)
    labels = rc.assign(x, cents)
    counts = np.bincount(labels, minlength=params.n_clusters)
    offsets = np.zeros(params.n_clusters + 1, dtype=np.uint64)
    offsets[1:] = np.cumsum(counts)
    order = np.argsort(labels, kind="stable")
    rot32 = rlin.gen_rotation(dims, params.seed).matrix.astype(np.float32)
    cent32 = cents.values.astype(np.float32)
    cent_rot = (cent32 @ rot32.T).astype(np.float32)
    resid, dist = rcodec.normalize_residuals(x[order], cent32[labels[order]])
    o_rot = (resid @ rot32.T.astype(np.float64)).astype(np.float32)
    codes = np.zeros((n, dims), dtype=np.uint8)
    tvals = np.zeros(n, dtype=np.float32)
    for c in range(params.n_clusters):
        lo, hi = int(offsets[c]), int(offsets[c + 1])
        if hi > lo:
            u, t = rcodec.quantize_batch(o_rot[lo:hi], params.quant)
            codes[lo:hi] = u
            tvals[lo:hi] = t
    return dict(
        train_rows=rows.astype(np.int64),
        km_seed=np.int64(km_seed),
        pp_centers=pp,
        centroids64=cents.values,
        centroids64_sqnorms=cents.squared_norms,
        labels=labels.astype(np.int64),
        counts=counts.astype(np.int64),
        order=order.astype(np.int64),
        cent32=cent32,
        o_rot=o_rot,
        dist=dist,
        codes=codes,
        t=tvals,
    )


def gen_subops(indexes: dict) -> None:
    """Reference outputs of the per-call sub-operators (search.py:84-375, codec.py:118-151, 262-303, 322-401)."""
    rng = np.random.default_rng(77)
    out = {}
    # quantize_oracle: small vectors, every width the enumeration guard admits
    qo = []
    for i, (dims, bits) in enumerate([(d, b) for d in (1, 3, 5, 8, 12, 31) for b in (1, 2, 3, 4, 6)]):
        if dims * 2 ** (bits - 1) > rcodec._ORACLE_MAX_FACTORS:
            continue
        for j in range(4):
            o = rng.standard_normal(dims)
            if j == 1:
                o[rng.integers(0, dims)] = 0.0  # a zero coordinate (u_zero)
            if j == 3:
                o = np.round(o * 2) / 2  # exact ties between coordinates
            nrm = np.linalg.norm(o)
            o = o / nrm if nrm > 0 else o
            out[f"qo{len(qo)}_o"] = o
            out[f"qo{len(qo)}_u"] = rcodec.quantize_oracle(o, bits)
            qo.append(bits)
    out["qo_bits"] = np.array(qo, dtype=np.int64)
    # compute_factors_batch
    for bits in (1, 4, 7):
        n, dims = 40, 24
        o = rng.standard_normal((n, dims))
        o /= np.linalg.norm(o, axis=1)[:, None]
        u, _ = rcodec.quantize_batch(o, rcodec.QuantizationParams(bits=bits))
        dd = rng.uniform(0.0, 3.0, n)
        dd[3] = 0.0
        c = rng.standard_normal((n, dims))
        sh, lg, lowq = rcodec.compute_factors_batch(u, o, dd, c, rcodec.QuantizationParams(bits=bits))
        out.update({f"cf{bits}_u": u, f"cf{bits}_o": o, f"cf{bits}_d": dd, f"cf{bits}_c": c,
                    f"cf{bits}_short": sh, f"cf{bits}_long": lg, f"cf{bits}_lowq": lowq})
    # normalize_residuals (einsum order: host independent)
    x = rng.standard_normal((30, 20))
    c = rng.standard_normal((30, 20))
    c[4] = x[4]
    o, dd = rcodec.normalize_residuals(x, c)
    out.update(nr_x=x, nr_c=c, nr_o=o, nr_d=dd)
    # cluster_local_search on two golden indexes, both ip modes, open and finite thresholds
    for name, (idx, queries) in indexes.items():
        for mode in ("bitwise", "lut"):
            sp = rs.SearchParams(k=7, n_probe=1, ip_mode=mode)
            for qi in range(3):
                st = rs.prepare_query(np.asarray(queries[qi], dtype=np.float64), idx, sp)
                for cl in range(idx.n_clusters):
                    for ti, thr in enumerate((math.inf, None)):
                        if thr is None:  # a threshold that prunes part of the list
                            ids0, d0 = rs.cluster_local_search(st, idx, cl, rs.SearchParams(k=1000, n_probe=1,
                                                                                           ip_mode=mode))
                            thr = float(np.median(d0)) if d0.size else 0.0
                        ids, dists = rs.cluster_local_search(st, idx, cl, sp, thr)
                        key = f"cls_{name}_{mode}_{qi}_{cl}_{ti}"
                        out[key + "_thr"] = np.float64(thr)
                        out[key + "_ids"] = ids
                        out[key + "_dists"] = dists
                out[f"cls_{name}_{mode}_{qi}_qrot"] = st.q_rot
    np.savez_compressed(HERE / "subops.npz", **out)
    print("subops ok", (HERE / "subops.npz").stat().st_size, "bytes")


def main() -> None:
    make_dataset = _make_dataset()
    only = set(sys.argv[1:])
    sub_indexes = {}
    for case in CASES:
        if only and case["name"] not in only and "subops" not in only:
            continue
        x, queries = _data(case, make_dataset)
        params = rindex.BuildParams(
            n_clusters=case["nlist"],
            quant=rcodec.QuantizationParams(bits=case["bits"]),
            kmeans_iters=case["iters"],
            train_fraction=case["tf"],
            seed=case["seed"],
        )
        idx = rindex.build_index(x, params)
        if case["name"] in ("b4_d48", "b8_d128"):
            sub_indexes[case["name"]] = (idx, queries)
        if only and case["name"] not in only:
            continue
        st = _stage_build(x, params)
        # the staged pipeline must reproduce build_index bit for bit
        assert np.array_equal(st["order"].astype(np.uint64), idx.pids)
        out = {
            "queries": queries,
            "params": np.array(
                [case["nlist"], case["bits"], case["iters"], case["seed"]], dtype=np.int64
            ),
            "train_fraction": np.float64(case["tf"]),
            "eps_bound": np.float64(idx.eps_bound),
            "rotation": idx.rotation,
            "centroids": idx.centroids.values,
            "centroid_sqnorms": idx.centroids.squared_norms,
            "offsets": idx.offsets,
            "packed_msb": idx.packed_msb,
            "excodes": idx.excodes,
            "short_factors": idx.short_factors,
            "long_factors": idx.long_factors,
            "pids": idx.pids,
        }
        if case["gen"] != "mix":
            out["x"] = x
        out["gen"] = np.array([case["gen"], str(case["n"]), str(case["nq"]), str(case["dims"]), str(case["seed"])])
        for key, val in st.items():
            out["stage_" + key] = val
        q64 = np.ascontiguousarray(queries, dtype=np.float64)
        q_rot = q64 @ idx.rotation.T.astype(np.float64)
        out["q_rot"] = q_rot
        for si, sp_kw in enumerate(SEARCHES):
            sp = rs.SearchParams(**sp_kw)
            if sp.n_probe > idx.n_clusters:
                continue
            res = rs.search_batch(queries, idx, sp)
            k = sp.k
            ids = np.full((len(res), k), -1, dtype=np.int64)
            dists = np.full((len(res), k), np.inf)
            cnt = np.zeros(len(res), dtype=np.int32)
            for i, (a, b) in enumerate(res):
                ids[i, : a.size] = a
                dists[i, : b.size] = b
                cnt[i] = a.size
            out[f"s{si}_ids"] = ids
            out[f"s{si}_dists"] = dists
            out[f"s{si}_counts"] = cnt
            pid, pd2 = rs.select_clusters(q_rot, idx.centroids, sp.n_probe)
            out[f"s{si}_probe_ids"] = pid
            out[f"s{si}_probe_d2"] = pd2
            # per-query state scalars
            scal = np.zeros((q_rot.shape[0], 4))
            planes = []
            luts = []
            for i in range(q_rot.shape[0]):
                qs = rs._prepare_from_rotated(q_rot[i], idx.dims, sp, idx.eps_bound)
                scal[i] = (qs.sum_q, qs.delta_q, qs.code_sum_q, qs.ip_margin)
                if sp.ip_mode == "bitwise":
                    planes.append(qs.planes)
                else:
                    luts.append(qs.luts)
            out[f"s{si}_qstate"] = scal
            if planes:
                out[f"s{si}_planes"] = np.stack(planes)
            if luts:  # 16 queries' tables are enough to pin build_luts (they dominate the fixture size)
                out[f"s{si}_luts"] = np.stack(luts[:16])
        np.savez_compressed(HERE / f"{case['name']}.npz", **out)
        print(case["name"], "ok", (HERE / f"{case['name']}.npz").stat().st_size, "bytes")
    if not only or "subops" in only:
        gen_subops(sub_indexes)
    # known-answer vectors for the reduction orders (host-independent NumPy semantics)
    rng = np.random.default_rng(5)
    red = {}
    for d in (1, 7, 8, 13, 32, 96, 100, 128, 768, 1536):
        a = rng.standard_normal((16, d))
        b = rng.standard_normal((16, d)).astype(np.float32)
        red[f"einsum_a_{d}"] = a
        red[f"einsum_b_{d}"] = b
        red[f"einsum_ab_{d}"] = np.einsum("ij,ij->i", a, b, dtype=np.float64)
        red[f"einsum_aa_{d}"] = np.einsum("ij,ij->i", a, a)
        v = rng.standard_normal(d) * np.exp(rng.uniform(-8, 8, d))
        red[f"sum_v_{d}"] = v
        red[f"sum_{d}"] = np.float64(v.sum())
    np.savez_compressed(HERE / "reductions.npz", **red)
    print("reductions ok")


if __name__ == "__main__":
    sys.exit(main())
