"""CPU oracle for the IVF-RaBitQ build + search path -- TEST INFRASTRUCTURE ONLY.

This module restates the reference algorithm (the ``ivfrabitq`` package under
/root/reference/pkg/src/ivfrabitq, pure NumPy) so that the CUDA product can
be checked against it on the same seeded inputs.  It is imported only by
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm -- never by the product package, which has no CPU path.

Parity status: PINNED.  ``tests/test_oracle_golden.py`` checks every stage
here against golden vectors produced by running the reference itself
(tests/golden/gen_golden.py): bit-exact for labels, CSR order, codes, packed
planes, ex-codes, probe ids, query planes and returned neighbour ids; float
values bit-exact where the reference's arithmetic is host independent and to
<= 1e-12 relative where it goes through an OpenBLAS GEMM.

Each function cites the reference lines it follows.  Arithmetic is float64
through NumPy exactly where the reference uses float64, with the reference's
dtype rules (the grid search runs in the dtype of ``o``, float32 for built
indexes, because of NumPy 2 promotion of Python scalars).
"""

from __future__ import annotations

import math

import numpy as np

# ---------------------------------------------------------------- numerics


def rowdot(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Row-wise float64 dot with NumPy's einsum reduction order (used at every einsum site)."""
    return np.einsum("ij,ij->i", a, b, dtype=np.float64)


# ---------------------------------------------------------------- k-means (clustering.py)


def nearest_centre(x64: np.ndarray, centres: np.ndarray, c_sq: np.ndarray, block: int = 8192):
    """Labels and clamped distance to the chosen centre (clustering.py:41-57)."""
    n = x64.shape[0]
    lab = np.empty(n, dtype=np.int64)
    best = np.empty(n, dtype=np.float64)
    for s in range(0, n, block):
        xb = x64[s : s + block]
        dist = rowdot(xb, xb)[:, None] + c_sq[None, :] - 2.0 * (xb @ centres.T)
        j = dist.argmin(axis=1)
        lab[s : s + block] = j
        best[s : s + block] = np.maximum(dist[np.arange(xb.shape[0]), j], 0.0)
    return lab, best


def _sqdist_rows(x64: np.ndarray, c: np.ndarray, pool=None) -> np.ndarray:
    """rowdot(x - c, x - c); with a thread pool, row blocks in parallel (rows are independent,
    so the values are those of the single call -- einsum drops the GIL in its inner loop)."""
    if pool is None:
        gap = x64 - c
        return rowdot(gap, gap)
    out = np.empty(x64.shape[0])
    bounds = np.linspace(0, x64.shape[0], 4 * pool._max_workers + 1).astype(np.int64)

    def part(a, b):
        g = x64[a:b] - c
        out[a:b] = rowdot(g, g)

    list(pool.map(lambda ab: part(*ab), zip(bounds[:-1], bounds[1:])))
    return out


def seed_centres(x64: np.ndarray, k: int, rng: np.random.Generator, pool=None) -> np.ndarray:
    """k-means++ seeding (clustering.py:60-79)."""
    n, d = x64.shape
    out = np.empty((k, d))
    out[0] = x64[int(rng.integers(n))]
    dmin = _sqdist_rows(x64, out[0], pool)
    for j in range(1, k):
        tot = float(dmin.sum())
        if tot > 0.0:
            pick = min(int(np.searchsorted(np.cumsum(dmin), rng.random() * tot)), n - 1)
        else:
            pick = int(rng.integers(n))
        out[j] = x64[pick]
        np.minimum(dmin, _sqdist_rows(x64, out[j], pool), out=dmin)
    return out


def kmeans(x: np.ndarray, k: int, iters: int, seed: int, pool=None) -> np.ndarray:
    """Lloyd iterations with empty-cluster reseeding (clustering.py:82-113); float64 centres."""
    x64 = np.ascontiguousarray(x, dtype=np.float64)
    n = x64.shape[0]
    rng = np.random.default_rng(seed)
    centres = seed_centres(x64, k, rng, pool)
    for _ in range(iters):
        lab, dmin = nearest_centre(x64, centres, rowdot(centres, centres))
        cnt = np.bincount(lab, minlength=k)
        for j in np.flatnonzero(cnt == 0):
            far = int(np.argmax(dmin))
            lab[far] = j
            dmin[far] = -1.0
        cnt = np.bincount(lab, minlength=k)
        perm = np.argsort(lab, kind="stable")
        first = np.concatenate(([0], np.cumsum(cnt)[:-1]))
        centres = np.add.reduceat(x64[perm], first, axis=0) / cnt[:, None]
    return centres


# ---------------------------------------------------------------- rotation (linalg.py)


def rotation(dims: int, seed: int) -> np.ndarray:
    """Seeded Gaussian -> QR -> sign-fixed Q (linalg.py:25-40), float64."""
    q, r = np.linalg.qr(np.random.default_rng(seed).standard_normal((dims, dims)))
    s = np.sign(np.diag(r))
    s[s == 0] = 1.0
    return q * s[None, :]


# ---------------------------------------------------------------- encoder (codec.py)


def normalise(x_rows: np.ndarray, c_rows: np.ndarray):
    """(o, d): unit residual directions and norms; zero rows stay zero (codec.py:138-151)."""
    diff = np.asarray(x_rows, dtype=np.float64) - np.asarray(c_rows, dtype=np.float64)
    d = np.sqrt(rowdot(diff, diff))
    o = diff / np.where(d == 0.0, 1.0, d)[:, None]
    o[d == 0.0] = 0.0
    return o, d


def _grid_codes(o: np.ndarray, t: np.ndarray, bits: int) -> np.ndarray:
    """floor(t*o + 2^(B-1)) clipped to [0, 2^B - 1], in o's dtype (codec.py:163-174)."""
    v = t[:, None] * o
    v += (2**bits - 1) / 2.0 + 0.5
    return np.clip(np.floor(v), 0.0, float(2**bits - 1))


def _scan_grid(o, lo, hi, count, bits, best_val, best_t):
    """Evaluate ``count`` evenly spaced factors, strict-> updates (codec.py:177-201)."""
    half_range = (2**bits - 1) / 2.0
    step = (hi - lo) / (count - 1)
    for s in range(count):
        t = lo + s * step
        c = _grid_codes(o, t, bits) - half_range
        score = rowdot(c, o) / np.sqrt(rowdot(c, c))
        better = score > best_val
        best_val[better] = score[better]
        best_t[better] = t[better]


def quantize(o: np.ndarray, bits: int, n_coarse: int = 64, n_fine: int = 32):
    """Two-phase rescaling search; returns (u uint8, t) (codec.py:204-244)."""
    o = np.atleast_2d(np.asarray(o))
    norms = np.sqrt(rowdot(o, o))
    if np.any((norms != 0.0) & (np.abs(norms - 1.0) > 1e-4)):
        raise ValueError("input rows must be unit vectors (or zero)")
    n, d = o.shape
    peak = np.abs(o).max(axis=1) if d else np.zeros(n)
    flat = peak == 0.0
    if bits == 1:
        u = (o > 0).astype(np.uint8)
        u[flat] = 1
        return u, np.where(flat, 0.0, 0.5 / np.where(flat, 1.0, peak))
    denom = np.where(flat, 1.0, peak)  # keeps o's dtype (NumPy 2 weak scalar promotion)
    first = 0.5 / denom
    last = (2 ** (bits - 1) - 0.5) * (1.0 + 6.0 / 2 ** (bits - 1)) / denom
    best_val = np.full(n, -np.inf)
    best_t = first.copy()
    _scan_grid(o, first, last, n_coarse, bits, best_val, best_t)
    width = (last - first) / (n_coarse - 1)
    _scan_grid(o, np.maximum(first, best_t - width), np.minimum(last, best_t + width), n_fine, bits, best_val, best_t)
    u = _grid_codes(o, best_t, bits).astype(np.uint8)
    u[flat] = np.uint8(2 ** (bits - 1))
    return u, np.where(flat, 0.0, best_t)


def factors(u: np.ndarray, o: np.ndarray, d: np.ndarray, c_rows: np.ndarray, bits: int, eps: float):
    """Short (add, scale, err) and long (add, scale) factors, float64 (codec.py:322-380)."""
    o = np.asarray(o, dtype=np.float64)
    c_rows = np.asarray(c_rows, dtype=np.float64)
    n, dims = o.shape
    xb = (u >> (bits - 1)).astype(np.float64) - 0.5
    xf = u.astype(np.float64) - (2**bits - 1) / 2.0
    nb = 0.5 * math.sqrt(dims)
    cb = rowdot(xb, o) / nb
    nx = np.sqrt(rowdot(xf, xf))
    cx = rowdot(xf, o) / nx
    cb = np.maximum(cb, 1e-6)
    cx = np.maximum(cx, 1e-6)
    sb = 2.0 * d / (nb * cb)
    sx = 2.0 * d / (nx * cx)
    var = np.maximum(1.0 - cb * cb, 0.0) / (cb * cb * max(dims - 1, 1))
    short = np.stack([d * d + sb * rowdot(xb, c_rows), sb, 2.0 * d * eps * np.sqrt(var)], axis=1)
    long = np.stack([d * d + sx * rowdot(xf, c_rows), sx], axis=1)
    dead = ~(d > 0.0)
    short[dead] = 0.0
    long[dead] = 0.0
    return short, long


def msb_words(msb: np.ndarray) -> np.ndarray:
    """Interleaved 32-dim words of one list: word (g, v) at g*n + v (codec.py:404-413)."""
    n, dims = msb.shape
    groups = (dims + 31) // 32
    padded = np.zeros((n, groups * 32), dtype=np.uint8)
    padded[:, :dims] = msb
    per_vec = np.packbits(padded, axis=1, bitorder="little").view("<u4")
    return np.ascontiguousarray(per_vec.T).ravel()


def ex_bytes(ex: np.ndarray, bits: int) -> np.ndarray:
    """LSB-first (bits-1)-bit fields per vector, byte padded (codec.py:432-444)."""
    n, dims = ex.shape
    if bits == 1:
        return np.zeros((n, 0), dtype=np.uint8)
    w = bits - 1
    stream = ((ex[:, :, None] >> np.arange(w, dtype=np.uint8)) & 1).reshape(n, dims * w)
    return np.packbits(stream, axis=1, bitorder="little")


# ---------------------------------------------------------------- build (index.py:190-281)


def _encode_lists(c_lo, c_hi, offsets, o_rot, d, crot, bits, n_coarse, n_fine, eps, g, out):
    """Encode lists [c_lo, c_hi) into the output arrays (index.py:247-264, one _quantize_cluster each)."""
    dims = o_rot.shape[1]
    packed, exb, short, long, codes = out
    for c in range(c_lo, c_hi):
        lo, hi = int(offsets[c]), int(offsets[c + 1])
        if hi == lo:
            continue
        u, _ = quantize(o_rot[lo:hi], bits, n_coarse, n_fine)
        if codes is not None:
            codes[lo:hi] = u
        sh, lg = factors(u, o_rot[lo:hi], d[lo:hi], np.broadcast_to(crot[c].astype(np.float64), (hi - lo, dims)), bits, eps)
        packed[lo * g : hi * g] = msb_words(u >> (bits - 1))
        exb[lo:hi] = ex_bytes(u & ((1 << (bits - 1)) - 1), bits)
        short[lo:hi] = sh
        long[lo:hi] = lg


_FORK_STATE: dict = {}


def _encode_worker(span):
    st = _FORK_STATE
    _encode_lists(span[0], span[1], st["offsets"], st["o_rot"], st["d"], st["crot"], st["bits"], st["n_coarse"],
                  st["n_fine"], st["eps"], st["g"], st["out"])
    return span


def _shared(shape, dtype):
    """A zeroed array in anonymous shared memory (visible to forked workers)."""
    import mmap

    nbytes = max(1, int(np.prod(shape, dtype=np.int64)) * np.dtype(dtype).itemsize)
    buf = mmap.mmap(-1, nbytes)
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape, dtype=np.int64))).reshape(shape)


def build(x, nlist, bits, iters=25, train_fraction=1.0, seed=0, n_coarse=64, n_fine=32, eps=1.9, inject=None,
          workers=1, timings=None):
    """Index arrays of ``build_index``; ``inject`` may pin centroids64/rotation/cent_rot/o_rot.

    ``workers > 1`` (bench.py's CPU arm only): the k-means++ distance passes run on a thread
    pool and the per-list encoder on forked processes writing shared memory -- every value is
    computed by the same expressions on the same rows, so the arrays equal ``workers=1``'s
    (the reference's own build parallelises the same per-list loop, index.py:259-264).
    """
    import time as _time

    inject = inject or {}
    tick = _time.perf_counter()

    def lap(name):
        nonlocal tick
        if timings is not None:
            now = _time.perf_counter()
            timings[name] = round(now - tick, 3)
            tick = now

    pool = None
    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor

        pool = ThreadPoolExecutor(workers)
    x = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float32)
    n, dims = x.shape
    seeds = np.random.SeedSequence(seed).spawn(2)
    if "centroids64" in inject:
        centres = np.asarray(inject["centroids64"], dtype=np.float64)
    else:
        if train_fraction < 1.0:
            m = max(1, math.ceil(train_fraction * n), min(n, nlist))
            rows = np.sort(np.random.default_rng(seeds[0]).choice(n, size=m, replace=False))
            xt = x[rows]
        else:
            xt = x
        centres = kmeans(xt, nlist, iters, int(seeds[1].generate_state(1)[0]), pool)
    lap("kmeans")
    lab, _ = nearest_centre(x.astype(np.float64), centres, rowdot(centres, centres))
    lap("assign")
    cnt = np.bincount(lab, minlength=nlist)
    offsets = np.concatenate(([0], np.cumsum(cnt))).astype(np.uint64)
    perm = np.argsort(lab, kind="stable")
    rot = inject.get("rotation")
    rot = np.asarray(rot, dtype=np.float32) if rot is not None else rotation(dims, seed).astype(np.float32)
    c32 = centres.astype(np.float32)
    crot = inject.get("cent_rot")
    crot = np.asarray(crot, dtype=np.float32) if crot is not None else (c32 @ rot.T).astype(np.float32)
    o, d = normalise(x[perm], c32[lab[perm]])
    o_rot = inject.get("o_rot")
    o_rot = np.asarray(o_rot, dtype=np.float32) if o_rot is not None else (o @ rot.T.astype(np.float64)).astype(np.float32)
    lap("normalize_rotate")
    g = (dims + 31) // 32
    bpv = (dims * (bits - 1) + 7) // 8
    alloc = _shared if workers > 1 else (lambda shape, dt: np.zeros(shape, dtype=dt))
    packed = alloc((n * g,), np.uint32)
    exb = alloc((n, bpv), np.uint8)
    short = alloc((n, 3), np.float32)
    long = alloc((n, 2), np.float32)
    codes = alloc((n, dims), np.uint8) if workers == 1 else None
    out = (packed, exb, short, long, codes)
    if workers > 1:
        import multiprocessing as mp

        _FORK_STATE.update(offsets=offsets, o_rot=o_rot, d=d, crot=crot, bits=bits, n_coarse=n_coarse,
                           n_fine=n_fine, eps=eps, g=g, out=out)
        # lists in contiguous spans of about equal row count, several per worker
        cuts = np.searchsorted(offsets.astype(np.int64), np.linspace(0, n, 8 * workers + 1)[1:-1])
        edges = np.unique(np.concatenate(([0], cuts, [nlist])))
        with mp.get_context("fork").Pool(workers) as pp:
            list(pp.imap_unordered(_encode_worker, list(zip(edges[:-1], edges[1:]))))
        _FORK_STATE.clear()
        pool.shutdown()
    else:
        _encode_lists(0, nlist, offsets, o_rot, d, crot, bits, n_coarse, n_fine, eps, g, out)
    lap("encode")
    return dict(
        dims=dims, bits=bits, n_clusters=nlist, size=n, eps_bound=eps, rotation=rot, centroids=crot,
        centroid_sqnorms=rowdot(crot.astype(np.float64), crot.astype(np.float64)), offsets=offsets,
        packed_msb=packed, excodes=exb, short_factors=short, long_factors=long, pids=perm.astype(np.uint64),
        labels=lab, centroids64=centres, o_rot=o_rot, dist=d, codes=codes,
    )


# ---------------------------------------------------------------- search (search.py)


def probe(q_rot: np.ndarray, centroids: np.ndarray, c_sq: np.ndarray, n_probe: int):
    """n_probe nearest centroids, ascending (distance, id) (search.py:226-244)."""
    q = np.atleast_2d(np.asarray(q_rot, dtype=np.float64))
    dist = rowdot(q, q)[:, None] + c_sq[None, :] - 2.0 * (q @ np.asarray(centroids, dtype=np.float64).T)
    np.maximum(dist, 0.0, out=dist)
    sel = np.argsort(dist, axis=1, kind="stable")[:, :n_probe]
    return sel, np.take_along_axis(dist, sel, axis=1)


def query_state(q_rot: np.ndarray, mode: str, query_bits: int, eps: float):
    """Per-query derived values (search.py:186-214, 115-132, 84-104)."""
    dims = q_rot.size
    st = {"q_rot": q_rot, "sum_q": float(q_rot.sum()), "delta": 1.0, "ip_margin": 0.0}
    groups = (dims + 31) // 32
    if mode == "lut":
        pad = np.zeros(groups * 32)
        pad[:dims] = q_rot
        keys = np.arange(16)
        sel = ((keys[:, None] >> np.arange(4)) & 1).astype(np.float64)
        st["luts"] = (pad.reshape(-1, 4) @ sel.T).astype(np.float32)
        st["code_sum"] = st["sum_q"]
        return st
    half = 1 << (query_bits - 1)
    peak = float(np.abs(q_rot).max()) if dims else 0.0
    delta = peak / (half - 1) if peak > 0.0 else 1.0
    qh = np.clip(np.round(q_rot / delta), -half, half - 1).astype(np.int32)
    twos = (qh & ((1 << query_bits) - 1)).astype(np.uint32)
    bitrows = np.zeros((query_bits, groups * 32), dtype=np.uint8)
    for j in range(query_bits):
        bitrows[j, :dims] = (twos >> j) & 1
    st["planes"] = np.packbits(bitrows, axis=1, bitorder="little").view("<u4")
    st["q_hat"] = qh
    st["delta"] = delta
    st["code_sum"] = delta * float(qh.sum())
    st["ip_margin"] = eps * delta * math.sqrt(dims / 24.0)
    return st


def binary_ip_bitwise(words_gn: np.ndarray, planes: np.ndarray, query_bits: int) -> np.ndarray:
    """Integer <msb, q_hat> from AND + popcount (search.py:163-183)."""
    per_plane = np.bitwise_count(words_gn[None, :, :] & planes[:, :, None]).sum(axis=1, dtype=np.int64)
    w = 1 << np.arange(query_bits, dtype=np.int64)
    w[-1] = -w[-1]
    return w @ per_plane


def binary_ip_lut(words_gn: np.ndarray, luts: np.ndarray) -> np.ndarray:
    """Sum of table entries picked by the 4-bit nibbles, float64 (search.py:146-160)."""
    g, n = words_gn.shape
    nib = np.empty((n, 8 * g), dtype=np.int64)
    for s in range(8):
        nib[:, s::8] = ((words_gn >> np.uint32(4 * s)) & np.uint32(15)).T
    flat = luts.reshape(-1)
    return np.take(flat, nib + 16 * np.arange(8 * g)).sum(axis=1, dtype=np.float64)


def decode_codes(ix: dict) -> np.ndarray:
    """Full unsigned codes as float32 (index.py:142-166)."""
    n, dims, bits = ix["size"], ix["dims"], ix["bits"]
    g = (dims + 31) // 32
    out = np.zeros((n, dims), dtype=np.float32)
    off = ix["offsets"]
    for c in range(ix["n_clusters"]):
        lo, hi = int(off[c]), int(off[c + 1])
        if hi == lo:
            continue
        per_vec = np.ascontiguousarray(ix["packed_msb"][lo * g : hi * g].reshape(g, hi - lo).T)
        out[lo:hi] = np.unpackbits(per_vec.view(np.uint8).reshape(hi - lo, 4 * g), axis=1, bitorder="little")[:, :dims]
    out *= float(2 ** (bits - 1))
    if bits > 1:
        w = bits - 1
        stream = np.unpackbits(ix["excodes"], axis=1, bitorder="little")[:, : dims * w].reshape(n, dims, w)
        out += (stream.astype(np.float32) * (1 << np.arange(w))).sum(axis=2)
    return out


def search(queries, ix: dict, k: int, n_probe: int, ip_mode="lut", query_bits=4, refine=True, prune=True, q_rot=None,
           codes=None, stats=None, list_range=None, init=None):
    """Per-query two-stage scan, lists in ascending id with a carried threshold (search.py:390-454).

    Shard semantics for the multi-GPU tests: ``list_range=(lo, hi)`` restricts
    the walk to those cluster ids; ``init`` = [(ids, dists)] per query seeds
    each pool (and its threshold) as if the lower-id lists had been visited.
    """
    q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float64)
    if q_rot is None:
        q_rot = q @ np.asarray(ix["rotation"]).T.astype(np.float64)
    sel, d2 = probe(q_rot, ix["centroids"], ix["centroid_sqnorms"], n_probe)
    g = (ix["dims"] + 31) // 32
    bits = ix["bits"]
    use_refine = refine and bits >= 2
    if use_refine and codes is None:
        codes = decode_codes(ix)
    sf = ix["short_factors"].astype(np.float64)
    lf = ix["long_factors"].astype(np.float64)
    pids = ix["pids"].astype(np.int64)
    off = ix["offsets"]
    kb = (2**bits - 1) / 2.0
    results = []
    for qi in range(q.shape[0]):
        st = query_state(q_rot[qi], ip_mode, query_bits, ix["eps_bound"])
        pool_i = np.empty(0, dtype=np.int64)
        pool_d = np.empty(0)
        if init is not None:
            pool_i = np.asarray(init[qi][0], dtype=np.int64)
            pool_d = np.asarray(init[qi][1], dtype=np.float64)
        thr = float(pool_d[k - 1]) if pool_i.size >= k else math.inf
        for j in np.argsort(sel[qi], kind="stable"):
            c = int(sel[qi, j])
            if list_range is not None and not (list_range[0] <= c < list_range[1]):
                continue
            dq = float(d2[qi, j])
            lo, hi = int(off[c]), int(off[c + 1])
            if hi == lo:
                continue
            words = ix["packed_msb"][lo * g : hi * g].reshape(g, hi - lo)
            if ip_mode == "lut":
                ipb = binary_ip_lut(words, st["luts"])
            else:
                ipb = st["delta"] * binary_ip_bitwise(words, st["planes"], query_bits)
            add, scale, err = sf[lo:hi, 0], sf[lo:hi, 1], sf[lo:hi, 2]
            est = np.maximum(add + dq - scale * (ipb - 0.5 * st["code_sum"]), 0.0)
            margin = err * np.sqrt(dq)
            if st["ip_margin"]:
                margin = np.sqrt(margin * margin + (scale * st["ip_margin"]) ** 2)
            lower = np.maximum(est - margin, 0.0)
            alive = np.flatnonzero(lower <= (thr if prune else math.inf))
            if stats is not None:
                stats["probed"] = stats.get("probed", 0) + (hi - lo)
                stats["survivors"] = stats.get("survivors", 0) + alive.size
            if alive.size == 0:
                continue
            if use_refine:
                ipu = codes[lo + alive] @ st["q_rot"]
                dist = np.maximum(lf[lo + alive, 0] + dq - lf[lo + alive, 1] * (ipu - kb * st["sum_q"]), 0.0)
            else:
                dist = est[alive]
            cand_i = np.concatenate([pool_i, pids[lo + alive]])
            cand_d = np.concatenate([pool_d, dist])
            keep = np.lexsort((cand_i, cand_d))[:k]
            pool_i, pool_d = cand_i[keep], cand_d[keep]
            if pool_i.size >= k:
                thr = float(pool_d[k - 1])
        results.append((pool_i, pool_d))
    return results


def recall_at_k(results, gt_ids: np.ndarray, k: int) -> float:
    """Mean |top-k result ∩ top-k truth| / k (cli.py:41-56)."""
    hits = 0
    for (ids, _), truth in zip(results, gt_ids):
        hits += len(set(np.asarray(ids)[:k].tolist()) & set(truth[:k].tolist()))
    return hits / (len(results) * k)


def exact_knn(base: np.ndarray, queries: np.ndarray, k: int, block: int = 256):
    """Brute-force float64 k-NN, ties to the smaller id (linalg.py:53-90)."""
    b = np.ascontiguousarray(base, dtype=np.float64)
    q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float64)
    kk = min(k, b.shape[0])
    b_sq = rowdot(b, b)
    ids = np.empty((q.shape[0], kk), dtype=np.int64)
    dd = np.empty((q.shape[0], kk))
    for s in range(0, q.shape[0], block):
        qb = q[s : s + block]
        dist = np.maximum(rowdot(qb, qb)[:, None] + b_sq[None, :] - 2.0 * (qb @ b.T), 0.0)
        o = np.argsort(dist, axis=1, kind="stable")[:, :kk]
        ids[s : s + block] = o
        dd[s : s + block] = np.take_along_axis(dist, o, axis=1)
    return ids, dd
