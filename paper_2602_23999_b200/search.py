"""Batched search on the GPU: rotation, coarse probe, query prep and the fused scan.

Mirrors ``ivfrabitq.search`` (reference search.py).  ``search_batch``
(search.py:390-454) is four launches of libivrq_b200.so on the current stream:

1. ``ivrq_rotate_queries``       q_rot = q @ R^T, float64           (search.py:422)
2. ``ivrq_select_clusters_ordered`` exact n_probe nearest centroids,
   handed to the scan in ascending cluster id                      (search.py:226-244, 429)
3. ``ivrq_prepare_queries``      QueryState: planes / LUTs, sums    (search.py:186-214)
4. ``ivrq_search_scan``          per query, lists in ascending id: stage-1
   estimate + lower bound, prune against the running threshold, ex-code
   refinement of survivors, top-k merge, threshold update           (search.py:326-387, 425-448)

Results are identical for every ``workers`` value (the argument is accepted
for API compatibility; GPU parallelism does not change the per-query
threshold trajectory).
"""

from __future__ import annotations

import math
import os
import threading
from dataclasses import dataclass

import numpy as np
import torch

from paper_2602_23999_b200 import _device as dev
from paper_2602_23999_b200 import _lib
from paper_2602_23999_b200.clustering import Centroids, row_sqnorms
from paper_2602_23999_b200.index import IvfRabitqIndex, default_workers

__all__ = [
    "SearchParams",
    "QueryState",
    "build_luts",
    "nibbles_from_bits",
    "ip_lut",
    "ip_bitwise",
    "prepare_query",
    "estimate_stage1",
    "refine_stage2",
    "cluster_local_search",
    "select_clusters",
    "search_batch",
    "search_device",
    "schedule_probes",
    "merge_topk",
]


@dataclass(frozen=True)
class SearchParams:
    """Per-search knobs (search.py:56-81)."""

    k: int
    n_probe: int
    ip_mode: str = "lut"
    query_bits: int = 4
    refine: bool = True
    prune: bool = True

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ValueError(f"k must be >= 1, got {self.k}")
        if self.n_probe < 1:
            raise ValueError(f"n_probe must be >= 1, got {self.n_probe}")
        if self.ip_mode not in ("lut", "bitwise"):
            raise ValueError(f"ip_mode must be 'lut' or 'bitwise', got {self.ip_mode!r}")
        if not 2 <= self.query_bits <= 8:
            raise ValueError(f"query_bits must be in [2, 8], got {self.query_bits}")

    def to_c(self) -> _lib.SearchParamsC:
        return _lib.SearchParamsC(
            k=self.k,
            n_probe=self.n_probe,
            ip_mode=_lib.IVRQ_IP_BITWISE if self.ip_mode == "bitwise" else _lib.IVRQ_IP_LUT,
            query_bits=self.query_bits,
            refine=1 if self.refine else 0,
            prune=1 if self.prune else 0,
        )


def schedule_probes(pairs):
    """Stable sort of (query, cluster, ...) pairs by (cluster, query) (search.py:247-253)."""
    return sorted(pairs, key=lambda p: (p[1], p[0]))


def merge_topk(lists, k: int):
    """K smallest (dist, id) of the concatenated candidate lists (search.py:378-387).

    Host helper for API compatibility; the GPU scan merges in shared memory.
    """
    if not lists:
        return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.float64)
    ids = np.concatenate([np.asarray(i, dtype=np.int64) for i, _ in lists])
    dists = np.concatenate([np.asarray(d, dtype=np.float64) for _, d in lists])
    order = np.lexsort((ids, dists))[:k]
    return ids[order], dists[order]


# ---------------------------------------------------------------- per-query sub-operators
# The reference exports the pieces of its per-query scan (search.py:84-375).  Each
# one here is a launch of libivrq_b200.so on the current stream (ivrq_ops.cu);
# host code only validates shapes and moves the small operands.

_LUT_BLOCK = 4


@dataclass
class QueryState:
    """Per-query derived data reused across the query's probes (search.py:84-104)."""

    q_rot: np.ndarray
    sum_q: float
    delta_q: float = 1.0
    q_hat: np.ndarray | None = None
    planes: np.ndarray | None = None
    luts: np.ndarray | None = None
    code_sum_q: float = 0.0
    ip_margin: float = 0.0
    threshold: float = math.inf

    def __post_init__(self) -> None:
        if not self.code_sum_q:
            self.code_sum_q = self.sum_q

    def scalars(self) -> np.ndarray:
        sc = np.zeros(_lib.QS_COUNT, dtype=np.float64)
        sc[_lib.QS_SUM_Q] = self.sum_q
        sc[_lib.QS_DELTA] = self.delta_q
        sc[_lib.QS_CODE_SUM] = self.code_sum_q
        sc[_lib.QS_IP_MARGIN] = self.ip_margin
        return sc


def _prepare_one(q_rot: np.ndarray, params: SearchParams, eps_bound: float, bits: int = 1):
    """ivrq_prepare_queries for one rotated query; host copies of scalars / planes / luts."""
    q = np.ascontiguousarray(np.asarray(q_rot, dtype=np.float64).reshape(1, -1))
    d = q.shape[1]
    g = (d + 31) // 32
    device = dev.require_cuda()
    qd = dev.to_device(q, device)
    scal = torch.empty((1, _lib.QS_COUNT), dtype=torch.float64, device=device)
    planes = luts = None
    if params.ip_mode == "bitwise":
        planes = torch.empty((params.query_bits, g), dtype=torch.int32, device=device)
    else:
        luts = torch.empty((8 * g, 16), dtype=torch.float32, device=device)
    cp = _lib.SearchParamsC(k=params.k, n_probe=params.n_probe,
                            ip_mode=_lib.IVRQ_IP_BITWISE if params.ip_mode == "bitwise" else _lib.IVRQ_IP_LUT,
                            query_bits=params.query_bits, refine=0, prune=1 if params.prune else 0)
    _lib.call("ivrq_prepare_queries", dev.ptr(qd), 1, d, cp, bits, float(eps_bound), dev.ptr(scal), dev.ptr(planes),
              dev.ptr(luts), None, dev.stream_ptr())
    sc = dev.to_host(scal)[0]
    return sc, (dev.to_host(planes).view(np.uint32) if planes is not None else None), (
        dev.to_host(luts) if luts is not None else None)


def _q_hat_from_planes(planes: np.ndarray, dims: int, qb: int) -> np.ndarray:
    """The quantized query from its two's-complement bit planes (format view)."""
    bits = np.unpackbits(np.ascontiguousarray(planes).view(np.uint8).reshape(qb, -1), axis=1,
                         bitorder="little")[:, :dims].astype(np.int32)
    w = (1 << np.arange(qb, dtype=np.int32))
    w[-1] = -w[-1]
    return (w[:, None] * bits).sum(axis=0).astype(np.int32)


def _prepare_from_rotated(q_rot: np.ndarray, dims: int, params: SearchParams, eps_bound: float = 0.0) -> QueryState:
    """QueryState of an already rotated query (search.py:186-214) on the GPU."""
    q_rot = np.asarray(q_rot, dtype=np.float64)
    sc, planes, luts = _prepare_one(q_rot, params, eps_bound)
    st = QueryState(q_rot=q_rot, sum_q=float(sc[_lib.QS_SUM_Q]))
    if params.ip_mode == "lut":
        st.luts = luts
        return st
    st.delta_q = float(sc[_lib.QS_DELTA])
    st.planes = planes
    st.q_hat = _q_hat_from_planes(planes, dims, params.query_bits)
    st.code_sum_q = float(sc[_lib.QS_CODE_SUM])
    st.ip_margin = float(sc[_lib.QS_IP_MARGIN])
    return st


def prepare_query(q: np.ndarray, index: IvfRabitqIndex, params: SearchParams) -> QueryState:
    """Rotate one query on the GPU and derive its QueryState (search.py:217-223)."""
    q = np.asarray(q, dtype=np.float64)
    if q.shape != (index.dims,):
        raise ValueError(f"query shape {q.shape} != ({index.dims},)")
    qd = dev.to_device(np.ascontiguousarray(q[None, :]))
    q_rot = dev.to_host(rotate_queries_device(qd, index))[0]
    return _prepare_from_rotated(q_rot, index.dims, params, index.eps_bound)


def build_luts(q_rot: np.ndarray, block: int = _LUT_BLOCK) -> np.ndarray:
    """Per-query lookup tables ``L[j][key]`` over 4-dim blocks, float32 (search.py:115-132)."""
    if block != _LUT_BLOCK:
        raise ValueError(f"the packed-nibble layout uses {_LUT_BLOCK}-dim blocks, got block={block}")
    q = np.asarray(q_rot, dtype=np.float64).ravel()
    if q.size == 0:
        return np.zeros((1, 16), dtype=np.float32)
    _, _, luts = _prepare_one(q, SearchParams(k=1, n_probe=1, ip_mode="lut"), 0.0)
    return luts


def nibbles_from_bits(bits_matrix: np.ndarray) -> np.ndarray:
    """(n, dims) 0/1 rows -> (n, blocks) 4-dim nibble keys, zero padded (search.py:135-143; format view)."""
    m = np.atleast_2d(np.asarray(bits_matrix, dtype=np.uint8))
    n, dims = m.shape
    padded_dims = ((dims + 31) // 32) * 32 if dims % 32 else dims
    buf = np.zeros((n, max(padded_dims, _LUT_BLOCK)), dtype=np.uint8)
    buf[:, :dims] = m
    return (buf.reshape(n, -1, _LUT_BLOCK) @ (1 << np.arange(_LUT_BLOCK)).astype(np.uint8)).astype(np.uint8)


def ip_lut(nibbles: np.ndarray, luts: np.ndarray):
    """Binary code x real query via table lookups (search.py:146-160); float64."""
    nib = np.asarray(nibbles)
    single = nib.ndim == 1
    nib2 = np.ascontiguousarray(np.atleast_2d(nib).astype(np.uint8))
    luts = np.ascontiguousarray(np.asarray(luts, dtype=np.float32))
    blocks = luts.shape[0]
    if nib2.shape[1] != blocks:
        raise ValueError(f"nibble count {nib2.shape[1]} != table count {blocks}")
    n = nib2.shape[0]
    out = dev.empty(n, torch.float64)
    nd, ld = dev.to_device(nib2), dev.to_device(luts)  # alive until the launch is queued
    _lib.call("ivrq_ip_lut", dev.ptr(nd), n, blocks, dev.ptr(ld), dev.ptr(out), dev.stream_ptr())
    res = dev.to_host(out)
    return float(res[0]) if single else res


def ip_bitwise(words: np.ndarray, planes: np.ndarray, query_bits: int):
    """Binary code x quantized query via AND + popcount (search.py:163-183); exact int."""
    w = np.asarray(words, dtype=np.uint32)
    single = w.ndim == 1
    w2 = w[:, None] if single else w
    planes = np.asarray(planes, dtype=np.uint32)
    if planes.shape != (query_bits, w2.shape[0]):
        raise ValueError(f"planes shape {planes.shape} != ({query_bits}, {w2.shape[0]})")
    groups, n = w2.shape
    out = dev.empty(n, torch.int64)
    wd, pd = dev.to_device(np.ascontiguousarray(w2)), dev.to_device(np.ascontiguousarray(planes))
    _lib.call("ivrq_ip_bitwise", dev.ptr(wd), groups, n, dev.ptr(pd), query_bits, dev.ptr(out), dev.stream_ptr())
    res = dev.to_host(out)
    return int(res[0]) if single else res


def _short_cols(sf) -> np.ndarray:
    from paper_2602_23999_b200.codec import ShortFactors

    if isinstance(sf, ShortFactors):
        return np.array([sf.add, sf.scale, sf.err], dtype=np.float64)
    return np.asarray(sf, dtype=np.float64)


def _long_cols(lf) -> np.ndarray:
    from paper_2602_23999_b200.codec import LongFactors

    if isinstance(lf, LongFactors):
        return np.array([lf.add, lf.scale], dtype=np.float64)
    return np.asarray(lf, dtype=np.float64)


def estimate_stage1(ip_binary, sf, state: QueryState, d_qc2):
    """1-bit estimate and pruning lower bound, both clamped at 0 (search.py:270-287)."""
    cols = _short_cols(sf)
    ip = np.asarray(ip_binary, dtype=np.float64)
    dq = np.asarray(d_qc2, dtype=np.float64)
    shape = np.broadcast_shapes(ip.shape, cols.shape[:-1], dq.shape)
    n = int(np.prod(shape, dtype=np.int64))
    ipb = np.ascontiguousarray(np.broadcast_to(ip, shape).reshape(n))
    sfb = np.ascontiguousarray(np.broadcast_to(cols, shape + (3,)).reshape(n, 3))
    dqb = np.ascontiguousarray(np.broadcast_to(dq, shape).reshape(n))
    est = dev.empty(n, torch.float64)
    lb = dev.empty(n, torch.float64)
    ipd, sfd, dqd = dev.to_device(ipb), dev.to_device(sfb), dev.to_device(dqb)
    _lib.call("ivrq_estimate_stage1", dev.ptr(ipd), dev.ptr(sfd), n,
              dev.ptr(dqd), float(state.code_sum_q), float(state.ip_margin or 0.0), dev.ptr(est),
              dev.ptr(lb), dev.stream_ptr())
    e, lo = dev.to_host(est).reshape(shape), dev.to_host(lb).reshape(shape)
    if shape == ():
        return np.float64(e), np.float64(lo)
    return e, lo


def refine_stage2(excode, ip_binary, lf, state: QueryState, d_qc2, bits: int):
    """Refined estimate from the full code, clamped at 0 (search.py:290-310)."""
    if bits < 2:
        raise ValueError("refinement requires bits >= 2 (no ex-code exists for 1-bit indexes)")
    ex = np.ascontiguousarray(np.atleast_2d(np.asarray(excode, dtype=np.float64)))
    n, d = ex.shape
    ipb = np.ascontiguousarray(np.broadcast_to(np.asarray(ip_binary, dtype=np.float64), (n,)))
    lfb = np.ascontiguousarray(np.broadcast_to(_long_cols(lf), (n, 2)))
    dqb = np.ascontiguousarray(np.broadcast_to(np.asarray(d_qc2, dtype=np.float64), (n,)))
    q = np.ascontiguousarray(np.asarray(state.q_rot, dtype=np.float64))
    out = dev.empty(n, torch.float64)
    exd, ipd, lfd, qd, dqd = (dev.to_device(a) for a in (ex, ipb, lfb, q, dqb))
    _lib.call("ivrq_refine_stage2", dev.ptr(exd), n, d, dev.ptr(ipd), dev.ptr(lfd), dev.ptr(qd), float(state.sum_q),
              dev.ptr(dqd), bits, dev.ptr(out), dev.stream_ptr())
    res = dev.to_host(out)
    if np.asarray(excode).ndim == 1:
        return float(res[0])
    return res


def cluster_local_search(
    state: QueryState,
    index: IvfRabitqIndex,
    cluster: int,
    params: SearchParams,
    threshold: float = math.inf,
    d_qc2: float | None = None,
) -> tuple[np.ndarray, np.ndarray]:
    """One query, one cluster: stage 1, prune, refine, local top-K by (dist, id) (search.py:326-375)."""
    lo, hi = index.cluster_range(cluster)
    n_c = hi - lo
    if n_c == 0:
        return np.empty(0, dtype=np.int64), np.empty(0, dtype=np.float64)
    device = dev.require_cuda()
    bitwise = params.ip_mode == "bitwise"
    q = dev.to_device(np.ascontiguousarray(np.asarray(state.q_rot, dtype=np.float64)), device)
    planes = dev.to_device(np.ascontiguousarray(state.planes, dtype=np.uint32), device) if bitwise else None
    luts = None if bitwise else dev.to_device(np.ascontiguousarray(state.luts, dtype=np.float32), device)
    if (planes if bitwise else luts) is None:
        raise ValueError(f"the query state has no {'planes' if bitwise else 'tables'} for ip_mode={params.ip_mode!r}")
    import ctypes

    sc = (ctypes.c_double * _lib.QS_COUNT)(*state.scalars().tolist())  # host scalars
    dq = ctypes.byref(ctypes.c_double(float(d_qc2))) if d_qc2 is not None else None
    k = params.k
    out_i = torch.empty(k, dtype=torch.int64, device=device)
    out_d = torch.empty(k, dtype=torch.float64, device=device)
    cnt = torch.zeros(1, dtype=torch.int32, device=device)
    ws_bytes = int(_lib.load().ivrq_cluster_local_search_workspace(n_c))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    _lib.call("ivrq_cluster_local_search", index.view(), int(cluster), dev.ptr(q), dev.ptr(planes), dev.ptr(luts),
              sc, params.to_c(), float(threshold), dq, dev.ptr(out_i), dev.ptr(out_d),
              dev.ptr(cnt), dev.ptr(ws), ws_bytes, n_c, dev.stream_ptr())
    m = int(cnt.item())
    return dev.to_host(out_i[:m]).copy(), dev.to_host(out_d[:m]).copy()


def _probe_device(q_rot: torch.Tensor, cent: torch.Tensor, c_sq: torch.Tensor, n_probe: int, order_by_id: bool,
                  out: tuple[torch.Tensor, torch.Tensor] | None = None, ws: torch.Tensor | None = None):
    nq, d = q_rot.shape
    nlist = cent.shape[0]
    if out is None:
        ids = torch.empty((nq, n_probe), dtype=torch.int64, device=q_rot.device)
        d2 = torch.empty((nq, n_probe), dtype=torch.float64, device=q_rot.device)
    else:
        ids, d2 = out
    lib = _lib.load()
    ws_bytes = int(lib.ivrq_select_clusters_workspace(nq, nlist))
    if ws is None or ws.numel() < ws_bytes:
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q_rot.device)
    _lib.call(
        "ivrq_select_clusters_ordered",
        dev.ptr(q_rot), nq, d, dev.ptr(cent), dev.ptr(c_sq), nlist, n_probe, 1 if order_by_id else 0,
        dev.ptr(ids), dev.ptr(d2), dev.ptr(ws), ws_bytes, dev.stream_ptr(),
    )
    return ids, d2


def select_clusters(q_rot: np.ndarray, centroids: Centroids, n_probe: int) -> tuple[np.ndarray, np.ndarray]:
    """Exact n_probe nearest centroids, ascending (distance, id) (search.py:226-244)."""
    q = np.atleast_2d(np.asarray(q_rot, dtype=np.float64))
    if n_probe > centroids.n_clusters:
        raise ValueError(f"n_probe={n_probe} exceeds {centroids.n_clusters} clusters")
    vals = np.asarray(centroids.values)
    v32 = vals.astype(np.float32)
    qd = dev.to_device(q)
    csq = dev.to_device(np.asarray(centroids.squared_norms, dtype=np.float64))
    if vals.dtype == np.float32 or np.array_equal(v32.astype(vals.dtype), vals):
        ids, d2 = _probe_device(qd, dev.to_device(v32), csq, n_probe, order_by_id=False)
        return dev.to_host(ids), dev.to_host(d2)
    # float64 centroids (e.g. train_kmeans output): the float64 GEMM probe
    cd = dev.to_device(np.ascontiguousarray(vals, dtype=np.float64))
    nq, d = q.shape
    ncl = cd.shape[0]
    ids = torch.empty((nq, n_probe), dtype=torch.int64, device=qd.device)
    d2 = torch.empty((nq, n_probe), dtype=torch.float64, device=qd.device)
    ws_bytes = int(_lib.load().ivrq_select_clusters_workspace(nq, ncl))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=qd.device)
    _lib.call("ivrq_select_clusters_f64", dev.ptr(qd), nq, d, dev.ptr(cd), dev.ptr(csq), ncl, n_probe, 0,
              dev.ptr(ids), dev.ptr(d2), dev.ptr(ws), ws_bytes, dev.stream_ptr())
    return dev.to_host(ids), dev.to_host(d2)


@dataclass
class DeviceResult:
    """Device-resident output of one search batch."""

    ids: torch.Tensor  # (nq, k) int64, -1 padded
    dists: torch.Tensor  # (nq, k) float64, +inf padded
    counts: torch.Tensor  # (nq,) int32
    stats: torch.Tensor | None  # (nq, 2) int64: vectors probed, stage-1 survivors


def rotate_queries_device(q: torch.Tensor, index: IvfRabitqIndex, out: torch.Tensor | None = None) -> torch.Tensor:
    nq, d = q.shape
    q_rot = torch.empty((nq, d), dtype=torch.float64, device=q.device) if out is None else out
    if nq:
        _lib.call(
            "ivrq_rotate_queries",
            dev.ptr(q), 1 if q.dtype == torch.float64 else 0, nq, d, dev.ptr(index.device["rotation"]),
            dev.ptr(q_rot), dev.stream_ptr(),
        )
    return q_rot


def _query_state_buffers(nq: int, d: int, index: IvfRabitqIndex, params: SearchParams, device):
    """scalars, planes, luts, qslices as ivrq_prepare_queries writes them (None when unused)."""
    g = (d + 31) // 32
    scalars = torch.empty((nq, _lib.QS_COUNT), dtype=torch.float64, device=device)
    planes = luts = qslices = None
    if params.refine and index.bits >= 2:
        kpad = (d + 63) // 64 * 64
        qslices = torch.empty((nq, 8, kpad), dtype=torch.int8, device=device)
    if params.ip_mode == "bitwise":
        planes = torch.empty((nq, params.query_bits, g), dtype=torch.int32, device=device)
    else:
        luts = torch.empty((nq, 8 * g, 16), dtype=torch.float32, device=device)
    return scalars, planes, luts, qslices


def prepare_queries_device(q_rot: torch.Tensor, index: IvfRabitqIndex, params: SearchParams, out=None):
    """QueryState scalars + planes/LUTs for every query (device tensors); ``out`` = row slices
    of buffers from _query_state_buffers."""
    nq, d = q_rot.shape
    scalars, planes, luts, qslices = out if out is not None else _query_state_buffers(nq, d, index, params,
                                                                                      q_rot.device)
    cp = params.to_c()
    _lib.call(
        "ivrq_prepare_queries",
        dev.ptr(q_rot), nq, d, cp, index.bits, float(index.eps_bound),
        dev.ptr(scalars), dev.ptr(planes), dev.ptr(luts), dev.ptr(qslices), dev.stream_ptr(),
    )
    return scalars, planes, luts, qslices


def search_device(
    q: torch.Tensor,
    index: IvfRabitqIndex,
    params: SearchParams,
    *,
    q_rot: torch.Tensor | None = None,
    with_stats: bool = False,
    events: dict[str, torch.cuda.Event] | None = None,
) -> DeviceResult:
    """The whole search on device tensors (queries already in HBM).

    ``q_rot`` (tests only) injects precomputed rotated queries, the
    reference's own, to compare everything downstream bit-exactly.
    ``events`` (bench only) receives CUDA events recorded on the current
    stream at the stage boundaries: start, rotated, probed, prepared, scanned.
    """

    def mark(name: str) -> None:
        if events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            events[name] = ev

    mark("start")
    nq = q.shape[0] if q_rot is None else q_rot.shape[0]
    if q_rot is None:
        q_rot = rotate_queries_device(q, index)
    mark("rotated")
    t = index.device
    # query prep on the side stream beside the probe (both only read q_rot); the "probed"
    # stage mark therefore covers both, "prepared" follows it at once
    state = _query_state_buffers(nq, q_rot.shape[1], index, params, q_rot.device)
    # (measured on C3: beside the probe 3.28 ms per step, after it 3.31; a high-priority side stream 3.28)
    with _forked() as side:
        with torch.cuda.stream(side):
            scalars, planes, luts, qslices = prepare_queries_device(q_rot, index, params, out=state)
        probe_ids, probe_d2 = _probe_device(q_rot, t["centroids"], t["centroid_sqnorms"], params.n_probe, True)
    mark("probed")
    mark("prepared")
    res = _scan_device(q_rot, index, params, probe_ids, probe_d2, (scalars, planes, luts, qslices), with_stats)
    mark("scanned")
    return res


def _scan_device(q_rot, index: IvfRabitqIndex, params: SearchParams, probe_ids, probe_d2, state,
                 with_stats: bool = False) -> DeviceResult:
    """ivrq_search_scan over the whole batch (the per-query loop, search.py:425-448)."""
    nq = q_rot.shape[0]
    scalars, planes, luts, qslices = state
    k = params.k
    out_ids = torch.empty((nq, k), dtype=torch.int64, device=q_rot.device)
    out_d = torch.empty((nq, k), dtype=torch.float64, device=q_rot.device)
    counts = torch.empty(nq, dtype=torch.int32, device=q_rot.device)
    stats = torch.empty((nq, 2), dtype=torch.int64, device=q_rot.device) if with_stats else None
    cp = params.to_c()
    _lib.call(
        "ivrq_search_scan",
        index.view(), dev.ptr(q_rot), dev.ptr(probe_ids), dev.ptr(probe_d2), dev.ptr(scalars), dev.ptr(planes),
        dev.ptr(luts), dev.ptr(qslices), nq, cp, dev.ptr(out_ids), dev.ptr(out_d), dev.ptr(counts), dev.ptr(stats),
        dev.stream_ptr(),
    )
    return DeviceResult(ids=out_ids, dists=out_d, counts=counts, stats=stats)


def _rows_to_lists(ids: np.ndarray, dists: np.ndarray, counts: np.ndarray) -> list[tuple[np.ndarray, np.ndarray]]:
    """One (ids, dists) pair per row, trimmed to the row's count.

    The pairs are row views of ``ids`` / ``dists``, which must be fresh arrays
    owned by the caller (rows are disjoint, so the views are independent).
    """
    k = ids.shape[1]
    if counts.size and int(counts.min()) == k:
        return list(zip(list(ids), list(dists)))
    return [(ids[i, :n], dists[i, :n]) for i, n in enumerate(counts.tolist())]


def results_to_lists(res: DeviceResult) -> list[tuple[np.ndarray, np.ndarray]]:
    return _rows_to_lists(dev.to_host(res.ids), dev.to_host(res.dists), dev.to_host(res.counts))


# ------------------------------------------------------------------ host pipeline
_PINNED = threading.local()  # per calling thread: concurrent readers never share staging memory


def _pinned(device: torch.device, name: str, nbytes: int) -> torch.Tensor:
    """A page-locked staging buffer (uint8), grown on demand, kept per device and per thread.

    The index is immutable and ``search_batch`` may be called from several
    threads at once (reference index.py:7-8), so each thread stages its queries
    and results in its own buffers.
    """
    bufs = getattr(_PINNED, "bufs", None)
    if bufs is None:
        bufs = _PINNED.bufs = {}
    key = (device.index or 0, name)
    buf = bufs.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        bufs[key] = buf
    return buf


def _env_int(name: str, default: int) -> int:
    v = os.environ.get(name)
    return int(v) if v else default


_STAGE_THREADS = max(1, _env_int("IVRQ_STAGE_THREADS", min(8, os.cpu_count() or 4)))
_POOL = None


def _stage_pieces(nq: int) -> int:
    """Host->device pieces of a single-batch search (copy / transfer / rotation overlap):
    pieces of >= 1024 queries keep every rotation GEMM at least a wave of tiles."""
    return max(1, min(_env_int("IVRQ_STAGE_PIECES", 4), nq // 1024))


def _stage_pool():
    """Threads for the pinned-memory staging copies (np.copyto drops the GIL)."""
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _POOL = ThreadPoolExecutor(_STAGE_THREADS, thread_name_prefix="ivrq-stage")
    return _POOL


def _chunk_bounds(nq: int) -> list[int]:
    """Query chunks of the host pipeline: big enough that each keeps the GPU busy
    (the first-list phase shares list passes between queries of one chunk),
    small enough that host work on one chunk hides behind the next chunk's kernels."""
    import os

    split = os.environ.get("IVRQ_E2E_SPLIT")  # e.g. "0.7": two chunks, the first 70% of the queries
    if split and nq >= 4096:
        a = int(nq * float(split))
        return [0, a, nq] if 0 < a < nq else [0, nq]
    env = os.environ.get("IVRQ_E2E_CHUNKS")
    n = int(env) if env else 1  # each chunk re-streams the index (list-major kernels): one batch
    n = max(1, min(n, nq))
    return [nq * i // n for i in range(n + 1)]


_WAIT_OK: bool | None = None


def _stream_wait_supported(flag_ptr: int) -> bool:
    """Whether the driver takes stream waits on a host flag (probed once, value 0 always holds)."""
    global _WAIT_OK
    if _WAIT_OK is None:
        if os.environ.get("IVRQ_STREAM_WAIT", "1") == "0":
            _WAIT_OK = False
        else:
            try:
                _lib.call("ivrq_stream_wait_flag", flag_ptr, 0, dev.stream_ptr())
                _WAIT_OK = True
            except Exception:
                _WAIT_OK = False
    return _WAIT_OK


def _copy_stream(device) -> torch.cuda.Stream:
    """The calling thread's host->device copy stream on ``device``."""
    streams = getattr(_PINNED, "copy_streams", None)
    if streams is None:
        streams = _PINNED.copy_streams = {}
    key = device.index or 0
    if key not in streams:
        streams[key] = torch.cuda.Stream(device)
    return streams[key]


class _forked:
    """Fork the current stream into the calling thread's side stream and join it back on exit.

    Buffers used on the side stream must be allocated before the fork (they are then
    free on the current stream's timeline, which the side stream joins first)."""

    def __enter__(self) -> torch.cuda.Stream:
        self.main = torch.cuda.current_stream()
        dev_ = self.main.device
        streams = getattr(_PINNED, "side_streams", None)
        if streams is None:
            streams = _PINNED.side_streams = {}
        key = dev_.index or 0
        if key not in streams:
            streams[key] = torch.cuda.Stream(dev_)
        self.side = streams[key]
        self.side.wait_stream(self.main)
        return self.side

    def __exit__(self, *exc) -> None:
        self.main.wait_stream(self.side)


def _native_copy(pairs) -> None:
    """np.copyto(dst, src) for C-contiguous pairs of equal shape, on the native staging threads."""
    import ctypes

    handles = []
    flags = np.zeros(len(pairs) * _STAGE_THREADS, dtype=np.uint32)
    try:
        for i, (dst, src) in enumerate(pairs):
            if dst.nbytes < (256 << 10):
                np.copyto(dst, src)
                continue
            h = ctypes.c_void_p()
            rows = dst.shape[0]
            _lib.call("ivrq_stage_rows", dst.ctypes.data, src.ctypes.data, rows, dst.nbytes // max(rows, 1), 1,
                      _STAGE_THREADS, flags.ctypes.data + 4 * i * _STAGE_THREADS, ctypes.byref(h))
            handles.append(h)
    finally:
        for h in handles:
            _lib.call("ivrq_stage_join", h)


class _PieceStager:
    """Host copy of a query batch into pinned memory, in row pieces, on native threads.

    ivrq_stage_rows splits every piece over all threads, which copy the pieces in
    order and raise one page-locked flag word per piece; piece 0 is staged after 1/P
    of the copy.  When the driver supports stream memory operations the stream waits
    on the piece's flag (ivrq_stream_wait_flag), so the whole search is enqueued while
    the copy runs; otherwise ``wait(p)`` blocks the host on piece p.  Nothing on the
    publish path needs the interpreter: a GPU-synchronising call made while the GIL is
    held (an allocation, say) cannot deadlock against the staging.
    """

    def __init__(self, q: np.ndarray, pin_np: np.ndarray, device) -> None:
        import ctypes

        nq = q.shape[0]
        npieces = _stage_pieces(nq)
        edges = [nq * p // npieces for p in range(npieces + 1)]  # the same split as ivrq_stage_rows
        self.pieces = list(zip(edges[:-1], edges[1:]))
        self.max_piece = max(y - x for x, y in self.pieces)
        self.nthreads = _STAGE_THREADS
        flags_t = _pinned(device, "flag", 4 * npieces)[: 4 * npieces]
        self.flags_ptr = flags_t.data_ptr()
        self.stream_wait = _stream_wait_supported(self.flags_ptr)
        self._q = q  # kept alive until the threads are joined
        self._handle = ctypes.c_void_p()
        _lib.call("ivrq_stage_rows", pin_np.ctypes.data, q.ctypes.data, nq, q.strides[0], npieces, self.nthreads,
                  self.flags_ptr, ctypes.byref(self._handle))

    def wait(self, p: int) -> None:
        if self.stream_wait:
            _lib.call("ivrq_stream_wait_flag", self.flags_ptr + 4 * p, self.nthreads, dev.stream_ptr())
        else:
            _lib.call("ivrq_stage_wait", self.flags_ptr, p, self.nthreads)

    def finish(self) -> None:
        """Join the copy threads (every flag then holds its final value: no wait stays pending)."""
        if self._handle:
            _lib.call("ivrq_stage_join", self._handle)
            self._handle = None


class _Front:
    """Rotation, probe and query state for row pieces of one batch, into whole-batch buffers."""

    def __init__(self, nq: int, d: int, index: IvfRabitqIndex, params: SearchParams, device, max_piece: int):
        self.index, self.params = index, params
        t = index.device
        self.cent, self.c_sq = t["centroids"], t["centroid_sqnorms"]
        self.q_rot = torch.empty((nq, d), dtype=torch.float64, device=device)
        self.probe_ids = torch.empty((nq, params.n_probe), dtype=torch.int64, device=device)
        self.probe_d2 = torch.empty((nq, params.n_probe), dtype=torch.float64, device=device)
        self.state = _query_state_buffers(nq, d, index, params, device)
        ws_bytes = int(_lib.load().ivrq_select_clusters_workspace(max_piece, self.cent.shape[0]))
        self.ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)

    def run(self, qd: torch.Tensor, x: int, y: int) -> None:
        if y <= x:
            return
        q_rot = self.q_rot[x:y]
        rotate_queries_device(qd, self.index, out=q_rot)
        with _forked() as side:  # query prep beside the probe (both only read q_rot)
            with torch.cuda.stream(side):
                prepare_queries_device(q_rot, self.index, self.params,
                                       out=tuple(None if b is None else b[x:y] for b in self.state))
            _probe_device(q_rot, self.cent, self.c_sq, self.params.n_probe, True,
                          out=(self.probe_ids[x:y], self.probe_d2[x:y]), ws=self.ws)


def _search_pipelined(q: np.ndarray, index: IvfRabitqIndex, params: SearchParams, t_enter: float = 0.0):
    """search_batch for host queries, pipelined over query chunks on one stream.

    Per chunk: host memcpy into a pinned buffer, async H2D, the four search
    launches, async D2H of (ids, dists, counts) into pinned memory, an event.
    While the GPU runs chunk i the host stages chunk i+1's queries and turns
    chunk i-1's results into the per-query lists.
    """
    device = dev.require_cuda()
    nq, d = q.shape
    k = params.k
    bounds = _chunk_bounds(nq)
    stream = torch.cuda.current_stream(device)
    tdt = torch.float32 if q.dtype == np.float32 else torch.float64
    pin_q_t = _pinned(device, "q", q.nbytes)[: q.nbytes].view(tdt).view(nq, d)
    pin_q_np = pin_q_t.numpy()
    nk = nq * k
    pin_o = _pinned(device, "out", nk * 16 + nq * 4)
    ids_t = pin_o[: nk * 8].view(torch.int64).view(nq, k)
    dists_t = pin_o[nk * 8 : nk * 16].view(torch.float64).view(nq, k)
    counts_t = pin_o[nk * 16 : nk * 16 + nq * 4].view(torch.int32)
    ids_h, dists_h, counts_h = ids_t.numpy(), dists_t.numpy(), counts_t.numpy()
    qd = torch.empty((nq, d), dtype=pin_q_t.dtype, device=device)
    # the previous call's D2H into the same pinned buffers has been consumed
    # (search_batch returns only after its last event), so no wait is needed here
    ids_out = np.empty((nq, k), dtype=np.int64)
    dists_out = np.empty((nq, k), dtype=np.float64)
    counts_out = np.empty(nq, dtype=np.int32)
    done: list[tuple[int, int, torch.cuda.Event]] = []
    results: list[tuple[np.ndarray, np.ndarray]] = []

    def finish(a: int, b: int, ev: torch.cuda.Event) -> None:
        ev.synchronize()
        np.copyto(ids_out[a:b], ids_h[a:b])
        np.copyto(dists_out[a:b], dists_h[a:b])
        np.copyto(counts_out[a:b], counts_h[a:b])
        results.extend(_rows_to_lists(ids_out[a:b], dists_out[a:b], counts_out[a:b]))

    def stage(i: int) -> list:
        # host copy of chunk i into pinned memory, split over the staging threads
        a, b = bounds[i], bounds[i + 1]
        parts = np.linspace(a, b, _STAGE_THREADS + 1).astype(np.int64)
        pool = _stage_pool()
        return [pool.submit(np.copyto, pin_q_np[x:y], q[x:y]) for x, y in zip(parts[:-1], parts[1:]) if y > x]

    if len(bounds) == 2:  # one batch: staging, transfer, rotation, probe and prep overlap piecewise
        import time

        trace = os.environ.get("IVRQ_E2E_TRACE")
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            stager = _PieceStager(q, pin_q_np, device)
            try:
                front = _Front(nq, d, index, params, device, stager.max_piece)
                tev = []

                def tmark(name):
                    if trace:
                        e = torch.cuda.Event(enable_timing=True)
                        e.record(stream)
                        tev.append((name, e))

                tmark("start")
                # H2D copies on a copy stream (each behind its piece's flag), so the transfer of
                # piece p+1 overlaps the rotation / probe / prep of piece p on the compute stream
                cstream = _copy_stream(device)
                ready = torch.cuda.Event()
                ready.record(stream)  # qd's memory is free on the compute stream from here
                cstream.wait_event(ready)
                qd.record_stream(cstream)
                for p, (x, y) in enumerate(stager.pieces):
                    with torch.cuda.stream(cstream):
                        stager.wait(p)  # a stream wait on the published flag (or a host wait)
                        qd[x:y].copy_(pin_q_t[x:y], non_blocking=True)
                        landed = torch.cuda.Event()
                        landed.record(cstream)
                    stream.wait_event(landed)
                    tmark(f"h{p}")
                    front.run(qd[x:y], x, y)
                    tmark(f"f{p}")
                t1 = time.perf_counter()
                res = _scan_device(front.q_rot, index, params, front.probe_ids, front.probe_d2, front.state)
                tmark("scan")
                ids_t.copy_(res.ids, non_blocking=True)
                dists_t.copy_(res.dists, non_blocking=True)
                counts_t.copy_(res.counts, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            finally:
                stager.finish()  # every piece published (releases the stream on any error), copies joined
            t2 = time.perf_counter()
            # the per-query row views are made while the GPU searches; the results are copied
            # into the viewed arrays once the event fires, short rows (count < k) re-cut after
            rows = list(zip(list(ids_out), list(dists_out)))
            ev.synchronize()
            t3 = time.perf_counter()
            _native_copy([(ids_out, ids_h), (dists_out, dists_h), (counts_out, counts_h)])
            if nq and int(counts_out.min()) < k:
                for i in np.flatnonzero(counts_out < k).tolist():
                    n = int(counts_out[i])
                    rows[i] = (ids_out[i, :n], dists_out[i, :n])
            results.extend(rows)
            t4 = time.perf_counter()
        if trace:
            import sys

            print(f"[e2e] setup {1e3*(t0-t_enter):.2f} front enqueued {1e3*(t1-t0):.2f} scan enqueued + staged {1e3*(t2-t1):.2f} "
                  f"row views + gpu-wait {1e3*(t3-t2):.2f} copy-out {1e3*(t4-t3):.2f} ms "
                  f"(stream wait {'on' if stager.stream_wait else 'off'})", file=sys.stderr)
            print("[e2e] gpu timeline ms: " + " ".join(f"{n} {tev[0][1].elapsed_time(e):.2f}" for n, e in tev[1:]),
                  file=sys.stderr)
        return results

    with torch.cuda.stream(stream):
        pending = stage(0)
        for i in range(len(bounds) - 1):
            a, b = bounds[i], bounds[i + 1]
            for f in pending:
                f.result()
            qd[a:b].copy_(pin_q_t[a:b], non_blocking=True)
            res = search_device(qd[a:b], index, params)
            ids_t[a:b].copy_(res.ids, non_blocking=True)
            dists_t[a:b].copy_(res.dists, non_blocking=True)
            counts_t[a:b].copy_(res.counts, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            done.append((a, b, ev))
            pending = stage(i + 1) if i + 2 < len(bounds) else []
            if i > 0:
                finish(*done[i - 1])
        finish(*done[-1])
    return results


def _validate(q: np.ndarray, index: IvfRabitqIndex, params: SearchParams) -> None:
    if q.shape[1] != index.dims:
        raise ValueError(f"query dims {q.shape[1]} != index dims {index.dims}")
    if params.n_probe > index.n_clusters:
        raise ValueError(f"n_probe={params.n_probe} exceeds {index.n_clusters} clusters")


def search_batch(
    queries: np.ndarray,
    index: IvfRabitqIndex,
    params: SearchParams,
    workers: int | None = None,
) -> list[tuple[np.ndarray, np.ndarray]]:
    """Approximate K nearest neighbours per query row (search.py:390-454).

    Returns one ``(ids int64, dists float64)`` pair per query, ascending by
    (distance, id), with fewer than K entries when the probed lists hold fewer.
    """
    import time

    t_enter = time.perf_counter()
    q = np.atleast_2d(np.asarray(queries))
    if q.dtype not in (np.float32, np.float64):
        q = q.astype(np.float64)
    q = np.ascontiguousarray(q)
    _validate(q, index, params)
    if workers is None:
        default_workers()
    if q.shape[0] == 0:
        return []
    return _search_pipelined(q, index, params, t_enter)
