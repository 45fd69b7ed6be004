"""Multi-GPU IVF-RaBitQ: list-sharded index, all-gather merge and the exact chain.

The index shards naturally by inverted list: rank r owns the
contiguous cluster-id range ``ranges[r]``, balanced by vector count, and keeps
those lists renumbered from 0.  Every rank holds all centroids and the
rotation, so probing is local.  Two search protocols:

* ``merge`` -- each rank scans its lists for all queries (fresh pools), the
  per-query top-k are all-gathered and merged by (dist, pid).  Exact when the
  result does not depend on the probe order: 1-bit indexes (pruning is safe)
  or ``prune=False``.  For B >= 2 with pruning it is "recall-parity mode".
* ``chain`` -- exact for every configuration.  The reference visits a query's
  lists in ascending id carrying its pool and threshold (search.py:429-447);
  since ranks own ascending id ranges, rank r continues the pool handed over
  by rank r-1 (NCCL send/recv over NVLink).  Queries are split into
  micro-batches so ranks work on different micro-batches concurrently; the
  last rank broadcasts the final pools.

The protocols take the per-shard scan as a callable so the host-side logic is
exercised with gloo on CPU (tests/test_distributed_gloo.py).  On GPUs the
scan is ``ivrq_search_scan_shard`` and the merge ``ivrq_merge_topk``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch
import torch.distributed as tdist

from paper_2602_23999_b200 import _device as dev
from paper_2602_23999_b200 import _lib

__all__ = [
    "cluster_ranges",
    "merge_protocol",
    "chain_protocol",
    "ShardedIndex",
    "build_sharded",
    "train_kmeans_sharded",
    "search_sharded",
]

Pools = tuple[torch.Tensor, torch.Tensor, torch.Tensor]  # ids (nq,k) int64, dists (nq,k) f64, counts (nq,) int32


def cluster_ranges(counts: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous cluster-id ranges, one per rank, with balanced vector counts."""
    counts = np.asarray(counts, dtype=np.int64)
    nlist = counts.size
    if world < 1 or world > nlist:
        raise ValueError(f"cannot shard {nlist} lists over {world} ranks")
    prefix = np.concatenate(([0], np.cumsum(counts)))
    total = prefix[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        cut = int(np.searchsorted(prefix, target, side="left"))
        cut = max(cut, bounds[-1] + 1)  # every rank owns >= 1 list
        cut = min(cut, nlist - (world - r))
        bounds.append(cut)
    bounds.append(nlist)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


# ---------------------------------------------------------------- protocols


def _host_staged(group) -> bool:
    """Collectives of non-NCCL backends (gloo: the CPU tests) go through host tensors."""
    return tdist.get_backend(group) != "nccl"


def merge_protocol(local: Pools, k: int, group, merge_fn: Callable[[Pools, int, int], Pools]) -> Pools:
    """All-gather every rank's per-query top-k and merge them (exact for order-independent searches)."""
    world = tdist.get_world_size(group)
    host = _host_staged(group)
    device = local[0].device
    outs = []
    for t in local:
        x = t.cpu() if host else t.contiguous()
        g = [torch.empty_like(x) for _ in range(world)]
        tdist.all_gather(g, x, group=group)
        outs.append(torch.stack(g).to(device))
    return merge_fn(tuple(outs), world, k)  # [parts, nq, k]


def chain_protocol(
    scan_fn: Callable[[slice, Pools | None], Pools],
    nq: int,
    k: int,
    group,
    n_micro: int = 4,
    device: torch.device | str = "cpu",
) -> Pools:
    """Ascending-id chain over ranks: rank r continues rank r-1's pools, exactly.

    ``scan_fn(query_slice, init)`` scans this rank's lists for the queries in the slice
    starting from ``init`` pools (None on rank 0) and returns pools.  Micro-batches pipeline
    the chain: rank r scans micro-batch m + 1 while rank r + 1 continues micro-batch m
    (sends are asynchronous; on NCCL they are ordered after the scan on the device).
    """
    rank = tdist.get_rank(group)
    world = tdist.get_world_size(group)
    host = _host_staged(group)
    out_ids = torch.empty((nq, k), dtype=torch.int64, device=device)
    out_d = torch.empty((nq, k), dtype=torch.float64, device=device)
    out_c = torch.empty(nq, dtype=torch.int32, device=device)
    n_micro = max(1, min(n_micro, nq))
    edges = np.linspace(0, nq, n_micro + 1).astype(np.int64)
    src = (tdist.get_global_rank(group, rank - 1) if group is not None else rank - 1) if rank > 0 else None
    dst = (tdist.get_global_rank(group, rank + 1) if group is not None else rank + 1) if rank < world - 1 else None
    pending = []
    for m in range(n_micro):
        sl = slice(int(edges[m]), int(edges[m + 1]))
        nm = sl.stop - sl.start
        init = None
        if src is not None:
            bufs = (
                torch.empty((nm, k), dtype=torch.int64, device="cpu" if host else device),
                torch.empty((nm, k), dtype=torch.float64, device="cpu" if host else device),
                torch.empty(nm, dtype=torch.int32, device="cpu" if host else device),
            )
            for b in bufs:
                tdist.recv(b, src=src, group=group)
            init = tuple(b.to(device) for b in bufs)
        ids, dists, counts = scan_fn(sl, init)
        if dst is not None:
            for t in (ids, dists, counts):
                x = t.cpu() if host else t.contiguous()
                pending.append((tdist.isend(x, dst=dst, group=group), x))
        else:
            out_ids[sl] = ids
            out_d[sl] = dists
            out_c[sl] = counts
    for req, _ in pending:
        req.wait()
    last = tdist.get_global_rank(group, world - 1) if group is not None else world - 1
    res = []
    for t in (out_ids, out_d, out_c):
        x = t.cpu() if host else t
        tdist.broadcast(x, src=last, group=group)
        res.append(x.to(device))
    return tuple(res)  # type: ignore[return-value]


# ---------------------------------------------------------------- GPU implementation


@dataclass
class ShardedIndex:
    """This rank's lists of a list-sharded index plus the shared probe data."""

    local: "object"  # IvfRabitqIndex over clusters [list_lo, list_hi), renumbered from 0
    list_lo: int
    list_hi: int
    n_clusters: int
    centroids: torch.Tensor  # all rotated centroids (nlist, D) float32
    centroid_sqnorms: torch.Tensor
    ranges: list[tuple[int, int]]


def slice_lists(full, lo: int, hi: int, ranges: list[tuple[int, int]] | None = None) -> ShardedIndex:
    """The lists [lo, hi) of a device index as a renumbered shard (device copies)."""
    from paper_2602_23999_b200.index import IvfRabitqIndex

    t = full.device
    off = dev.to_host(t["offsets"]).astype(np.int64)
    r0, r1 = int(off[lo]), int(off[hi])
    g = full.words_per_vector
    rb = int(_lib.load().ivrq_rcode_row_bytes(full.dims, full.bits))
    local_off = torch.as_tensor(off[lo : hi + 1] - off[lo], dtype=torch.int64, device=t["offsets"].device)
    local = {
        "offsets": local_off,
        "packed_msb": t["packed_msb"][g * r0 : g * r1].clone(),
        "short_add": t["short_add"][r0:r1].clone(),
        "short_scale": t["short_scale"][r0:r1].clone(),
        "short_err": t["short_err"][r0:r1].clone(),
        "long_factors": t["long_factors"][r0:r1].clone(),
        "rcodes": t["rcodes"][rb * r0 : rb * r1].clone(),
        "pids": t["pids"][r0:r1].clone(),
        "centroids": t["centroids"][lo:hi].clone(),
        "centroid_sqnorms": t["centroid_sqnorms"][lo:hi].clone(),
        "rotation": t["rotation"],
    }
    shard = IvfRabitqIndex(
        dims=full.dims, bits=full.bits, n_clusters=hi - lo, size=r1 - r0, eps_bound=full.eps_bound,
        seed=full.seed, device_arrays=local,
    )
    return ShardedIndex(
        local=shard, list_lo=lo, list_hi=hi, n_clusters=full.n_clusters, centroids=t["centroids"],
        centroid_sqnorms=t["centroid_sqnorms"], ranges=ranges or [(lo, hi)],
    )


class _Comm:
    """Collectives for the sharded build and search: NCCL on device tensors, or any other
    backend (gloo: the multi-process tests) through host copies."""

    def __init__(self, group=None):
        self.group = group
        self.on = tdist.is_available() and tdist.is_initialized()
        self.rank = tdist.get_rank(group) if self.on else 0
        self.world = tdist.get_world_size(group) if self.on else 1
        self.host = self.on and tdist.get_backend(group) != "nccl"

    def _g(self, r: int) -> int:
        return tdist.get_global_rank(self.group, r) if self.group is not None else r

    def _out(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.host else t.contiguous()

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if not self.on:
            return t
        x = self._out(t).clone()
        tdist.all_reduce(x, op=tdist.ReduceOp.SUM, group=self.group)
        return x.to(t.device)

    def all_gather(self, t: torch.Tensor) -> list[torch.Tensor]:
        """Same-shape tensors from every rank, in rank order."""
        if not self.on:
            return [t]
        x = self._out(t)
        outs = [torch.empty_like(x) for _ in range(self.world)]
        tdist.all_gather(outs, x, group=self.group)
        return [o.to(t.device) for o in outs]

    def all_gather_rows(self, t: torch.Tensor) -> list[torch.Tensor]:
        """Tensors whose first dimension differs per rank, in rank order."""
        if not self.on:
            return [t]
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        sizes = [int(v.item()) for v in self.all_gather(n)]
        m = max(sizes)
        pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        return [g[:sz] for g, sz in zip(self.all_gather(pad), sizes)]

    def broadcast(self, t: torch.Tensor, src: int) -> torch.Tensor:
        if not self.on:
            return t
        x = self._out(t).clone()
        tdist.broadcast(x, src=self._g(src), group=self.group)
        return x.to(t.device)

    def send(self, t: torch.Tensor, dst: int) -> None:
        tdist.send(self._out(t), dst=self._g(dst), group=self.group)

    def recv_like(self, t: torch.Tensor, src: int) -> torch.Tensor:
        x = torch.empty_like(self._out(t))
        tdist.recv(x, src=self._g(src), group=self.group)
        return x.to(t.device)

    def exchange_rows(self, parts: list[torch.Tensor]) -> list[torch.Tensor]:
        """All-to-all of row blocks: parts[d] goes to rank d; returns the blocks received, in
        source-rank order (so rows keep their global order when sources own ascending rows)."""
        if not self.on:
            return parts
        sizes = torch.tensor([p.shape[0] for p in parts], dtype=torch.int64, device=parts[0].device)
        recv_sizes = [int(v) for v in torch.stack(self.all_gather(sizes))[:, self.rank].tolist()]
        tail = tuple(parts[0].shape[1:])
        if not self.host:  # NCCL: one all-to-all over the concatenated blocks
            out = torch.empty((sum(recv_sizes),) + tail, dtype=parts[0].dtype, device=parts[0].device)
            tdist.all_to_all_single(out, torch.cat(parts).contiguous(), output_split_sizes=recv_sizes,
                                    input_split_sizes=[p.shape[0] for p in parts], group=self.group)
            return list(torch.split(out, recv_sizes))
        got: list[torch.Tensor | None] = [None] * self.world
        reqs = []
        for d in range(self.world):
            if d == self.rank:
                got[d] = parts[d]
                continue
            reqs.append(tdist.isend(parts[d].cpu().contiguous(), dst=self._g(d), group=self.group))
        bufs = {}
        for src in range(self.world):
            if src != self.rank:
                bufs[src] = torch.empty((recv_sizes[src],) + tail, dtype=parts[0].dtype)
                reqs.append(tdist.irecv(bufs[src], src=self._g(src), group=self.group))
        for r in reqs:
            r.wait()
        for src, b in bufs.items():
            got[src] = b.to(parts[0].device)
        return got  # type: ignore[return-value]


def _reseed_distributed(comm: _Comm, labels: torch.Tensor, dmin: torch.Tensor, counts_g: torch.Tensor) -> None:
    """Empty-cluster reseeding over rows spread across ranks (clustering.py:100-107): for each
    empty cluster in ascending id, the first row (in global row order) with maximal dmin."""
    for j in torch.nonzero(counts_g == 0).flatten().tolist():
        if dmin.numel():
            val, idx = torch.max(dmin, 0)  # first occurrence of the maximum
            mine = torch.stack([val.to(torch.float64), idx.to(torch.float64)])
        else:
            mine = torch.tensor([-math.inf, 0.0], dtype=torch.float64, device=labels.device)
        cand = torch.stack(comm.all_gather(mine)).cpu().numpy()
        best = max(range(comm.world), key=lambda r: (cand[r, 0], -r))  # ties: the earlier rank's rows
        if best == comm.rank:
            i = int(cand[best, 1])
            labels[i] = j
            dmin[i] = -1.0


def train_kmeans_sharded(x_train_local: torch.Tensor, n_clusters: int, iters: int, seed: int,
                         comm: _Comm) -> torch.Tensor:
    """k-means over training rows split across ranks in ascending row blocks.

    The k-means++ seeding (clustering.py:60-79) is a chain of n_clusters dependent draws over
    the whole training set: every rank runs it on the all-gathered rows (identical result).
    The Lloyd iterations (clustering.py:82-113) are data parallel: labels of local rows, global
    counts by all-reduce, reseeding over all ranks, and the centroid sums as a chain over the
    ranks in row order (ivrq_kmeans_chain_sums), which reproduces np.add.reduceat exactly.
    """
    from paper_2602_23999_b200.clustering import _kmeanspp_device, assign_device, counting_sort, row_sqnorms

    device = x_train_local.device
    d = x_train_local.shape[1]
    xt_all = torch.cat(comm.all_gather_rows(x_train_local))
    centers = _kmeanspp_device(xt_all, n_clusters, seed)
    del xt_all
    n_loc = x_train_local.shape[0]
    for _ in range(iters):
        c_sq = row_sqnorms(centers)
        if n_loc:
            labels, dmin = assign_device(x_train_local, centers, c_sq, with_dmin=True)
        else:
            labels = torch.empty(0, dtype=torch.int32, device=device)
            dmin = torch.empty(0, dtype=torch.float64, device=device)
        counts_l = torch.bincount(labels.long(), minlength=n_clusters)
        counts_g = comm.all_reduce_sum(counts_l)
        if bool((counts_g == 0).any()):
            _reseed_distributed(comm, labels, dmin, counts_g)
            counts_l = torch.bincount(labels.long(), minlength=n_clusters)
            counts_g = comm.all_reduce_sum(counts_l)
        if n_loc:
            _, offsets, order = counting_sort(labels, n_clusters)
        else:
            offsets = torch.zeros(n_clusters + 1, dtype=torch.int64, device=device)
            order = torch.empty(0, dtype=torch.int64, device=device)
        init_s = init_c = None
        if comm.rank > 0:
            init_s = comm.recv_like(torch.empty((n_clusters, d), dtype=torch.float64, device=device), comm.rank - 1)
            init_c = comm.recv_like(torch.empty(n_clusters, dtype=torch.int64, device=device), comm.rank - 1)
        last = comm.rank == comm.world - 1
        out = torch.empty((n_clusters, d), dtype=torch.float64, device=device)
        out_c = torch.empty(n_clusters, dtype=torch.int64, device=device)
        _lib.call(
            "ivrq_kmeans_chain_sums", dev.ptr(x_train_local), dev.ptr(order), dev.ptr(offsets), n_clusters, d,
            dev.ptr(init_s), dev.ptr(init_c), dev.ptr(counts_g) if last else None, dev.ptr(out), dev.ptr(out_c),
            dev.stream_ptr(),
        )
        if not last:
            comm.send(out, comm.rank + 1)
            comm.send(out_c, comm.rank + 1)
            centers = torch.empty((n_clusters, d), dtype=torch.float64, device=device)
        else:
            centers = out
        centers = comm.broadcast(centers, comm.world - 1)
    return centers


def build_sharded(x_local: torch.Tensor, params, group=None, timings: dict | None = None) -> ShardedIndex:
    """List-sharded build (index.py:190-281 across ranks).

    ``x_local`` holds this rank's block of rows; ranks hold ascending, contiguous blocks of
    the dataset (rank r's rows follow rank r-1's in the global order).  Training (sharded
    k-means, see train_kmeans_sharded) yields the reference's centroids on every rank; each
    rank assigns its own rows; the rows are exchanged (all-to-all) to the rank owning their
    cluster (contiguous cluster-id ranges balanced by vector count); each rank then encodes
    only its lists.  Shard r equals lists [lo_r, hi_r) of the single-GPU build, bit for bit.
    """
    import time

    from paper_2602_23999_b200.clustering import assign_device, counting_sort, row_sqnorms
    from paper_2602_23999_b200.codec import encode_rows
    from paper_2602_23999_b200.index import IvfRabitqIndex
    from paper_2602_23999_b200.linalg import gen_rotation

    comm = _Comm(group)
    device = x_local.device
    k = params.n_clusters
    n_loc, d = x_local.shape
    t0 = [time.perf_counter()]

    def tick(name: str) -> None:
        if timings is not None:
            torch.cuda.synchronize()
            now = time.perf_counter()
            timings[name] = round(now - t0[0], 3)
            t0[0] = now

    sizes = [int(v.item()) for v in comm.all_gather(torch.tensor([n_loc], dtype=torch.int64, device=device))]
    n = sum(sizes)
    row0 = sum(sizes[: comm.rank])
    if k > n:
        raise ValueError(f"n_clusters={k} exceeds dataset size {n}")
    seeds = np.random.SeedSequence(params.seed).spawn(2)
    if params.train_fraction < 1.0:
        n_train = max(1, math.ceil(params.train_fraction * n))
        n_train = max(n_train, min(n, k))
        rows = np.sort(np.random.default_rng(seeds[0]).choice(n, size=n_train, replace=False))
    else:
        rows = np.arange(n)
    mine = rows[(rows >= row0) & (rows < row0 + n_loc)] - row0
    x_train = x_local.index_select(0, dev.to_device(mine.astype(np.int64), device)) if mine.size else \
        torch.empty((0, d), dtype=torch.float32, device=device)
    km_seed = int(seeds[1].generate_state(1)[0])
    centers = train_kmeans_sharded(x_train, k, params.kmeans_iters, km_seed, comm)
    del x_train
    tick("kmeans")
    # assignment of the local rows, cluster ranges from the global counts
    c_sq = row_sqnorms(centers)
    labels = assign_device(x_local, centers, c_sq) if n_loc else torch.empty(0, dtype=torch.int32, device=device)
    counts_g = comm.all_reduce_sum(torch.bincount(labels.long(), minlength=k))
    ranges = cluster_ranges(counts_g.cpu().numpy(), comm.world)
    lo, hi = ranges[comm.rank]
    tick("assign")
    # rows to their list owners (ascending global row order kept: sources in rank order)
    bounds = torch.tensor([r[1] for r in ranges[:-1]], dtype=torch.int64, device=device)
    owner = torch.bucketize(labels.long(), bounds, right=True)
    gid = torch.arange(row0, row0 + n_loc, dtype=torch.int64, device=device)
    sel = [torch.nonzero(owner == r).flatten() for r in range(comm.world)]
    xs = torch.cat(comm.exchange_rows([x_local.index_select(0, i) for i in sel]))
    ls = torch.cat(comm.exchange_rows([labels.index_select(0, i) for i in sel]))
    gs = torch.cat(comm.exchange_rows([gid.index_select(0, i) for i in sel]))
    tick("exchange")
    # local CSR (stable: ascending global row within each list), then this rank's lists only
    local_labels = (ls.long() - lo).to(torch.int32)
    counts, offsets, order = counting_sort(local_labels, hi - lo)
    pids = gs.index_select(0, order)
    rot32 = dev.to_device(gen_rotation(d, params.seed).matrix.astype(np.float32), device)
    cent32 = centers.to(torch.float32)
    cent_rot = torch.empty((k, d), dtype=torch.float32, device=device)
    _lib.call("ivrq_rotate_rows_f32", dev.ptr(cent32), k, d, dev.ptr(rot32), dev.ptr(cent_rot), dev.stream_ptr())
    m = xs.shape[0]
    o_rot = torch.empty((m, d), dtype=torch.float32, device=device)
    dist = torch.empty(m, dtype=torch.float64, device=device)
    cent32_local = cent32[lo:hi].contiguous()
    if m:
        _lib.call(
            "ivrq_normalize_rotate", dev.ptr(xs), dev.ptr(order), dev.ptr(local_labels), dev.ptr(cent32_local),
            dev.ptr(rot32), m, d, dev.ptr(o_rot), dev.ptr(dist), dev.stream_ptr(),
        )
    cent_rot_local = cent_rot[lo:hi].contiguous()
    enc = encode_rows(o_rot, dist, cent_rot_local, offsets, params.quant)
    tick("encode")
    local = {
        "offsets": offsets,
        "packed_msb": enc["packed_msb"],
        "short_add": enc["short_add"],
        "short_scale": enc["short_scale"],
        "short_err": enc["short_err"],
        "long_factors": enc["long_factors"],
        "rcodes": enc["rcodes"],
        "pids": pids,
        "centroids": cent_rot_local,
        "centroid_sqnorms": row_sqnorms(cent_rot_local),
        "rotation": rot32,
    }
    shard = IvfRabitqIndex(
        dims=d, bits=params.quant.bits, n_clusters=hi - lo, size=m, eps_bound=params.quant.eps_bound,
        seed=params.seed, device_arrays=local,
    )
    return ShardedIndex(local=shard, list_lo=lo, list_hi=hi, n_clusters=k, centroids=cent_rot,
                        centroid_sqnorms=row_sqnorms(cent_rot), ranges=ranges)


def _merge_gpu(stacked: Pools, parts: int, k: int) -> Pools:
    ids, dists, counts = stacked
    nq = ids.shape[1]
    out_i = torch.empty((nq, k), dtype=torch.int64, device=ids.device)
    out_d = torch.empty((nq, k), dtype=torch.float64, device=ids.device)
    out_c = torch.empty(nq, dtype=torch.int32, device=ids.device)
    _lib.call(
        "ivrq_merge_topk", dev.ptr(ids), dev.ptr(dists), dev.ptr(counts), nq, parts, k,
        dev.ptr(out_i), dev.ptr(out_d), dev.ptr(out_c), dev.stream_ptr(),
    )
    return out_i, out_d, out_c


def search_sharded(q: torch.Tensor, sidx: ShardedIndex, params, group=None, mode: str = "auto",
                   n_micro: int | None = None) -> Pools:
    """Search a list-sharded index; every rank returns the final (ids, dists, counts).

    ``n_micro`` (chain mode) defaults to the number of ranks: enough micro-batches to keep every
    rank busy once the chain is full, and no more (each micro-batch streams the rank's lists again).
    """
    from paper_2602_23999_b200.search import _probe_device, prepare_queries_device, rotate_queries_device

    shard = sidx.local
    if mode == "auto":
        mode = "merge" if (shard.bits == 1 or not params.prune) else "chain"
    q_rot = rotate_queries_device(q, shard)
    probe_ids, probe_d2 = _probe_device(q_rot, sidx.centroids, sidx.centroid_sqnorms, params.n_probe, True)
    scalars, planes, luts, qslices = prepare_queries_device(q_rot, shard, params)
    nq, k = q.shape[0], params.k
    cp = params.to_c()

    def scan(sl: slice, init: Pools | None) -> Pools:
        n = sl.stop - sl.start
        ids = torch.empty((n, k), dtype=torch.int64, device=q.device)
        dists = torch.empty((n, k), dtype=torch.float64, device=q.device)
        counts = torch.empty(n, dtype=torch.int32, device=q.device)
        g = (shard.dims + 31) // 32
        _lib.call(
            "ivrq_search_scan_shard",
            shard.view(), sidx.list_lo, sidx.list_hi, None,
            dev.ptr(probe_ids[sl]), dev.ptr(probe_d2[sl]), dev.ptr(scalars[sl]),
            dev.ptr(planes[sl]) if planes is not None else None,
            dev.ptr(luts[sl]) if luts is not None else None,
            dev.ptr(qslices[sl]) if qslices is not None else None,
            n, cp,
            dev.ptr(init[0]) if init else None, dev.ptr(init[1]) if init else None,
            dev.ptr(init[2]) if init else None,
            dev.ptr(ids), dev.ptr(dists), dev.ptr(counts), None, dev.stream_ptr(),
        )
        del g
        return ids, dists, counts

    if mode == "merge":
        return merge_protocol(scan(slice(0, nq), None), k, group, _merge_gpu)
    if mode == "chain":
        if n_micro is None:
            n_micro = tdist.get_world_size(group) if tdist.is_initialized() else 1
        return chain_protocol(scan, nq, k, group, n_micro=n_micro, device=q.device)
    raise ValueError(f"unknown mode {mode!r}")
