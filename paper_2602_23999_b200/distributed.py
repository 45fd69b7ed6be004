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


def merge_protocol(local: Pools, k: int, group, merge_fn: Callable[[Pools, int, int], Pools]) -> Pools:
    """All-gather every rank's per-query top-k and merge them (exact for order-independent searches)."""
    world = tdist.get_world_size(group)
    ids, dists, counts = local
    g_ids = [torch.empty_like(ids) for _ in range(world)]
    g_d = [torch.empty_like(dists) for _ in range(world)]
    g_c = [torch.empty_like(counts) for _ in range(world)]
    tdist.all_gather(g_ids, ids.contiguous(), group=group)
    tdist.all_gather(g_d, dists.contiguous(), group=group)
    tdist.all_gather(g_c, counts.contiguous(), group=group)
    stacked = (torch.stack(g_ids), torch.stack(g_d), torch.stack(g_c))  # [parts, nq, k]
    return merge_fn(stacked, world, k)


def chain_protocol(
    scan_fn: Callable[[slice, Pools | None], Pools],
    nq: int,
    k: int,
    group,
    n_micro: int = 4,
    device: torch.device | str = "cpu",
) -> Pools:
    """Ascending-id chain over ranks: rank r continues rank r-1's pools, exactly.

    ``scan_fn(query_slice, init)`` scans this rank's lists for the queries in
    the slice starting from ``init`` pools (None on rank 0) and returns pools.
    """
    rank = tdist.get_rank(group)
    world = tdist.get_world_size(group)
    out_ids = torch.empty((nq, k), dtype=torch.int64, device=device)
    out_d = torch.empty((nq, k), dtype=torch.float64, device=device)
    out_c = torch.empty(nq, dtype=torch.int32, device=device)
    n_micro = max(1, min(n_micro, nq))
    edges = np.linspace(0, nq, n_micro + 1).astype(np.int64)
    for m in range(n_micro):
        sl = slice(int(edges[m]), int(edges[m + 1]))
        nm = sl.stop - sl.start
        init = None
        if rank > 0:
            ri = torch.empty((nm, k), dtype=torch.int64, device=device)
            rd = torch.empty((nm, k), dtype=torch.float64, device=device)
            rc = torch.empty(nm, dtype=torch.int32, device=device)
            src = tdist.get_global_rank(group, rank - 1) if group is not None else rank - 1
            tdist.recv(ri, src=src, group=group)
            tdist.recv(rd, src=src, group=group)
            tdist.recv(rc, src=src, group=group)
            init = (ri, rd, rc)
        ids, dists, counts = scan_fn(sl, init)
        if rank < world - 1:
            dst = tdist.get_global_rank(group, rank + 1) if group is not None else rank + 1
            tdist.send(ids.contiguous(), dst=dst, group=group)
            tdist.send(dists.contiguous(), dst=dst, group=group)
            tdist.send(counts.contiguous(), dst=dst, group=group)
        else:
            out_ids[sl] = ids
            out_d[sl] = dists
            out_c[sl] = counts
    last = tdist.get_global_rank(group, world - 1) if group is not None else world - 1
    tdist.broadcast(out_ids, src=last, group=group)
    tdist.broadcast(out_d, src=last, group=group)
    tdist.broadcast(out_c, src=last, group=group)
    return out_ids, out_d, out_c


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


def build_sharded(x: torch.Tensor, params, group=None) -> ShardedIndex:
    """Every rank trains the same centroids (deterministic for a seed), assigns the
    rows and keeps the lists of its cluster range (balanced by vector count)."""
    from paper_2602_23999_b200.index import build_index_device

    rank = tdist.get_rank(group) if tdist.is_initialized() else 0
    world = tdist.get_world_size(group) if tdist.is_initialized() else 1
    keep: dict = {}
    full = build_index_device(x, params, keep=keep)
    ranges = cluster_ranges(dev.to_host(keep["counts"]), world)
    lo, hi = ranges[rank]
    return slice_lists(full, lo, hi, ranges)


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
                   n_micro: int = 4) -> Pools:
    """Search a list-sharded index; every rank returns the final (ids, dists, counts)."""
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
        return chain_protocol(scan, nq, k, group, n_micro=n_micro, device=q.device)
    raise ValueError(f"unknown mode {mode!r}")
