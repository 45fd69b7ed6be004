"""Multi-process (gloo, world_size 2) tests of the list-sharded search protocols.

The per-shard scan is the oracle restricted to the rank's cluster range (the
GPU kernel takes the same (list range, initial pools) inputs); what is tested
here is the host-side logic: the balanced cluster ranges, the all-gather
merge, and the ascending-id chain with micro-batches.  The chain must equal
the single-process reference bit for bit (B >= 2 with pruning); the merge
must equal it for 1-bit indexes and for prune=False.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from conftest import SEARCHES, golden_index_arrays, load_case, padded
from oracle import ivrq_oracle as orc
from paper_2602_23999_b200.distributed import chain_protocol, cluster_ranges, merge_protocol


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _to_pools(results, k):
    ids, dists, cnt = padded(results, k)
    return torch.from_numpy(ids), torch.from_numpy(dists), torch.from_numpy(cnt)


def _merge_host(stacked, parts, k):
    ids, dists, counts = (t.numpy() for t in stacked)
    nq = ids.shape[1]
    out = []
    for q in range(nq):
        lists = [(ids[p, q, : counts[p, q]], dists[p, q, : counts[p, q]]) for p in range(parts)]
        cat_i = np.concatenate([a for a, _ in lists])
        cat_d = np.concatenate([b for _, b in lists])
        o = np.lexsort((cat_i, cat_d))[:k]
        out.append((cat_i[o], cat_d[o]))
    return _to_pools(out, k)


def _worker(rank, world, port, case, si, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_case(case)
        sp = dict(SEARCHES[si])
        k = sp["k"]
        ix = golden_index_arrays(g)
        counts = np.diff(ix["offsets"].astype(np.int64))
        lo, hi = cluster_ranges(counts, world)[rank]
        nq = g["queries"].shape[0]
        codes = orc.decode_codes(ix) if ix["bits"] > 1 else None

        def scan(sl, init):
            init_l = None
            if init is not None:
                ii, dd, cc = (t.numpy() for t in init)
                init_l = [(ii[j, : cc[j]], dd[j, : cc[j]]) for j in range(ii.shape[0])]
            res = orc.search(g["queries"][sl], ix, q_rot=g["q_rot"][sl], codes=codes, list_range=(lo, hi),
                             init=init_l, **sp)
            return _to_pools(res, k)

        if mode == "chain":
            ids, dists, cnt = chain_protocol(scan, nq, k, None, n_micro=3)
        else:
            ids, dists, cnt = merge_protocol(scan(slice(0, nq), None), k, None, _merge_host)
        q.put((rank, ids.numpy(), dists.numpy(), cnt.numpy()))
    finally:
        tdist.destroy_process_group()


def _run(case, si, mode, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, si, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_cluster_ranges_balanced_and_contiguous():
    counts = np.array([5, 1, 1, 30, 2, 2, 2, 9, 0, 4])
    for world in (1, 2, 3, 4):
        rs = cluster_ranges(counts, world)
        assert rs[0][0] == 0 and rs[-1][1] == counts.size
        assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(rs, rs[1:]))
    with pytest.raises(ValueError):
        cluster_ranges(counts, 11)


@pytest.mark.parametrize("case,si", [("b8_d128", 0), ("b4_d48", 1), ("b3_d96", 2)])
def test_chain_is_exact_for_pruned_multibit(case, si):
    g = load_case(case)
    outs = _run(case, si, "chain")
    for _, ids, dists, cnt in outs:  # every rank holds the final result
        np.testing.assert_array_equal(cnt, g[f"s{si}_counts"])
        np.testing.assert_array_equal(ids, g[f"s{si}_ids"])
        np.testing.assert_allclose(dists, g[f"s{si}_dists"], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("case,si", [("b1_d32", 0), ("b1_d32", 1), ("b8_d128", 4)])
def test_merge_is_exact_when_order_independent(case, si):
    # 1-bit indexes (safe pruning) and prune=False (search 4)
    g = load_case(case)
    outs = _run(case, si, "merge")
    for _, ids, dists, cnt in outs:
        np.testing.assert_array_equal(cnt, g[f"s{si}_counts"])
        np.testing.assert_array_equal(ids, g[f"s{si}_ids"])
        np.testing.assert_allclose(dists, g[f"s{si}_dists"], rtol=1e-12, atol=1e-12)
