"""The list-sharded GPU build and search with two ranks.

Two processes share cuda:0 and talk over gloo (host-staged collectives): the
boxes this runs on have one GPU, and the code path is the one an 8-GPU NCCL run
takes, minus the transport.  Bar: every shard equals the corresponding lists of
the single-GPU build bit for bit (data-parallel k-means, row exchange, local
encode), the chain search equals the single-GPU search exactly (B >= 2 with
pruning), and the merge search does for prune=False.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(kind: str):
    rng = np.random.default_rng(7)
    if kind == "dup":  # duplicated points: empty clusters during training (reseeding across ranks)
        x = np.zeros((60, 8), dtype=np.float32)
        x[30:] = 1.0
        x[-1] = 5.0
        x[17] = 3.0
        q = rng.standard_normal((16, 8))
        return x, q, dict(nlist=4, bits=3, iters=3, tf=1.0, seed=0)
    centres = rng.standard_normal((12, 64)) * 2.0
    x = (centres[rng.integers(0, 12, 20000)] + rng.standard_normal((20000, 64))).astype(np.float32)
    q = centres[rng.integers(0, 12, 400)] + rng.standard_normal((400, 64))
    return x, q, dict(nlist=40, bits=4, iters=4, tf=0.5, seed=3)


def _params(p):
    import paper_2602_23999_b200 as iv

    return iv.BuildParams(n_clusters=p["nlist"], quant=iv.QuantizationParams(bits=p["bits"]), kmeans_iters=p["iters"],
                          train_fraction=p["tf"], seed=p["seed"])


def _worker(rank, world, port, kind, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist

    import paper_2602_23999_b200 as iv
    from paper_2602_23999_b200 import _device as dev
    from paper_2602_23999_b200.distributed import build_sharded, search_sharded

    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, q, p = _data(kind)
        blocks = np.array_split(np.arange(x.shape[0]), world)
        xl = dev.to_device(x[blocks[rank]])
        sh = build_sharded(xl, _params(p))
        loc = sh.local
        arrays = {name: dev.to_host(t) for name, t in loc.device.items() if name != "rotation"}
        res = {}
        qd = dev.to_device(q)
        for mode, prune in (("chain", True), ("merge", False)):
            sp = iv.SearchParams(k=10, n_probe=min(6, p["nlist"]), ip_mode="bitwise", prune=prune)
            ids, dists, cnt = search_sharded(qd, sh, sp, mode=mode, n_micro=3)
            res[mode] = (dev.to_host(ids), dev.to_host(dists), dev.to_host(cnt))
        out_q.put((rank, sh.list_lo, sh.list_hi, arrays, dev.to_host(sh.centroids), res))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("kind", ["mix", "dup"])
def test_sharded_build_and_search_match_single_gpu(kind):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    outs = sorted([q.get(timeout=600) for _ in range(world)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0

    import paper_2602_23999_b200 as iv
    from paper_2602_23999_b200 import _device as dev
    from paper_2602_23999_b200.index import build_index_device
    from paper_2602_23999_b200.search import search_device

    x, queries, p = _data(kind)
    full = build_index_device(dev.to_device(x), _params(p))
    t = {name: dev.to_host(v) for name, v in full.device.items()}
    off = t["offsets"].astype(np.int64)
    g = full.words_per_vector
    rb = full.device["rcodes"].numel() // max(full.size, 1)
    assert outs[0][1] == 0 and outs[-1][2] == p["nlist"] and outs[0][2] == outs[1][1]
    for rank, lo, hi, arr, cent_all, _ in outs:
        r0, r1 = int(off[lo]), int(off[hi])
        np.testing.assert_array_equal(cent_all, t["centroids"], err_msg="rotated centroids")
        np.testing.assert_array_equal(arr["offsets"], off[lo : hi + 1] - off[lo])
        np.testing.assert_array_equal(arr["pids"], t["pids"][r0:r1])
        np.testing.assert_array_equal(arr["packed_msb"], t["packed_msb"][g * r0 : g * r1])
        np.testing.assert_array_equal(arr["rcodes"], t["rcodes"][rb * r0 : rb * r1])
        for name in ("short_add", "short_scale", "short_err", "long_factors"):
            np.testing.assert_array_equal(arr[name], t[name][r0:r1], err_msg=name)
    qd = dev.to_device(queries)
    for mode, prune in (("chain", True), ("merge", False)):
        sp = iv.SearchParams(k=10, n_probe=min(6, p["nlist"]), ip_mode="bitwise", prune=prune)
        r = search_device(qd, full, sp)
        want = (dev.to_host(r.ids), dev.to_host(r.dists), dev.to_host(r.counts))
        for _, _, _, _, _, res in outs:  # every rank holds the final result
            got = res[mode]
            np.testing.assert_array_equal(got[2], want[2], err_msg=mode)
            np.testing.assert_array_equal(got[0], want[0], err_msg=mode)
            np.testing.assert_array_equal(got[1], want[1], err_msg=mode)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (NCCL)")
def test_nccl_two_gpus_chain_equals_single_gpu(tmp_path):
    """Same check over NCCL when the box has >= 2 GPUs (bench.py --gpus N takes this path)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "nccl_chain.py"
    script.write_text(
        "import os, sys, torch, torch.distributed as tdist, numpy as np\n"
        f"sys.path[:0] = [{root!r}, {os.path.join(root, 'tests')!r}]\n"
        "import paper_2602_23999_b200 as iv\n"
        "from paper_2602_23999_b200 import _device as dev\n"
        "from paper_2602_23999_b200.distributed import build_sharded, search_sharded\n"
        "from test_distributed_gpu import _data, _params\n"
        "r = int(os.environ['RANK']); torch.cuda.set_device(r)\n"
        "tdist.init_process_group('nccl', device_id=torch.device('cuda', r))\n"
        "x, q, p = _data('mix'); blocks = np.array_split(np.arange(x.shape[0]), 2)\n"
        "sh = build_sharded(dev.to_device(x[blocks[r]]), _params(p))\n"
        "sp = iv.SearchParams(k=10, n_probe=6, ip_mode='bitwise')\n"
        "ids, d, c = search_sharded(dev.to_device(q), sh, sp)\n"
        f"np.save(os.path.join({str(tmp_path)!r}, f'ids_{{r}}.npy'), dev.to_host(ids))\n"
        "tdist.destroy_process_group()\n"
    )
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), str(script)]
    subprocess.run(cmd, check=True, timeout=600, cwd=root)

    import paper_2602_23999_b200 as iv
    from paper_2602_23999_b200 import _device as dev
    from paper_2602_23999_b200.index import build_index_device
    from paper_2602_23999_b200.search import search_device

    x, queries, p = _data("mix")
    full = build_index_device(dev.to_device(x), _params(p))
    r = search_device(dev.to_device(queries), full, iv.SearchParams(k=10, n_probe=6, ip_mode="bitwise"))
    for rank in range(2):
        np.testing.assert_array_equal(np.load(tmp_path / f"ids_{rank}.npy"), dev.to_host(r.ids))
