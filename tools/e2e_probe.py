"""Break the public search_batch() call into its host/device parts (C3 by default).

    python tools/e2e_probe.py --config c3 --nprobe 8
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_23999_b200 as iv  # noqa: E402
from paper_2602_23999_b200 import _device as dev  # noqa: E402
from paper_2602_23999_b200 import search as S  # noqa: E402
from paper_2602_23999_b200.index import build_index_device  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--nprobe", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    d0 = torch.device("cuda", 0)
    x, q = bench.make_dataset_gpu(cfg["n"], bench.NQ, cfg["d"], d0)
    params = iv.BuildParams(
        n_clusters=cfg["nlist"], quant=iv.QuantizationParams(bits=cfg["bits"]), kmeans_iters=25,
        train_fraction=bench.train_fraction(cfg["n"], cfg["nlist"]), seed=0,
    )
    ix = build_index_device(x, params)
    q_host = q.cpu().numpy()
    sp = iv.SearchParams(k=bench.K, n_probe=args.nprobe, ip_mode="bitwise")
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        qd = dev.to_device(q_host)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        res = S.search_device(qd, ix, sp)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ids, dists, counts = dev.to_host(res.ids), dev.to_host(res.dists), dev.to_host(res.counts)
        t3 = time.perf_counter()
        out = S.results_to_lists(res)
        t4 = time.perf_counter()
        out2 = iv.search_batch(q_host, ix, sp)
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        print(
            f"h2d {1e3*(t1-t0):.2f} ms  device {1e3*(t2-t1):.2f}  d2h {1e3*(t3-t2):.2f}  "
            f"lists(+d2h) {1e3*(t4-t3):.2f}  search_batch {1e3*(t5-t4):.2f}",
            file=sys.stderr,
        )
    assert len(out) == len(out2)
    import os

    for nqs in (2000, 3000, 5000, 7000, 10000):
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            S.search_device(q[:nqs], ix, sp)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        print(f"device search of {nqs} queries: {1e3*np.median(ts):.2f} ms", file=sys.stderr)
    # host enqueue time of one search (no sync) vs its device time
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S.search_device(q, ix, sp)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"enqueue {1e3*(t1-t0):.2f} ms, until done {1e3*(t2-t0):.2f} ms", file=sys.stderr)
    # per C-ABI call host time within one search (enqueue only)
    from paper_2602_23999_b200 import _lib
    orig = _lib.call
    acc = {}

    def timed(name, *a):
        t0 = time.perf_counter()
        orig(name, *a)
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0

    _lib.call = timed
    S._lib.call = timed
    for _ in range(3):
        torch.cuda.synchronize()
        acc.clear()
        t0 = time.perf_counter()
        S.search_device(q, ix, sp)
        tot = time.perf_counter() - t0
        torch.cuda.synchronize()
    _lib.call = orig
    S._lib.call = orig
    print("enqueue split (ms): " + ", ".join(f"{k} {1e3*v:.3f}" for k, v in acc.items()) + f", python rest {1e3*(tot-sum(acc.values())):.3f}", file=sys.stderr)
    # host-side pieces of the pipeline
    pin = torch.empty(q_host.nbytes, dtype=torch.uint8, pin_memory=True).numpy().view(np.float32).reshape(q_host.shape)
    t0 = time.perf_counter(); np.copyto(pin, q_host); t1 = time.perf_counter()
    print(f"host memcpy into pinned (1 thread): {1e3*(t1-t0):.2f} ms", file=sys.stderr)
    ids_h, d_h, c_h = dev.to_host(res.ids), dev.to_host(res.dists), dev.to_host(res.counts)
    t0 = time.perf_counter(); out4 = S._rows_to_lists(ids_h.copy(), d_h.copy(), c_h.copy()); t1 = time.perf_counter()
    print(f"result lists: {1e3*(t1-t0):.2f} ms", file=sys.stderr)
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    for _ in range(3):
        iv.search_batch(q_host, ix, sp)
    pr.disable()
    pstats.Stats(pr, stream=sys.stderr).sort_stats("tottime").print_stats(12)
    for thr in (4, 8, 16):
        S._STAGE_THREADS = thr
        S._POOL = None
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            iv.search_batch(q_host, ix, sp)
            ts.append(time.perf_counter() - t0)
        print(f"stage threads {thr}: search_batch {1e3*np.median(ts):.2f} ms", file=sys.stderr)
    S._STAGE_THREADS = 4
    S._POOL = None
    for split in ():
        os.environ["IVRQ_E2E_SPLIT"] = split
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out3 = iv.search_batch(q_host, ix, sp)
            ts.append(time.perf_counter() - t0)
        print(f"split {split}: search_batch {1e3*np.median(ts):.2f} ms", file=sys.stderr)
    os.environ.pop("IVRQ_E2E_SPLIT", None)
    for chunks in (1, 2, 3):
        os.environ["IVRQ_E2E_CHUNKS"] = str(chunks)
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out3 = iv.search_batch(q_host, ix, sp)
            ts.append(time.perf_counter() - t0)
        same = all(np.array_equal(a[0], b[0]) for a, b in zip(out3, out2))
        print(f"chunks {chunks}: search_batch {1e3*np.median(ts):.2f} ms  identical={same}", file=sys.stderr)




def host_register_probe():
    """cudaHostRegister of a 30 MB numpy buffer vs staging copies (run standalone)."""
    import ctypes

    q = np.random.rand(10000, 768).astype(np.float32)
    cud = ctypes.CDLL("libcudart.so") if False else None
    rt = torch.cuda.cudart()
    dst = torch.empty(q.shape, dtype=torch.float32, device="cuda")
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rt.cudaHostRegister(q.ctypes.data, q.nbytes, 0)
        t1 = time.perf_counter()
        dst.copy_(torch.from_numpy(q), non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rt.cudaHostUnregister(q.ctypes.data)
        t3 = time.perf_counter()
        print(f"register {1e3*(t1-t0):.2f} ms, dma {1e3*(t2-t1):.2f} ms, unregister {1e3*(t3-t2):.2f} ms", file=sys.stderr)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.copy_(torch.from_numpy(q))
        torch.cuda.synchronize()
        print(f"pageable copy {1e3*(time.perf_counter()-t0):.2f} ms", file=sys.stderr)


if __name__ == "__main__":
    if "--register" in sys.argv:
        host_register_probe()
    else:
        main()
