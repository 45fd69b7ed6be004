"""Profiling driver: build one synthetic config and run the search a few times.

    ncu --profile-from-start off --set full -k regex:scan_kernel -c 1 -o gpurun_out/prof \
        python tools/prof_search.py --config c3 --nprobe 8
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_23999_b200 as iv  # noqa: E402
from paper_2602_23999_b200.index import build_index_device  # noqa: E402
from paper_2602_23999_b200.search import search_device  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--nprobe", type=int, default=8)
    ap.add_argument("--mode", default="bitwise")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nq", type=int, default=bench.NQ)
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    x, q = bench.make_dataset_gpu(cfg["n"], args.nq, cfg["d"], dev)
    params = iv.BuildParams(
        n_clusters=cfg["nlist"], quant=iv.QuantizationParams(bits=cfg["bits"]), kmeans_iters=25,
        train_fraction=bench.train_fraction(cfg["n"], cfg["nlist"]), seed=0,
    )
    t = time.perf_counter()
    ix = build_index_device(x, params)
    torch.cuda.synchronize()
    print(f"build {time.perf_counter() - t:.2f}s", file=sys.stderr)
    sp = iv.SearchParams(k=bench.K, n_probe=args.nprobe, ip_mode=args.mode)
    search_device(q, ix, sp)  # warm-up (allocator pools, tensor maps) outside the profiled range
    torch.cuda.synchronize()
    import ctypes
    import os

    from paper_2602_23999_b200 import _lib

    timing = os.environ.get("IVRQ_KERNEL_TIMING") == "1"
    if timing:
        _lib.call("ivrq_kernel_timing", 1)
    torch.cuda.profiler.start()  # ncu --profile-from-start off: only the searches below are captured
    for _ in range(args.reps):
        ev: dict = {}
        search_device(q, ix, sp, events=ev)
        ev["scanned"].synchronize()
        print(
            "step ms %.3f (rotate %.3f probe %.3f prep %.3f scan %.3f)"
            % (
                ev["start"].elapsed_time(ev["scanned"]),
                ev["start"].elapsed_time(ev["rotated"]),
                ev["rotated"].elapsed_time(ev["probed"]),
                ev["probed"].elapsed_time(ev["prepared"]),
                ev["prepared"].elapsed_time(ev["scanned"]),
            ),
            file=sys.stderr,
        )
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    if timing:
        _lib.call("ivrq_kernel_timing", 0)
        for kn in ("tc_refine_kernel", "tc_ip_kernel", "ip_list_kernel", "scan_rd_kernel", "scan_warp_kernel"):
            tot, n = ctypes.c_double(0.0), ctypes.c_int64(0)
            _lib.call("ivrq_kernel_time", kn.encode(), ctypes.byref(tot), ctypes.byref(n))
            if n.value:
                print(f"{kn} {tot.value / n.value:.4f} ms x{n.value}", file=sys.stderr)


if __name__ == "__main__":
    main()
