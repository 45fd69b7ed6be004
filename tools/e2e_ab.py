"""A/B of the public search_batch() host pipeline settings on one index (C3 by default).

    python tools/e2e_ab.py --config c3 --nprobe 8 --threads 4,8,16 --pieces 1,4,8

Prints the mean / median wall time of search_batch(numpy queries) per setting,
with the L2 flushed before each call as bench.py does, and one traced call
(IVRQ_E2E_TRACE) per setting.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2602_23999_b200 as iv  # noqa: E402
from paper_2602_23999_b200 import search as S  # noqa: E402
from paper_2602_23999_b200.index import build_index_device  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--nprobe", type=int, default=8)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--threads", default="4,8")
    ap.add_argument("--pieces", default="4,8")
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
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=d0)
    print(f"host cores {os.cpu_count()}", file=sys.stderr)
    ref = None
    for th in [int(t) for t in args.threads.split(",")]:
        S._STAGE_THREADS = th
        S._POOL = None
        for pc in [int(p) for p in args.pieces.split(",")]:
            os.environ["IVRQ_STAGE_PIECES"] = str(pc)
            for _ in range(3):
                out = iv.search_batch(q_host, ix, sp)
            ts = []
            for _ in range(args.reps):
                flush.zero_()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                out = iv.search_batch(q_host, ix, sp)
                ts.append(time.perf_counter() - t0)
            if ref is None:
                ref = out
            same = all(np.array_equal(a[0], b[0]) for a, b in zip(out, ref))
            os.environ["IVRQ_E2E_TRACE"] = "1"
            flush.zero_()
            torch.cuda.synchronize()
            iv.search_batch(q_host, ix, sp)
            os.environ.pop("IVRQ_E2E_TRACE")
            if os.environ.get("E2E_CPROFILE") and pc == 4:
                import cProfile
                import pstats

                pr = cProfile.Profile()
                pr.enable()
                for _ in range(5):
                    iv.search_batch(q_host, ix, sp)
                pr.disable()
                pstats.Stats(pr, stream=sys.stderr).sort_stats("tottime").print_stats(18)
            print(f"threads {th:2d} pieces {pc:2d}: mean {1e3*np.mean(ts):.2f} ms  median {1e3*np.median(ts):.2f} ms "
                  f"-> {bench.NQ/np.mean(ts)/1e6:.3f}M QPS  same={same}", file=sys.stderr)


if __name__ == "__main__":
    main()
