"""Benchmark: IVF-RaBitQ search QPS at recall@10 ~ 0.95 (and build seconds) on B200.

    python bench.py [--gpus N --steps K --warmup W --config c3 --impl ours|reference]

One JSON line on rank 0 (driver contract).  A "step" is one search of a
10,000-query batch (rotation, coarse probe, query prep, fused scan + top-k)
against the resident index.  ``value`` times steps whose queries already sit
in HBM; ``e2e`` times the public ``search_batch`` call with host NumPy
queries (H2D of the queries and D2H of ids/dists inside the timed region).

Data: the reference's synthetic Gaussian-mixture recipe (reference
pkg/tests/conftest.py:26-51: 50 anisotropic blobs, log-uniform sigma,
exp(-i/tau) axis decay, Dirichlet(5) weights, seed 20260810) generated on the
GPU with a seeded torch generator (same recipe, different RNG stream), so the
1M x 768 dataset does not cost minutes of host BLAS.  Ground truth is exact
float64 k-NN on the GPU.

N > 1 GPUs: each rank holds a replica built from the same seed and searches
its own 10,000-query batch (weak scaling, no data-path collective); the time
is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (N, D, nlist, bits, nprobe (None -> smallest sweep value with recall >= target))
    "c1": dict(n=100_000, d=128, nlist=256, bits=1, nprobe=16, desc="synthetic 100Kx128, nlist 256, 1-bit, nprobe 16"),
    "c2": dict(n=1_000_000, d=128, nlist=1024, bits=4, nprobe=None, desc="synthetic 1Mx128, nlist 1024, 4-bit"),
    "c3": dict(n=1_000_000, d=768, nlist=1024, bits=8, nprobe=None, desc="synthetic 1Mx768, nlist 1024, 8-bit"),
    "c4": dict(n=10_000_000, d=96, nlist=16384, bits=4, nprobe=None, desc="synthetic 10Mx96, nlist 16384, 4-bit"),
    "c5": dict(n=5_000_000, d=1536, nlist=8192, bits=4, nprobe=None, desc="synthetic 5Mx1536, nlist 8192, 4-bit"),
}
SWEEP = (1, 2, 4, 8, 16, 32, 64, 128)
TARGET_RECALL = 0.95
NQ = 10_000
K = 10


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- data


def make_dataset_gpu(n, nq, d, device, n_blobs=50, seed=20260810, tau=12.0):
    """The reference conftest.make_dataset recipe, sampled on the GPU (float32 rows)."""
    import torch

    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, 1.0, (n_blobs, d))
    sigmas = np.exp(rng.uniform(np.log(0.5), np.log(1.5), n_blobs))
    decay = np.exp(-np.arange(d) / tau)
    weights = rng.dirichlet(np.full(n_blobs, 5.0))
    counts = rng.multinomial(n, weights)
    q_counts = rng.multinomial(nq, weights)
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    base = torch.empty((n, d), dtype=torch.float32, device=device)
    queries = torch.empty((nq, d), dtype=torch.float32, device=device)
    pb = pq = 0
    for j in range(n_blobs):
        g = torch.randn((d, d), generator=gen, device=device, dtype=torch.float64)
        basis, _ = torch.linalg.qr(g)
        cov_sqrt = basis * torch.from_numpy(sigmas[j] * decay).to(device)[None, :]
        c = torch.from_numpy(centers[j]).to(device)
        for dst, cnt, off in ((base, int(counts[j]), pb), (queries, int(q_counts[j]), pq)):
            if cnt:
                z = torch.randn((cnt, d), generator=gen, device=device, dtype=torch.float64)
                dst[off : off + cnt] = (c[None, :] + z @ cov_sqrt.T).to(torch.float32)
        pb += int(counts[j])
        pq += int(q_counts[j])
    perm = torch.randperm(n, generator=gen, device=device)
    base = base[perm].contiguous()
    qperm = torch.randperm(nq, generator=gen, device=device)
    queries = queries[qperm].contiguous()
    return base, queries


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = (
        "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
        "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    )

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            t0 = time.perf_counter()  # the sampler is live before the timed region starts
            while not self.lines and time.perf_counter() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.005)
            del self.lines[:-1]  # keep the sample taken just before the region (short regions may see no other)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {
            "sm_mhz": float(np.median(sm)),
            "sm_max_mhz": float(max(mx)),
            "reasons": sorted(reasons),
            "samples": len(sm),
        }


# ---------------------------------------------------------------- helpers


def train_fraction(n, nlist):
    return min(n, max(math.ceil(n / 10), 10 * nlist)) / n


def recall_at_k(ids: np.ndarray, gt: np.ndarray, k: int) -> float:
    hits = 0
    for a, b in zip(ids[:, :k], gt[:, :k]):
        hits += len(set(a[a >= 0].tolist()) & set(b.tolist()))
    return hits / (ids.shape[0] * k)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"hbm_gbs": 6650.0, "_fallback": True}


def count_launches(step_fn) -> tuple[int, list[str]]:
    """Kernels one search step launches, counted by CUPTI (torch.profiler), ours and library."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step_fn()
        torch.cuda.synchronize()
    names: dict[str, int] = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA and not ev.name.startswith(("Memcpy", "Memset")):
            names[ev.name] = names.get(ev.name, 0) + 1
    ours = {k: v for k, v in names.items() if "ivrq" in k or "scan::" in k or "gemm::" in k or "enc::" in k}
    short = sorted({k.split("(")[0].replace("void ", "")[:60] for k in ours})
    return int(sum(ours.values())), short


def ncu_traffic(cfg_name: str, nprobe: int, kernel: str | None = None):
    """DRAM bytes (read + write) per launch of `kernel` (and of the whole scan stage) from the
    committed ncu capture (profiles/<round>/traffic_<cfg>.json, written by tools/ncu_traffic.py), or None."""
    for p in sorted((ROOT / "profiles").glob(f"*/traffic_{cfg_name}.json"), reverse=True):
        try:
            t = json.loads(p.read_text())
        except ValueError:
            continue
        if t.get("n_probe") != nprobe:
            continue
        kb = None
        if kernel:
            kb = sum(v for k, v in (t.get("kernels") or {}).items() if k.split("<")[0].endswith(kernel)) or None
        return {"dram_bytes": kb, "kernel": kernel, "scan_stage_dram_bytes": t["dram_bytes"],
                "source": str(p.relative_to(ROOT)), "kernels": t.get("kernels")}
    return None


def kernel_roofline(kernel_ms: dict, peaks: dict, probed: int, survivors: int, d: int, bits: int) -> dict:
    """Roofline of the scan's dominant kernel (largest CUDA-event time in the timed region).

    Algorithmic work per launch:
      tc_refine_kernel  int8 tensor ops 2 * probed * kpad * 8 (8 digit slices of every probed pair)
      tc_ip/ip_list     int8 tensor ops 2 * probed * 32 ceil(D/32) * 4 (4-bit query planes)
      scan_rd_kernel    bytes probed * (2 + 12) + survivors * 8 (ip, factors; refined distance)
      scan_warp_kernel  bytes probed * (2 + 12) + survivors * (rcode row + 8) (ip, factors; codes, long factors)
    """
    if not kernel_ms:
        return {"bound": None, "kernel": None, "note": "no timed kernel"}
    name, (avg_ms, launches) = max(kernel_ms.items(), key=lambda kv: kv[1][0] * kv[1][1])
    kpad = -(-d // 64) * 64
    g = -(-d // 32)
    rb = -(-d * (8 if bits > 4 else 4) // 8)
    bf16 = float(peaks.get("bf16_tflops", 1590.0))
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    src = "MEASURED_PEAKS.json" if "_fallback" not in peaks else "fallback"
    if name in ("tc_refine_kernel", "tc_ip_kernel", "ip_list_kernel"):
        work = 2.0 * probed * (kpad * 8 if name == "tc_refine_kernel" else 32 * g * 4)
        achieved = work / (avg_ms / 1e3) / 1e12
        peak = 2.0 * bf16
        out = {"bound": "tensor", "unit": "TFLOP/s", "op": "int8 multiply-add (x2), TOP/s",
               "peak_source": f"2 x {src} bf16_tflops (dense int8 tcgen05 rate = 2 x bf16 on sm_100; "
                              "no int8 measurement in the file)",
               "work_formula": "2*probed*kpad*8" if name == "tc_refine_kernel" else "2*probed*32*ceil(D/32)*4"}
    else:
        work = probed * 14.0 + survivors * (8.0 if name == "scan_rd_kernel" else rb + 8.0)
        achieved = work / (avg_ms / 1e3) / 1e9
        peak = hbm
        out = {"bound": "hbm", "unit": "GB/s", "peak_source": f"{src} hbm_gbs",
               "work_formula": "probed*14 + survivors*" + ("8" if name == "scan_rd_kernel" else f"({rb}+8)")}
    out.update({"kernel": name, "achieved": round(achieved, 1), "peak": round(peak, 1),
                "frac": round(achieved / peak, 4), "work_per_launch": int(work),
                "kernel_ms_per_launch": round(avg_ms, 4), "launches_timed": launches,
                "timing": "CUDA events on the kernel's launching stream (ivrq_kernel_timing), timed region",
                "other_kernels_ms": {k: round(v[0], 4) for k, v in kernel_ms.items() if k != name}})
    return out


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------- our arm


def run_ours(args, cfg_name: str) -> dict:
    import torch
    import torch.distributed as tdist

    import ctypes

    import paper_2602_23999_b200 as iv
    from paper_2602_23999_b200 import _device as dev
    from paper_2602_23999_b200 import _lib
    from paper_2602_23999_b200.index import build_index_device
    from paper_2602_23999_b200.linalg import exact_knn_device
    from paper_2602_23999_b200.search import search_device

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=device)
    cfg = CONFIGS[cfg_name]
    n, d, nlist, bits = cfg["n"], cfg["d"], cfg["nlist"], cfg["bits"]
    t0 = time.perf_counter()
    x, queries = make_dataset_gpu(n, NQ, d, device, seed=20260810 + 0)
    torch.cuda.synchronize()
    log(f"[bench] data {n}x{d} generated in {time.perf_counter() - t0:.1f}s")
    params = iv.BuildParams(
        n_clusters=nlist, quant=iv.QuantizationParams(bits=bits), kmeans_iters=25,
        train_fraction=train_fraction(n, nlist), seed=0,
    )
    # ---- build (device-resident input)
    torch.cuda.synchronize()
    tb = time.perf_counter()
    index = build_index_device(x, params)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - tb
    log(f"[bench] build {build_s:.2f}s")
    build_stages: dict = {}
    if args.build_breakdown:
        del index
        torch.cuda.empty_cache()
        index = build_index_device(x, params, timings=build_stages)
        log(f"[bench] build stages {build_stages}")
    # ---- ground truth + nprobe choice
    tg = time.perf_counter()
    n_gt = NQ if args.gt_queries <= 0 else min(NQ, args.gt_queries)
    gt_ids, _ = exact_knn_device(x, queries[:n_gt].to(torch.float64), K)
    gt = gt_ids.cpu().numpy()
    log(f"[bench] ground truth ({n_gt} queries) {time.perf_counter() - tg:.1f}s")
    sweep = []
    nprobe = cfg["nprobe"]
    mode = args.mode
    if nprobe is None:
        for p in SWEEP:
            if p > nlist:
                break
            r = search_device(queries, index, iv.SearchParams(k=K, n_probe=p, ip_mode=mode))
            rec = recall_at_k(r.ids.cpu().numpy()[:n_gt], gt, K)
            sweep.append({"n_probe": p, "recall": round(rec, 4)})
            if rec >= TARGET_RECALL:
                nprobe = p
                break
            if len(sweep) >= 2 and rec - sweep[-2]["recall"] < 0.002:
                nprobe = sweep[-2]["n_probe"]  # recall saturated below the target (code width bound)
                break
        if nprobe is None:
            nprobe = sweep[-1]["n_probe"]
    sp = iv.SearchParams(k=K, n_probe=nprobe, ip_mode=mode)
    res = search_device(queries, index, sp, with_stats=True)
    recall = recall_at_k(res.ids.cpu().numpy()[:n_gt], gt, K)
    stats = res.stats.cpu().numpy()
    probed, survivors = int(stats[:, 0].sum()), int(stats[:, 1].sum())
    g = (d + 31) // 32
    bpv = (d * (bits - 1) + 7) // 8
    stage1_b = 4 * g + 12
    surv_b = (bpv + 16) if bits > 1 else 8
    alg_bytes = probed * stage1_b + survivors * surv_b
    log(f"[bench] nprobe={nprobe} recall={recall:.4f} probed/q={probed / NQ:.0f} surv/q={survivors / NQ:.0f}")

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # > 126 MB L2
    for _ in range(args.warmup):
        search_device(queries, index, sp)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    step_ms, scan_ms, stage_ms = [], [], {"rotate": 0.0, "probe": 0.0, "prepare": 0.0, "scan": 0.0}
    klib = _lib.load()
    prof_range = os.environ.get("BENCH_PROFILE_RANGE") == "1"  # ncu --profile-from-start off: timed steps only
    if prof_range:
        torch.cuda.profiler.start()
    _lib.call("ivrq_kernel_timing", 1)  # CUDA events around the scan's dominant kernels, on their streams
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            ev: dict = {}
            search_device(queries, index, sp, events=ev)
            ev["scanned"].synchronize()
            step_ms.append(ev["start"].elapsed_time(ev["scanned"]))
            scan_ms.append(ev["prepared"].elapsed_time(ev["scanned"]))
            stage_ms["rotate"] += ev["start"].elapsed_time(ev["rotated"])
            stage_ms["probe"] += ev["rotated"].elapsed_time(ev["probed"])
            stage_ms["prepare"] += ev["probed"].elapsed_time(ev["prepared"])
            stage_ms["scan"] += scan_ms[-1]
    torch.cuda.synchronize()
    if prof_range:
        torch.cuda.profiler.stop()
    _lib.call("ivrq_kernel_timing", 0)
    kernel_ms = {}
    for kn in ("tc_refine_kernel", "scan_rd_kernel", "scan_warp_kernel", "tc_ip_kernel", "ip_list_kernel"):
        tot, nl_ = ctypes.c_double(0.0), ctypes.c_int64(0)
        _lib.call("ivrq_kernel_time", kn.encode(), ctypes.byref(tot), ctypes.byref(nl_))
        if nl_.value:
            kernel_ms[kn] = (tot.value / nl_.value, int(nl_.value))
    del klib
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=device, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        total_ms = float(t.item())
        tdist.barrier()
    ms_per_step = total_ms / args.steps
    qps = world * NQ / (ms_per_step / 1e3)
    # ---- end to end through the public API (host queries, D2H results)
    q_host = queries.cpu().numpy()
    for _ in range(max(1, args.warmup // 2)):
        iv.search_batch(q_host, index, sp)
    torch.cuda.synchronize()
    e2e_times = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        te = time.perf_counter()
        out = iv.search_batch(q_host, index, sp)
        e2e_times.append(time.perf_counter() - te)
    e2e_s = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], device=device, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_s = float(t.item())
    assert len(out) == NQ
    launches_per_step, kernel_names = count_launches(lambda: search_device(queries, index, sp))
    scan_mean_ms = float(np.mean(scan_ms))
    peaks = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg_bytes / (scan_mean_ms / 1e3) / 1e9
    roofline = kernel_roofline(kernel_ms, peaks, probed=probed, survivors=survivors, d=d, bits=bits)
    roofline["traffic"] = ncu_traffic(cfg_name, nprobe, roofline.get("kernel"))
    roofline["scan_stage"] = {
        "note": "whole scan stage against the per-query-equivalent bytes of the reference's scan "
                "(list-major sharing of code reads lets this exceed the copy peak; context, not the roofline)",
        "ms": round(scan_mean_ms, 4),
        "per_query_equivalent_bytes": int(alg_bytes),
        "bytes_formula": f"probed*(4*ceil(D/32)+12) + survivors*({surv_b})",
        "effective_gbs": round(achieved, 1),
        "probed_per_query": round(probed / NQ, 1),
        "survivors_per_query": round(survivors / NQ, 1),
    }
    result = {
        "metric": "search QPS @ recall@10~0.95 (10K-query batch)",
        "value": round(qps, 1),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 estimator / int popcount / u8 codes",
        "data": "synthetic Gaussian mixture (reference conftest recipe, torch RNG), L2 flushed between steps",
        "config": {
            "workload": cfg_name + ": " + cfg["desc"],
            "n_probe": nprobe,
            "k": K,
            "n_queries": NQ,
            "ip_mode": mode,
            "query_bits": 4,
            "recall_at_10": round(recall, 4),
            "recall_queries": n_gt,
            "nprobe_sweep": sweep,
            "build_seconds": round(build_s, 3),
            "build_stage_seconds": {k2: round(v, 3) for k2, v in build_stages.items()},
            "build_params": {"kmeans_iters": 25, "train_fraction": round(params.train_fraction, 5), "seed": 0},
            "stage_ms_per_step": {k2: round(v / args.steps, 4) for k2, v in stage_ms.items()},
            "l2": "flushed (256 MB write) between timed steps",
        },
        "e2e": {
            "value": round(world * NQ / e2e_s, 1),
            "unit": "queries/s",
            "h2d_bytes_per_step": int(q_host.nbytes),
            "d2h_bytes_per_step": int(NQ * K * 16 + NQ * 4),
        },
        "gpu_launches": args.steps * launches_per_step,
        "gpu_launches_per_step": launches_per_step,
        "gpu_kernels": kernel_names,
        "roofline": roofline,
        "clocks": clocks.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(index, q_host, gt, sp, budget_s=args.cpu_budget)
    if world > 1:
        tdist.destroy_process_group()
    return result if rank == 0 else {}


def _host_index_arrays(index) -> dict:
    return dict(
        dims=index.dims, bits=index.bits, n_clusters=index.n_clusters, size=index.size,
        eps_bound=index.eps_bound, rotation=index.rotation, centroids=index.centroids.values,
        centroid_sqnorms=index.centroids.squared_norms, offsets=index.offsets, packed_msb=index.packed_msb,
        excodes=index.excodes, short_factors=index.short_factors, long_factors=index.long_factors,
        pids=index.pids,
    )


def cpu_baseline(index, q_host, gt, sp, budget_s=20.0) -> dict:
    """The oracle (NumPy restatement of the reference) on a bounded query sample, 1 host thread."""
    from oracle import ivrq_oracle as orc

    from threadpoolctl import threadpool_limits

    ix = _host_index_arrays(index)
    codes = orc.decode_codes(ix) if ix["bits"] > 1 else None
    with threadpool_limits(1):  # 1 host thread, BLAS included (the reference default, IVRQ_THREADS=1)
        return _cpu_baseline_timed(orc, ix, codes, q_host, gt, sp, budget_s)


def _cpu_baseline_timed(orc, ix, codes, q_host, gt, sp, budget_s) -> dict:
    t = time.perf_counter()
    orc.search(q_host[:4], ix, sp.k, sp.n_probe, ip_mode=sp.ip_mode, query_bits=sp.query_bits, codes=codes)
    per_q = max((time.perf_counter() - t) / 4, 1e-4)
    m = int(min(len(q_host), max(8, budget_s / per_q)))
    t = time.perf_counter()
    res = orc.search(q_host[:m], ix, sp.k, sp.n_probe, ip_mode=sp.ip_mode, query_bits=sp.query_bits, codes=codes)
    dt = time.perf_counter() - t
    ids = np.full((m, sp.k), -1, dtype=np.int64)
    for i, (a, _) in enumerate(res):
        ids[i, : len(a)] = a
    return {
        "value": round(m / dt, 2),
        "unit": "queries/s",
        "cores": 1,
        "kind": "port",
        "sample": f"first {m} of {len(q_host)} queries, same index/params (oracle/ivrq_oracle.py search)",
        "recall_at_10_sample": round(recall_at_k(ids, gt[:m], K), 4),
    }


# ---------------------------------------------------------------- reference arm


_REF_INDEX: dict = {}  # set before the worker pool forks: the index is inherited, never pickled per task


def _ref_worker(payload):
    from oracle import ivrq_oracle as orc

    from threadpoolctl import threadpool_limits

    qs, k, nprobe, mode, qbits = payload
    with threadpool_limits(1):  # one BLAS thread per process (the reference's fastest setting)
        t = time.perf_counter()
        orc.search(qs, _REF_INDEX["ix"], k, nprobe, ip_mode=mode, query_bits=qbits, codes=_REF_INDEX["codes"])
        return len(qs), time.perf_counter() - t


def run_reference(args, cfg_name: str) -> dict:
    """The reference algorithm on the host (oracle port), all cores, bounded query samples."""
    world, rank, local = dist_setup()
    if rank != 0:
        return {}
    import multiprocessing as mp

    import torch

    import paper_2602_23999_b200 as iv
    from oracle import ivrq_oracle as orc
    from paper_2602_23999_b200.index import build_index_device

    cfg = CONFIGS[cfg_name]
    n, d, nlist, bits = cfg["n"], cfg["d"], cfg["nlist"], cfg["bits"]
    device = torch.device("cuda", local)
    torch.cuda.set_device(local)
    x, queries = make_dataset_gpu(n, NQ, d, device)
    params = iv.BuildParams(
        n_clusters=nlist, quant=iv.QuantizationParams(bits=bits), kmeans_iters=25,
        train_fraction=train_fraction(n, nlist), seed=0,
    )
    # untimed setup: the index arrays (identical to the reference's build up to
    # float ulps, see tests/test_gpu_parity.py), handed to the CPU search
    index = build_index_device(x, params)
    ix = _host_index_arrays(index)
    q_host = queries.cpu().numpy()
    nprobe = cfg["nprobe"] or args.ref_nprobe
    codes = orc.decode_codes(ix) if bits > 1 else None
    cores = os.cpu_count() or 1
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    per_step = max(cores, int(args.ref_queries_per_step))
    ctx = mp.get_context("fork")
    step_qps = []
    _REF_INDEX["ix"], _REF_INDEX["codes"] = ix, codes
    with ctx.Pool(cores) as pool:
        for step in range(args.warmup + args.steps):
            lo = (step * per_step) % NQ
            qs = q_host[lo : lo + per_step]
            chunks = np.array_split(qs, cores)
            t = time.perf_counter()
            pool.map(_ref_worker, [(c, K, nprobe, args.mode, 4) for c in chunks if len(c)])
            dt = time.perf_counter() - t
            if step >= args.warmup:
                step_qps.append(len(qs) / dt)
    value = float(np.mean(step_qps))
    return {
        "impl": "reference",
        "metric": "search QPS @ recall@10~0.95 (10K-query batch)",
        "value": round(value, 2),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "higher_is_better": True,
        "config": {"workload": cfg_name + ": " + cfg["desc"], "n_probe": nprobe, "k": K, "ip_mode": args.mode},
        "cpu_baseline": {
            "value": round(value, 2),
            "unit": "queries/s",
            "cores": cores,
            "kind": "port",
            "sample": f"{per_step} queries per step across {cores} processes (oracle/ivrq_oracle.py search)",
        },
        "e2e": {"value": round(value, 2), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--mode", default="bitwise", choices=("bitwise", "lut"))
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-nprobe", type=int, default=8)
    ap.add_argument("--ref-queries-per-step", type=int, default=1024)
    ap.add_argument("--gt-queries", type=int, default=0, help="queries with exact ground truth (0 = all)")
    ap.add_argument("--build-breakdown", action="store_true", help="rebuild once with per-stage timings")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        out = run_reference(args, args.config)
    else:
        out = run_ours(args, args.config)
    if out:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
