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

Both arms print the same ``config`` (the workload: shape, nlist, bits, n_probe,
k, query batch); measured quantities (recall, nprobe sweep, build seconds,
stage times) are separate keys.  ``--impl reference`` never imports
paper_2602_23999_b200: it builds the index on the host (the reference's own
``build_index`` for the 100K-row config, the oracle port with a parallel
per-list encoder otherwise) and times the unmodified reference ``search_batch``
from baseline/_ref in one forked process per host core.
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
    # n_probe: the smallest sweep value with recall@10 >= 0.95 (C3, C5), or where recall saturates
    # below it (C2, C4: 4-bit codes), measured by this script's sweep (reported under "quality")
    "c1": dict(n=100_000, d=128, nlist=256, bits=1, nprobe=16, desc="synthetic 100Kx128, nlist 256, 1-bit"),
    "c2": dict(n=1_000_000, d=128, nlist=1024, bits=4, nprobe=16, desc="synthetic 1Mx128, nlist 1024, 4-bit"),
    "c3": dict(n=1_000_000, d=768, nlist=1024, bits=8, nprobe=8, desc="synthetic 1Mx768, nlist 1024, 8-bit"),
    "c4": dict(n=10_000_000, d=96, nlist=16384, bits=4, nprobe=64, desc="synthetic 10Mx96, nlist 16384, 4-bit"),
    "c5": dict(n=5_000_000, d=1536, nlist=8192, bits=4, nprobe=32, desc="synthetic 5Mx1536, nlist 8192, 4-bit"),
}
METRIC = "search QPS @ recall@10~0.95 (10K-query batch)"
DATA_NOTE = "synthetic Gaussian mixture (reference conftest recipe, torch RNG on cuda:0)"
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


def config_dict(cfg_name: str, mode: str) -> dict:
    """The workload, identical for both arms (--impl ours / reference)."""
    cfg = CONFIGS[cfg_name]
    return {
        "workload": cfg_name + ": " + cfg["desc"],
        "n": cfg["n"], "dims": cfg["d"], "nlist": cfg["nlist"], "bits": cfg["bits"],
        "n_probe": cfg["nprobe"], "k": K, "n_queries": NQ, "ip_mode": mode, "query_bits": 4,
        "build_params": {"kmeans_iters": 25, "train_fraction": round(train_fraction(cfg["n"], cfg["nlist"]), 5),
                         "seed": 0},
    }


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


def int8_peak(peaks: dict) -> tuple[float, str]:
    """Dense int8 tcgen05 peak: the committed tools/tc_probe.cu measurement, else 2 x bf16."""
    for p in sorted((ROOT / "profiles").glob("*/int8_peak.json"), reverse=True):
        try:
            t = json.loads(p.read_text())
            return float(t["tops"]), f"{p.relative_to(ROOT)} (tools/tc_probe.cu, measured on a B200)"
        except (ValueError, KeyError):
            continue
    src = "MEASURED_PEAKS.json" if "_fallback" not in peaks else "fallback"
    return 2.0 * float(peaks.get("bf16_tflops", 1590.0)), f"2 x {src} bf16_tflops (no int8 measurement committed)"


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


def kernel_roofline(kernel_ms: dict, peaks: dict, probed: int, survivors: int, d: int, bits: int,
                    mode: str = "bitwise", n_vectors: int = 0, n_pairs: int = 0) -> dict:
    """Roofline of the scan's dominant kernel (largest CUDA-event time in the timed region).

    Algorithmic work per launch:
      tc_refine_kernel  int8 tensor ops 2 * probed * kpad * R: R = 4 leading query digits, plus the fused
                        stage 1 (8-bit and <= 4-bit codes): 2 qhat rows (bitwise) or the 4 digit rows again
                        read as signed bytes (LUT); and bytes N * rcode_bytes (every code row once) +
                        probed * 8 (the (distance, stage-1) pair) + pairs * (B rows) * kpad; the roofline
                        with the larger time at peak is the one reported
      tc_ip/ip_list     int8 tensor ops 2 * probed * 32 ceil(D/32) * 4 (4-bit query planes)
      scan_rd_kernel    bytes probed * (2 + 12) + survivors * 4 (ip, factors; float32 refined distance)
                        (1-bit indexes: probed * 14)
      scan_warp_kernel  bytes probed * (2 + 12) + survivors * (rcode row + 8) (ip, factors; codes, long factors)
    """
    if not kernel_ms:
        return {"bound": None, "kernel": None, "note": "no timed kernel"}
    name, (avg_ms, launches) = max(kernel_ms.items(), key=lambda kv: kv[1][0] * kv[1][1])
    kpad = -(-d // 64) * 64
    g = -(-d // 32)
    rb = -(-d * (8 if bits > 4 else 4) // 8)
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    src = "MEASURED_PEAKS.json" if "_fallback" not in peaks else "fallback"
    if name == "tc_refine_kernel":
        # Two rooflines for the refine: its int8 MMA work and its bytes (every index code row streamed
        # at least once, the (distance, stage-1) float pair written per probed vector, the groups' B rows
        # read once per probed pair); the binding one (the larger time at peak) is reported.
        fused = bits == 8 or bits <= 4
        rows = 4 + ((4 if mode == "lut" else 2) if fused else 0)
        work = 2.0 * probed * kpad * rows
        peak_t, psrc = int8_peak(peaks)
        code_bytes = float(n_vectors) * rb
        io_bytes = code_bytes + probed * (8.0 if fused else 4.0) + n_pairs * (rows if mode == "lut" else rows - 1) * kpad
        t_tensor, t_hbm = work / (peak_t * 1e12), io_bytes / (hbm * 1e9)
        secs = avg_ms / 1e3
        other = {"bound": "tensor", "unit": "TFLOP/s", "achieved": round(work / secs / 1e12, 1),
                 "peak": round(peak_t, 1), "frac": round(work / secs / 1e12 / peak_t, 4),
                 "work_formula": f"2*probed*kpad*{rows}"}
        if t_hbm >= t_tensor:
            work, achieved, peak = io_bytes, io_bytes / secs / 1e9, hbm
            out = {"bound": "hbm", "unit": "GB/s", "peak_source": f"{src} hbm_gbs",
                   "work_formula": f"N*rcode_bytes + probed*{8 if fused else 4} + pairs*{rows if mode == 'lut' else rows - 1}*kpad",
                   "other_roofline": other}
        else:
            achieved, peak = work / secs / 1e12, peak_t
            out = {"bound": "tensor", "unit": "TFLOP/s", "op": "int8 multiply-add (x2), TOP/s", "peak_source": psrc,
                   "work_formula": f"2*probed*kpad*{rows}",
                   "other_roofline": {"bound": "hbm", "unit": "GB/s", "achieved": round(io_bytes / secs / 1e9, 1),
                                      "peak": round(hbm, 1), "frac": round(io_bytes / secs / 1e9 / hbm, 4)}}
    elif name in ("tc_ip_kernel", "ip_list_kernel"):
        work = 2.0 * probed * 32 * g * 4
        achieved = work / (avg_ms / 1e3) / 1e12
        peak, psrc = int8_peak(peaks)
        out = {"bound": "tensor", "unit": "TFLOP/s", "op": "int8 multiply-add (x2), TOP/s",
               "peak_source": psrc, "work_formula": "2*probed*32*ceil(D/32)*4"}
    else:
        per_surv = (4.0 if bits > 1 else 0.0) if name == "scan_rd_kernel" else rb + 8.0
        work = probed * 14.0 + survivors * per_surv
        achieved = work / (avg_ms / 1e3) / 1e9
        peak = hbm
        out = {"bound": "hbm", "unit": "GB/s", "peak_source": f"{src} hbm_gbs",
               "work_formula": f"probed*14 + survivors*{per_surv:g}"}
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
    import ctypes

    import torch
    import torch.distributed as tdist

    import paper_2602_23999_b200 as iv
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
    # ---- ground truth (exact float64 k-NN on the GPU) and the recall sweep around the config's n_probe
    tg = time.perf_counter()
    n_gt = NQ if args.gt_queries <= 0 else min(NQ, args.gt_queries)
    gt_ids, _ = exact_knn_device(x, queries[:n_gt].to(torch.float64), K)
    gt = gt_ids.cpu().numpy()
    log(f"[bench] ground truth ({n_gt} queries) {time.perf_counter() - tg:.1f}s")
    nprobe = cfg["nprobe"]
    mode = args.mode
    sweep = []
    for p in SWEEP:
        if p > nlist or p > 2 * nprobe:
            break
        r = search_device(queries[:n_gt], index, iv.SearchParams(k=K, n_probe=p, ip_mode=mode))
        sweep.append({"n_probe": p, "recall": round(recall_at_k(r.ids.cpu().numpy(), gt, K), 4)})
    sp = iv.SearchParams(k=K, n_probe=nprobe, ip_mode=mode)
    res = search_device(queries, index, sp, with_stats=True)
    res_ids = res.ids.cpu().numpy()
    res_dists = res.dists.cpu().numpy()
    recall = recall_at_k(res_ids[:n_gt], gt, K)
    stats = res.stats.cpu().numpy()
    probed, survivors = int(stats[:, 0].sum()), int(stats[:, 1].sum())
    log(f"[bench] nprobe={nprobe} recall={recall:.4f} probed/q={probed / NQ:.0f} surv/q={survivors / NQ:.0f}")

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)  # > 126 MB L2
    for _ in range(args.warmup):
        search_device(queries, index, sp)
    torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    step_ms, scan_ms, stage_ms = [], [], {"rotate": 0.0, "probe": 0.0, "prepare": 0.0, "scan": 0.0}
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
    assert all(np.array_equal(out[i][0], res_ids[i, : len(out[i][0])]) for i in range(0, NQ, 97))
    launches_per_step, kernel_names = count_launches(lambda: search_device(queries, index, sp))
    scan_mean_ms = float(np.mean(scan_ms))
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    roofline = kernel_roofline(kernel_ms, peaks, probed=probed, survivors=survivors, d=d, bits=bits, mode=args.mode,
                               n_vectors=n, n_pairs=NQ * nprobe)
    traffic = ncu_traffic(cfg_name, nprobe, roofline.get("kernel"))
    roofline["traffic"] = traffic
    g = (d + 31) // 32
    surv_b = ((d * (bits - 1) + 7) // 8 + 16) if bits > 1 else 8
    roofline["scan_stage"] = {
        "ms": round(scan_mean_ms, 4),
        "probed_per_query": round(probed / NQ, 1),
        "survivors_per_query": round(survivors / NQ, 1),
        "alg_bytes_formula": f"probed*(4*ceil(D/32)+12) + survivors*({surv_b})  (SURVEY 8(d), per query)",
        "alg_bytes": int(probed * (4 * g + 12) + survivors * surv_b),
    }
    if traffic and traffic.get("scan_stage_dram_bytes"):
        dram = float(traffic["scan_stage_dram_bytes"])
        roofline["scan_dram_frac"] = round(dram / (scan_mean_ms / 1e3) / 1e9 / hbm, 4)
        roofline["scan_stage"]["dram_bytes"] = int(dram)
        roofline["scan_stage"]["dram_gbs"] = round(dram / (scan_mean_ms / 1e3) / 1e9, 1)
    result = {
        "metric": METRIC,
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
        "data": DATA_NOTE + ", L2 flushed (256 MB write) between timed steps",
        "config": config_dict(cfg_name, mode),
        "quality": {"recall_at_10": round(recall, 4), "recall_queries": n_gt, "nprobe_sweep": sweep},
        "build": {"seconds": round(build_s, 3), "stage_seconds": {k2: round(v, 3) for k2, v in build_stages.items()},
                  "note": "build_index_device on the device-resident dataset (H2D excluded, cli.py:78-80)"},
        "stage_ms_per_step": {k2: round(v / args.steps, 4) for k2, v in stage_ms.items()},
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
        result["gt_parity"] = gt_parity(x, queries, gt_ids, n_check=args.gt_check)
        result["cpu_baseline"] = cpu_baseline(index, q_host, gt, sp, res_ids, res_dists, budget_s=args.cpu_budget)
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


def gt_parity(x, queries, gt_ids, n_check: int = 100) -> dict:
    """exact_knn_device against the oracle's float64 brute force on the first n_check queries."""
    from oracle import ivrq_oracle as orc

    if n_check <= 0:
        return {"queries": 0}
    t = time.perf_counter()
    ids_o, _ = orc.exact_knn(x.cpu().numpy(), queries[:n_check].cpu().numpy().astype(np.float64), K)
    got = gt_ids[:n_check].cpu().numpy()
    return {"queries": int(n_check), "id_mismatch_rows": int((ids_o != got).any(axis=1).sum()),
            "oracle_seconds": round(time.perf_counter() - t, 1)}


def cpu_baseline(index, q_host, gt, sp, gpu_ids, gpu_dists, budget_s=20.0) -> dict:
    """The oracle (NumPy restatement of the reference) on a bounded query sample, 1 host thread,
    with its results compared id for id against the GPU search of the same queries."""
    from oracle import ivrq_oracle as orc

    from threadpoolctl import threadpool_limits

    ix = _host_index_arrays(index)
    codes = orc.decode_codes(ix) if ix["bits"] > 1 else None
    with threadpool_limits(1):  # 1 host thread, BLAS included (the reference default, IVRQ_THREADS=1)
        out = _cpu_baseline_timed(orc, ix, codes, q_host, gt, sp, budget_s, gpu_ids, gpu_dists)
    return out


def _cpu_baseline_timed(orc, ix, codes, q_host, gt, sp, budget_s, gpu_ids, gpu_dists) -> dict:
    kw = dict(ip_mode=sp.ip_mode, query_bits=sp.query_bits, codes=codes)
    t = time.perf_counter()
    orc.search(q_host[:4], ix, sp.k, sp.n_probe, **kw)
    per_q = max((time.perf_counter() - t) / 4, 1e-4)
    m = int(min(len(q_host), max(8, budget_s / per_q)))
    t = time.perf_counter()
    res = orc.search(q_host[:m], ix, sp.k, sp.n_probe, **kw)
    dt = time.perf_counter() - t
    ids = np.full((m, sp.k), -1, dtype=np.int64)
    dists = np.full((m, sp.k), np.inf)
    for i, (a, b) in enumerate(res):
        ids[i, : len(a)] = a
        dists[i, : len(b)] = b
    bad = np.flatnonzero((ids != gpu_ids[:m]).any(axis=1))
    fin = np.isfinite(dists) & (ids == gpu_ids[:m])
    rel = np.abs(dists[fin] - gpu_dists[:m][fin]) / np.maximum(np.abs(dists[fin]), 1e-300)
    parity = {"queries": m, "id_mismatch": int(bad.size), "max_rel_dist": float(rel.max()) if rel.size else 0.0,
              "note": "oracle search on the host (its own float64 query rotation) vs the GPU search, same index"}
    return {
        "value": round(m / dt, 2),
        "unit": "queries/s",
        "cores": 1,
        "kind": "port",
        "sample": f"first {m} of {len(q_host)} queries, same index/params (oracle/ivrq_oracle.py search)",
        "recall_at_10_sample": round(recall_at_k(ids, gt[:m], K), 4) if m <= len(gt) else None,
        "parity": parity,
    }


# ---------------------------------------------------------------- reference arm


_REF: dict = {}  # set before the worker pool forks: the index is inherited, never pickled per task


def _ref_import():
    """The unmodified reference package from baseline/_ref (pip install --target), or None."""
    ref_dir = ROOT / "baseline" / "_ref"
    if (ref_dir / "ivfrabitq" / "__init__.py").exists():
        sys.path.insert(0, str(ref_dir))
        import ivfrabitq

        return ivfrabitq
    return None


def _ref_worker(payload):
    from threadpoolctl import threadpool_limits

    qs, k, nprobe, mode, qbits = payload
    with threadpool_limits(1):  # one BLAS thread per process (the reference's fastest setting)
        t = time.perf_counter()
        ref = _REF.get("pkg")
        if ref is not None:
            sp = ref.SearchParams(k=k, n_probe=nprobe, ip_mode=mode, query_bits=qbits)
            ref.search_batch(qs, _REF["index"], sp, workers=1)
        else:
            from oracle import ivrq_oracle as orc

            orc.search(qs, _REF["ix"], k, nprobe, ip_mode=mode, query_bits=qbits, codes=_REF["codes"])
        return len(qs), time.perf_counter() - t


def run_reference(args, cfg_name: str) -> dict:
    """The reference on the host: its build (or the oracle port's, parallel) and its own search_batch,
    one forked process per host core over bounded query samples.  Does not import the product package."""
    world, rank, local = dist_setup()
    if rank != 0:
        return {}
    import multiprocessing as mp

    import torch

    from oracle import ivrq_oracle as orc

    cfg = CONFIGS[cfg_name]
    n, d, nlist, bits, nprobe = cfg["n"], cfg["d"], cfg["nlist"], cfg["bits"], cfg["nprobe"]
    cores = os.cpu_count() or 1
    device = torch.device("cuda", local)
    torch.cuda.set_device(local)
    xt, qt = make_dataset_gpu(n, NQ, d, device)  # the same synthetic data as our arm (torch RNG only)
    x, q_host = xt.cpu().numpy(), qt.cpu().numpy()
    del xt, qt
    torch.cuda.empty_cache()
    ref = _ref_import()
    tf = train_fraction(n, nlist)
    tb = time.perf_counter()
    stages: dict = {}
    if ref is not None and n <= 200_000:
        # the reference's own build_index (small config: minutes would be needed at 1M rows)
        index = ref.build_index(x, ref.BuildParams(n_clusters=nlist, quant=ref.QuantizationParams(bits=bits),
                                                   kmeans_iters=25, train_fraction=tf, seed=0), workers=1)
        build_kind, build_cores = "reference build_index (baseline/_ref)", 1
        ix = None
    else:
        ix = orc.build(x, nlist, bits, 25, tf, 0, workers=cores, timings=stages)
        build_kind, build_cores = "port (oracle build: k-means++ passes on a thread pool, per-list encoder " \
                                  "in forked processes)", cores
        index = None
    build_s = time.perf_counter() - tb
    log(f"[bench:reference] build {build_s:.1f}s ({build_kind})")
    if ref is not None:
        if index is None:
            index = ref.IvfRabitqIndex(
                dims=d, bits=bits, n_clusters=nlist, size=n, eps_bound=float(ix["eps_bound"]), seed=0,
                rotation=ix["rotation"], centroids=ref.Centroids.from_values(ix["centroids"]),
                offsets=ix["offsets"], packed_msb=ix["packed_msb"], excodes=ix["excodes"],
                short_factors=ix["short_factors"], long_factors=ix["long_factors"], pids=ix["pids"],
            )
        if bits > 1:
            _ = index.code_values  # materialised once, inherited by the forked workers
        if args.mode == "lut":
            _ = index.msb_nibbles
        _REF["pkg"], _REF["index"] = ref, index
        search_kind = "reference search_batch (baseline/_ref, unmodified)"
    else:
        _REF["ix"], _REF["codes"] = ix, (orc.decode_codes(ix) if bits > 1 else None)
        search_kind = "port (oracle/ivrq_oracle.py search; baseline/_ref not installed)"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    per_step = max(cores, int(args.ref_queries_per_step))
    step_qps = []
    with mp.get_context("fork").Pool(cores) as pool:
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
    kind = "reference" if ref is not None else "port"
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * per_step / value, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64 estimator / int popcount / u8 codes",
        "data": DATA_NOTE + " (copied to the host)",
        "config": config_dict(cfg_name, args.mode),
        "build": {"seconds": round(build_s, 3), "kind": build_kind, "cores": build_cores,
                  "stage_seconds": stages},
        "cpu_baseline": {
            "value": round(value, 2),
            "unit": "queries/s",
            "cores": cores,
            "kind": kind,
            "sample": f"{per_step} queries per step across {cores} forked processes ({search_kind})",
        },
        "e2e": {"value": round(value, 2), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_sharded(args, cfg_name: str) -> dict:
    """`--sharded`: the north star's list-sharded design, strong scaling.  The dataset's rows are split
    in ascending blocks over the ranks, `build_sharded` trains shared centroids (data-parallel Lloyd)
    and leaves each rank a contiguous cluster-id range; every step searches ONE shared 10K-query batch
    with `search_sharded` (the exact ascending-id chain for B >= 2, the all-gather merge otherwise)."""
    import torch
    import torch.distributed as tdist

    import paper_2602_23999_b200 as iv
    from paper_2602_23999_b200.distributed import build_sharded, search_sharded
    from paper_2602_23999_b200.linalg import exact_knn_device

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    for key, val in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", "0"), ("WORLD_SIZE", "1")):
        os.environ.setdefault(key, val)  # a one-rank NCCL group when not launched by torchrun
    tdist.init_process_group("nccl", device_id=device)
    cfg = CONFIGS[cfg_name]
    n, d, nlist, bits = cfg["n"], cfg["d"], cfg["nlist"], cfg["bits"]
    x, queries = make_dataset_gpu(n, NQ, d, device, seed=20260810 + 0)
    lo, hi = n * rank // world, n * (rank + 1) // world
    x_local = x[lo:hi].contiguous()
    params = iv.BuildParams(n_clusters=nlist, quant=iv.QuantizationParams(bits=bits), kmeans_iters=25,
                            train_fraction=train_fraction(n, nlist), seed=0)
    tdist.barrier()
    torch.cuda.synchronize()
    tb = time.perf_counter()
    sidx = build_sharded(x_local, params)
    torch.cuda.synchronize()
    tdist.barrier()
    build_s = time.perf_counter() - tb
    sp = iv.SearchParams(k=K, n_probe=cfg["nprobe"], ip_mode=args.mode)
    n_gt = min(NQ, 1000)
    gt = exact_knn_device(x, queries[:n_gt].to(torch.float64), K)[0].cpu().numpy() if rank == 0 else None
    del x
    for _ in range(args.warmup):
        ids, dists, counts = search_sharded(queries, sidx, sp)
    torch.cuda.synchronize()
    tdist.barrier()
    stream = torch.cuda.current_stream(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ids, dists, counts = search_sharded(queries, sidx, sp)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    # end to end: host queries in, host ids out, every step
    q_host = queries.cpu().numpy()
    tdist.barrier()
    te = time.perf_counter()
    for _ in range(args.steps):
        qd = torch.from_numpy(q_host).to(device, non_blocking=False)
        ids_e, _, _ = search_sharded(qd, sidx, sp)
        ids_e = ids_e.cpu()
    e2e_s = (time.perf_counter() - te) / args.steps
    te_t = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if world > 1:
        tdist.all_reduce(te_t, op=tdist.ReduceOp.MAX)
    e2e_s = float(te_t.item())
    out = None
    if rank == 0:
        got = ids[:n_gt].cpu().numpy()
        out = {
            "metric": "search QPS @ recall@10~0.95 (10K-query batch)", "value": round(NQ / (ms / 1e3), 1),
            "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 estimator / int popcount / u8 codes", "data": DATA_NOTE,
            "config": dict(config_dict(cfg_name, args.mode), parallelism=f"list-sharded x{world}",
                           search_protocol="chain" if bits > 1 and sp.prune else "merge"),
            "quality": {"recall_at_10": recall_at_k(got, gt, K), "recall_queries": n_gt},
            "build": {"seconds": round(build_s, 3), "note": "build_sharded, device-resident rows"},
            "e2e": {"value": round(NQ / e2e_s, 1), "unit": "queries/s", "h2d_bytes_per_step": int(q_host.nbytes),
                    "d2h_bytes_per_step": int(NQ * K * 8)},
        }
    tdist.destroy_process_group()
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--mode", default="bitwise", choices=("bitwise", "lut"))
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-queries-per-step", type=int, default=1024)
    ap.add_argument("--gt-queries", type=int, default=2000, help="queries with exact ground truth (0 = all)")
    ap.add_argument("--gt-check", type=int, default=100, help="ground-truth rows checked against the oracle")
    ap.add_argument("--build-breakdown", action="store_true", help="rebuild once with per-stage timings")
    ap.add_argument("--sharded", action="store_true",
                    help="list-sharded build + search of one shared batch (strong scaling) instead of replicas")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    # stdout carries exactly the one JSON line: everything else written to fd 1 while the bench runs
    # (NCCL's version banner, library chatter) goes to stderr
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        out = run_reference(args, args.config)
    elif args.sharded:
        out = run_sharded(args, args.config)
    else:
        out = run_ours(args, args.config)
    sys.stdout.flush()
    if out:
        os.write(json_fd, (json.dumps(out) + "\n").encode())
    os.close(json_fd)


if __name__ == "__main__":
    main()
