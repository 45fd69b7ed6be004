"""bench.py's measurement helpers (no GPU): the roofline of the dominant kernel and the peaks."""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402

PEAKS = {"hbm_gbs": 6500.0, "bf16_tflops": 1700.0}


def test_int8_peak_is_the_committed_measurement():
    tops, src = bench.int8_peak(PEAKS)
    assert tops > 4000 and "tc_probe" in src


def test_refine_roofline_reports_the_binding_bound():
    kms = {"tc_refine_kernel": (1.0, 10), "scan_rd_kernel": (0.5, 10)}
    # C3-like: the bytes bind (1.9 GB at 6.5 TB/s > 0.94 TOP at 4.8 POP/s)
    r = bench.kernel_roofline(kms, PEAKS, probed=101_450_000, survivors=20_000_000, d=768, bits=8,
                              n_vectors=1_000_000, n_pairs=80_000)
    assert r["kernel"] == "tc_refine_kernel" and r["bound"] == "hbm"
    assert r["other_roofline"]["bound"] == "tensor"
    assert abs(r["achieved"] - r["work_per_launch"] / 1e-3 / 1e9) < 1.0
    assert 0 < r["frac"] < 1
    # a tiny index probed by many pairs: the MMA work binds
    r2 = bench.kernel_roofline(kms, PEAKS, probed=10_000_000_000, survivors=0, d=768, bits=8,
                               n_vectors=1000, n_pairs=10)
    assert r2["bound"] == "tensor" and r2["other_roofline"]["bound"] == "hbm"


def test_pass_roofline_counts_float32_distances():
    kms = {"scan_rd_kernel": (1.0, 5)}
    r = bench.kernel_roofline(kms, PEAKS, probed=1000, survivors=100, d=128, bits=4)
    assert r["bound"] == "hbm" and r["work_per_launch"] == 1000 * 14 + 100 * 4
    r1 = bench.kernel_roofline(kms, PEAKS, probed=1000, survivors=100, d=128, bits=1)
    assert r1["work_per_launch"] == 1000 * 14


def test_bench_accepts_the_sharded_mode():
    import subprocess

    out = subprocess.run([sys.executable, str(Path(bench.__file__)), "--help"], capture_output=True, text=True).stdout
    assert "--sharded" in out and "--impl" in out
