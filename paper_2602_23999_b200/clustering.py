"""Coarse IVF partitioning on the GPU: k-means++ seeding, Lloyd iterations, assignment.

Mirrors ``ivfrabitq.clustering`` (reference clustering.py).  Host NumPy only
draws the random numbers, in the reference's order (so the same seed yields
the same draws); every distance, reduction and update runs in
libivrq_b200.so with the reference's float64 arithmetic and reduction orders:
  * point-to-centre distances use the identity ``(|x|^2 + |c|^2) - 2<x,c>``
    with NumPy's einsum order for the squared norms (clustering.py:41-57);
  * k-means++ totals use NumPy's pairwise summation and the sampling uses the
    sequential cumsum + searchsorted (clustering.py:60-79);
  * centroid sums run in stable label order (np.add.reduceat, clustering.py:108-112);
  * empty clusters are reseeded to the farthest point (clustering.py:100-107).
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2602_23999_b200 import _device as dev
from paper_2602_23999_b200 import _lib

__all__ = ["Centroids", "train_kmeans", "assign", "row_sqnorms", "train_kmeans_device", "assign_device"]


def row_sqnorms(x: torch.Tensor) -> torch.Tensor:
    """einsum("ij,ij->i", x, x) in float64 on the device, NumPy-order exact."""
    n, d = x.shape
    out = torch.empty(n, dtype=torch.float64, device=x.device)
    if n:
        _lib.call(
            "ivrq_row_sqnorms", dev.ptr(x), 1 if x.dtype == torch.float64 else 0, n, d, dev.ptr(out), dev.stream_ptr()
        )
    return out


class Centroids:
    """Cluster centroids plus their cached squared norms (clustering.py:19-38).

    ``squared_norms`` (einsum order, float64) is computed on the GPU the first
    time it is needed when not supplied.
    """

    __slots__ = ("values", "_sq")

    def __init__(self, values: np.ndarray, squared_norms: np.ndarray | None = None) -> None:
        self.values = values
        self._sq = squared_norms

    @property
    def squared_norms(self) -> np.ndarray:
        if self._sq is None:
            t = dev.to_device(np.asarray(self.values, dtype=np.float64))
            self._sq = dev.to_host(row_sqnorms(t))
        return self._sq

    @classmethod
    def from_values(cls, values: np.ndarray) -> "Centroids":
        return cls(values=np.atleast_2d(np.asarray(values)))

    @property
    def n_clusters(self) -> int:
        return self.values.shape[0]

    @property
    def dims(self) -> int:
        return self.values.shape[1]


def assign_device(x: torch.Tensor, centers: torch.Tensor, c_sq: torch.Tensor, with_dmin: bool = False):
    """Nearest-centre labels (int32) [and clamped distances] for float32 rows ``x``."""
    n, d = x.shape
    k = centers.shape[0]
    labels = torch.empty(n, dtype=torch.int32, device=x.device)
    dmin = torch.empty(n, dtype=torch.float64, device=x.device) if with_dmin else None
    _lib.call(
        "ivrq_assign",
        dev.ptr(x),
        n,
        d,
        dev.ptr(centers),
        dev.ptr(c_sq),
        k,
        dev.ptr(labels),
        dev.ptr(dmin),
        dev.stream_ptr(),
    )
    return (labels, dmin) if with_dmin else labels


def counting_sort(labels: torch.Tensor, k: int):
    """Stable CSR of labels: (counts int64[k], offsets int64[k+1], order int64[n])."""
    n = labels.numel()
    counts = torch.empty(k, dtype=torch.int64, device=labels.device)
    offsets = torch.empty(k + 1, dtype=torch.int64, device=labels.device)
    order = torch.empty(n, dtype=torch.int64, device=labels.device)
    _lib.call(
        "ivrq_counting_sort", dev.ptr(labels), n, k, dev.ptr(counts), dev.ptr(offsets), dev.ptr(order), dev.stream_ptr()
    )
    return counts, offsets, order


def _kmeanspp_device(x: torch.Tensor, n_clusters: int, seed: int) -> torch.Tensor:
    n, d = x.shape
    rng = np.random.default_rng(seed)
    draws = np.empty(n_clusters, dtype=np.float64)
    draws[0] = float(int(rng.integers(n)))
    for j in range(1, n_clusters):
        draws[j] = rng.random()
    centers = torch.empty((n_clusters, d), dtype=torch.float64, device=x.device)
    d2 = torch.empty(n, dtype=torch.float64, device=x.device)
    zero_step = torch.full((1,), -1, dtype=torch.int32, device=x.device)
    d_draws = dev.to_device(draws, x.device)
    _lib.call(
        "ivrq_kmeanspp",
        dev.ptr(x), n, d, n_clusters, 0, n_clusters, dev.ptr(d_draws), 0,
        dev.ptr(centers), dev.ptr(d2), dev.ptr(zero_step), dev.stream_ptr(),
    )
    j0 = int(zero_step.item()) if n_clusters > 1 else -1
    if j0 >= 0:
        # total <= 0 from step j0 on: the reference draws rng.integers(n)
        # instead of rng.random() for every remaining centre; replay the stream.
        rng = np.random.default_rng(seed)
        rng.integers(n)
        for _ in range(1, j0):
            rng.random()
        for j in range(j0, n_clusters):
            draws[j] = float(int(rng.integers(n)))
        d_draws = dev.to_device(draws, x.device)
        _lib.call(
            "ivrq_kmeanspp",
            dev.ptr(x), n, d, n_clusters, j0, n_clusters, dev.ptr(d_draws), 1,
            dev.ptr(centers), dev.ptr(d2), dev.ptr(zero_step), dev.stream_ptr(),
        )
    return centers


def train_kmeans_device(x: torch.Tensor, n_clusters: int, iters: int, seed: int,
                        timings: dict | None = None) -> torch.Tensor:
    """Lloyd's k-means with k-means++ seeding on float32 device rows; returns float64 centres."""
    import time

    n, d = x.shape
    if n_clusters < 1 or n_clusters > n:
        raise ValueError(f"n_clusters must be in [1, {n}], got {n_clusters}")
    if iters < 1:
        raise ValueError(f"iters must be >= 1, got {iters}")
    t0 = time.perf_counter()
    centers = _kmeanspp_device(x, n_clusters, seed)
    if timings is not None:
        torch.cuda.synchronize()
        timings["kmeans_pp"] = time.perf_counter() - t0
        t0 = time.perf_counter()
    n_empty = torch.zeros(1, dtype=torch.int32, device=x.device)
    for _ in range(iters):
        c_sq = row_sqnorms(centers)
        labels, dmin = assign_device(x, centers, c_sq, with_dmin=True)
        counts, offsets, order = counting_sort(labels, n_clusters)
        _lib.call(
            "ivrq_kmeans_reseed",
            dev.ptr(labels), dev.ptr(dmin), n, dev.ptr(counts), n_clusters, dev.ptr(n_empty), dev.stream_ptr(),
        )
        counts, offsets, order = counting_sort(labels, n_clusters)
        new_centers = torch.empty_like(centers)
        _lib.call(
            "ivrq_kmeans_update",
            dev.ptr(x), n, dev.ptr(order), dev.ptr(offsets), n_clusters, d, dev.ptr(new_centers), dev.stream_ptr(),
        )
        centers = new_centers
    if timings is not None:
        torch.cuda.synchronize()
        timings["lloyd"] = time.perf_counter() - t0
    return centers


def train_kmeans(x: np.ndarray, n_clusters: int, iters: int, seed: int) -> Centroids:
    """Train centroids (clustering.py:82-113); the arithmetic runs on the GPU.

    ``x`` is used at float32 precision on the device; float64 inputs that are
    not float32-representable are rejected rather than silently rounded.
    """
    arr = np.ascontiguousarray(np.atleast_2d(x))
    x32 = arr.astype(np.float32)
    if arr.dtype != np.float32 and not np.array_equal(x32.astype(arr.dtype), arr):
        raise ValueError("train_kmeans on the GPU takes float32-representable data")
    n = x32.shape[0]
    if n_clusters < 1 or n_clusters > n:
        raise ValueError(f"n_clusters must be in [1, {n}], got {n_clusters}")
    if iters < 1:
        raise ValueError(f"iters must be >= 1, got {iters}")
    xd = dev.to_device(x32)
    centers = train_kmeans_device(xd, n_clusters, iters, seed)
    return Centroids(values=dev.to_host(centers), squared_norms=dev.to_host(row_sqnorms(centers)))


def assign(x: np.ndarray, centroids: Centroids) -> np.ndarray:
    """Nearest-centroid label per row, ties to the smaller id (clustering.py:116-125)."""
    arr = np.atleast_2d(np.asarray(x))
    if arr.shape[1] != centroids.dims:
        raise ValueError(
            f"dimension mismatch: x is {arr.shape[1]}-d, centroids are {centroids.dims}-d"
        )
    x32 = arr.astype(np.float32)
    if arr.dtype != np.float32 and not np.array_equal(x32.astype(arr.dtype), arr):
        raise ValueError("assign on the GPU takes float32-representable data")
    xd = dev.to_device(x32)
    cd = dev.to_device(np.asarray(centroids.values, dtype=np.float64))
    csq = dev.to_device(np.asarray(centroids.squared_norms, dtype=np.float64))
    labels = assign_device(xd, cd, csq)
    return dev.to_host(labels).astype(np.int64)
