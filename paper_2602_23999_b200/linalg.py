"""Seeded random rotations, rotation of row vectors and the exact k-NN oracle.

Mirrors ``ivfrabitq.linalg`` (reference linalg.py).  ``gen_rotation`` draws
the seeded Gaussian matrix and runs its QR factorisation with host NumPy/LAPACK
once per index (an O(D^3) setup step, kept on the host so the matrix is the
reference's own for a given (dims, seed)); it is stored in the index.
``rotate`` and ``exact_knn`` run on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from paper_2602_23999_b200 import _device as dev
from paper_2602_23999_b200 import _lib

__all__ = ["Rotation", "gen_rotation", "rotate", "exact_knn", "matmul_nt"]


@dataclass(frozen=True)
class Rotation:
    """A random orthogonal matrix reproducible from ``(dims, seed)`` (linalg.py:18-23)."""

    dims: int
    matrix: np.ndarray
    seed: int


def gen_rotation(dims: int, seed: int) -> Rotation:
    """Seeded Gaussian -> QR -> column signs fixed by diag(R) (linalg.py:25-40)."""
    if dims < 1:
        raise ValueError(f"dims must be >= 1, got {dims}")
    gauss = np.random.default_rng(seed).standard_normal((dims, dims))
    q, r = np.linalg.qr(gauss)
    sign = np.sign(np.diagonal(r)).copy()
    sign[sign == 0] = 1.0
    return Rotation(dims=dims, matrix=q * sign[np.newaxis, :], seed=seed)


def matmul_nt(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """float64 ``a @ b.T`` on the device (a: (m, k), b: (n, k), float32/float64)."""
    m, k = a.shape
    n = b.shape[0]
    out = torch.empty((m, n), dtype=torch.float64, device=a.device)
    if m and n:
        _lib.call(
            "ivrq_matmul_nt",
            dev.ptr(a), 1 if a.dtype == torch.float64 else 0,
            dev.ptr(b), 1 if b.dtype == torch.float64 else 0,
            m, n, k, dev.ptr(out), dev.stream_ptr(),
        )
    return out


def rotate(rot: Rotation, x: np.ndarray) -> np.ndarray:
    """Row i of the result is ``R @ x[i]`` (linalg.py:43-50), float64 on the GPU."""
    arr = np.asarray(x)
    if arr.shape[-1] != rot.dims:
        raise ValueError(f"dimension mismatch: rotation is {rot.dims}-d, input is {arr.shape[-1]}-d")
    single = arr.ndim == 1
    rows = np.atleast_2d(arr)
    a = dev.to_device(rows if rows.dtype in (np.float32, np.float64) else rows.astype(np.float64))
    m = np.asarray(rot.matrix)
    b = dev.to_device(m if m.dtype in (np.float32, np.float64) else m.astype(np.float64))
    out = dev.to_host(matmul_nt(a, b))
    return out[0] if single else out


def exact_knn(base: np.ndarray, queries: np.ndarray, k: int, chunk: int = 256) -> tuple[np.ndarray, np.ndarray]:
    """Exact k-NN under squared L2 with ties to the smaller id (linalg.py:53-90).

    float64 distance identity on the GPU (the same kernels as the coarse
    probe); ``chunk`` is accepted for API compatibility.
    """
    del chunk
    b = np.ascontiguousarray(base)
    q = np.ascontiguousarray(np.atleast_2d(queries))
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    if b.ndim != 2 or b.shape[0] == 0:
        raise ValueError("base must be a nonempty 2-d array")
    if b.shape[1] != q.shape[1]:
        raise ValueError(f"dimension mismatch: base is {b.shape[1]}-d, queries are {q.shape[1]}-d")
    b32 = b.astype(np.float32)
    if b.dtype != np.float32 and not np.array_equal(b32.astype(b.dtype), b):
        raise ValueError("exact_knn on the GPU takes a float32-representable base")
    k_eff = min(k, b.shape[0])
    bd = dev.to_device(b32)
    qd = dev.to_device(q.astype(np.float64))
    ids, d2 = exact_knn_device(bd, qd, k_eff)
    return dev.to_host(ids), dev.to_host(d2)


def exact_knn_device(base: torch.Tensor, queries: torch.Tensor, k: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Device exact k-NN: base float32 (n, d), queries float64 (nq, d)."""
    from paper_2602_23999_b200.clustering import row_sqnorms

    n, d = base.shape
    nq = queries.shape[0]
    b_sq = row_sqnorms(base)
    ids = torch.empty((nq, k), dtype=torch.int64, device=base.device)
    d2 = torch.empty((nq, k), dtype=torch.float64, device=base.device)
    lib = _lib.load()
    ws_bytes = int(lib.ivrq_select_clusters_workspace(nq, n))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=base.device)
    _lib.call(
        "ivrq_select_clusters",
        dev.ptr(queries), nq, d, dev.ptr(base), dev.ptr(b_sq), n, k,
        dev.ptr(ids), dev.ptr(d2), dev.ptr(ws), ws_bytes, dev.stream_ptr(),
    )
    return ids, d2
