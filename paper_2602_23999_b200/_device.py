"""Device plumbing: CUDA tensors, streams and pointer handling via PyTorch.

PyTorch provides device memory (the caching allocator), streams and
torch.distributed; every computation on the IVF-RaBitQ path is a kernel of
libivrq_b200.so.  Nothing here falls back to the CPU: without a CUDA device
the compute entry points raise.
"""

from __future__ import annotations

import numpy as np
import torch

_NP_TO_TORCH = {
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.uint8): torch.uint8,
    np.dtype(np.uint32): torch.int32,  # bit-reinterpreted (torch has no uint32 arithmetic need)
    np.dtype(np.uint64): torch.int64,  # bit-reinterpreted
}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "the B200 IVF-RaBitQ kernels need a CUDA device; none is visible "
            "(there is no CPU implementation of this path)"
        )
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return int(t.data_ptr()) if t.numel() else None


def to_device(arr: np.ndarray, device: torch.device | None = None, non_blocking: bool = False) -> torch.Tensor:
    """Copy a host array to the device, keeping its bit pattern (uint32/uint64 reinterpreted)."""
    device = device or require_cuda()
    a = np.ascontiguousarray(arr)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    elif a.dtype == np.uint64:
        a = a.view(np.int64)
    t = torch.from_numpy(a)
    if non_blocking:
        t = t.pin_memory()
    return t.to(device, non_blocking=non_blocking)


def to_host(t: torch.Tensor, dtype: np.dtype | None = None) -> np.ndarray:
    a = t.detach().to("cpu").numpy()
    if dtype is not None and np.dtype(dtype) != a.dtype:
        a = a.view(dtype) if np.dtype(dtype).itemsize == a.dtype.itemsize else a.astype(dtype)
    return a


def empty(shape, dtype: torch.dtype, device: torch.device | None = None) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device or require_cuda())


def zeros(shape, dtype: torch.dtype, device: torch.device | None = None) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device or require_cuda())
