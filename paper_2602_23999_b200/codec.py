"""RaBitQ code parameters, code/plane formats and the GPU quantizer.

Mirrors ``ivfrabitq.codec`` (reference codec.py).  The quantizer itself (the
two-phase rescaling-factor grid search, factor computation and bit packing)
is one warp-per-vector CUDA kernel (``ivrq_encode``); the helpers below that
only move bits between the IVRQ1 storage formats (``split_planes``,
``pack_interleaved``/``unpack_interleaved``, ``pack_excodes``/``unpack_excodes``)
are host-side data-format utilities used for file I/O and views.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from paper_2602_23999_b200 import _device as dev
from paper_2602_23999_b200 import _lib

__all__ = [
    "QuantizationParams",
    "ShortFactors",
    "LongFactors",
    "PackedPlane",
    "excode_bytes_per_vector",
    "split_planes",
    "pack_interleaved",
    "unpack_interleaved",
    "pack_excodes",
    "unpack_excodes",
    "quantize_batch",
    "quantize_vector",
    "quantize_oracle",
    "normalize_residual",
    "normalize_residuals",
    "compute_factors",
    "compute_factors_batch",
    "encode_rows",
    "rcode_row_bytes",
]

_ORACLE_MAX_FACTORS = 1 << 15


@dataclass(frozen=True)
class QuantizationParams:
    """Code width and rescaling-search parameters (reference codec.py:52-72)."""

    bits: int
    n_coarse: int = 64
    n_fine: int = 32
    eps_bound: float = 1.9

    def __post_init__(self) -> None:
        if not 1 <= self.bits <= 8:
            raise ValueError(f"bits must be in [1, 8], got {self.bits}")
        if self.n_coarse < 2 or self.n_fine < 2:
            raise ValueError("n_coarse and n_fine must both be >= 2")
        if not math.isfinite(self.eps_bound) or self.eps_bound < 0:
            raise ValueError(f"eps_bound must be finite and >= 0, got {self.eps_bound}")


@dataclass(frozen=True)
class ShortFactors:
    """Per-vector scalars of the 1-bit estimate: additive term, ip scale, error scale."""

    add: float
    scale: float
    err: float


@dataclass(frozen=True)
class LongFactors:
    """Per-vector scalars of the full-code (refinement) estimate."""

    add: float
    scale: float


@dataclass(frozen=True)
class PackedPlane:
    """One bit per (vector, dim), 32 dims per word, word (g, v) at ``g * n + v`` (codec.py:98-115)."""

    n: int
    dims: int
    words: np.ndarray

    @property
    def words_per_vector(self) -> int:
        return (self.dims + 31) // 32


def excode_bytes_per_vector(dims: int, bits: int) -> int:
    """Bytes of one vector's (bits-1)-bit ex-code stream (codec.py:427-429)."""
    return (dims * (bits - 1) + 7) // 8


# ---------------------------------------------------------------- formats


def split_planes(u: np.ndarray, bits: int) -> tuple[np.ndarray, np.ndarray | None]:
    """MSB plane and low-bit ex-code of unsigned codes (codec.py:306-319)."""
    codes = np.asarray(u, dtype=np.uint8)
    if codes.size and int(codes.max()) >= (1 << bits):
        raise ValueError(f"code value out of range for bits={bits}")
    shift = np.uint8(bits - 1)
    msb = np.right_shift(codes, shift).astype(np.uint8)
    if bits == 1:
        return msb, None
    return msb, np.bitwise_and(codes, np.uint8((1 << (bits - 1)) - 1)).astype(np.uint8)


def _bits_to_words(bits_matrix: np.ndarray) -> np.ndarray:
    """(n, dims) 0/1 -> (n, groups) little-endian uint32 words, zero padded."""
    n, dims = bits_matrix.shape
    groups = (dims + 31) // 32
    buf = np.zeros((n, groups * 32), dtype=np.uint8)
    buf[:, :dims] = bits_matrix
    return np.packbits(buf.reshape(n, groups, 32), axis=2, bitorder="little").reshape(n, groups * 4).view("<u4")


def pack_interleaved(bits_matrix: np.ndarray) -> PackedPlane:
    """(n, dims) 0/1 matrix -> interleaved words (codec.py:404-413)."""
    m = np.atleast_2d(np.asarray(bits_matrix, dtype=np.uint8))
    n, dims = m.shape
    per_vec = _bits_to_words(m)  # (n, groups)
    return PackedPlane(n=n, dims=dims, words=np.ascontiguousarray(per_vec.T).ravel())


def unpack_interleaved(plane: PackedPlane) -> np.ndarray:
    """Inverse of :func:`pack_interleaved` (codec.py:416-424)."""
    groups = plane.words_per_vector
    if plane.n == 0:
        return np.zeros((0, plane.dims), dtype=np.uint8)
    per_vec = np.ascontiguousarray(np.asarray(plane.words, dtype="<u4").reshape(groups, plane.n).T)
    flat = np.unpackbits(per_vec.view(np.uint8).reshape(plane.n, groups * 4), axis=1, bitorder="little")
    return flat[:, : plane.dims]


def pack_excodes(ex: np.ndarray, bits: int) -> np.ndarray:
    """(n, dims) ex-codes -> LSB-first bit stream per vector, byte padded (codec.py:432-444)."""
    e = np.atleast_2d(np.asarray(ex, dtype=np.uint8))
    n, dims = e.shape
    width = bits - 1
    if width == 0:
        return np.zeros((n, 0), dtype=np.uint8)
    planes = np.stack([(e >> np.uint8(b)) & np.uint8(1) for b in range(width)], axis=2)
    return np.packbits(planes.reshape(n, dims * width), axis=1, bitorder="little")


def unpack_excodes(packed: np.ndarray, dims: int, bits: int) -> np.ndarray:
    """Inverse of :func:`pack_excodes` (codec.py:447-456)."""
    p = np.atleast_2d(np.asarray(packed, dtype=np.uint8))
    n = p.shape[0]
    width = bits - 1
    if width == 0:
        return np.zeros((n, dims), dtype=np.uint8)
    stream = np.unpackbits(p, axis=1, bitorder="little")[:, : dims * width].reshape(n, dims, width)
    out = np.zeros((n, dims), dtype=np.uint8)
    for b in range(width):
        out |= (stream[:, :, b] << np.uint8(b)).astype(np.uint8)
    return out


# ---------------------------------------------------------------- refine code rows


def kpad64(dims: int) -> int:
    return (dims + 63) // 64 * 64


def rcode_row_bytes(dims: int, bits: int) -> int:
    """Bytes per vector of the device ``rcodes`` rows (see include/ivrq_b200.h)."""
    if bits <= 1:
        return 0
    return kpad64(dims) // 2 if bits <= 4 else kpad64(dims)


def codes_from_rcodes(rcodes: np.ndarray, dims: int, bits: int) -> np.ndarray:
    """Full unsigned codes (n, dims) from rcodes rows (host view)."""
    rc = np.asarray(rcodes, dtype=np.uint8).reshape(-1, rcode_row_bytes(dims, bits))
    if bits <= 4:
        u = np.empty((rc.shape[0], rc.shape[1] * 2), dtype=np.uint8)
        u[:, 0::2] = rc & 15
        u[:, 1::2] = rc >> 4
    else:
        u = rc
    return np.ascontiguousarray(u[:, :dims])


def excodes_from_rcodes(rcodes: np.ndarray, dims: int, bits: int) -> np.ndarray:
    """IVRQ1 ex-code bytes (codec.py:432-444) derived from rcodes rows."""
    u = codes_from_rcodes(rcodes, dims, bits)
    return pack_excodes(u & np.uint8((1 << (bits - 1)) - 1), bits)


# ---------------------------------------------------------------- GPU encoder


def encode_rows(
    o_rot: torch.Tensor,
    dist: torch.Tensor,
    cent_rot: torch.Tensor,
    offsets: torch.Tensor,
    params: QuantizationParams,
    want_codes: bool = False,
) -> dict[str, torch.Tensor]:
    """Run the warp-per-vector encoder over CSR-ordered rows (device tensors).

    Returns the device list layout (packed_msb, rcodes rows, short SoA, long
    float2) plus optionally the full codes ``u`` and factors ``t``.
    """
    n, d = o_rot.shape
    n_clusters = offsets.numel() - 1
    g = (d + 31) // 32
    eb = params.bits - 1
    device = o_rot.device
    out = {
        "packed_msb": torch.empty(n * g, dtype=torch.int32, device=device),
        "rcodes": torch.empty(n * rcode_row_bytes(d, params.bits), dtype=torch.uint8, device=device),
        "short_add": torch.empty(n, dtype=torch.float32, device=device),
        "short_scale": torch.empty(n, dtype=torch.float32, device=device),
        "short_err": torch.empty(n, dtype=torch.float32, device=device),
        "long_factors": torch.empty((n, 2), dtype=torch.float32, device=device),
        "bad_rows": torch.zeros(1, dtype=torch.int32, device=device),
    }
    if want_codes:
        out["codes"] = torch.empty((n, d), dtype=torch.uint8, device=device)
        out["t"] = torch.empty(n, dtype=torch.float64, device=device)
    _lib.call(
        "ivrq_encode",
        dev.ptr(o_rot),
        1 if o_rot.dtype == torch.float64 else 0,
        dev.ptr(dist),
        dev.ptr(cent_rot),
        dev.ptr(offsets),
        n_clusters,
        n,
        d,
        params.bits,
        params.n_coarse,
        params.n_fine,
        float(params.eps_bound),
        dev.ptr(out["packed_msb"]),
        dev.ptr(out["rcodes"]) if eb else None,
        dev.ptr(out["short_add"]),
        dev.ptr(out["short_scale"]),
        dev.ptr(out["short_err"]),
        dev.ptr(out["long_factors"]),
        dev.ptr(out.get("codes")),
        dev.ptr(out.get("t")),
        dev.ptr(out["bad_rows"]),
        dev.stream_ptr(),
    )
    return out


def quantize_batch(o: np.ndarray, params: QuantizationParams) -> tuple[np.ndarray, np.ndarray]:
    """Quantize unit rows on the GPU; returns ``(codes uint8, t)`` (codec.py:204-244).

    The grid search runs in the dtype of ``o`` (float32 or float64) exactly
    as the reference's NumPy expressions do.
    """
    arr = np.atleast_2d(np.asarray(o))
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    n, d = arr.shape
    device = dev.require_cuda()
    if n == 0:
        return np.zeros((0, d), dtype=np.uint8), np.zeros(0, dtype=arr.dtype)
    o_d = dev.to_device(arr, device)
    dist = torch.ones(n, dtype=torch.float64, device=device)
    cent = torch.zeros((1, d), dtype=torch.float32, device=device)
    offsets = torch.tensor([0, n], dtype=torch.int64, device=device)
    out = encode_rows(o_d, dist, cent, offsets, params, want_codes=True)
    if int(out["bad_rows"].item()) > 0:
        norms = np.sqrt(np.einsum("ij,ij->i", arr, arr, dtype=np.float64))
        bad = (norms != 0.0) & (np.abs(norms - 1.0) > 1e-4)
        raise ValueError(f"input rows must be unit vectors (or zero): worst norm {norms[bad].max():.6f}")
    codes = dev.to_host(out["codes"])
    t = dev.to_host(out["t"]).astype(arr.dtype)
    return codes, t


def quantize_vector(o_prime: np.ndarray, params: QuantizationParams) -> tuple[np.ndarray, float]:
    """Single-vector :func:`quantize_batch` (codec.py:247-253)."""
    v = np.asarray(o_prime)
    if v.ndim != 1:
        raise ValueError(f"expected a 1-d vector, got shape {v.shape}")
    u, t = quantize_batch(v[np.newaxis, :], params)
    return u[0], float(t[0])


# ---------------------------------------------------------------- per-vector sub-operators


def _check_finite_pair(a: np.ndarray, b: np.ndarray) -> None:
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if not (np.isfinite(a).all() and np.isfinite(b).all()):
        raise ValueError("non-finite input")


def _normalize(x: np.ndarray, c: np.ndarray, dd_norm: int) -> tuple[np.ndarray, np.ndarray]:
    n, d = x.shape
    device = dev.require_cuda()
    o = torch.empty((n, d), dtype=torch.float64, device=device)
    dist = torch.empty(n, dtype=torch.float64, device=device)
    if n:
        xd, cd = dev.to_device(x, device), dev.to_device(c, device)  # alive until the launch is queued
        _lib.call("ivrq_normalize_residuals", dev.ptr(xd), dev.ptr(cd), n, d, dd_norm, dev.ptr(o), dev.ptr(dist),
                  dev.stream_ptr())
    return dev.to_host(o), dev.to_host(dist)


def normalize_residual(o_r: np.ndarray, c: np.ndarray) -> tuple[np.ndarray, float]:
    """Unit direction and distance of ``o_r`` from ``c``; zero vector when d == 0 (codec.py:118-135)."""
    x = np.asarray(o_r, dtype=np.float64)
    cc = np.asarray(c, dtype=np.float64)
    _check_finite_pair(x, cc)
    o, d = _normalize(np.ascontiguousarray(x.reshape(1, -1)), np.ascontiguousarray(cc.reshape(1, -1)), 1)
    return o[0].reshape(x.shape), float(d[0])


def normalize_residuals(x: np.ndarray, centers: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Row-wise :func:`normalize_residual`, einsum-order norms (codec.py:138-151)."""
    xx = np.ascontiguousarray(np.atleast_2d(np.asarray(x, dtype=np.float64)))
    cc = np.ascontiguousarray(np.atleast_2d(np.asarray(centers, dtype=np.float64)))
    _check_finite_pair(xx, cc)
    return _normalize(xx, cc, 0)


def compute_factors_batch(u: np.ndarray, o: np.ndarray, d: np.ndarray, c_prime: np.ndarray, params: QuantizationParams):
    """Per-vector estimator factors ``(short (n,3), long (n,2), low_quality)`` in float64 (codec.py:322-380)."""
    uu = np.ascontiguousarray(np.atleast_2d(np.asarray(u, dtype=np.uint8)))
    oo = np.ascontiguousarray(np.atleast_2d(np.asarray(o, dtype=np.float64)))
    cc = np.ascontiguousarray(np.atleast_2d(np.asarray(c_prime, dtype=np.float64)))
    dd = np.ascontiguousarray(np.atleast_1d(np.asarray(d, dtype=np.float64)))
    n, dims = oo.shape
    if uu.shape != (n, dims) or cc.shape != (n, dims) or dd.shape != (n,):
        raise ValueError("inconsistent shapes across codes, vectors, and centers")
    device = dev.require_cuda()
    short = torch.zeros((n, 3), dtype=torch.float64, device=device)
    long = torch.zeros((n, 2), dtype=torch.float64, device=device)
    lowq = torch.zeros(n, dtype=torch.uint8, device=device)
    if n:
        ud, od, ddd, cd = (dev.to_device(a, device) for a in (uu, oo, dd, cc))
        _lib.call("ivrq_compute_factors", dev.ptr(ud), dev.ptr(od), dev.ptr(ddd), dev.ptr(cd), n, dims, params.bits,
                  float(params.eps_bound), dev.ptr(short), dev.ptr(long), dev.ptr(lowq), dev.stream_ptr())
    return dev.to_host(short), dev.to_host(long), dev.to_host(lowq).astype(bool)


def compute_factors(u: np.ndarray, o_prime: np.ndarray, d: float, c_prime: np.ndarray, params: QuantizationParams):
    """Single-vector :func:`compute_factors_batch` (codec.py:383-401)."""
    short, long, _ = compute_factors_batch(np.asarray(u)[None, :], np.asarray(o_prime)[None, :], np.array([d]),
                                           np.asarray(c_prime)[None, :], params)
    return (
        ShortFactors(add=float(short[0, 0]), scale=float(short[0, 1]), err=float(short[0, 2])),
        LongFactors(add=float(long[0, 0]), scale=float(long[0, 1])),
    )


def quantize_oracle(o_prime: np.ndarray, bits: int) -> np.ndarray:
    """Exhaustive critical-factor quantizer of one vector (codec.py:262-303), one CTA on the GPU."""
    o = np.ascontiguousarray(np.asarray(o_prime, dtype=np.float64))
    if o.ndim != 1:
        raise ValueError(f"expected a 1-d vector, got shape {o.shape}")
    dims = o.size
    if dims * 2 ** (bits - 1) > _ORACLE_MAX_FACTORS:
        raise ValueError(
            f"critical-factor count {dims * 2 ** (bits - 1)} exceeds the enumeration guard ({_ORACLE_MAX_FACTORS})"
        )
    device = dev.require_cuda()
    out = torch.empty(dims, dtype=torch.uint8, device=device)
    ws_bytes = int(_lib.load().ivrq_quantize_oracle_workspace(dims, bits))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    od = dev.to_device(o, device)
    _lib.call("ivrq_quantize_oracle", dev.ptr(od), dims, bits, dev.ptr(out), dev.ptr(ws),
              ws_bytes, dev.stream_ptr())
    return dev.to_host(out)
