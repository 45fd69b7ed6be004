"""GPU-resident IVF-RaBitQ index: build pipeline, device layout and IVRQ1 files.

Mirrors ``ivfrabitq.index`` (reference index.py).  ``build_index`` runs the
reference pipeline (index.py:190-281) with every arithmetic stage in
libivrq_b200.so; host NumPy only draws the seeded random numbers (subsample,
k-means++ draws) and the once-per-index rotation QR, so a seed gives the
reference's random stream.  The built index lives in HBM in the layout of
include/ivrq_b200.h; the reference's NumPy attributes (``packed_msb``,
``excodes``, ``short_factors`` ...) are materialised from it on access and
``save_index``/``load_index`` read and write the reference's IVRQ1 format
byte for byte.
"""

from __future__ import annotations

import math
import os
import struct
from dataclasses import dataclass

import numpy as np
import torch

from paper_2602_23999_b200 import _device as dev
from paper_2602_23999_b200 import _lib
from paper_2602_23999_b200.clustering import (
    Centroids,
    assign_device,
    counting_sort,
    row_sqnorms,
    train_kmeans_device,
)
from paper_2602_23999_b200.codec import (
    PackedPlane,
    QuantizationParams,
    encode_rows,
    excode_bytes_per_vector,
    excodes_from_rcodes,
    rcode_row_bytes,
    unpack_excodes,
    unpack_interleaved,
)
from paper_2602_23999_b200.linalg import gen_rotation

__all__ = [
    "BuildParams",
    "IvfRabitqIndex",
    "IndexFormatError",
    "build_index",
    "save_index",
    "load_index",
    "default_workers",
]

_MAGIC = b"IVRQ1\x00"
_VERSION = 1
_SECTIONS = (
    "rotation",
    "centroids",
    "offsets",
    "packed_msb",
    "excodes",
    "short_factors",
    "long_factors",
    "pids",
)


class IndexFormatError(ValueError):
    """A malformed index file; the message names the offending section (index.py:49-50)."""


def default_workers() -> int:
    """IVRQ_THREADS semantics of the reference (index.py:53-66).

    The GPU path does not use host worker threads; the value is validated and
    accepted for API compatibility (results never depend on it).
    """
    env = os.environ.get("IVRQ_THREADS")
    if env:
        workers = int(env)
        if workers < 1:
            raise ValueError(f"IVRQ_THREADS must be >= 1, got {workers}")
        return workers
    return 1


@dataclass(frozen=True)
class BuildParams:
    """Index construction parameters (index.py:69-85)."""

    n_clusters: int
    quant: QuantizationParams
    kmeans_iters: int = 25
    train_fraction: float = 1.0
    seed: int = 0

    def __post_init__(self) -> None:
        if self.n_clusters < 1:
            raise ValueError(f"n_clusters must be >= 1, got {self.n_clusters}")
        if self.kmeans_iters < 1:
            raise ValueError(f"kmeans_iters must be >= 1, got {self.kmeans_iters}")
        if not 0.0 < self.train_fraction <= 1.0:
            raise ValueError(f"train_fraction must be in (0, 1], got {self.train_fraction}")


_HOST_FIELDS = ("rotation", "offsets", "packed_msb", "excodes", "short_factors", "long_factors", "pids")


class IvfRabitqIndex:
    """Built index (index.py:88-166).  Immutable after construction.

    Holds the device layout (``device`` dict of CUDA tensors) and serves the
    reference's NumPy attributes from it.  Constructing it from NumPy arrays
    (as ``load_index`` does, or as a caller of the reference dataclass would)
    uploads them on first use.
    """

    def __init__(
        self,
        dims: int,
        bits: int,
        n_clusters: int,
        size: int,
        eps_bound: float,
        seed: int,
        rotation: np.ndarray | None = None,
        centroids: Centroids | None = None,
        offsets: np.ndarray | None = None,
        packed_msb: np.ndarray | None = None,
        excodes: np.ndarray | None = None,
        short_factors: np.ndarray | None = None,
        long_factors: np.ndarray | None = None,
        pids: np.ndarray | None = None,
        *,
        device_arrays: dict[str, torch.Tensor] | None = None,
    ) -> None:
        self.dims = int(dims)
        self.bits = int(bits)
        self.n_clusters = int(n_clusters)
        self.size = int(size)
        self.eps_bound = float(eps_bound)
        self.seed = int(seed)
        self._host: dict[str, np.ndarray] = {}
        self._centroids = centroids
        for name, val in (
            ("rotation", rotation),
            ("offsets", offsets),
            ("packed_msb", packed_msb),
            ("excodes", excodes),
            ("short_factors", short_factors),
            ("long_factors", long_factors),
            ("pids", pids),
        ):
            if val is not None:
                self._host[name] = np.asarray(val)
        self._dev: dict[str, torch.Tensor] | None = device_arrays
        self._view = None

    # ------------------------------------------------------------ geometry
    @property
    def words_per_vector(self) -> int:
        return (self.dims + 31) // 32

    def cluster_range(self, cluster: int) -> tuple[int, int]:
        off = self.offsets
        return int(off[cluster]), int(off[cluster + 1])

    def cluster_words(self, cluster: int) -> np.ndarray:
        lo, hi = self.cluster_range(cluster)
        g = self.words_per_vector
        return self.packed_msb[lo * g : hi * g].reshape(g, hi - lo)

    # ------------------------------------------------------------ device layout
    @property
    def device(self) -> dict[str, torch.Tensor]:
        """The HBM layout (see include/ivrq_b200.h), uploading host arrays if needed."""
        if self._dev is None:
            self._dev = self._upload()
        return self._dev

    def _upload(self) -> dict[str, torch.Tensor]:
        d = dev.require_cuda()
        g = self.words_per_vector
        eb = self.bits - 1
        n = self.size
        sf = np.asarray(self._host["short_factors"], dtype=np.float32).reshape(n, 3)
        lf = np.asarray(self._host["long_factors"], dtype=np.float32).reshape(n, 2)
        cent = self.centroids
        cvals = np.ascontiguousarray(np.asarray(cent.values, dtype=np.float32))
        out = {
            "offsets": dev.to_device(np.asarray(self._host["offsets"], dtype=np.uint64), d),
            "packed_msb": dev.to_device(np.asarray(self._host["packed_msb"], dtype=np.uint32), d),
            "short_add": dev.to_device(np.ascontiguousarray(sf[:, 0]), d),
            "short_scale": dev.to_device(np.ascontiguousarray(sf[:, 1]), d),
            "short_err": dev.to_device(np.ascontiguousarray(sf[:, 2]), d),
            "long_factors": dev.to_device(np.ascontiguousarray(lf), d),
            "pids": dev.to_device(np.asarray(self._host["pids"], dtype=np.uint64), d),
            "centroids": dev.to_device(cvals, d),
            "rotation": dev.to_device(np.asarray(self._host["rotation"], dtype=np.float32), d),
        }
        out["centroid_sqnorms"] = dev.to_device(np.asarray(cent.squared_norms, dtype=np.float64), d)
        rb = rcode_row_bytes(self.dims, self.bits)
        out["rcodes"] = torch.empty(n * rb, dtype=torch.uint8, device=d)
        if eb and n:
            bpv = excode_bytes_per_vector(self.dims, self.bits)
            ex = dev.to_device(np.ascontiguousarray(np.asarray(self._host["excodes"], dtype=np.uint8).reshape(n, bpv)), d)
            _lib.call(
                "ivrq_make_rcodes",
                dev.ptr(out["packed_msb"]), dev.ptr(out["offsets"]), self.n_clusters, dev.ptr(ex),
                n, self.dims, self.bits, dev.ptr(out["rcodes"]), dev.stream_ptr(),
            )
        del g
        return out

    def view(self) -> _lib.IndexView:
        """C-ABI view of the device layout (kept alive with the index)."""
        if self._view is None:
            t = self.device
            self._view = _lib.IndexView(
                dims=self.dims,
                bits=self.bits,
                n_clusters=self.n_clusters,
                max_list=int(torch.diff(t["offsets"]).max().item()) if self.n_clusters else 0,
                size=self.size,
                eps_bound=self.eps_bound,
                offsets=dev.ptr(t["offsets"]),
                packed_msb=dev.ptr(t["packed_msb"]),
                short_add=dev.ptr(t["short_add"]),
                short_scale=dev.ptr(t["short_scale"]),
                short_err=dev.ptr(t["short_err"]),
                long_factors=dev.ptr(t["long_factors"]),
                rcodes=dev.ptr(t["rcodes"]),
                rcode_bytes=rcode_row_bytes(self.dims, self.bits),
                pids=dev.ptr(t["pids"]),
                centroids=dev.ptr(t["centroids"]),
                centroid_sqnorms=dev.ptr(t["centroid_sqnorms"]),
                rotation=dev.ptr(t["rotation"]),
            )
        return self._view

    # ------------------------------------------------------------ reference attributes
    def _materialise(self, name: str) -> np.ndarray:
        if name in self._host:
            return self._host[name]
        t = self._dev
        if t is None:
            raise AttributeError(name)
        n = self.size
        if name == "rotation":
            a = dev.to_host(t["rotation"])
        elif name == "offsets":
            a = dev.to_host(t["offsets"]).view(np.uint64)
        elif name == "packed_msb":
            a = dev.to_host(t["packed_msb"]).view(np.uint32)
        elif name == "excodes":
            if self.bits == 1:
                a = np.zeros((n, 0), dtype=np.uint8)
            else:
                a = excodes_from_rcodes(dev.to_host(t["rcodes"]), self.dims, self.bits)
        elif name == "short_factors":
            a = np.stack(
                [dev.to_host(t["short_add"]), dev.to_host(t["short_scale"]), dev.to_host(t["short_err"])], axis=1
            ).astype(np.float32)
        elif name == "long_factors":
            a = dev.to_host(t["long_factors"]).reshape(n, 2)
        elif name == "pids":
            a = dev.to_host(t["pids"]).view(np.uint64)
        else:
            raise AttributeError(name)
        self._host[name] = a
        return a

    rotation = property(lambda self: self._materialise("rotation"))
    offsets = property(lambda self: self._materialise("offsets"))
    packed_msb = property(lambda self: self._materialise("packed_msb"))
    excodes = property(lambda self: self._materialise("excodes"))
    short_factors = property(lambda self: self._materialise("short_factors"))
    long_factors = property(lambda self: self._materialise("long_factors"))
    pids = property(lambda self: self._materialise("pids"))

    @property
    def centroids(self) -> Centroids:
        if self._centroids is None:
            t = self._dev
            self._centroids = Centroids(
                values=dev.to_host(t["centroids"]), squared_norms=dev.to_host(t["centroid_sqnorms"])
            )
        return self._centroids

    @property
    def msb_nibbles(self) -> np.ndarray:
        """1-bit codes as 4-dim nibble indices (size, 8g) (index.py:120-140)."""
        if "msb_nibbles" not in self._host:
            g = self.words_per_vector
            out = np.zeros((self.size, 8 * g), dtype=np.uint8)
            for c in range(self.n_clusters):
                lo, hi = self.cluster_range(c)
                if hi == lo:
                    continue
                w = self.cluster_words(c).T  # (n_c, g)
                for s in range(8):
                    out[lo:hi, s::8] = ((w >> np.uint32(4 * s)) & np.uint32(15)).astype(np.uint8)
            self._host["msb_nibbles"] = out
        return self._host["msb_nibbles"]

    @property
    def code_values(self) -> np.ndarray:
        """Full unsigned codes as float32 (size, dims) (index.py:142-166)."""
        if "code_values" not in self._host:
            out = np.empty((self.size, self.dims), dtype=np.float32)
            g = self.words_per_vector
            for c in range(self.n_clusters):
                lo, hi = self.cluster_range(c)
                if hi == lo:
                    continue
                plane = PackedPlane(n=hi - lo, dims=self.dims, words=self.packed_msb[lo * g : hi * g])
                out[lo:hi] = unpack_interleaved(plane)
            out *= float(2 ** (self.bits - 1))
            if self.bits > 1:
                out += unpack_excodes(self.excodes, self.dims, self.bits)
            self._host["code_values"] = out
        return self._host["code_values"]

    def __repr__(self) -> str:
        return (
            f"IvfRabitqIndex(dims={self.dims}, bits={self.bits}, n_clusters={self.n_clusters}, "
            f"size={self.size}, eps_bound={self.eps_bound}, seed={self.seed})"
        )


# ---------------------------------------------------------------- build


def build_index_device(
    x: torch.Tensor,
    params: BuildParams,
    *,
    inject: dict | None = None,
    keep: dict | None = None,
    timings: dict | None = None,
) -> IvfRabitqIndex:
    """Build from float32 rows already on the device (the bench's resident path).

    ``inject`` (tests only) may replace intermediate results with the
    reference's own -- ``centroids64`` (float64 (k, d)), ``rotation`` (float32),
    ``cent_rot`` (float32), ``o_rot`` (float32, CSR order) -- to check the
    downstream stages bit-exactly "given identical rotated vectors and
    centroids".  ``keep`` receives intermediate device tensors when given;
    ``timings`` (bench) receives per-stage seconds (synchronising between stages).
    """
    import time

    t_last = [time.perf_counter()]

    def tick(name: str) -> None:
        if timings is not None:
            torch.cuda.synchronize()
            now = time.perf_counter()
            timings[name] = timings.get(name, 0.0) + now - t_last[0]
            t_last[0] = now

    inject = inject or {}
    n, dims = x.shape
    quant = params.quant
    device = x.device
    seeds = np.random.SeedSequence(params.seed).spawn(2)
    if "centroids64" in inject:
        centers = dev.to_device(np.asarray(inject["centroids64"], dtype=np.float64), device)
    else:
        if params.train_fraction < 1.0:
            n_train = max(1, math.ceil(params.train_fraction * n))
            n_train = max(n_train, min(n, params.n_clusters))
            rows = np.sort(np.random.default_rng(seeds[0]).choice(n, size=n_train, replace=False))
            x_train = x.index_select(0, dev.to_device(rows.astype(np.int64), device))
        else:
            x_train = x
        km_seed = int(seeds[1].generate_state(1)[0])
        centers = train_kmeans_device(x_train, params.n_clusters, params.kmeans_iters, km_seed, timings=timings)
        t_last[0] = time.perf_counter()
    c_sq = row_sqnorms(centers)
    labels = assign_device(x, centers, c_sq)
    counts, offsets, order = counting_sort(labels, params.n_clusters)
    tick("assign_csr")

    if "rotation" in inject:
        rot32_np = np.asarray(inject["rotation"], dtype=np.float32)
    else:
        rot32_np = gen_rotation(dims, params.seed).matrix.astype(np.float32)
    rot32 = dev.to_device(rot32_np, device)
    cent32 = centers.to(torch.float32)
    if "cent_rot" in inject:
        cent_rot = dev.to_device(np.asarray(inject["cent_rot"], dtype=np.float32), device)
    else:
        cent_rot = torch.empty((params.n_clusters, dims), dtype=torch.float32, device=device)
        _lib.call(
            "ivrq_rotate_rows_f32", dev.ptr(cent32), params.n_clusters, dims, dev.ptr(rot32), dev.ptr(cent_rot),
            dev.stream_ptr(),
        )
    o_rot = torch.empty((n, dims), dtype=torch.float32, device=device)
    dist = torch.empty(n, dtype=torch.float64, device=device)
    _lib.call(
        "ivrq_normalize_rotate",
        dev.ptr(x), dev.ptr(order), dev.ptr(labels), dev.ptr(cent32), dev.ptr(rot32),
        n, dims, dev.ptr(o_rot), dev.ptr(dist), dev.stream_ptr(),
    )
    if "o_rot" in inject:
        o_rot = dev.to_device(np.asarray(inject["o_rot"], dtype=np.float32), device)
    tick("rotations")
    enc = encode_rows(o_rot, dist, cent_rot, offsets, quant, want_codes=keep is not None)
    tick("encode")
    if keep is not None:
        keep.update(
            centers=centers, labels=labels, counts=counts, offsets=offsets, order=order,
            cent_rot=cent_rot, o_rot=o_rot, dist=dist, codes=enc.get("codes"), t=enc.get("t"),
        )
    device_arrays = {
        "offsets": offsets,
        "packed_msb": enc["packed_msb"],
        "short_add": enc["short_add"],
        "short_scale": enc["short_scale"],
        "short_err": enc["short_err"],
        "long_factors": enc["long_factors"],
        "rcodes": enc["rcodes"],
        "pids": order,
        "centroids": cent_rot,
        "centroid_sqnorms": row_sqnorms(cent_rot),
        "rotation": rot32,
    }
    return IvfRabitqIndex(
        dims=dims,
        bits=quant.bits,
        n_clusters=params.n_clusters,
        size=n,
        eps_bound=quant.eps_bound,
        seed=params.seed,
        device_arrays=device_arrays,
    )


def build_index(x: np.ndarray, params: BuildParams, workers: int | None = None) -> IvfRabitqIndex:
    """Build an index over the rows of ``x`` on the GPU (index.py:190-281).

    ``workers`` is accepted for API compatibility; the result never depends on it.
    """
    arr = np.ascontiguousarray(np.atleast_2d(x), dtype=np.float32)
    n, _ = arr.shape
    if n == 0:
        raise ValueError("cannot build an index over an empty dataset")
    if params.n_clusters > n:
        raise ValueError(f"n_clusters={params.n_clusters} exceeds dataset size {n}")
    if workers is None:
        default_workers()
    xd = dev.to_device(arr)
    if not bool(torch.isfinite(xd).all().item()):
        raise ValueError("dataset contains non-finite values")
    return build_index_device(xd, params)


# ---------------------------------------------------------------- IVRQ1 files


def save_index(index: IvfRabitqIndex, path: str) -> None:
    """Write the IVRQ1 file (little-endian), byte-identical to the reference (index.py:296-325)."""
    arrays = {
        "rotation": np.asarray(index.rotation, dtype="<f4"),
        "centroids": np.asarray(index.centroids.values, dtype="<f4"),
        "offsets": np.asarray(index.offsets, dtype="<u8"),
        "packed_msb": np.asarray(index.packed_msb, dtype="<u4"),
        "excodes": np.asarray(index.excodes, dtype="<u1"),
        "short_factors": np.asarray(index.short_factors, dtype="<f4"),
        "long_factors": np.asarray(index.long_factors, dtype="<f4"),
        "pids": np.asarray(index.pids, dtype="<u8"),
    }
    header = struct.pack(
        "<IIIQfQ", index.dims, index.bits, index.n_clusters, index.size, index.eps_bound, index.seed
    )
    with open(path, "wb") as f:
        f.write(_MAGIC + struct.pack("<H", _VERSION) + header)
        for name in _SECTIONS:
            blob = np.ascontiguousarray(arrays[name]).tobytes()
            f.write(struct.pack("<Q", len(blob)))
            f.write(blob)


def _read(f, count: int, section: str) -> bytes:
    data = f.read(count)
    if len(data) != count:
        raise IndexFormatError(f"file truncated in section '{section}'")
    return data


def load_index(path: str) -> IvfRabitqIndex:
    """Read an IVRQ1 file (index.py:335-388); the device copy is made on first search."""
    with open(path, "rb") as f:
        magic = f.read(len(_MAGIC))
        if magic != _MAGIC:
            raise IndexFormatError(f"bad magic {magic!r}, not an index file")
        (version,) = struct.unpack("<H", _read(f, 2, "header"))
        if version != _VERSION:
            raise IndexFormatError(f"unsupported version {version}")
        dims, bits, n_clusters, size, eps_bound, seed = struct.unpack("<IIIQfQ", _read(f, 32, "header"))
        g = (dims + 31) // 32
        bpv = excode_bytes_per_vector(dims, bits)
        layout = {
            "rotation": ("<f4", (dims, dims)),
            "centroids": ("<f4", (n_clusters, dims)),
            "offsets": ("<u8", (n_clusters + 1,)),
            "packed_msb": ("<u4", (size * g,)),
            "excodes": ("<u1", (size, bpv)),
            "short_factors": ("<f4", (size, 3)),
            "long_factors": ("<f4", (size, 2)),
            "pids": ("<u8", (size,)),
        }
        arrays: dict[str, np.ndarray] = {}
        for name in _SECTIONS:
            dtype, shape = layout[name]
            nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
            (length,) = struct.unpack("<Q", _read(f, 8, name))
            if length != nbytes:
                raise IndexFormatError(f"section '{name}' has {length} bytes, expected {nbytes}")
            arrays[name] = np.frombuffer(_read(f, nbytes, name), dtype=dtype).reshape(shape).copy()
    off = arrays["offsets"]
    if off[0] != 0 or off[-1] != size or np.any(np.diff(off.astype(np.int64)) < 0):
        raise IndexFormatError("section 'offsets' is not a valid row-pointer array")
    return IvfRabitqIndex(
        dims=dims,
        bits=bits,
        n_clusters=n_clusters,
        size=size,
        eps_bound=eps_bound,
        seed=seed,
        rotation=arrays["rotation"],
        centroids=Centroids.from_values(arrays["centroids"]),
        offsets=off,
        packed_msb=arrays["packed_msb"],
        excodes=arrays["excodes"],
        short_factors=arrays["short_factors"],
        long_factors=arrays["long_factors"],
        pids=arrays["pids"],
    )
