"""ctypes binding of ``libivrq_b200.so`` (the C ABI in include/ivrq_b200.h).

The library is the product: there is no CPU implementation behind this
module.  Importing it without the shared library raises; calling a compute
entry point without a CUDA device raises.  Error codes are mapped to the
reference's exception types (``ValueError`` for bad arguments).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_uint8, c_uint32, c_void_p
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
HEADER = PKG_DIR.parent / "include" / "ivrq_b200.h"

IVRQ_OK = 0
IVRQ_EINVAL = -1
IVRQ_ECUDA = -2
IVRQ_ENOMEM = -3
IVRQ_EUNSUP = -4

IVRQ_IP_LUT = 0
IVRQ_IP_BITWISE = 1

QS_SUM_Q, QS_DELTA, QS_CODE_SUM, QS_IP_MARGIN, QS_KB_SUM, QS_HALF_CODE, QS_SLICE_EXP = range(7)
QS_COUNT = 8


class IndexView(ctypes.Structure):
    _fields_ = [
        ("dims", c_int32),
        ("bits", c_int32),
        ("n_clusters", c_int32),
        ("max_list", c_int32),
        ("size", c_int64),
        ("eps_bound", c_double),
        ("offsets", c_void_p),
        ("packed_msb", c_void_p),
        ("short_add", c_void_p),
        ("short_scale", c_void_p),
        ("short_err", c_void_p),
        ("long_factors", c_void_p),
        ("rcodes", c_void_p),
        ("rcode_bytes", c_int64),
        ("pids", c_void_p),
        ("centroids", c_void_p),
        ("centroid_sqnorms", c_void_p),
        ("rotation", c_void_p),
    ]


class SearchParamsC(ctypes.Structure):
    _fields_ = [
        ("k", c_int32),
        ("n_probe", c_int32),
        ("ip_mode", c_int32),
        ("query_bits", c_int32),
        ("refine", c_int32),
        ("prune", c_int32),
    ]


P = c_void_p  # device pointers are passed as integers

# name -> (restype, argtypes)
_SIGNATURES: dict[str, tuple[object, list[object]]] = {
    "ivrq_abi_version": (c_int, []),
    "ivrq_kernel_timing": (c_int, [ctypes.c_int32]),
    "ivrq_kernel_time": (c_int, [ctypes.c_char_p, POINTER(ctypes.c_double), POINTER(ctypes.c_int64)]),
    "ivrq_last_error": (ctypes.c_char_p, []),
    "ivrq_device_sm_count": (c_int, [c_int, POINTER(c_int)]),
    "ivrq_release_memory": (c_int, [P]),
    "ivrq_stream_wait_flag": (c_int, [P, ctypes.c_uint32, P]),
    "ivrq_stage_rows": (c_int, [P, P, c_int64, c_int64, c_int32, c_int32, P, POINTER(c_void_p)]),
    "ivrq_stage_wait": (c_int, [P, c_int32, c_int32]),
    "ivrq_stage_join": (c_int, [P]),
    "ivrq_row_sqnorms": (c_int, [P, c_int, c_int64, c_int32, P, P]),
    "ivrq_matmul_nt": (c_int, [P, c_int, P, c_int, c_int64, c_int64, c_int32, P, P]),
    "ivrq_rotate_queries": (c_int, [P, c_int, c_int64, c_int32, P, P, P]),
    "ivrq_select_clusters_workspace": (c_size_t, [c_int64, c_int32]),
    "ivrq_select_clusters": (
        c_int,
        [P, c_int64, c_int32, P, P, c_int32, c_int32, P, P, P, c_size_t, P],
    ),
    "ivrq_select_clusters_ordered": (
        c_int,
        [P, c_int64, c_int32, P, P, c_int32, c_int32, c_int32, P, P, P, c_size_t, P],
    ),
    "ivrq_select_clusters_f64": (
        c_int,
        [P, c_int64, c_int32, P, P, c_int32, c_int32, c_int32, P, P, P, c_size_t, P],
    ),
    "ivrq_prepare_queries": (
        c_int,
        [P, c_int64, c_int32, POINTER(SearchParamsC), c_int32, c_double, P, P, P, P, P],
    ),
    "ivrq_search_scan": (
        c_int,
        [POINTER(IndexView), P, P, P, P, P, P, P, c_int64, POINTER(SearchParamsC), P, P, P, P, P],
    ),
    "ivrq_search_scan_shard": (
        c_int,
        [POINTER(IndexView), c_int64, c_int64, P, P, P, P, P, P, P, c_int64, POINTER(SearchParamsC),
         P, P, P, P, P, P, P, P],
    ),
    "ivrq_merge_topk": (c_int, [P, P, P, c_int64, c_int32, c_int32, P, P, P, P]),
    "ivrq_ip_bitwise": (c_int, [P, c_int32, c_int64, P, c_int32, P, P]),
    "ivrq_ip_lut": (c_int, [P, c_int64, c_int32, P, P, P]),
    "ivrq_estimate_stage1": (c_int, [P, P, c_int64, P, c_double, c_double, P, P, P]),
    "ivrq_refine_stage2": (c_int, [P, c_int64, c_int32, P, P, P, c_double, P, c_int32, P, P]),
    "ivrq_cluster_local_search_workspace": (c_size_t, [c_int64]),
    "ivrq_cluster_local_search": (
        c_int,
        [POINTER(IndexView), c_int64, P, P, P, POINTER(c_double), POINTER(SearchParamsC), c_double,
         POINTER(c_double), P, P, P, P, c_size_t, c_int64, P],
    ),
    "ivrq_compute_factors": (c_int, [P, P, P, P, c_int64, c_int32, c_int32, c_double, P, P, P, P]),
    "ivrq_normalize_residuals": (c_int, [P, P, c_int64, c_int32, c_int32, P, P, P]),
    "ivrq_quantize_oracle_workspace": (c_size_t, [c_int32, c_int32]),
    "ivrq_quantize_oracle": (c_int, [P, c_int32, c_int32, P, P, c_size_t, P]),
    "ivrq_rcode_row_bytes": (c_int64, [c_int32, c_int32]),
    "ivrq_make_rcodes": (c_int, [P, P, c_int32, P, c_int64, c_int32, c_int32, P, P]),
    "ivrq_kmeanspp": (
        c_int,
        [P, c_int64, c_int32, c_int32, c_int32, c_int32, P, c_int32, P, P, P, P],
    ),
    "ivrq_assign": (c_int, [P, c_int64, c_int32, P, P, c_int32, P, P, P]),
    "ivrq_counting_sort": (c_int, [P, c_int64, c_int32, P, P, P, P]),
    "ivrq_kmeans_reseed": (c_int, [P, P, c_int64, P, c_int32, P, P]),
    "ivrq_kmeans_update": (c_int, [P, c_int64, P, P, c_int32, c_int32, P, P]),
    "ivrq_kmeans_chain_sums": (c_int, [P, P, P, c_int32, c_int32, P, P, P, P, P, P]),
    "ivrq_normalize_rotate": (c_int, [P, P, P, P, P, c_int64, c_int32, P, P, P]),
    "ivrq_rotate_rows_f32": (c_int, [P, c_int64, c_int32, P, P, P]),
    "ivrq_encode": (
        c_int,
        [
            P, c_int32, P, P, P, c_int32, c_int64, c_int32, c_int32, c_int32, c_int32, c_double,
            P, P, P, P, P, P, P, P, P, P,
        ],
    ),
}

_lib: ctypes.CDLL | None = None


def library_path() -> Path:
    return PKG_DIR / "libivrq_b200.so"


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load (building it first if needed and possible) the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if build_if_missing and os.environ.get("IVRQ_NO_AUTOBUILD") != "1":
        from paper_2602_23999_b200 import _build

        try:
            if _build.needs_build():
                _build.build()
        except RuntimeError:
            if not path.exists():
                raise
    if not path.exists():
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_2602_23999_b200._build` "
            "(the IVF-RaBitQ path has no CPU implementation)"
        )
    lib = ctypes.CDLL(str(path))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def check(rc: int, what: str = "") -> None:
    if rc == IVRQ_OK:
        return
    lib = load()
    msg = lib.ivrq_last_error().decode(errors="replace")
    if rc == IVRQ_EINVAL:
        raise ValueError(msg)
    if rc == IVRQ_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"{what or 'ivrq'} failed ({rc}): {msg}")


def call(name: str, *args) -> None:
    lib = load()
    check(getattr(lib, name)(*args), name)
