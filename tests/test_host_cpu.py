"""Host-side logic that runs without a GPU: parameter validation, storage
formats, IVRQ1 files and the C-ABI library surface."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2602_23999_b200 as iv
from conftest import ROOT, golden_index_arrays, load_case
from oracle import ivrq_oracle as orc
from paper_2602_23999_b200 import _lib
from paper_2602_23999_b200.clustering import Centroids
from paper_2602_23999_b200.index import IvfRabitqIndex


def _host_index(g) -> IvfRabitqIndex:
    a = golden_index_arrays(g)
    return IvfRabitqIndex(
        dims=a["dims"], bits=a["bits"], n_clusters=a["n_clusters"], size=a["size"], eps_bound=a["eps_bound"],
        seed=int(g["params"][3]), rotation=a["rotation"],
        centroids=Centroids(a["centroids"], a["centroid_sqnorms"]), offsets=a["offsets"],
        packed_msb=a["packed_msb"], excodes=a["excodes"], short_factors=a["short_factors"],
        long_factors=a["long_factors"], pids=a["pids"],
    )


# ---------------------------------------------------------------- ABI


def _header_symbols() -> list[str]:
    text = (ROOT / "include" / "ivrq_b200.h").read_text()
    return sorted(set(re.findall(r"IVRQ_API\s+[\w\s\*]+?\b(ivrq_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = _header_symbols()
    for name in ("ivrq_search_scan", "ivrq_select_clusters", "ivrq_encode", "ivrq_kmeanspp", "ivrq_assign"):
        assert name in syms


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    for name in _header_symbols():
        assert hasattr(lib, name), name
    assert set(_header_symbols()) == set(_lib.exported_symbols())
    assert lib.ivrq_abi_version() == 1
    assert lib.ivrq_last_error() is not None


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(
        ["cuobjdump", "--list-elf", str(_lib.library_path())], capture_output=True, text=True
    ).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out


# ---------------------------------------------------------------- params


def test_params_validation():
    with pytest.raises(ValueError):
        iv.QuantizationParams(bits=0)
    with pytest.raises(ValueError):
        iv.QuantizationParams(bits=9)
    with pytest.raises(ValueError):
        iv.QuantizationParams(bits=4, n_coarse=1)
    with pytest.raises(ValueError):
        iv.QuantizationParams(bits=4, eps_bound=-1.0)
    with pytest.raises(ValueError):
        iv.BuildParams(n_clusters=0, quant=iv.QuantizationParams(bits=1))
    with pytest.raises(ValueError):
        iv.BuildParams(n_clusters=2, quant=iv.QuantizationParams(bits=1), kmeans_iters=0)
    with pytest.raises(ValueError):
        iv.BuildParams(n_clusters=2, quant=iv.QuantizationParams(bits=1), train_fraction=0.0)
    with pytest.raises(ValueError):
        iv.SearchParams(k=0, n_probe=1)
    with pytest.raises(ValueError):
        iv.SearchParams(k=1, n_probe=0)
    with pytest.raises(ValueError):
        iv.SearchParams(k=1, n_probe=1, ip_mode="simd")
    with pytest.raises(ValueError):
        iv.SearchParams(k=1, n_probe=1, query_bits=1)
    assert iv.SearchParams(k=1, n_probe=1).ip_mode == "lut"


def test_default_workers_env(monkeypatch):
    monkeypatch.setenv("IVRQ_THREADS", "3")
    assert iv.default_workers() == 3
    monkeypatch.setenv("IVRQ_THREADS", "0")
    with pytest.raises(ValueError):
        iv.default_workers()


def test_search_batch_validates_before_touching_the_device():
    g = load_case("b4_d48")
    ix = _host_index(g)
    with pytest.raises(ValueError):
        iv.search_batch(np.zeros((1, ix.dims)), ix, iv.SearchParams(k=1, n_probe=ix.n_clusters + 1))
    with pytest.raises(ValueError):
        iv.search_batch(np.zeros((1, ix.dims + 1)), ix, iv.SearchParams(k=1, n_probe=2))


# ---------------------------------------------------------------- formats


def test_pack_interleaved_word_order():
    plane = iv.pack_interleaved(np.ones((1, 32), dtype=np.uint8))
    assert plane.words.tolist() == [0xFFFFFFFF]
    bits = np.zeros((2, 64), dtype=np.uint8)
    bits[0, 0] = 1
    bits[1, 1] = 1
    bits[0, 32] = 1
    bits[1, 63] = 1
    assert iv.pack_interleaved(bits).words.tolist() == [1, 2, 1, 1 << 31]


@pytest.mark.parametrize("dims", [1, 31, 32, 33, 70, 128])
def test_pack_roundtrips(dims):
    rng = np.random.default_rng(dims)
    b = rng.integers(0, 2, (7, dims)).astype(np.uint8)
    plane = iv.pack_interleaved(b)
    assert np.array_equal(iv.unpack_interleaved(plane), b)
    assert int(np.bitwise_count(plane.words).sum()) == int(b.sum())
    np.testing.assert_array_equal(plane.words, orc.msb_words(b))
    for bits in (2, 3, 5, 8):
        ex = rng.integers(0, 2 ** (bits - 1), (6, dims)).astype(np.uint8)
        packed = iv.pack_excodes(ex, bits)
        assert packed.shape == (6, iv.excode_bytes_per_vector(dims, bits))
        np.testing.assert_array_equal(packed, orc.ex_bytes(ex, bits))
        assert np.array_equal(iv.unpack_excodes(packed, dims, bits), ex)


def test_split_planes():
    msb, ex = iv.split_planes(np.array([5], dtype=np.uint8), 3)
    assert msb.tolist() == [1] and ex.tolist() == [1]
    msb, ex = iv.split_planes(np.array([0, 1, 1], dtype=np.uint8), 1)
    assert ex is None and msb.tolist() == [0, 1, 1]
    with pytest.raises(ValueError):
        iv.split_planes(np.array([4], dtype=np.uint8), 2)


# ---------------------------------------------------------------- IVRQ1 files


def test_save_load_roundtrip_is_byte_identical(tmp_path):
    for name in ("b4_d48", "b1_d32", "b2_dup"):
        g = load_case(name)
        ix = _host_index(g)
        p1 = tmp_path / f"{name}.idx"
        iv.save_index(ix, str(p1))
        loaded = iv.load_index(str(p1))
        for field in ("rotation", "offsets", "packed_msb", "excodes", "short_factors", "long_factors", "pids"):
            assert np.array_equal(getattr(loaded, field), getattr(ix, field)), field
        assert np.array_equal(loaded.centroids.values, ix.centroids.values)
        assert loaded.eps_bound == np.float32(ix.eps_bound)
        p2 = tmp_path / f"{name}.2.idx"
        iv.save_index(loaded, str(p2))
        assert p1.read_bytes() == p2.read_bytes()


def test_load_rejects_malformed_files(tmp_path):
    g = load_case("b4_d48")
    path = tmp_path / "a.idx"
    iv.save_index(_host_index(g), str(path))
    data = path.read_bytes()
    bad = tmp_path / "bad.idx"
    bad.write_bytes(b"NOTIDX" + b"\x00" * 64)
    with pytest.raises(iv.IndexFormatError, match="magic"):
        iv.load_index(str(bad))
    cut = tmp_path / "cut.idx"
    cut.write_bytes(data[:-17])
    with pytest.raises(iv.IndexFormatError, match="pids"):
        iv.load_index(str(cut))
    head = tmp_path / "head.idx"
    head.write_bytes(data[:10])
    with pytest.raises(iv.IndexFormatError, match="header"):
        iv.load_index(str(head))
    raw = bytearray(data)
    raw[40:48] = (999).to_bytes(8, "little")
    wrong = tmp_path / "wrong.idx"
    wrong.write_bytes(bytes(raw))
    with pytest.raises(iv.IndexFormatError, match="rotation"):
        iv.load_index(str(wrong))


def test_index_views_match_oracle_decode():
    g = load_case("b3_d96")
    ix = _host_index(g)
    a = golden_index_arrays(g)
    np.testing.assert_array_equal(ix.code_values, orc.decode_codes(a))
    lo, hi = ix.cluster_range(0)
    assert ix.cluster_words(0).shape == (ix.words_per_vector, hi - lo)
    assert ix.msb_nibbles.shape == (ix.size, 8 * ix.words_per_vector)


# ---------------------------------------------------------------- drop-in API surface

# the reference's public names (reference pkg/src/ivfrabitq/__init__.py:57-101)
REFERENCE_ALL = [
    "Centroids", "assign", "train_kmeans", "LongFactors", "PackedPlane", "QuantizationParams", "ShortFactors",
    "compute_factors", "normalize_residual", "pack_excodes", "pack_interleaved", "quantize_oracle",
    "quantize_vector", "split_planes", "unpack_excodes", "unpack_interleaved", "BuildParams", "IndexFormatError",
    "IvfRabitqIndex", "build_index", "load_index", "save_index", "read_fvecs", "read_ivecs", "write_fvecs",
    "write_ivecs", "Rotation", "exact_knn", "gen_rotation", "rotate", "QueryState", "SearchParams", "build_luts",
    "cluster_local_search", "estimate_stage1", "ip_bitwise", "ip_lut", "merge_topk", "prepare_query",
    "refine_stage2", "schedule_probes", "search_batch", "select_clusters",
]


def test_reference_public_names_all_exported():
    missing = [n for n in REFERENCE_ALL if not hasattr(iv, n)]
    assert not missing, missing
    assert set(REFERENCE_ALL) <= set(iv.__all__)


def test_query_state_defaults_follow_reference():
    st = iv.QueryState(q_rot=np.ones(4), sum_q=4.0)
    assert st.code_sum_q == 4.0 and st.delta_q == 1.0 and st.threshold == float("inf")
    assert st.q_hat is None and st.planes is None and st.luts is None


def test_nibbles_from_bits_layout():
    bits = np.zeros((2, 8), dtype=np.uint8)
    bits[0, 0] = 1
    bits[1, 4:8] = 1
    nib = iv.nibbles_from_bits(bits)
    # 8 dims are padded to one 32-dim word: 8 nibbles per row
    assert nib.shape == (2, 8)
    assert nib[0, 0] == 1 and nib[1, 1] == 15 and nib[1, 0] == 0


def test_fvecs_ivecs_round_trip_and_errors(tmp_path):
    x = np.arange(12, dtype=np.float32).reshape(3, 4) / 7.0
    p = tmp_path / "a.fvecs"
    iv.write_fvecs(str(p), x)
    np.testing.assert_array_equal(iv.read_fvecs(str(p)), x)
    ids = np.arange(6, dtype=np.int32).reshape(2, 3)
    pi = tmp_path / "a.ivecs"
    iv.write_ivecs(str(pi), ids)
    np.testing.assert_array_equal(iv.read_ivecs(str(pi)), ids)
    # 4 + 4*4 bytes per record: drop the last 4 bytes -> truncated record at the second record's offset
    raw = p.read_bytes()
    bad = tmp_path / "bad.fvecs"
    bad.write_bytes(raw[:-4])
    with pytest.raises(ValueError, match="truncated record at byte offset 40"):
        iv.read_fvecs(str(bad))
    mixed = tmp_path / "mixed.fvecs"
    mixed.write_bytes(raw[:20] + np.array([3], dtype="<i4").tobytes() + raw[24:])
    with pytest.raises(ValueError, match="inconsistent dimension 3 at byte offset 20"):
        iv.read_fvecs(str(mixed))
    empty = tmp_path / "e.fvecs"
    empty.write_bytes(b"")
    assert iv.read_fvecs(str(empty)).shape == (0, 0)


@pytest.mark.parametrize("rows,pieces,threads", [(10000, 8, 8), (7, 3, 4), (0, 1, 2), (4900, 4, 16)])
def test_native_staging_copies_pieces_and_raises_flags(rows, pieces, threads):
    """ivrq_stage_rows (search_batch's host staging, no interpreter on the publish path): every row
    copied, every piece's flag == the thread count, host waits return, join is clean."""
    import ctypes

    rng = np.random.default_rng(rows)
    q = rng.standard_normal((rows, 96)).astype(np.float32)
    dst = np.zeros_like(q)
    flags = np.full(pieces, 77, dtype=np.uint32)  # zeroed by the call
    h = ctypes.c_void_p()
    _lib.call("ivrq_stage_rows", dst.ctypes.data, q.ctypes.data, rows, 96 * 4, pieces, threads,
              flags.ctypes.data, ctypes.byref(h))
    for p in range(pieces):
        _lib.call("ivrq_stage_wait", flags.ctypes.data, p, threads)
    _lib.call("ivrq_stage_join", h)
    np.testing.assert_array_equal(dst, q)
    assert (flags == threads).all()
    with pytest.raises(ValueError):
        _lib.call("ivrq_stage_rows", dst.ctypes.data, q.ctypes.data, rows, 0, pieces, threads,
                  flags.ctypes.data, ctypes.byref(h))


def test_native_staging_after_fork():
    """The staging pool is rebuilt in a forked child (its workers are not inherited): a copy there
    completes instead of waiting on threads that do not exist."""
    import ctypes
    import os

    q = np.arange(4096 * 8, dtype=np.float32).reshape(4096, 8)
    dst = np.zeros_like(q)
    flags = np.zeros(2, dtype=np.uint32)
    h = ctypes.c_void_p()
    _lib.call("ivrq_stage_rows", dst.ctypes.data, q.ctypes.data, 4096, 32, 2, 4, flags.ctypes.data, ctypes.byref(h))
    _lib.call("ivrq_stage_join", h)  # the parent's pool has started its workers
    pid = os.fork()
    if pid == 0:  # child: copy again through the library, exit 0 on success
        code = 1
        try:
            d2 = np.zeros_like(q)
            h2 = ctypes.c_void_p()
            _lib.call("ivrq_stage_rows", d2.ctypes.data, q.ctypes.data, 4096, 32, 2, 4, flags.ctypes.data,
                      ctypes.byref(h2))
            _lib.call("ivrq_stage_join", h2)
            code = 0 if np.array_equal(d2, q) else 2
        finally:
            os._exit(code)
    import time

    deadline = time.time() + 60
    while time.time() < deadline:
        done, status = os.waitpid(pid, os.WNOHANG)
        if done:
            assert os.waitstatus_to_exitcode(status) == 0
            return
        time.sleep(0.05)
    os.kill(pid, 9)
    os.waitpid(pid, 0)
    raise AssertionError("staging in the forked child did not complete")
