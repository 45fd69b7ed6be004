"""Build the sm_100a shared library ``libivrq_b200.so`` in-tree with nvcc.

The library is plain C ABI (include/ivrq_b200.h) with the CUDA runtime linked
statically, so it loads on a machine without a GPU (the CPU test suite checks
its exported symbols) and travels to the GPU box with the repository snapshot.
"""

from __future__ import annotations

import concurrent.futures
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
INCLUDE = PKG_DIR.parent / "include"
BUILD_DIR = PKG_DIR / "_build"
LIB_NAME = "libivrq_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "-DIVRQ_BUILD",
    f"-I{INCLUDE}",
]


def _nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libivrq_b200.so")
    return cand


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


BUILDINFO = LIB_PATH.with_name(LIB_PATH.name + ".buildinfo")  # travels with the library


def _source_digest(extra_flags: list[str] | None = None) -> str:
    """sha256 of the nvcc flags and every source, header and this script: what the library is built from."""
    import hashlib

    flags = [f.replace(str(INCLUDE), "<include>") for f in ARCH_FLAGS + NVCC_FLAGS + list(extra_flags or [])]
    h = hashlib.sha256(" ".join(flags).encode())  # location independent: the repo root differs per machine
    for p in _sources() + _headers() + [Path(__file__)]:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def needs_build(extra_flags: list[str] | None = None) -> bool:
    """Whether libivrq_b200.so is missing or was built from other sources / flags.

    Decided by content (the digest recorded beside the library), not by file times: a
    snapshot of the repo copied to another machine may not keep the files' mtimes."""
    if not LIB_PATH.exists():
        return True
    if BUILDINFO.exists():
        return BUILDINFO.read_text().strip() != _source_digest(extra_flags)
    lib_m = LIB_PATH.stat().st_mtime
    deps = _sources() + _headers() + [Path(__file__)]
    return any(p.stat().st_mtime > lib_m for p in deps)


def build(force: bool = False, verbose: bool = False, extra_flags: list[str] | None = None) -> Path:
    """Compile every ``csrc/*.cu`` for sm_100a and link ``libivrq_b200.so``."""
    if not force and not needs_build(extra_flags):
        return LIB_PATH
    nvcc = _nvcc()
    BUILD_DIR.mkdir(exist_ok=True)
    flags = ARCH_FLAGS + NVCC_FLAGS + list(extra_flags or [])
    srcs = _sources()
    hdr_m = max((p.stat().st_mtime for p in _headers()), default=0.0)
    # cached objects are reused only when they were compiled with these exact flags (a variant
    # build with -D switches must never leave its objects behind for the next default build)
    stamp = BUILD_DIR / "flags.txt"
    if not stamp.exists() or stamp.read_text() != " ".join(flags):
        force = True
        stamp.unlink(missing_ok=True)  # rewritten once every object has been compiled with these flags

    def compile_one(src: Path) -> Path:
        obj = BUILD_DIR / (src.stem + ".o")
        if (
            not force
            and obj.exists()
            and obj.stat().st_mtime > max(src.stat().st_mtime, hdr_m, Path(__file__).stat().st_mtime)
        ):
            return obj
        cmd = [nvcc, *flags, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stderr}")
        if verbose and res.stderr:
            print(res.stderr, file=sys.stderr)
        return obj

    workers = max(1, min(len(srcs), os.cpu_count() or 1))
    with concurrent.futures.ThreadPoolExecutor(max_workers=workers) as ex:
        objs = list(ex.map(compile_one, srcs))
    stamp.write_text(" ".join(flags))
    tmp = LIB_PATH.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH_FLAGS, "-shared", "-cudart", "static", "-o", str(tmp), *map(str, objs)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{res.stderr}")
    os.replace(tmp, LIB_PATH)
    BUILDINFO.write_text(_source_digest(extra_flags) + "\n")
    return LIB_PATH


if __name__ == "__main__":
    force = "--force" in sys.argv
    print(build(force=force, verbose="-v" in sys.argv))
