"""Builds the native libraries in-tree (they travel to the GPU box with the
repo snapshot):

* ``libpbg.so``      — the sm_100a kernels + C-ABI (include/pbg.h), nvcc;
* ``libpbg_host.so`` — host input preparation (include/pbg_host.h), g++/OpenMP;
* ``libspgemm_b200.so`` — the C++ drop-in ``spgemm::pb_multiply`` over the
  C-ABI (include/spgemm_b200/pb_spgemm.hpp);
* ``libpbg_checked.so`` — libpbg with PBG_CHECKED device bounds checks (trap
  on an out-of-range store index), run by tests/test_gpu_checked.py in place
  of compute-sanitizer memcheck, which the GPU pool does not run.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]

LIBPBG = PKG / "libpbg.so"
LIBHOST = PKG / "libpbg_host.so"
LIBSHIM = PKG / "libspgemm_b200.so"
LIBCHECKED = PKG / "libpbg_checked.so"


def _newer(target: Path, deps) -> bool:
    if not target.exists():
        return False
    t = target.stat().st_mtime
    return all(Path(d).stat().st_mtime <= t for d in deps)


def _run(cmd):
    print("+", " ".join(str(c) for c in cmd), file=sys.stderr)
    subprocess.run([str(c) for c in cmd], check=True)


def _build_cu(target: Path, defines, force: bool) -> Path:
    deps = [CSRC / "pbg.cu", *sorted(CSRC.glob("*.cuh")), INCLUDE / "pbg.h"]
    if force or not _newer(target, deps):
        tmp = target.with_suffix(".so.tmp")
        _run([NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-Wall", "-shared", *defines, "-I", INCLUDE, "-I", CSRC,
              "-o", tmp, CSRC / "pbg.cu", "-lcudart"])
        tmp.replace(target)
    return target


def build_pbg(force: bool = False) -> Path:
    return _build_cu(LIBPBG, [], force)


def build_checked(force: bool = False) -> Path:
    return _build_cu(LIBCHECKED, ["-DPBG_CHECKED"], force)


def build_host(force: bool = False) -> Path:
    deps = [CSRC / "pbg_host.cpp", INCLUDE / "pbg_host.h"]
    if force or not _newer(LIBHOST, deps):
        tmp = LIBHOST.with_suffix(".so.tmp")
        _run(["g++", "-std=c++17", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared",
              "-Wall", "-I", INCLUDE, "-o", tmp, CSRC / "pbg_host.cpp"])
        tmp.replace(LIBHOST)
    return LIBHOST


def build_shim(force: bool = False) -> Path:
    deps = [CSRC / "pb_spgemm_shim.cpp", *sorted((INCLUDE / "spgemm_b200").glob("*.hpp")),
            INCLUDE / "pbg.h", INCLUDE / "pbg_host.h", LIBPBG, LIBHOST]
    if force or not _newer(LIBSHIM, deps):
        tmp = LIBSHIM.with_suffix(".so.tmp")
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-I", INCLUDE,
              "-o", tmp, CSRC / "pb_spgemm_shim.cpp", "-L", PKG, "-lpbg", "-l:libpbg_host.so",
              f"-Wl,-rpath,$ORIGIN"])
        tmp.replace(LIBSHIM)
    return LIBSHIM


def build_all(force: bool = False) -> None:
    import threading
    build_host(force)
    # the checked variant compiles alongside the product library
    errs = []
    t = threading.Thread(target=lambda: _catch(errs, build_checked, force))
    t.start()
    build_pbg(force)
    t.join()
    if errs:
        raise errs[0]
    build_shim(force)


def _catch(errs, fn, *args):
    try:
        fn(*args)
    except Exception as e:  # re-raised by the caller's thread
        errs.append(e)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
