"""The C-ABI boundary: libraries load, export every declared symbol, and keep
the reference's error contract even without a GPU (no CPU fallback)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2002_11302_b200 import _native, api, build, matrices as M

ROOT = Path(__file__).resolve().parents[1]


def declared(header: str, prefix: str):
    text = (ROOT / "include" / header).read_text()
    return sorted(set(re.findall(rf"\b({prefix}[a-z0-9_]+)\s*\(", text)))


def test_libpbg_exports_every_declared_symbol():
    build.build_pbg()
    lib = C.CDLL(str(build.LIBPBG))
    names = declared("pbg.h", "pbg_")
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(_native.PBG_EXPORTS), "ctypes table misses a symbol"


def test_libpbg_host_exports_every_declared_symbol():
    lib = C.CDLL(str(build.build_host()))
    for n in declared("pbg_host.h", "pbgh_"):
        assert hasattr(lib, n), n


def test_kernels_are_sm100a_with_tma():
    """The product .so carries sm_100a SASS, and the sort kernel stages bins
    with TMA bulk copies (UBLKCP)."""
    so = build.build_pbg()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(so)],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    for k in ("k_expand", "k_sortmerge", "k_bincount", "k_scan"):
        assert k in out, k
    assert "UBLKCP" in out


def test_choose_nbins_matches_reference_rule():
    lib = _native.pbg()
    assert lib.pbg_choose_nbins(16 << 20, 1 << 20, 1 << 20, 12) == 512
    assert lib.pbg_choose_nbins(0, 1 << 20, 1 << 20, 12) == 64
    assert lib.pbg_choose_nbins(0, 10, 1 << 20, 12) == 8
    assert lib.pbg_choose_nbins(1 << 40, 1 << 30, 1 << 20, 12) == 8192


def _eye(n):
    csr = M.coo_to_csr(n, n, np.arange(n), np.arange(n))
    return M.csr_to_csc(csr), csr


def test_parameter_errors_before_device():
    a, b = _eye(4)
    bad = M.CscMatrix(4, 3, np.zeros(4, np.uint64), np.zeros(0, np.uint32), np.zeros(0))
    with pytest.raises(api.ParameterError, match="dimension mismatch"):
        api.pb_multiply(bad, b)
    with pytest.raises(api.ParameterError, match="power of two"):
        api.pb_multiply(a, b, api.PbConfig(nbins=3))
    with pytest.raises(api.ParameterError, match="multiple of 16"):
        api.pb_multiply(a, b, api.PbConfig(lbin_bytes=24))


@pytest.mark.skipif(api.device_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    a, b = _eye(8)
    with pytest.raises(api.DeviceError, match="no CUDA device"):
        api.pb_multiply(a, b)


def test_cpp_dropin_compiles_and_keeps_error_contract(tmp_path):
    shim = build.build_shim()
    exe = tmp_path / "dropin_test"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "dropin_test.cpp"), "-L", str(shim.parent),
                    "-lspgemm_b200", f"-Wl,-rpath,{shim.parent}", "-o", str(exe)], check=True)
    if not api.device_available():
        r = subprocess.run([str(exe), "nodevice"], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr


def _build_report_test(tmp_path):
    shim = build.build_shim()
    exe = tmp_path / "report_test"
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "report_test.cpp"), "-L", str(shim.parent),
                    "-lspgemm_b200", f"-Wl,-rpath,{shim.parent}", "-o", str(exe)], check=True)
    return exe


def test_cpp_report_roofline_headers(tmp_path):
    """report.hpp / roofline.hpp / validate(): the reference's measurement
    callers compile against include/spgemm_b200 and the roofline KATs of
    test_roofline.cpp hold (no device needed for these)."""
    exe = _build_report_test(tmp_path)
    if not api.device_available():
        r = subprocess.run([str(exe), "nodevice"], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_report_run_once_on_gpu(tmp_path):
    exe = _build_report_test(tmp_path)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_hash_multiply_rejects_wrong_types_before_native_views():
    a_csr = M.make_matrix("er", 6, 2, 1)
    a = M.csr_to_csc(a_csr)
    with pytest.raises(TypeError):
        api.hash_multiply(a_csr, a)  # CSR left operand
    with pytest.raises(TypeError):
        api.hash_multiply(a, a_csr)  # CSR right operand
    bad = M.CscMatrix(a.nrows, a.ncols, a.colptr, a.rowids.astype(np.int64), a.values)
    with pytest.raises(TypeError):
        api.hash_multiply(bad, a)
    with pytest.raises(TypeError):
        api.pb_multiply(a_csr, a_csr)
