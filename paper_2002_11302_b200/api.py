"""Python mirror of the reference's PB-SpGEMM entry point.

``pb_multiply(a_csc, b_csr, cfg)`` has the meaning, arguments and error
behaviour of ``spgemm::pb_multiply`` (proj/include/spgemm/pb_spgemm.hpp:116,
proj/src/pb_spgemm.cpp:330-361), computed on the B200 through the C-ABI
(include/pbg.h). ``ParameterError`` / ``InternalError`` stand for the
reference's ``parameter_error`` / ``internal_error`` (types.hpp:80-91).

``DeviceContext`` is the device-resident path the benchmark times: inputs
already in HBM (torch tensors as plumbing), one multiply per call.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .matrices import CscMatrix, CsrMatrix


class ParameterError(ValueError):
    """spgemm::parameter_error (types.hpp:80-83)."""


class InternalError(RuntimeError):
    """spgemm::internal_error (types.hpp:89-91)."""


class DeviceError(RuntimeError):
    """CUDA failure or no device (the GPU path has no CPU fallback)."""


def _raise(rc: int):
    msg = _native.last_error()
    if rc in (_native.PBG_ERR_DIM, _native.PBG_ERR_NBINS, _native.PBG_ERR_LBIN,
              _native.PBG_ERR_FLOP_OVERFLOW):
        raise ParameterError(msg)
    if rc == _native.PBG_ERR_INTERNAL:
        raise InternalError(msg)
    if rc == _native.PBG_ERR_UNIMPLEMENTED:
        raise NotImplementedError(msg)
    raise DeviceError(f"[pbg {rc}] {msg}")


@dataclass
class PbConfig:
    """spgemm::PbConfig (pb_spgemm.hpp:11-17) + GPU fields."""
    nbins: int = 0
    lbin_bytes: int = 512
    l2_bytes: int = 1 << 20
    nthreads: int = 0
    balanced_bins: bool = False
    device: int = -1
    bin_cap: int = 0  # GPU shared-memory bin capacity in tuples (0 = 4096)
    max_round_tuples: int = 0  # host path: tuples per bounded-memory round (0 = from free HBM)
    expand_bands: int = 0  # row bands of the expand (0 = auto, 1 = one pass)
    ngpus: int = 0  # host path: devices to split C's rows over (0/1 = one, -1 = all)
    wrap_devices: bool = False  # test hook: more bands than devices wrap around them

    def to_c(self) -> _native.Config:
        c = _native.Config()
        _native.pbg().pbg_default_config(C.byref(c))
        c.nbins, c.lbin_bytes, c.l2_bytes = self.nbins, self.lbin_bytes, self.l2_bytes
        c.nthreads, c.balanced_bins = self.nthreads, int(self.balanced_bins)
        c.device, c.bin_cap = self.device, self.bin_cap
        c.reserved[0] = self.max_round_tuples
        c.reserved[1] = self.expand_bands
        c.ngpus = self.ngpus
        c.flags = _native.PBG_FLAG_WRAP_DEVICES if self.wrap_devices else 0
        return c


@dataclass
class SymbolicResult:
    """spgemm::SymbolicResult (pb_spgemm.hpp:48-55) on the reference bin layout."""
    flop: int = 0
    per_column_flop: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    nbins: int = 1
    per_bin_flop: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    bin_row_starts: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


@dataclass
class PbResult:
    c: CsrMatrix
    sym: SymbolicResult
    phases: dict
    tuples_into_sort: int
    merged_total: int
    report: dict


def _view(nrows, ncols, ptr, idx, val) -> _native.CsxView:
    v = _native.CsxView()
    v.nrows, v.ncols, v.nnz = nrows, ncols, int(idx.size)
    v.ptr = ptr.ctypes.data
    v.idx = idx.ctypes.data if idx.size else None
    v.val = val.ctypes.data if val.size else None
    return v


def _host_arrays(m):
    if isinstance(m, CscMatrix):
        return m.colptr, m.rowids, m.values
    return m.rowptr, m.colids, m.values


def _checked_arrays(a, b):
    """Host arrays of both operands with the reference's element types (u64
    pointers, u32 indices, f64 values); anything else is a TypeError before
    any native view is built."""
    ap, ai, av = (np.ascontiguousarray(x) for x in _host_arrays(a))
    bp, bi, bv = (np.ascontiguousarray(x) for x in _host_arrays(b))
    if ap.dtype != np.uint64 or bp.dtype != np.uint64 or ai.dtype != np.uint32 \
            or bi.dtype != np.uint32 or av.dtype != np.float64 or bv.dtype != np.float64:
        raise TypeError("expected u64 pointers, u32 indices, f64 values")
    return (ap, ai, av), (bp, bi, bv)


def pb_multiply(a: CscMatrix, b: CsrMatrix, cfg: PbConfig | None = None,
                symbolic: bool = True, out=None) -> PbResult:
    """C = A·B on the GPU, A in CSC, B in CSR, C in CSR (host buffers in/out).

    ``out`` = (rowptr, colids, values) caller-owned host arrays (e.g. pinned):
    C is written straight into them by pbg_multiply_into (row bands whose
    copies overlap the next band's multiply; no host staging, so products
    whose C exceeds HBM work too). The returned CsrMatrix views them."""
    cfg = cfg or PbConfig()
    lib = _native.pbg()
    if not isinstance(a, CscMatrix) or not isinstance(b, CsrMatrix):
        raise TypeError("pb_multiply takes A in CSC and B in CSR")
    (ap, ai, av), (bp, bi, bv) = _checked_arrays(a, b)
    va = _view(a.nrows, a.ncols, ap, ai, av)
    vb = _view(b.nrows, b.ncols, bp, bi, bv)
    c_cfg = cfg.to_c()
    if out is not None:
        rowptr, colids, values = out
        if rowptr.size < a.nrows + 1 or rowptr.dtype != np.uint64 or colids.dtype != np.uint32 \
                or values.dtype != np.float64 or colids.size != values.size:
            raise TypeError("out = (u64 rowptr[nrows+1], u32 colids[cap], f64 values[cap])")
        nnz = C.c_uint64(0)
        rep = _native.Report()
        rc = lib.pbg_multiply_into(C.byref(va), C.byref(vb), C.byref(c_cfg), rowptr.ctypes.data,
                                   colids.ctypes.data, values.ctypes.data, colids.size,
                                   C.byref(nnz), C.byref(rep))
        if rc:
            _raise(rc)
        k = nnz.value
        r = rep.as_dict()
        phases = {key: r[key] for key in ("t_symbolic", "t_expand", "t_sort", "t_compress",
                                          "t_convert", "t_total", "t_h2d", "t_d2h")}
        c = CsrMatrix(a.nrows, b.ncols, rowptr[:a.nrows + 1], colids[:k], values[:k])
        if c.nnz != rep.merged_total:
            raise InternalError("compressed counts disagree with output nnz")
        return PbResult(c, SymbolicResult(flop=rep.flop, nbins=rep.nbins), phases,
                        rep.tuples_into_sort, rep.merged_total, r)
    h = C.c_void_p()
    nnz = C.c_uint64(0)
    rc = lib.pbg_multiply_begin(C.byref(va), C.byref(vb), C.byref(c_cfg), C.byref(h), C.byref(nnz))
    if rc:
        _raise(rc)
    try:
        k = nnz.value
        rowptr = np.empty(a.nrows + 1, np.uint64)
        colids = np.empty(max(k, 1), np.uint32)
        values = np.empty(max(k, 1), np.float64)
        rep = _native.Report()
        rc = lib.pbg_multiply_fetch(h, rowptr.ctypes.data, colids.ctypes.data,
                                    values.ctypes.data, C.byref(rep))
        if rc:
            _raise(rc)
        sym = SymbolicResult(flop=rep.flop, nbins=rep.nbins)
        if symbolic:
            sym.per_column_flop = np.zeros(max(a.ncols, 1), np.uint64)
            sym.per_bin_flop = np.zeros(max(rep.nbins, 1), np.uint64)
            sym.bin_row_starts = np.zeros(rep.nbins + 1, np.uint32)
            rc = lib.pbg_symbolic_fetch(h, sym.per_column_flop.ctypes.data,
                                        sym.per_bin_flop.ctypes.data,
                                        sym.bin_row_starts.ctypes.data)
            if rc:
                _raise(rc)
            sym.per_column_flop = sym.per_column_flop[:a.ncols]
            sym.per_bin_flop = sym.per_bin_flop[:rep.nbins]
    finally:
        lib.pbg_release(h)
    r = rep.as_dict()
    phases = {key: r[key] for key in ("t_symbolic", "t_expand", "t_sort", "t_compress",
                                      "t_convert", "t_total", "t_h2d", "t_d2h")}
    c = CsrMatrix(a.nrows, b.ncols, rowptr[:a.nrows + 1], colids[:k], values[:k])
    if c.nnz != rep.merged_total:
        raise InternalError("compressed counts disagree with output nnz")
    return PbResult(c, sym, phases, rep.tuples_into_sort, rep.merged_total, r)


@dataclass
class HashResult:
    c: CscMatrix
    flop: int
    phases: dict


def hash_multiply(a: CscMatrix, b: CscMatrix, cfg: PbConfig | None = None) -> HashResult:
    """spgemm::hash_multiply (baseline.hpp:21-24, baseline.cpp:141-200) on the
    GPU: C = A·B, A, B and C in CSC — the column hash SpGEMM the paper finds
    faster than PB-SpGEMM above a compression factor of ~4 (SURVEY.md §8f
    f3). Hub columns of more than 4096 products (RMAT) are summed in a dense
    per-CTA accumulator in global memory instead of a shared-memory table."""
    cfg = cfg or PbConfig()
    lib = _native.pbg()
    if not isinstance(a, CscMatrix) or not isinstance(b, CscMatrix):
        raise TypeError("hash_multiply takes A and B in CSC")
    (ap, ai, av), (bp, bi, bv) = _checked_arrays(a, b)
    va = _view(a.nrows, a.ncols, ap, ai, av)
    vb = _view(b.nrows, b.ncols, bp, bi, bv)
    c_cfg = cfg.to_c()
    h = C.c_void_p()
    nnz = C.c_uint64(0)
    rc = lib.pbg_hash_multiply_begin(C.byref(va), C.byref(vb), C.byref(c_cfg), C.byref(h),
                                     C.byref(nnz))
    if rc:
        _raise(rc)
    try:
        k = nnz.value
        colptr = np.empty(b.ncols + 1, np.uint64)
        rowids = np.empty(max(k, 1), np.uint32)
        values = np.empty(max(k, 1), np.float64)
        rep = _native.Report()
        rc = lib.pbg_multiply_fetch(h, colptr.ctypes.data, rowids.ctypes.data,
                                    values.ctypes.data, C.byref(rep))
        if rc:
            _raise(rc)
    finally:
        lib.pbg_release(h)
    r = rep.as_dict()
    phases = {key: r[key] for key in ("t_symbolic", "t_sort", "t_total", "t_h2d", "t_d2h")}
    return HashResult(CscMatrix(a.nrows, b.ncols, colptr, rowids[:k], values[:k]), rep.flop, phases)


def _coo_convert(nrows, ncols, rows, cols, vals, to_csc, cfg):
    cfg = cfg or PbConfig()
    lib = _native.pbg()
    r = np.ascontiguousarray(rows, dtype=np.uint32)
    c = np.ascontiguousarray(cols, dtype=np.uint32)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    if not (r.size == c.size == v.size):
        raise ValueError("rows, cols and vals must have one entry each")
    nz = r.size
    h = C.c_void_p()
    out_nnz = C.c_uint64(0)
    c_cfg = cfg.to_c()
    p = lambda a: a.ctypes.data if a.size else None  # noqa: E731
    rc = lib.pbg_coo_convert_begin(nrows, ncols, nz, p(r), p(c), p(v), int(to_csc),
                                   C.byref(c_cfg), C.byref(h), C.byref(out_nnz))
    if rc:
        if rc == _native.PBG_ERR_ARG:
            raise ValueError(_native.last_error())
        _raise(rc)
    try:
        k = out_nnz.value
        nmajor = ncols if to_csc else nrows
        ptr = np.empty(nmajor + 1, np.uint64)
        idx = np.empty(max(k, 1), np.uint32)
        val = np.empty(max(k, 1), np.float64)
        rc = lib.pbg_multiply_fetch(h, ptr.ctypes.data, idx.ctypes.data, val.ctypes.data, None)
        if rc:
            _raise(rc)
    finally:
        lib.pbg_release(h)
    if to_csc:
        return CscMatrix(nrows, ncols, ptr, idx[:k], val[:k])
    return CsrMatrix(nrows, ncols, ptr, idx[:k], val[:k])


def coo_to_csr(nrows: int, ncols: int, rows, cols, vals, cfg: PbConfig | None = None) -> CsrMatrix:
    """coo_to_csr (convert.cpp:41-70, duplicates summed, columns sorted) on the
    GPU, run as the product of a one-entry-per-column CSC with a
    one-entry-per-row CSR through the same pipeline as pb_multiply."""
    return _coo_convert(nrows, ncols, rows, cols, vals, False, cfg)


def coo_to_csc(nrows: int, ncols: int, rows, cols, vals, cfg: PbConfig | None = None) -> CscMatrix:
    """coo_to_csc (convert.cpp:82-89) on the GPU (see coo_to_csr)."""
    return _coo_convert(nrows, ncols, rows, cols, vals, True, cfg)


class DeviceContext:
    """Device-resident multiply: views over CUDA memory (e.g. torch tensors)."""

    def __init__(self, device: int = 0):
        self._lib = _native.pbg()
        self._ctx = C.c_void_p()
        rc = self._lib.pbg_context_create(device, C.byref(self._ctx))
        if rc:
            _raise(rc)
        self.device = device

    def close(self):
        if self._ctx:
            self._lib.pbg_context_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def view(nrows: int, ncols: int, ptr, idx, val) -> _native.CsxView:
        """View over torch CUDA tensors (u64-as-int64 ptr, u32-as-int32 idx, f64 val)."""
        v = _native.CsxView()
        v.nrows, v.ncols, v.nnz = nrows, ncols, int(idx.numel())
        v.ptr, v.idx, v.val = ptr.data_ptr(), idx.data_ptr() or None, val.data_ptr() or None
        return v

    def multiply(self, a_view, b_view, cfg: PbConfig | None = None, stream: int = 0):
        cfg = cfg or PbConfig()
        c_cfg = cfg.to_c()
        nnz = C.c_uint64(0)
        rep = _native.Report()
        rc = self._lib.pbg_multiply_device(self._ctx, C.byref(a_view), C.byref(b_view),
                                           C.byref(c_cfg), C.c_void_p(stream or None),
                                           C.byref(nnz), C.byref(rep))
        if rc:
            _raise(rc)
        return nnz.value, rep.as_dict()

    def band_cuts(self, a_view, b_view, nbands: int, stream: int = 0, rows=None):
        """Flop-balanced cuts of rows [r0, r1) (default: all) of A*B into
        nbands bands, computed on the device (balanced_starts rule,
        pb_spgemm.cpp:58-82): (cuts, flop of the rows)."""
        r0, r1 = rows or (0, a_view.nrows)
        cuts = np.zeros(nbands + 1, np.uint32)
        flop = C.c_uint64(0)
        rc = self._lib.pbg_band_cuts_device(self._ctx, C.byref(a_view), C.byref(b_view), r0, r1,
                                            nbands, C.c_void_p(stream or None), cuts.ctypes.data,
                                            C.byref(flop))
        if rc:
            _raise(rc)
        return cuts, flop.value

    def row_slab(self, a_view, r0: int, r1: int, stream: int = 0):
        """A(r0:r1, :) as a CSC (rows renumbered) built on the device: torch
        tensors (colptr int64, rowids int32, values float64) and its view."""
        import torch
        nnz = C.c_uint64(0)
        s = C.c_void_p(stream or None)
        rc = self._lib.pbg_row_slab_device(self._ctx, C.byref(a_view), r0, r1, s, None, None,
                                           None, 0, C.byref(nnz))
        if rc:
            _raise(rc)
        dev = torch.device("cuda", self.device)
        k = nnz.value
        cp = torch.empty(a_view.ncols + 1, dtype=torch.int64, device=dev)
        ri = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
        vv = torch.empty(max(k, 1), dtype=torch.float64, device=dev)
        rc = self._lib.pbg_row_slab_device(self._ctx, C.byref(a_view), r0, r1, s, cp.data_ptr(),
                                           ri.data_ptr(), vv.data_ptr(), k, C.byref(nnz))
        if rc:
            _raise(rc)
        ri, vv = ri[:k], vv[:k]
        return (cp, ri, vv), self.view(r1 - r0, a_view.ncols, cp, ri, vv)

    def multiply_band(self, a_view, b_view, r0: int, r1: int, cfg: PbConfig | None = None,
                      stream: int = 0):
        """C(r0:r1, :) = A(r0:r1, :)·B with the row slab of the device-resident
        A extracted on the device; the band's CSR (r1 - r0 rows) stays in the
        context (result_pointers)."""
        cfg = cfg or PbConfig()
        c_cfg = cfg.to_c()
        nnz = C.c_uint64(0)
        rep = _native.Report()
        rc = self._lib.pbg_multiply_device_band(self._ctx, C.byref(a_view), C.byref(b_view), r0, r1,
                                                C.byref(c_cfg), C.c_void_p(stream or None),
                                                C.byref(nnz), C.byref(rep))
        if rc:
            _raise(rc)
        return nnz.value, rep.as_dict()

    def checksum(self, row_base: int = 0, stream: int = 0):
        """(nnz, row hash, (row, col) hash, value sum) of the last product; the
        hashes are sums, so the bands of a product add up to its checksum."""
        out = np.zeros(3, np.uint64)
        vs = C.c_double(0)
        rc = self._lib.pbg_context_checksum(self._ctx, row_base, C.c_void_p(stream or None),
                                            out.ctypes.data, C.byref(vs))
        if rc:
            _raise(rc)
        return int(out[0]), int(out[1]), int(out[2]), vs.value

    def workbins(self):
        """Development aid: (tuples, key bits, flags, distinct keys) arrays of
        the last product's work bins (the sort kernel's units of work)."""
        nw = C.c_uint64(0)
        rc = self._lib.pbg_context_workbins(self._ctx, 0, C.byref(nw), None, None, None, None)
        if rc:
            _raise(rc)
        c = nw.value
        n, nnz = np.zeros(c, np.uint64), np.zeros(c, np.uint64)
        kb, fl = np.zeros(c, np.uint32), np.zeros(c, np.uint32)
        rc = self._lib.pbg_context_workbins(self._ctx, c, C.byref(nw), n.ctypes.data, kb.ctypes.data,
                                            fl.ctypes.data, nnz.ctypes.data)
        if rc:
            _raise(rc)
        return n, kb, fl, nnz

    def result_pointers(self):
        rp, ci, va = C.c_void_p(), C.c_void_p(), C.c_void_p()
        rc = self._lib.pbg_context_result(self._ctx, C.byref(rp), C.byref(ci), C.byref(va))
        if rc:
            _raise(rc)
        return rp.value, ci.value, va.value

    def launches(self) -> int:
        return int(self._lib.pbg_context_launches(self._ctx))


def device_available() -> bool:
    return bool(_native.pbg().pbg_device_available())
