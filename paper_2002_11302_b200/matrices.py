"""Sparse matrix containers and benchmark inputs.

``CscMatrix`` / ``CsrMatrix`` mirror the reference's types
(proj/include/spgemm/types.hpp:51-69): u64 pointer arrays, u32 indices, f64
values, held as numpy arrays. Generators and conversions run in
``libpbg_host.so`` (C++/OpenMP) and follow the reference's algorithms
(proj/src/generate.cpp:20-90, proj/src/convert.cpp:41-98).

The benchmark configs (BASELINE.json ``configs``) square one
matrix, C = A·A, with A passed as CSC (left) and CSR (right):

====  ====================  ===========================================
name  config                 structure
====  ====================  ===========================================
C1    ER 2^16, d=4           gen_er(16, 4, seed) + U[0,1) values
C2    ER 2^20, d=16          gen_er(20, 16, seed) + U[0,1)
C3    RMAT s20 ef16          gen_rmat(20, 16, seed) minus self-loops + U[0,1)
C4    27-pt stencil 128^3    26 on the diagonal, -1 off it
C5a   ER 2^24, d=8           gen_er(24, 8, seed) + U[0,1)
C5b   RMAT s24 ef8           gen_rmat(24, 8, seed) minus self-loops + U[0,1)
====  ====================  ===========================================
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native

VALUE_SEED_XOR = 0x5EED5EED5EED5EED
RMAT_ABC = (0.57, 0.19, 0.19)  # Graph500 (generate.hpp:55-57); d = 0.05


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


@dataclass
class CscMatrix:
    nrows: int
    ncols: int
    colptr: np.ndarray  # u64 [ncols+1]
    rowids: np.ndarray  # u32 [nnz]
    values: np.ndarray  # f64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.rowids.size)


@dataclass
class CsrMatrix:
    nrows: int
    ncols: int
    rowptr: np.ndarray  # u64 [nrows+1]
    colids: np.ndarray  # u32 [nnz]
    values: np.ndarray  # f64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.colids.size)


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise ValueError(f"{what} failed (code {rc})")


def coo_to_csr(nrows: int, ncols: int, rows, cols, vals=None, combine: str = "sum",
               drop_diag: bool = False) -> CsrMatrix:
    """COO -> CSR. ``combine='sum'`` sums duplicates (coo_to_csr,
    convert.cpp:41-70); ``'collapse'`` keeps one entry of value 1.0 per
    (row, col) like gen_rmat's dedup (generate.cpp:83-88)."""
    rows = np.ascontiguousarray(rows, dtype=np.uint32)
    cols = np.ascontiguousarray(cols, dtype=np.uint32)
    nnz = rows.size
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.float64)
    rowptr = np.zeros(nrows + 1, dtype=np.uint64)
    colids = np.empty(max(nnz, 1), dtype=np.uint32)
    values = np.empty(max(nnz, 1), dtype=np.float64)
    out = C.c_uint64(0)
    rc = _native.host().pbgh_coo_to_csr(nrows, ncols, nnz, _p(rows), _p(cols), _p(v),
                                        1 if combine == "collapse" else 0, int(drop_diag),
                                        _p(rowptr), _p(colids), _p(values), C.byref(out))
    _check(rc, "coo_to_csr")
    k = out.value
    return CsrMatrix(nrows, ncols, rowptr, colids[:k].copy(), values[:k].copy())


def coo_to_csc(nrows: int, ncols: int, rows, cols, vals=None) -> CscMatrix:
    """COO -> CSC with duplicates summed (coo_to_csc, convert.cpp:82-89)."""
    return csr_to_csc(coo_to_csr(nrows, ncols, rows, cols, vals))


def csr_to_csc(m: CsrMatrix) -> CscMatrix:
    colptr = np.zeros(m.ncols + 1, dtype=np.uint64)
    rowids = np.empty(max(m.nnz, 1), dtype=np.uint32)
    values = np.empty(max(m.nnz, 1), dtype=np.float64)
    rc = _native.host().pbgh_csr_to_csc(m.nrows, m.ncols, _p(m.rowptr), _p(m.colids),
                                        _p(m.values), _p(colptr), _p(rowids), _p(values))
    _check(rc, "csr_to_csc")
    return CscMatrix(m.nrows, m.ncols, colptr, rowids[:m.nnz].copy(), values[:m.nnz].copy())


def csc_to_csr(m: CscMatrix) -> CsrMatrix:
    # the CSC of M is the CSR of M^T; transposing back gives the CSR of M
    t = csr_to_csc(CsrMatrix(m.ncols, m.nrows, m.colptr, m.rowids, m.values))
    return CsrMatrix(m.nrows, m.ncols, t.colptr, t.rowids, t.values)


def gen_er(scale: int, d: int, seed: int):
    """gen_er draws (generate.cpp:20-54): exactly d distinct rows per column."""
    n = 1 << scale
    rows = np.empty(n * d, dtype=np.uint32)
    cols = np.empty(n * d, dtype=np.uint32)
    _check(_native.host().pbgh_gen_er(scale, d, seed, _p(rows), _p(cols)), "gen_er")
    return rows, cols


def gen_rmat(scale: int, ef: int, seed: int, abc=RMAT_ABC):
    """gen_rmat quadrant-descent draws before dedup (generate.cpp:56-81)."""
    ne = ef << scale
    rows = np.empty(ne, dtype=np.uint32)
    cols = np.empty(ne, dtype=np.uint32)
    _check(_native.host().pbgh_gen_rmat(scale, ef, seed, abc[0], abc[1], abc[2],
                                        _p(rows), _p(cols)), "gen_rmat")
    return rows, cols


def fill_values(m: CsrMatrix, vseed: int) -> CsrMatrix:
    """U[0,1) value per (row, col): SplitMix64(split_seed(vseed, row<<32|col))
    .next_unit() (generate.hpp:35-40). Order-independent, so
    the CSC and CSR copies of A carry identical values."""
    _check(_native.host().pbgh_csr_fill_values(vseed, m.nrows, _p(m.rowptr), _p(m.colids),
                                               _p(m.values)), "fill_values")
    return m


def stencil27(nx: int, ny: int | None = None, nz: int | None = None) -> CsrMatrix:
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    out = C.c_uint64(0)
    h = _native.host()
    _check(h.pbgh_stencil27(nx, ny, nz, None, None, None, C.byref(out)), "stencil27")
    n = nx * ny * nz
    rowptr = np.zeros(n + 1, dtype=np.uint64)
    colids = np.empty(out.value, dtype=np.uint32)
    values = np.empty(out.value, dtype=np.float64)
    _check(h.pbgh_stencil27(nx, ny, nz, _p(rowptr), _p(colids), _p(values), C.byref(out)),
           "stencil27")
    return CsrMatrix(n, n, rowptr, colids, values)


def row_band(a: CscMatrix, r0: int, r1: int) -> CscMatrix:
    """Rows [r0, r1) of CSC A as a (r1-r0) x ncols CSC (rows renumbered)."""
    h = _native.host()
    out = C.c_uint64(0)
    _check(h.pbgh_csc_row_band(a.nrows, a.ncols, _p(a.colptr), _p(a.rowids), _p(a.values),
                               r0, r1, None, None, None, C.byref(out)), "row_band")
    colptr = np.zeros(a.ncols + 1, dtype=np.uint64)
    rowids = np.empty(max(out.value, 1), dtype=np.uint32)
    values = np.empty(max(out.value, 1), dtype=np.float64)
    _check(h.pbgh_csc_row_band(a.nrows, a.ncols, _p(a.colptr), _p(a.rowids), _p(a.values),
                               r0, r1, _p(colptr), _p(rowids), _p(values), C.byref(out)),
           "row_band")
    k = out.value
    return CscMatrix(r1 - r0, a.ncols, colptr, rowids[:k].copy(), values[:k].copy())


def row_flop(a: CscMatrix, b: CsrMatrix) -> np.ndarray:
    rf = np.zeros(max(a.nrows, 1), dtype=np.uint64)
    _check(_native.host().pbgh_row_flop(a.nrows, a.ncols, _p(a.colptr), _p(a.rowids),
                                        _p(b.rowptr), _p(rf)), "row_flop")
    return rf[:a.nrows]


def band_cuts(row_flop_arr: np.ndarray, g: int) -> np.ndarray:
    """Flop-balanced cuts of the rows into g bands."""
    rf = np.ascontiguousarray(row_flop_arr, dtype=np.uint64)
    cuts = np.zeros(g + 1, dtype=np.uint32)
    _check(_native.host().pbgh_band_cuts(rf.size, _p(rf), g, _p(cuts)), "band_cuts")
    return cuts


CONFIGS = {
    "C1": ("er", 16, 4),
    "C2": ("er", 20, 16),
    "C3": ("rmat", 20, 16),
    "C4": ("stencil", 128, None),
    "C5a": ("er", 24, 8),
    "C5b": ("rmat", 24, 8),
    # scaled-down development configs (same generators)
    "R16": ("rmat", 16, 16),
    "R18": ("rmat", 18, 16),
    "S64": ("stencil", 64, None),
    "E22": ("er", 22, 8),
}

CONFIG_NAMES = {
    "C1": "ER n=2^16 d=4, C=A*A, fp64 U[0,1)",
    "C2": "ER n=2^20 d=16, C=A*A, fp64 U[0,1)",
    "C3": "RMAT scale 20 ef 16 (a,b,c,d=.57,.19,.19,.05, dedup, no self-loops), C=A*A, fp64 U[0,1)",
    "C4": "27-point stencil 128^3 (26 / -1), C=A*A",
    "C5a": "ER n=2^24 d=8, C=A*A, fp64 U[0,1)",
    "C5b": "RMAT scale 24 ef 8 (dedup, no self-loops), C=A*A, fp64 U[0,1)",
    "R16": "dev: RMAT scale 16 ef 16, C=A*A",
    "R18": "dev: RMAT scale 18 ef 16, C=A*A",
    "S64": "dev: 27-point stencil 64^3, C=A*A",
    "E22": "dev: ER n=2^22 d=8, C=A*A",
}


class ParseError(ValueError):
    """spgemm::parse_error (types.hpp:84): malformed Matrix Market input."""


def read_mtx(path):
    """Matrix Market coordinate file -> (nrows, ncols, rows, cols, vals), the
    semantics of mm_read (mmio.cpp:33-105): real/integer/pattern, general/
    symmetric (expanded, mirror right after its source), pattern -> 1.0,
    0-based, file order. Parsed by the native host library."""
    lib = _native.host()
    h = C.c_void_p()
    nr, nc, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
    rc = lib.pbgh_mm_open(str(path).encode(), C.byref(h), C.byref(nr), C.byref(nc), C.byref(nnz))
    if rc:
        raise ParseError(lib.pbgh_last_error().decode())
    n = nnz.value
    rows = np.empty(n, np.uint32)
    cols = np.empty(n, np.uint32)
    vals = np.empty(n, np.float64)
    lib.pbgh_mm_fetch(h, _p(rows), _p(cols), _p(vals))
    lib.pbgh_mm_free(h)
    return nr.value, nc.value, rows, cols, vals


def write_mtx(path, nrows: int, ncols: int, rows, cols, vals=None) -> None:
    """mm_write (mmio.cpp:107-117): coordinate real general, %.17g values."""
    r = np.ascontiguousarray(rows, np.uint32)
    c = np.ascontiguousarray(cols, np.uint32)
    v = np.ascontiguousarray(np.ones(r.size) if vals is None else vals, np.float64)
    _check(_native.host().pbgh_mm_write(str(path).encode(), nrows, ncols, r.size, _p(r), _p(c),
                                        _p(v)), "pbgh_mm_write")


def matrix_from_mtx(path) -> CsrMatrix:
    """A Matrix Market file as CSR (duplicates summed, coo_to_csr), the
    reference bench's --matrix input (spgemm_bench.cpp:55-58)."""
    nr, nc, r, c, v = read_mtx(path)
    return coo_to_csr(nr, nc, r, c, v)


def make_matrix(kind: str, scale: int, ef: int | None, seed: int = 1) -> CsrMatrix:
    """One square input matrix in CSR (values included)."""
    vseed = seed ^ VALUE_SEED_XOR
    if kind == "er":
        r, c = gen_er(scale, ef, seed)
        m = coo_to_csr(1 << scale, 1 << scale, r, c)
        return fill_values(m, vseed)
    if kind == "rmat":
        r, c = gen_rmat(scale, ef, seed)
        m = coo_to_csr(1 << scale, 1 << scale, r, c, combine="collapse", drop_diag=True)
        return fill_values(m, vseed)
    if kind == "stencil":
        return stencil27(scale)
    raise ValueError(kind)


def _generate_gpu(kind: str, scale: int, ef: int, seed: int, to_csc: bool, device: int = 0):
    from . import api  # local: api imports this module
    lib = _native.pbg()
    h, nnz = C.c_void_p(), C.c_uint64(0)
    cfg = api.PbConfig(device=device).to_c()
    rc = lib.pbg_generate_begin(0 if kind == "er" else 1, scale, ef, seed, seed ^ VALUE_SEED_XOR,
                                int(to_csc), C.byref(cfg), C.byref(h), C.byref(nnz))
    if rc:
        api._raise(rc)
    try:
        n, k = 1 << scale, nnz.value
        ptr = np.empty(n + 1, np.uint64)
        idx = np.empty(max(k, 1), np.uint32)
        val = np.empty(max(k, 1), np.float64)
        rc = lib.pbg_multiply_fetch(h, ptr.ctypes.data, idx.ctypes.data, val.ctypes.data, None)
        if rc:
            api._raise(rc)
    finally:
        lib.pbg_release(h)
    if to_csc:
        return CscMatrix(n, n, ptr, idx[:k], val[:k])
    return CsrMatrix(n, n, ptr, idx[:k], val[:k])


def make_config_gpu(name: str, seed: int = 1, device: int = 0):
    """make_config with the ER / RMAT generators and both conversions run on
    the GPU (pbg_generate_begin); identical arrays, seconds faster at C5.
    The stencil (no RNG) is built on the host."""
    kind, scale, ef = CONFIGS[name]
    if kind == "stencil":
        return make_config(name, seed)
    return (_generate_gpu(kind, scale, ef, seed, True, device),
            _generate_gpu(kind, scale, ef, seed, False, device))


def make_config(name: str, seed: int = 1):
    """(A_csc, A_csr) of a benchmark config; the product is A_csc * A_csr."""
    kind, scale, ef = CONFIGS[name]
    csr = make_matrix(kind, scale, ef, seed)
    return csr_to_csc(csr), csr
