"""Host input preparation (libpbg_host.so) against the reference.

Generators must reproduce the reference's gen_er / gen_rmat draws exactly
(golden pins), conversions follow coo_to_csr's duplicate-summing semantics,
and the benchmark-only inputs (stencil, self-loop removal, row bands) have
the structural properties the configs need.
"""
import numpy as np
import pytest

from paper_2002_11302_b200 import bands, matrices as M

from helpers import assert_valid_csr, golden_generators


@pytest.mark.parametrize("gen", golden_generators(), ids=lambda g: f"{g[0]['kind']}{g[0]['scale']}")
def test_generators_match_reference(gen):
    meta, rows, cols = gen
    if meta["kind"] == "er":
        r, c = M.gen_er(meta["scale"], meta["ef"], meta["seed"])
        assert np.array_equal(r, rows) and np.array_equal(c, cols)
    else:
        r, c = M.gen_rmat(meta["scale"], meta["ef"], meta["seed"])
        # the reference returns the sorted, deduplicated list (generate.cpp:83-88)
        csr = M.coo_to_csr(1 << meta["scale"], 1 << meta["scale"], r, c, combine="collapse")
        rr = np.repeat(np.arange(csr.nrows, dtype=np.uint32), np.diff(csr.rowptr).astype(np.int64))
        assert np.array_equal(rr, rows) and np.array_equal(csr.colids, cols)
        assert np.all(csr.values == 1.0)


def test_er_exact_degree():
    # test_sparse_core.cpp: exactly d distinct rows per column
    r, c = M.gen_er(12, 4, 5)
    csc = M.coo_to_csc(1 << 12, 1 << 12, r, c)
    assert np.all(np.diff(csc.colptr) == 4)


def test_coo_to_csr_sums_duplicates():
    m = M.coo_to_csr(3, 3, [2, 0, 2, 0], [1, 2, 1, 0], [1.0, 2.0, 3.0, 4.0])
    assert list(m.rowptr) == [0, 2, 2, 3]
    assert list(m.colids) == [0, 2, 1]
    assert list(m.values) == [4.0, 2.0, 4.0]


def test_collapse_and_drop_diag():
    m = M.coo_to_csr(3, 3, [1, 1, 0, 2], [1, 2, 0, 2], [5.0, 6.0, 7.0, 8.0],
                     combine="collapse", drop_diag=True)
    assert list(m.rowptr) == [0, 0, 1, 1] and list(m.colids) == [2]
    assert list(m.values) == [1.0]


def test_out_of_range_rejected():
    with pytest.raises(ValueError):
        M.coo_to_csr(2, 2, [2], [0])


def test_csr_csc_roundtrip():
    r, c = M.gen_rmat(9, 6, 11)
    csr = M.fill_values(M.coo_to_csr(512, 512, r, c, combine="collapse"), 3)
    csc = M.csr_to_csc(csr)
    back = M.csc_to_csr(csc)
    assert np.array_equal(back.rowptr, csr.rowptr)
    assert np.array_equal(back.colids, csr.colids)
    assert np.array_equal(back.values, csr.values)
    assert_valid_csr(csr)


def test_values_order_independent():
    # the CSC and CSR copies of A carry identical values (value is f(row, col))
    csr = M.make_matrix("er", 8, 4, seed=9)
    csc = M.csr_to_csc(csr)
    for j in (0, 17, 255):
        for p in range(int(csc.colptr[j]), int(csc.colptr[j + 1])):
            i = int(csc.rowids[p])
            lo, hi = int(csr.rowptr[i]), int(csr.rowptr[i + 1])
            q = lo + int(np.searchsorted(csr.colids[lo:hi], j))
            assert csr.values[q] == csc.values[p]


def test_stencil27():
    s = M.stencil27(5)
    n = 125
    assert s.nrows == n and s.nnz == (3 * 5 - 2) ** 3  # 13^3 interior-truncated count
    assert_valid_csr(s)
    # symmetric pattern, 26 on the diagonal, -1 elsewhere
    dense = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(s.rowptr).astype(np.int64))
    dense[rows, s.colids] = s.values
    assert np.array_equal(dense, dense.T)
    assert np.all(np.diag(dense) == 26.0)
    assert set(np.unique(dense)) <= {0.0, -1.0, 26.0}
    assert M.stencil27(128).nnz == 55742968


def test_row_band_and_cuts():
    csr = M.make_matrix("rmat", 9, 8, seed=2)
    csc = M.csr_to_csc(csr)
    rf = M.row_flop(csc, csr)
    cuts = M.band_cuts(rf, 4)
    assert cuts[0] == 0 and cuts[-1] == csr.nrows and np.all(np.diff(cuts.astype(np.int64)) >= 0)
    total = int(rf.sum())
    for r in range(4):
        band = M.row_band(csc, int(cuts[r]), int(cuts[r + 1]))
        assert band.nrows == cuts[r + 1] - cuts[r]
        # a band's flop is within one row of the balanced share
        bf = int(rf[cuts[r]:cuts[r + 1]].sum())
        assert abs(bf - total / 4) <= int(rf.max()) + 1
    # the bands' entries partition A's entries
    assert sum(M.row_band(csc, int(cuts[r]), int(cuts[r + 1])).nnz for r in range(4)) == csc.nnz
    assert np.array_equal(bands.plan_bands(csc, csr, 4), cuts)


def test_row_band_unsorted_columns():
    """row_band keeps the entries of [r0, r1) in their column order even when
    the row ids inside a column are not sorted (the reference never requires
    sorted CSC columns)."""
    csr = M.make_matrix("er", 8, 5, seed=3)
    csc = M.csr_to_csc(csr)
    rev = M.CscMatrix(csc.nrows, csc.ncols, csc.colptr, csc.rowids.copy(), csc.values.copy())
    for j in range(csc.ncols):
        p0, p1 = int(csc.colptr[j]), int(csc.colptr[j + 1])
        rev.rowids[p0:p1] = csc.rowids[p0:p1][::-1]
        rev.values[p0:p1] = csc.values[p0:p1][::-1]
    r0, r1 = 60, 170
    got = M.row_band(rev, r0, r1)
    exp = M.row_band(csc, r0, r1)
    assert np.array_equal(got.colptr, exp.colptr)
    for j in range(csc.ncols):
        p0, p1 = int(exp.colptr[j]), int(exp.colptr[j + 1])
        assert np.array_equal(got.rowids[p0:p1], exp.rowids[p0:p1][::-1])
        assert np.array_equal(got.values[p0:p1], exp.values[p0:p1][::-1])
