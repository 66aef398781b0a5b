"""GPU parity: the sm_100a path, called through the C-ABI, against the
reference (golden fixtures and oracle/_ref) and the C restatement.

Bar (BASELINE.json north_star): rowptr / colids bit-exact, fp64 values within
1e-12 relative. Full-size configs that the CPU cannot multiply in seconds are
checked through size-independent properties (conservation, linearity, known
nnz, exact integer values) and band parity (rows of a band vs the oracle's
product of that band).
"""
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2002_11302_b200 import api, bands, matrices as M

from helpers import (RTOL, assert_csr_matches, assert_valid_csr, assert_values_close,
                     golden_cases)

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def gpu(a, b, **kw):
    return api.pb_multiply(a, b, api.PbConfig(device=0, **kw))


def check_vs(res, ref):
    assert_csr_matches(res.c.rowptr, res.c.colids, res.c.values, ref.rowptr, ref.colids,
                       ref.values)
    assert res.tuples_into_sort == ref.flop
    assert res.merged_total == ref.colids.size


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c[0]["name"])
def test_golden_reference_fixtures(case):
    meta, a, b, exp = case
    res = gpu(a, b, nbins=meta["nbins"], balanced_bins=meta["balanced"],
              l2_bytes=meta["l2_bytes"])
    assert_csr_matches(res.c.rowptr, res.c.colids, res.c.values, exp["c_rowptr"],
                       exp["c_colids"], exp["c_values"])
    assert res.sym.flop == meta["flop"]
    assert res.sym.nbins == meta["ref_nbins"]
    assert np.array_equal(res.sym.per_column_flop, exp["per_column_flop"])
    assert np.array_equal(res.sym.per_bin_flop, exp["per_bin_flop"])
    assert np.array_equal(res.sym.bin_row_starts, exp["bin_row_starts"])
    assert res.tuples_into_sort == meta["flop"]          # acceptance criterion 6
    assert res.merged_total == meta["nnz_c"] == res.c.nnz


def test_known_answers():
    d2 = M.coo_to_csr(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [1.0, 2.0, 3.0, 4.0])
    r = gpu(M.csr_to_csc(d2), d2)
    assert list(r.c.values) == [7.0, 10.0, 15.0, 22.0] and r.sym.flop == 8
    # cancellation keeps an exact zero as a structural nonzero
    a = M.coo_to_csr(2, 2, [0, 0], [0, 1], [1.0, -1.0])
    b = M.coo_to_csr(2, 2, [0, 1], [1, 1], [1.0, 1.0])
    z = gpu(M.csr_to_csc(a), b)
    assert z.c.nnz == 1 and z.c.values[0] == 0.0
    # empty product
    e = M.coo_to_csr(16, 16, [], [])
    r = gpu(M.csr_to_csc(e), e)
    assert r.c.nnz == 0 and r.sym.flop == 0 and np.all(r.c.rowptr == 0)


def test_identity_times_a():
    csr = M.make_matrix("rmat", 7, 5, seed=3)
    eye = M.coo_to_csr(csr.nrows, csr.nrows, np.arange(csr.nrows), np.arange(csr.nrows))
    r = gpu(M.csr_to_csc(eye), csr)
    assert_csr_matches(r.c.rowptr, r.c.colids, r.c.values, csr.rowptr, csr.colids, csr.values,
                       rtol=1e-15)


@pytest.mark.parametrize("seed", range(60))
def test_random_sweep_vs_oracle(seed):
    """acceptance.cpp:62-115 shape: random ER/RMAT pairs, scales 4..10."""
    rng = np.random.default_rng(1000 + seed)
    scale = int(rng.integers(4, 11))
    mats = []
    for k in range(2):
        kind = "er" if rng.integers(2) else "rmat"
        ef = int(min(rng.integers(2, 17), 1 << scale))
        mats.append(M.make_matrix(kind, scale, ef, seed=seed * 13 + k))
    a, b = M.csr_to_csc(mats[0]), mats[1]
    cap = [0, 2048, 1024, 512][seed % 4]
    res = gpu(a, b, bin_cap=cap)
    ref = oracle.multiply(a, b)
    check_vs(res, ref)
    assert_valid_csr(res.c)


def test_matrix_market_squaring(tmp_path):
    """The reference bench's --matrix path (spgemm_bench.cpp:55-58): a Matrix
    Market file (symmetric storage, mm_read semantics) squared on the GPU."""
    s = M.stencil27(6)
    rows = np.repeat(np.arange(s.nrows, dtype=np.uint32), np.diff(s.rowptr).astype(np.int64))
    lower = rows >= s.colids
    p = tmp_path / "st6_sym.mtx"
    with open(p, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n")
        f.write(f"{s.nrows} {s.ncols} {int(lower.sum())}\n")
        for r, c, v in zip(rows[lower], s.colids[lower], s.values[lower]):
            f.write(f"{r + 1} {c + 1} {v:.17g}\n")
    a = M.matrix_from_mtx(p)
    assert np.array_equal(a.rowptr, s.rowptr) and np.array_equal(a.colids, s.colids)
    res = gpu(M.csr_to_csc(a), a)
    check_vs(res, oracle.multiply(M.csr_to_csc(a), a))


def test_rectangular():
    r, c = M.gen_er(9, 4, 5)
    a = M.coo_to_csr(512, 512, r, c)
    a = M.CsrMatrix(300, 512, a.rowptr[:301].copy(), a.colids[:int(a.rowptr[300])].copy(),
                    np.linspace(0.5, 1.5, int(a.rowptr[300])))
    r2, c2 = M.gen_er(9, 3, 6)
    b = M.coo_to_csr(512, 512, r2, c2, np.ones(r2.size))
    b = M.CsrMatrix(512, 200, *_cols_below(b, 200))
    res = gpu(M.csr_to_csc(a), b)
    check_vs(res, oracle.multiply(M.csr_to_csc(a), b))


def _cols_below(m, ncols):
    keep = m.colids < ncols
    rows = np.repeat(np.arange(m.nrows), np.diff(m.rowptr).astype(np.int64))[keep]
    out = M.coo_to_csr(m.nrows, ncols, rows, m.colids[keep], m.values[keep])
    return out.rowptr, out.colids, out.values


def test_configuration_invariance():
    """acceptance.cpp:197-226: identical pattern across nbins / lbin_bytes /
    GPU bin capacity; values within tolerance."""
    a = M.make_matrix("er", 12, 4, seed=99)
    b = M.make_matrix("er", 12, 4, seed=100)
    ac = M.csr_to_csc(a)
    base = gpu(ac, b)
    for nbins in (0, 1, 16, 1024):
        for lbin in (16, 512, 4096):
            for cap in (0, 512, 1536):
                r = gpu(ac, b, nbins=nbins, lbin_bytes=lbin, bin_cap=cap)
                assert_csr_matches(r.c.rowptr, r.c.colids, r.c.values, base.c.rowptr,
                                   base.c.colids, base.c.values, rtol=1e-10)


def test_value_sum_conservation():
    """test_pb_spgemm.cpp:315-335 as linearity: sum(C) = sum_k colsum_A(k) * rowsum_B(k)."""
    a = M.make_matrix("rmat", 10, 8, seed=81)
    b = M.make_matrix("rmat", 10, 8, seed=82)
    ac = M.csr_to_csc(a)
    r = gpu(ac, b)
    colsum = np.bincount(np.repeat(np.arange(ac.ncols), np.diff(ac.colptr).astype(np.int64)),
                         weights=ac.values, minlength=ac.ncols)
    rowsum = np.bincount(np.repeat(np.arange(b.nrows), np.diff(b.rowptr).astype(np.int64)),
                         weights=b.values, minlength=b.nrows)
    assert abs(r.c.values.sum() - float(colsum @ rowsum)) <= 1e-9 * abs(float(colsum @ rowsum))


def test_row_bands_assemble_to_full_product():
    """The multi-GPU partitioning on one GPU: bands multiplied separately and
    concatenated equal the single product."""
    csr = M.make_matrix("er", 14, 8, seed=12)
    csc = M.csr_to_csc(csr)
    full = gpu(csc, csr)
    cuts = bands.plan_bands(csc, csr, 5)
    parts = [gpu(bands.band_slab(csc, cuts, r), csr).c for r in range(5)]
    asm = bands.assemble(parts, cuts, csr.ncols)
    assert_csr_matches(asm.rowptr, asm.colids, asm.values, full.c.rowptr, full.c.colids,
                       full.c.values)


def test_expand_row_bands_invariant():
    """Row-banded expand (forced 1..5 bands) gives the same product."""
    csr = M.make_matrix("er", 13, 8, seed=5)
    a = M.csr_to_csc(csr)
    base = gpu(a, csr, expand_bands=1)
    for g in (2, 3, 5):
        r = gpu(a, csr, expand_bands=g)
        assert r.report["expand_bands"] == g
        assert_csr_matches(r.c.rowptr, r.c.colids, r.c.values, base.c.rowptr, base.c.colids,
                           base.c.values)
    # row ids inside A's columns need not be sorted (the reference never
    # requires it): reverse every column and band again
    rev = M.CscMatrix(a.nrows, a.ncols, a.colptr, a.rowids.copy(), a.values.copy())
    for j in range(a.ncols):
        p0, p1 = int(a.colptr[j]), int(a.colptr[j + 1])
        rev.rowids[p0:p1] = a.rowids[p0:p1][::-1]
        rev.values[p0:p1] = a.values[p0:p1][::-1]
    for g in (1, 3):
        r = gpu(rev, csr, expand_bands=g)
        assert_csr_matches(r.c.rowptr, r.c.colids, r.c.values, base.c.rowptr, base.c.colids,
                           base.c.values)


def test_expand_bands_auto_many_bins():
    """The automatic band choice (> 200 K bins, short runs, no heavy row: C5a's
    regime) engages and gives the one-pass product. Tiny bins (bin_cap 32)
    on a sparse ER square reach that bin count at test size."""
    csr = M.make_matrix("er", 23, 1, seed=7)
    a = M.csr_to_csc(csr)
    auto = gpu(a, csr, bin_cap=32)
    one = gpu(a, csr, bin_cap=32, expand_bands=1)
    assert auto.report["heavy_bins"] == 0 and auto.report["gpu_bins"] > 200000
    assert auto.report["expand_bands"] == min(4, (auto.report["gpu_bins"] + 99999) // 100000)
    assert one.report["expand_bands"] == 1
    assert_csr_matches(auto.c.rowptr, auto.c.colids, auto.c.values, one.c.rowptr, one.c.colids,
                       one.c.values)


def test_bounded_memory_rounds_match_single_pass():
    """Forced row-band rounds (host path) give the single-pass product and
    the same reference-layout symbolic report."""
    for kind, scale in (("er", 13), ("rmat", 12)):
        csr = M.make_matrix(kind, scale, 8, seed=17)
        a = M.csr_to_csc(csr)
        one = gpu(a, csr)
        rounds = gpu(a, csr, max_round_tuples=max(one.sym.flop // 5, 1))
        assert_csr_matches(rounds.c.rowptr, rounds.c.colids, rounds.c.values, one.c.rowptr,
                           one.c.colids, one.c.values)
        assert rounds.sym.flop == one.sym.flop and rounds.sym.nbins == one.sym.nbins
        assert np.array_equal(rounds.sym.per_column_flop, one.sym.per_column_flop)
        assert np.array_equal(rounds.sym.per_bin_flop, one.sym.per_bin_flop)
        assert rounds.tuples_into_sort == one.sym.flop
        assert rounds.merged_total == one.c.nnz
        # unsorted row ids inside A's columns: the host slabs filter, not bisect
        rev = M.CscMatrix(a.nrows, a.ncols, a.colptr, a.rowids.copy(), a.values.copy())
        for j in range(a.ncols):
            p0, p1 = int(a.colptr[j]), int(a.colptr[j + 1])
            rev.rowids[p0:p1] = a.rowids[p0:p1][::-1]
            rev.values[p0:p1] = a.values[p0:p1][::-1]
        rr = gpu(rev, csr, max_round_tuples=max(one.sym.flop // 5, 1))
        assert_csr_matches(rr.c.rowptr, rr.c.colids, rr.c.values, one.c.rowptr, one.c.colids,
                           one.c.values)


def test_device_path_matches_host_path():
    import torch
    csr = M.make_matrix("er", 13, 6, seed=21)
    csc = M.csr_to_csc(csr)
    host = gpu(csc, csr)
    dev = torch.device("cuda", 0)
    t = lambda x, dt: torch.from_numpy(x.view(dt)).to(dev)  # noqa: E731
    A = (t(csc.colptr, np.int64), t(csc.rowids, np.int32), t(csc.values, np.float64))
    B = (t(csr.rowptr, np.int64), t(csr.colids, np.int32), t(csr.values, np.float64))
    ctx = api.DeviceContext(0)
    for _ in range(2):  # reuse of the grow-only workspace
        nnz, rep = ctx.multiply(ctx.view(csc.nrows, csc.ncols, *A),
                                ctx.view(csr.nrows, csr.ncols, *B), api.PbConfig(device=0))
    assert nnz == host.c.nnz and rep["flop"] == host.sym.flop
    assert ctx.launches() > 0
    import ctypes
    rp, ci, va = ctx.result_pointers()
    got_rp = torch.empty(csc.nrows + 1, dtype=torch.int64, device=dev)
    got_ci = torch.empty(nnz, dtype=torch.int32, device=dev)
    got_va = torch.empty(nnz, dtype=torch.float64, device=dev)
    cudart = ctypes.CDLL("libcudart.so.12")
    for dst, src, nbytes in ((got_rp, rp, (csc.nrows + 1) * 8), (got_ci, ci, nnz * 4),
                             (got_va, va, nnz * 8)):
        assert cudart.cudaMemcpy(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src),
                                 ctypes.c_size_t(nbytes), 3) == 0
    assert_csr_matches(got_rp.cpu().numpy().view(np.uint64), got_ci.cpu().numpy().view(np.uint32),
                       got_va.cpu().numpy(), host.c.rowptr, host.c.colids, host.c.values)


def test_parameter_errors_on_gpu():
    a = M.make_matrix("er", 6, 3, seed=1)
    ac = M.csr_to_csc(a)
    with pytest.raises(api.ParameterError):
        gpu(ac, a, nbins=6)
    with pytest.raises(api.ParameterError):
        gpu(ac, a, lbin_bytes=0)
    bad = M.CsrMatrix(32, 64, np.zeros(33, np.uint64), np.zeros(0, np.uint32), np.zeros(0))
    with pytest.raises(api.ParameterError):
        gpu(ac, bad)


# ---------------------------------------------------------------- configs --
def test_config_C1_vs_oracle():
    a, b = M.make_config("C1")
    res = gpu(a, b)
    ref = oracle.multiply(a, b)
    check_vs(res, ref)
    cf = ref.flop / ref.colids.size
    assert 1.0 <= cf <= 1.05  # acceptance criterion 4 (ER squared: cf in [1, 1.05])


@pytest.mark.slow
def test_config_C2_vs_reference():
    a, b = M.make_config("C2")
    res = gpu(a, b)
    impl = "reference" if oracle.ref_available() else "port"
    ref = oracle.multiply(a, b, impl=impl, nthreads=0, stepwise=False)
    assert res.sym.flop == 268435456
    check_vs(res, ref)


def _band_parity(a, b, res, nbands=3, rows=4096):
    """Rows of a few bands of the GPU product vs the oracle's band products
    (SURVEY.md §8c band parity)."""
    rng = np.random.default_rng(5)
    starts = sorted(rng.choice(a.nrows - rows, size=nbands, replace=False))
    for r0 in list(starts) + [a.nrows - rows]:
        slab = M.row_band(a, int(r0), int(r0) + rows)
        ref = oracle.multiply(slab, b, impl="reference" if oracle.ref_available() else "port",
                              nthreads=0 if oracle.ref_available() else 1)
        lo, hi = int(res.c.rowptr[r0]), int(res.c.rowptr[r0 + rows])
        assert np.array_equal(res.c.rowptr[r0:r0 + rows + 1] - res.c.rowptr[r0], ref.rowptr)
        assert np.array_equal(res.c.colids[lo:hi], ref.colids)
        assert_values_close(res.c.values[lo:hi], ref.values)


@pytest.mark.slow
def test_config_C4_stencil_properties_and_bands():
    a, b = M.make_config("C4")
    res = gpu(a, b)
    assert res.sym.flop == 1489355288 and res.c.nnz == 254840104
    assert res.tuples_into_sort == res.sym.flop and res.merged_total == res.c.nnz
    assert_valid_csr(res.c)
    # interior row of (27-pt)^2: 125 entries, diagonal 26*26 + 26*1 = 702, exact
    n = 128
    i = (64 * n + 64) * n + 64
    lo, hi = int(res.c.rowptr[i]), int(res.c.rowptr[i + 1])
    assert hi - lo == 125
    assert res.c.values[lo + int(np.searchsorted(res.c.colids[lo:hi], i))] == 702.0
    assert np.all(res.c.values == np.round(res.c.values))  # integer arithmetic stays exact
    _band_parity(a, b, res, rows=2048)


@pytest.mark.slow
def test_config_C5a_properties_and_bands():
    a, b = M.make_config("C5a")
    res = gpu(a, b)
    assert res.sym.flop == 1073741824 and res.c.nnz == 1073740073
    assert res.tuples_into_sort == res.sym.flop and res.merged_total == res.c.nnz
    rp = res.c.rowptr
    assert rp[0] == 0 and rp[-1] == res.c.nnz and np.all(rp[1:] >= rp[:-1])
    _band_parity(a, b, res, rows=8192)


def _rmat_band_parity(cfg_name, nrows_band):
    """SURVEY.md §8c band parity for the RMAT configs whose full tuple set
    exceeds one GPU: a few flop-balanced row bands of A (always including
    the heaviest row) multiplied by the full A on the GPU, against the
    reference's product of the same bands."""
    a, b = M.make_config(cfg_name)
    rf = M.row_flop(a, b)
    heavy = int(np.argmax(rf))
    rng = np.random.default_rng(7)
    starts = [max(0, heavy - nrows_band // 2)] + list(rng.integers(0, a.nrows - nrows_band, 3))
    impl = "reference" if oracle.ref_available() else "port"
    for r0 in starts:
        r0 = int(min(r0, a.nrows - nrows_band))
        slab = M.row_band(a, r0, r0 + nrows_band)
        res = gpu(slab, b)
        ref = oracle.multiply(slab, b, impl=impl, nthreads=0 if impl == "reference" else 1,
                              stepwise=False)
        assert res.sym.flop == int(rf[r0:r0 + nrows_band].sum())
        assert_csr_matches(res.c.rowptr, res.c.colids, res.c.values, ref.rowptr, ref.colids,
                           ref.values)


@pytest.mark.slow
def test_config_C3_band_parity():
    _rmat_band_parity("C3", 256)


@pytest.mark.slow
def test_config_C5b_band_parity():
    _rmat_band_parity("C5b", 64)


def test_rmat_heavy_rows_vs_oracle():
    """RMAT rows above the shared-memory capacity take the heavy-row split
    path (and uniform-key reduction for columns hit > capacity times)."""
    for scale in (10, 12, 14):
        csr = M.make_matrix("rmat", scale, 8, seed=scale)
        a = M.csr_to_csc(csr)
        res = gpu(a, csr)
        check_vs(res, oracle.multiply(a, csr))


@pytest.mark.parametrize("scale", [13, 15, 17])
@pytest.mark.parametrize("cap", [64, 1024, 0])
def test_heavy_split_digits_and_bin_caps(scale, cap):
    """Heavy-row split over column spaces of 2^13 / 2^15 / 2^17 (split digits
    of 1, 3 and 5 bits above the 4096-column dense range) and bin capacities
    from 64 tuples (nearly every row heavy, tiny unaligned sub-bins) up."""
    csr = M.make_matrix("rmat", scale, 6, seed=100 + scale)
    a = M.csr_to_csc(csr)
    res = gpu(a, csr, bin_cap=cap)
    check_vs(res, oracle.multiply(a, csr))
    assert_valid_csr(res.c)


def test_uniform_key_reduction():
    """One output entry receiving more tuples than a bin holds (6000 > 2048)."""
    K, n = 6000, 512
    a = M.coo_to_csr(4, K, np.r_[np.zeros(K, int), [1, 2]], np.r_[np.arange(K), [0, 1]],
                     np.r_[np.linspace(0.5, 1.5, K), [2.0, 3.0]])
    rows = np.r_[np.arange(K), np.arange(K)]
    cols = np.r_[np.zeros(K, int), np.arange(K) % 100 + 1]
    b = M.coo_to_csr(K, n, rows, cols, np.linspace(1.0, 2.0, 2 * K))
    ac = M.csr_to_csc(a)
    check_vs(gpu(ac, b), oracle.multiply(ac, b))


def test_distinct_count_paths_on_structured_duplicates():
    """The count-kernel shape is picked from the flop per row: a 2D 9-point
    stencil squared falls in the distinct-key class (81 products per row) yet
    every bin is duplicate-heavy (25 distinct of 81), and a sparse banded
    product has a few duplicates per bin: both must count exactly."""
    g = 96
    ii, jj = np.meshgrid(np.arange(g), np.arange(g), indexing="ij")
    rows, cols = [], []
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            ok = (ii + di >= 0) & (ii + di < g) & (jj + dj >= 0) & (jj + dj < g)
            rows.append((ii * g + jj)[ok])
            cols.append(((ii + di) * g + (jj + dj))[ok])
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    rng = np.random.default_rng(5)
    s9 = M.coo_to_csr(g * g, g * g, rows, cols, rng.uniform(0.5, 1.5, rows.size))
    a = M.csr_to_csc(s9)
    check_vs(gpu(a, s9), oracle.multiply(a, s9))
    n = 1 << 14  # 4 random entries per row within a band of 256 columns
    r = np.repeat(np.arange(n), 4)
    c = (r + rng.integers(0, 256, r.size)) % n
    bnd = M.coo_to_csr(n, n, r, c, rng.uniform(0.5, 1.5, r.size))
    a = M.csr_to_csc(bnd)
    check_vs(gpu(a, bnd), oracle.multiply(a, bnd))


def test_clustered_keys_rank_in_place_and_lsd_fallback():
    """One output row whose first 256 columns (one MSD bucket: 20 key bits,
    256 columns per bucket) receive `copies` tuples each, plus 600 single
    columns so that the bin is not pre-merged: 512 keys in the bucket are
    ranked in place (SM_BMAX = 512), 768 switch the bin to the LSD radix."""
    n = 1 << 20
    for copies, lsd in ((2, False), (3, True)):
        k = copies + 1
        a = M.coo_to_csc(n, k, np.zeros(k, int), np.arange(k), np.arange(2.0, 2.0 + k))
        rows = np.r_[np.repeat(np.arange(copies), 256), np.full(600, copies)]
        cols = np.r_[np.tile(np.arange(256), copies), 1000 + np.arange(600)]
        b = M.coo_to_csr(k, n, rows, cols, np.linspace(1.0, 2.0, rows.size))
        res = gpu(a, b, bin_cap=4096)  # (small products default to smaller bins)
        check_vs(res, oracle.multiply(a, b))
        assert (res.report["sort_fallbacks"] > 0) == lsd, res.report["sort_fallbacks"]


def test_tiny_bin_capacity_forces_heavy_split():
    csr = M.make_matrix("er", 11, 8, seed=3)
    a = M.csr_to_csc(csr)
    check_vs(gpu(a, csr, bin_cap=64), oracle.multiply(a, csr))


def test_cpp_dropin_on_gpu(tmp_path):
    import subprocess
    from paper_2002_11302_b200 import build
    shim = build.build_shim()
    exe = tmp_path / "dropin_test"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "dropin_test.cpp"), "-L", str(shim.parent),
                    "-lspgemm_b200", f"-Wl,-rpath,{shim.parent}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe), "gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_smoke_entry():
    import sys
    sys.path.insert(0, str(ROOT))
    import __graft_entry__
    __graft_entry__.smoke()


def _raw_csr(nrows, ncols, rows, cols, vals):
    """CSR straight from entry lists in the given order: duplicates and
    unsorted columns inside a row are kept (the reference accepts any CSR)."""
    rows = np.asarray(rows, np.int64)
    order = np.argsort(rows, kind="stable")
    rowptr = np.zeros(nrows + 1, np.uint64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.uint64)
    return M.CsrMatrix(nrows, ncols, rowptr, np.asarray(cols, np.uint32)[order],
                       np.asarray(vals, np.float64)[order])


def _raw_csc(nrows, ncols, rows, cols, vals):
    t = _raw_csr(ncols, nrows, cols, rows, vals)
    return M.CscMatrix(nrows, ncols, t.rowptr, t.colids, t.values)


def test_duplicate_and_unsorted_input_entries():
    """Repeated (row, col) entries in A or B and unsorted indices inside a
    column/row are summed like any other duplicate tuples."""
    rng = np.random.default_rng(7)
    n, nnz = 300, 4000
    ar, ac = rng.integers(0, n, nnz), rng.integers(0, n, nnz)
    br, bc = rng.integers(0, n, nnz), rng.integers(0, n, nnz)
    ar[:500], ac[:500] = ar[500:1000], ac[500:1000]  # explicit duplicates
    av, bv = rng.random(nnz), rng.random(nnz)
    a = _raw_csc(n, n, ar, ac, av)
    b = _raw_csr(n, n, br, bc, bv)
    res = gpu(a, b)
    check_vs(res, oracle.multiply(a, b))
    dense = np.zeros((n, n))
    np.add.at(dense, (ar, ac), av)
    db = np.zeros((n, n))
    np.add.at(db, (br, bc), bv)
    exp = dense @ db
    got = np.zeros((n, n))
    rows = np.repeat(np.arange(n), np.diff(res.c.rowptr).astype(np.int64))
    got[rows, res.c.colids] = res.c.values
    assert np.allclose(got, exp, rtol=1e-12, atol=0)


@pytest.mark.parametrize("ncols", [(1 << 31) - 1, 1 << 31, (1 << 32) - 1])
def test_widest_column_space(ncols):
    """col_bits 31 / 32: one row per GPU bin, keys are the columns themselves
    (the reference widens to 64-bit keys here, pb_spgemm.cpp:153)."""
    rng = np.random.default_rng(ncols & 0xffff)
    m, k, nnz = 50, 40, 600
    a = _raw_csc(m, k, rng.integers(0, m, nnz), rng.integers(0, k, nnz), rng.random(nnz))
    cols = np.concatenate([rng.integers(0, ncols, nnz - 20), np.full(20, ncols - 1)])
    b = _raw_csr(k, ncols, rng.integers(0, k, nnz), cols, rng.random(nnz))
    res = gpu(a, b)
    check_vs(res, oracle.multiply(a, b))
    assert res.c.colids.max() == ncols - 1


def test_empty_rows_and_columns():
    """Whole empty column bands of A, empty rows of B, empty output rows."""
    csr = M.make_matrix("er", 11, 6, seed=31)
    a = M.csr_to_csc(csr)
    keep = (np.arange(a.ncols) % 3) != 0
    nnz_per = np.diff(a.colptr).astype(np.int64) * keep
    colptr = np.concatenate([[0], np.cumsum(nnz_per)]).astype(np.uint64)
    mask = np.repeat(keep, np.diff(a.colptr).astype(np.int64))
    a2 = M.CscMatrix(a.nrows, a.ncols, colptr, a.rowids[mask], a.values[mask])
    rkeep = (np.arange(csr.nrows) % 5) != 0
    rn = np.diff(csr.rowptr).astype(np.int64) * rkeep
    rowptr = np.concatenate([[0], np.cumsum(rn)]).astype(np.uint64)
    rmask = np.repeat(rkeep, np.diff(csr.rowptr).astype(np.int64))
    b2 = M.CsrMatrix(csr.nrows, csr.ncols, rowptr, csr.colids[rmask], csr.values[rmask])
    res = gpu(a2, b2)
    check_vs(res, oracle.multiply(a2, b2))
    assert_valid_csr(res.c)


def test_coo_conversion_on_gpu():
    """coo_to_csr / coo_to_csc (convert.cpp:41-98) through the product path:
    duplicates summed, exact-zero sums kept, minor indices sorted; out-of-range
    entries rejected; empty input."""
    rng = np.random.default_rng(9)
    for (m, n, nnz) in ((300, 500, 20000), (1 << 14, 1 << 14, 300000), (7, 5, 0)):
        rows = rng.integers(0, m, nnz).astype(np.uint32)
        cols = rng.integers(0, n, nnz).astype(np.uint32)
        vals = rng.random(nnz)
        if nnz:
            rows[:50], cols[:50] = rows[50:100], cols[50:100]
            vals[:50] = -vals[50:100]  # cancellations -> exact zeros kept
        got = api.coo_to_csr(m, n, rows, cols, vals)
        exp = M.coo_to_csr(m, n, rows, cols, vals)
        assert_csr_matches(got.rowptr, got.colids, got.values, exp.rowptr, exp.colids, exp.values)
        gc = api.coo_to_csc(m, n, rows, cols, vals)
        ec = M.coo_to_csc(m, n, rows, cols, vals)
        assert_csr_matches(gc.colptr, gc.rowids, gc.values, ec.colptr, ec.rowids, ec.values)
        if oracle.ref_available() and nnz <= 50000:  # the reference's own convert.cpp
            rp, ri, rv = oracle.ref_convert(True, m, n, rows, cols, vals)
            assert_csr_matches(got.rowptr, got.colids, got.values, rp, ri, rv)
    with pytest.raises(ValueError):
        api.coo_to_csr(4, 4, np.array([1, 4], np.uint32), np.array([0, 0], np.uint32),
                       np.ones(2))


@pytest.mark.parametrize("name", ["C1", "R16", "E22"])
def test_gpu_generators_match_host(name):
    """pbg_generate_begin: the reference's ER / RMAT draws on the device,
    converted and valued there, bit-identical to the host build (whose
    generators are pinned against the reference)."""
    hc, hr = M.make_config(name)
    gc, gr = M.make_config_gpu(name)
    for g, h in ((gc.colptr, hc.colptr), (gc.rowids, hc.rowids), (gc.values, hc.values),
                 (gr.rowptr, hr.rowptr), (gr.colids, hr.colids), (gr.values, hr.values)):
        assert np.array_equal(g, h)


# ---- column hash SpGEMM: spgemm::hash_multiply ----------
def _hash_vs_reference(a, b):
    res = api.hash_multiply(a, b, api.PbConfig(device=0))
    if oracle.ref_available():
        cp, ri, v = oracle.ref_hash_multiply(a, b)
    else:  # CSC of C = (CSR of C^T): the oracle product of the transposes
        ref = oracle.multiply(M.csr_to_csc(_transpose(b)), _transpose(a))
        cp, ri, v = ref.rowptr, ref.colids, ref.values
    assert_csr_matches(res.c.colptr, res.c.rowids, res.c.values, cp, ri, v)
    return res


def _transpose(m):
    """CSC m as the CSR of its transpose (same arrays)."""
    return M.CsrMatrix(m.ncols, m.nrows, m.colptr, m.rowids, m.values)


@pytest.mark.parametrize("seed", range(16))
def test_hash_multiply_random_vs_reference(seed):
    rng = np.random.default_rng(500 + seed)
    scale = int(rng.integers(4, 11))
    mats = [M.make_matrix("er" if rng.integers(2) else "rmat", scale,
                          int(min(rng.integers(2, 12), 1 << scale)), seed=seed * 7 + k)
            for k in range(2)]
    a, b = M.csr_to_csc(mats[0]), M.csr_to_csc(mats[1])
    _hash_vs_reference(a, b)  # RMAT hub columns included (k_hash_hub)


def test_hash_multiply_stencil_and_edges():
    s = M.stencil27(12)   # cf ~5.8: the hash path's regime; exact integer values
    a = M.csr_to_csc(s)
    res = _hash_vs_reference(a, a)
    assert np.all(res.c.values == np.round(res.c.values))
    # big-table kernel: columns of 1025..4096 products
    r, c = M.gen_er(10, 40, 3)
    big = M.coo_to_csc(1 << 10, 1 << 10, r, c, np.linspace(0.5, 1.5, r.size))
    _hash_vs_reference(big, big)
    # empty columns, exact-zero cancellation kept
    x = M.coo_to_csc(2, 2, [0, 0], [0, 1], [1.0, -1.0])
    y = M.coo_to_csc(2, 2, [0, 1], [1, 1], [1.0, 1.0])
    z = api.hash_multiply(x, y, api.PbConfig(device=0)).c
    assert list(z.colptr) == [0, 0, 1] and z.values[0] == 0.0
    with pytest.raises(api.ParameterError):
        api.hash_multiply(M.coo_to_csc(2, 3, [0], [0]), x, api.PbConfig(device=0))


def test_hash_multiply_hub_columns():
    # one B column of 8000 products: above the shared-memory tables, summed in
    # the dense global-memory accumulator (k_hash_hub)
    k = 8000
    a = M.coo_to_csc(k, 1, np.arange(k), np.zeros(k, int), np.ones(k))
    b = M.coo_to_csc(1, 1, [0], [0], [2.0])
    c = _hash_vs_reference(a, b).c
    assert list(c.colptr) == [0, k] and np.all(c.values == 2.0)
    # hub column with an exact-zero cancellation kept in C: C(:,0) =
    # A(:,0) - A(:,1), and A(:,1) is a single 1 at row 5
    a2 = M.coo_to_csc(k, 2, np.r_[np.arange(k), [5]], np.r_[np.zeros(k, int), [1]], np.ones(k + 1))
    b2 = M.coo_to_csc(2, 1, [0, 1], [0, 0], [1.0, -1.0])
    c2 = _hash_vs_reference(a2, b2).c
    assert c2.nnz == k and c2.values[5] == 0.0 and np.all(np.delete(c2.values, 5) == 1.0)
    # RMAT scale 12 (hub columns of tens of thousands of products) against
    # the reference's own hash_multiply
    r = M.csr_to_csc(M.make_matrix("rmat", 12, 16, seed=3))
    assert np.diff(r.colptr).max() > 64
    _hash_vs_reference(r, r)


def test_speculative_graph_replay_matches_and_recovers():
    """run_pipeline's single-sync path: the same shape multiplied again on a
    context is launched with the previous symbolic scalars and replayed as a
    CUDA graph; results equal the synchronous multiply's. A different matrix
    of the same shape (different flop) is rejected by the guard kernel and
    recomputed synchronously — the result must still be exact."""
    import torch
    from paper_2002_11302_b200 import api

    def up(a, b):
        dev = torch.device("cuda", 0)
        t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x).view(dt)).to(dev)
        return ((t(a.colptr, np.int64), t(a.rowids, np.int32), t(a.values, np.float64)),
                (t(b.rowptr, np.int64), t(b.colids, np.int32), t(b.values, np.float64)))

    ctx = api.DeviceContext(0)
    csr = M.make_matrix("er", 12, 6, seed=21)
    a = M.csr_to_csc(csr)
    ref = oracle.multiply(a, csr)
    A, B = up(a, csr)
    va, vb = ctx.view(a.nrows, a.ncols, *A), ctx.view(csr.nrows, csr.ncols, *B)
    from test_gpu_bands import _download
    for it in range(5):
        nnz, rep = ctx.multiply(va, vb)
        assert nnz == ref.colids.size and rep["tuples_into_sort"] == ref.flop
        assert_csr_matches(*_download(ctx, a.nrows, nnz), ref.rowptr, ref.colids, ref.values)
        if it >= 2:  # replayed graph: one launch of the captured pipeline
            assert rep["t_total"] > 0
    # same shape, different structure: the plan's flop no longer holds
    csr2 = M.make_matrix("er", 12, 6, seed=22)
    a2 = M.csr_to_csc(csr2)
    A2, B2 = up(a2, csr2)
    assert a2.rowids.size == a.rowids.size
    ref2 = oracle.multiply(a2, csr2)
    va2, vb2 = ctx.view(a2.nrows, a2.ncols, *A2), ctx.view(csr2.nrows, csr2.ncols, *B2)
    for it in range(3):
        nnz2, rep2 = ctx.multiply(va2, vb2)
        assert nnz2 == ref2.colids.size and rep2["tuples_into_sort"] == ref2.flop
        assert_csr_matches(*_download(ctx, a2.nrows, nnz2), ref2.rowptr, ref2.colids, ref2.values)
    # and back to the first matrix (its plan was replaced)
    nnz, rep = ctx.multiply(va, vb)
    assert_csr_matches(*_download(ctx, a.nrows, nnz), ref.rowptr, ref.colids, ref.values)
