"""The CPU oracle (oracle/pb_oracle.c) pinned against the reference.

CPU only. Two pins: (1) the committed golden fixtures, produced by the
reference library itself (tests/golden/make_golden.py); (2) where the
reference is built here (oracle/_ref), a live port-vs-reference sweep.
The reference run with one thread is bit-reproducible, and so is the port:
they must agree bit for bit, values included.
"""
import numpy as np
import pytest

import oracle
from paper_2002_11302_b200 import matrices as M

from helpers import golden_cases, golden_values


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c[0]["name"])
def test_port_reproduces_reference_golden(case):
    meta, a, b, exp = case
    res = oracle.multiply(a, b, nbins=meta["nbins"], balanced=meta["balanced"],
                          l2_bytes=meta["l2_bytes"], impl="port")
    assert res.flop == meta["flop"]
    assert res.nbins == meta["ref_nbins"]
    assert res.tuples_into_sort == meta["tuples_into_sort"] == meta["flop"]
    assert res.merged_total == meta["merged_total"] == meta["nnz_c"]
    assert np.array_equal(res.per_column_flop, exp["per_column_flop"])
    assert np.array_equal(res.per_bin_flop, exp["per_bin_flop"])
    assert np.array_equal(res.bin_row_starts, exp["bin_row_starts"])
    # bit-exact, values included: same algorithm, same (1-thread) order
    assert np.array_equal(res.rowptr, exp["c_rowptr"])
    assert np.array_equal(res.colids, exp["c_colids"])
    assert np.array_equal(res.values, exp["c_values"])


def test_known_answers():
    # test_pb_spgemm.cpp:49-58: I4 flop 4, dense 2x2 flop 8
    eye = M.coo_to_csr(4, 4, np.arange(4), np.arange(4))
    r = oracle.multiply(M.csr_to_csc(eye), eye, nbins=1)
    assert r.flop == 4 and list(r.per_column_flop) == [1, 1, 1, 1]
    d2 = M.coo_to_csr(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [1.0, 2.0, 3.0, 4.0])
    r = oracle.multiply(M.csr_to_csc(d2), d2, nbins=1)
    assert r.flop == 8
    assert list(r.values) == [7.0, 10.0, 15.0, 22.0]


def test_choose_nbins_known_answers():
    # test_pb_spgemm.cpp:78-88
    assert oracle.choose_nbins(16 << 20, 1 << 20) == 512
    assert oracle.choose_nbins(0, 1 << 20) == 64
    assert oracle.choose_nbins(0, 10) == 8
    assert oracle.choose_nbins(1 << 40, 1 << 30) == 8192


def test_parameter_errors():
    e = M.coo_to_csr(4, 4, [], [])
    with pytest.raises(oracle.OracleError) as ei:  # non power-of-two nbins
        oracle.multiply(M.csr_to_csc(e), e, nbins=3)
    assert ei.value.code == 1
    with pytest.raises(oracle.OracleError) as ei:  # lbin not a multiple of 16
        oracle.multiply(M.csr_to_csc(e), e, lbin_bytes=24)
    assert ei.value.code == 1
    a = M.coo_to_csr(4, 3, [], [])
    with pytest.raises(oracle.OracleError):  # dims
        oracle.multiply(M.csr_to_csc(a), e)


def test_value_function_pins():
    r, c, v = golden_values()
    got = [oracle.value(99, int(x), int(y)) for x, y in zip(r, c)]
    assert np.array_equal(np.array(got), v)


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")


@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_port_equals_reference_live(seed):
    rng = np.random.default_rng(seed)
    scale = int(rng.integers(4, 10))
    mats = []
    for k in range(2):
        kind = "er" if rng.integers(2) else "rmat"
        ef = int(min(rng.integers(2, 17), 1 << scale))
        r, c, _ = oracle.ref_generate(kind, scale, ef, seed * 7 + k)
        mats.append(M.fill_values(M.coo_to_csr(1 << scale, 1 << scale, r, c,
                                               combine="collapse"), seed + k))
    a, b = M.csr_to_csc(mats[0]), mats[1]
    for nbins in (0, 1, 8):
        p = oracle.multiply(a, b, nbins=nbins, impl="port")
        q = oracle.multiply(a, b, nbins=nbins, impl="reference", nthreads=1)
        assert np.array_equal(p.rowptr, q.rowptr)
        assert np.array_equal(p.colids, q.colids)
        assert np.array_equal(p.values, q.values)
        assert np.array_equal(p.per_bin_flop, q.per_bin_flop)


@pytest.mark.parametrize("kind,scale,ef", [("er", 16, 4), ("rmat", 12, 8), ("stencil", 8, None)])
def test_reference_arm_inputs_match_product_inputs(kind, scale, ef):
    """bench.py --impl reference builds its inputs with the reference library
    alone (oracle.RefConfig); they must be the product's inputs bit for bit."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2002_11302_b200 import matrices as M
    rc = oracle.RefConfig(kind, scale, ef or 0, 1, 1 ^ M.VALUE_SEED_XOR)
    (ap, ai, av), (bp, bi, bv) = rc.arrays()
    csr = M.make_matrix(kind, scale, ef, 1)
    csc = M.csr_to_csc(csr)
    for x, y in [(ap, csc.colptr), (ai, csc.rowids), (av, csc.values), (bp, csr.rowptr),
                 (bi, csr.colids), (bv, csr.values)]:
        assert np.array_equal(x, y)
    assert rc.flop == int(M.row_flop(csc, csr).sum())
    t, flop, nnz = rc.multiply(2)
    assert flop == rc.flop and t[5] > 0
    r1, bf = rc.band(0.25)
    assert 0 < r1 < rc.nrows and 0 < bf < rc.flop
    _, flop_b, _ = rc.multiply(2)
    assert flop_b == bf
    rc.close()
