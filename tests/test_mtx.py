"""Matrix Market I/O: the native reader/writer against the
reference's own mm_read / mm_write (proj/src/mmio.cpp:33-117, compiled into
oracle/_ref), on fixture files covering every field/symmetry the reference
accepts and every parse_error it raises.
"""
import numpy as np
import pytest

import oracle
from paper_2002_11302_b200 import matrices as M

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")

CASES = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n"
                    "% a comment\n\n3 4 5\n1 1 1.5\n3 4 -2e-3\n2 2 0\n1 4 1e300\n3 1 .25\n",
    "symmetric_real": "%%MatrixMarket matrix coordinate real symmetric\n"
                      "4 4 4\n1 1 2.0\n2 1 -1.0\n4 2 3.5\n3 3 7\n",
    "pattern_general": "%%MatrixMarket matrix coordinate pattern general\n2 3 3\n1 2\n2 3\n1 1\n",
    "pattern_symmetric": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 3\n",
    "integer_upper": "%%MATRIXMARKET Matrix Coordinate Integer General\n2 2 2\n1 2 7\n2 1 -3\n",
    "crlf_comments": "%%MatrixMarket matrix coordinate real general\r\n%c\r\n2 2 2\r\n"
                     "% mid\r\n1 1 1\r\n\r\n2 2 2\r\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n1 1 2\n2 1 3\n",
    "one_by_one": "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 42\n",
    "trailing_tokens": "%%MatrixMarket matrix coordinate real general extra\n2 2 1 9\n2 1 0.5 x\n",
}

ERRORS = {
    "empty": "",
    "no_banner": "%MatrixMarket matrix coordinate real general\n1 1 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex_field": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n2 x 1\n",
    "zero_dims": "%%MatrixMarket matrix coordinate real general\n0 3 0\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "zero_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1.0\n",
    "missing_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "nan_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nan\n",
    "too_few": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n",
    "malformed_entry": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.5 1 1\n",
    "huge_dims": "%%MatrixMarket matrix coordinate real general\n4294967296 2 0\n",
}


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(text.encode())
    return p


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_known_entries(tmp_path, name):
    nr, nc, r, c, v = M.read_mtx(_write(tmp_path, name, CASES[name]))
    assert r.dtype == np.uint32 and v.dtype == np.float64
    assert np.all(r < nr) and np.all(c < nc)
    if name == "symmetric_real":  # mirror right after its source, diagonal single
        assert list(zip(r, c)) == [(0, 0), (1, 0), (0, 1), (3, 1), (1, 3), (2, 2)]
        assert list(v) == [2.0, -1.0, -1.0, 3.5, 3.5, 7.0]
    if name.startswith("pattern"):
        assert np.all(v == 1.0)


@needs_ref
@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference(tmp_path, name):
    p = _write(tmp_path, name, CASES[name])
    got = M.read_mtx(p)
    exp = oracle.ref_mm_read(p)
    assert got[:2] == exp[:2]
    for g, e in zip(got[2:], exp[2:]):
        assert np.array_equal(g, e)


@needs_ref
@pytest.mark.parametrize("name", sorted(ERRORS))
def test_parse_errors_match_reference(tmp_path, name):
    p = _write(tmp_path, name, ERRORS[name])
    with pytest.raises(M.ParseError) as ours:
        M.read_mtx(p)
    with pytest.raises(oracle.OracleError) as ref:
        oracle.ref_mm_read(p)
    assert str(ours.value) == ref.value.msg


def test_missing_file_is_a_parse_error(tmp_path):
    with pytest.raises(M.ParseError, match="cannot open"):
        M.read_mtx(tmp_path / "nope.mtx")


def test_writer_round_trip_and_bytes(tmp_path):
    rng = np.random.default_rng(5)
    n = 200
    r = rng.integers(0, 50, n).astype(np.uint32)
    c = rng.integers(0, 70, n).astype(np.uint32)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    ours = tmp_path / "ours.mtx"
    M.write_mtx(ours, 50, 70, r, c, v)
    nr, nc, r2, c2, v2 = M.read_mtx(ours)
    assert (nr, nc) == (50, 70)
    assert np.array_equal(r, r2) and np.array_equal(c, c2) and np.array_equal(v, v2)
    if oracle.ref_available():
        ref = tmp_path / "ref.mtx"
        oracle.ref_mm_write(ref, 50, 70, r, c, v)
        assert ours.read_bytes() == ref.read_bytes()


def test_matrix_from_mtx_sums_duplicates(tmp_path):
    csr = M.matrix_from_mtx(_write(tmp_path, "d", CASES["duplicates"]))
    assert list(csr.rowptr) == [0, 1, 2] and list(csr.colids) == [0, 0]
    assert list(csr.values) == [3.0, 3.0]
