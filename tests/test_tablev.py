"""Table V statistics check (reference acceptance.cpp:117-169): the check
logic on CPU (oracle as the multiply), the real check on the GPU when the
SuiteSparse files are mounted, and the same path on a generated matrix
file whose statistics are known."""
import numpy as np
import pytest

import oracle
from paper_2002_11302_b200 import matrices as M
from tablev import TABLE_V, TableVRow, check_rows, data_dir


def _stencil_file(tmp_path):
    s = M.stencil27(5)
    rows = np.repeat(np.arange(s.nrows, dtype=np.uint32), np.diff(s.rowptr).astype(np.int64))
    p = tmp_path / "st5.mtx"
    M.write_mtx(p, s.nrows, s.ncols, rows, s.colids, s.values)
    ref = oracle.multiply(M.csr_to_csc(s), s)
    flop, nnz_c = int(ref.flop), int(ref.colids.size)
    return p, TableVRow("st5", float(flop), float(nnz_c), flop / nnz_c, s.nrows, int(s.colids.size))


def _oracle_mult(a_csc, a_csr):
    r = oracle.multiply(a_csc, a_csr)
    return int(r.flop), int(r.colids.size)


def test_check_logic_on_known_file(tmp_path):
    p, row = _stencil_file(tmp_path)
    res = check_rows([row], tmp_path, _oracle_mult)
    assert res[0][1] and res[0][2], res
    bad = TableVRow(row.name, row.flop * 1.02, row.nnz_c, row.cf, row.nrows, row.nnz_a)
    assert check_rows([bad], tmp_path, _oracle_mult)[0][2] is False   # 2 % off flop
    meta = TableVRow(row.name, row.flop, row.nnz_c, row.cf, row.nrows + 1, row.nnz_a)
    assert check_rows([meta], tmp_path, _oracle_mult)[0][2] is False  # wrong metadata


def test_missing_files_are_skipped(tmp_path):
    res = check_rows(TABLE_V, tmp_path, _oracle_mult)
    assert [r[1] for r in res] == [False] * 4


def _gpu_mult(a_csc, a_csr):
    from paper_2002_11302_b200 import api
    r = api.pb_multiply(a_csc, a_csr, api.PbConfig(device=0))
    return int(r.sym.flop), int(r.c.rowptr[-1])


@pytest.mark.gpu
def test_table_v_known_file_on_gpu(tmp_path):
    p, row = _stencil_file(tmp_path)
    res = check_rows([row], tmp_path, _gpu_mult)
    assert res[0][1] and res[0][2], res


@pytest.mark.gpu
def test_table_v_suitesparse():
    res = check_rows(TABLE_V, data_dir(), _gpu_mult)
    found = [r for r in res if r[1]]
    if not found:
        pytest.skip(f"table statistics: no .mtx files under '{data_dir()}' "
                    "(set SPGEMM_DATA_DIR to a directory of SuiteSparse matrices)")
    assert all(r[2] for r in found), res
