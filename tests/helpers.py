"""Shared test helpers: golden fixtures and the parity comparison."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from paper_2002_11302_b200 import matrices as M

GOLDEN = Path(__file__).resolve().parent / "golden"
RTOL = 1e-12  # north_star: fp64 values within 1e-12 relative (summation order differs)


def golden_cases():
    idx = json.loads((GOLDEN / "index.json").read_text())
    z = np.load(GOLDEN / "golden.npz")
    out = []
    for c in idx["cases"]:
        k = c["key"]
        a = M.CscMatrix(c["a_dims"][0], c["a_dims"][1], z[f"{k}_a_colptr"], z[f"{k}_a_rowids"],
                        z[f"{k}_a_values"])
        b = M.CsrMatrix(c["b_dims"][0], c["b_dims"][1], z[f"{k}_b_rowptr"], z[f"{k}_b_colids"],
                        z[f"{k}_b_values"])
        exp = {kk: z[f"{k}_{kk}"] for kk in ("c_rowptr", "c_colids", "c_values", "per_column_flop",
                                              "per_bin_flop", "bin_row_starts")}
        out.append((c, a, b, exp))
    return out


def golden_generators():
    idx = json.loads((GOLDEN / "index.json").read_text())
    z = np.load(GOLDEN / "golden.npz")
    return [(g, z[f"{g['key']}_rows"], z[f"{g['key']}_cols"]) for g in idx["generators"]]


def golden_values():
    z = np.load(GOLDEN / "golden.npz")
    return z["values_rows"], z["values_cols"], z["values_seed99"]


def assert_values_close(got, exp, rtol=RTOL):
    got = np.asarray(got, dtype=np.float64)
    exp = np.asarray(exp, dtype=np.float64)
    assert got.shape == exp.shape
    scale = np.maximum(np.maximum(np.abs(got), np.abs(exp)), 1e-300)
    bad = np.abs(got - exp) > rtol * scale
    assert not bad.any(), f"{bad.sum()} values differ beyond {rtol}: first at {np.argmax(bad)}"


def assert_csr_matches(rowptr, colids, values, exp_rowptr, exp_colids, exp_values, rtol=RTOL):
    """rowptr / colids bit-exact, values within rtol (reference.cpp:37-51 semantics)."""
    assert np.array_equal(np.asarray(rowptr, np.uint64), np.asarray(exp_rowptr, np.uint64)), "rowptr"
    assert np.array_equal(np.asarray(colids, np.uint32), np.asarray(exp_colids, np.uint32)), "colids"
    assert_values_close(values, exp_values, rtol)


def assert_valid_csr(c: M.CsrMatrix):
    """Structural invariants (validate, convert.cpp:8-37): monotone rowptr,
    in-range and strictly increasing columns per row."""
    rp = c.rowptr.astype(np.int64)
    assert rp[0] == 0 and rp[-1] == c.nnz and np.all(np.diff(rp) >= 0)
    if c.nnz:
        assert int(c.colids.max()) < c.ncols
        d = np.diff(c.colids.astype(np.int64))
        row_start = np.zeros(c.nnz, dtype=bool)
        row_start[rp[:-1][rp[:-1] < c.nnz]] = True
        assert np.all((d > 0) | row_start[1:]), "columns not strictly increasing in a row"
