"""Regenerate the golden fixtures from the REFERENCE implementation.

Runs only where /root/reference exists (this build container): it builds the
unmodified reference library (oracle/build_ref.sh -> oracle/_ref/) and records
its outputs for small inputs, so the CPU oracle and the GPU path can be pinned
against the reference itself on boxes without /root/reference.

    python tests/golden/make_golden.py

Writes tests/golden/golden.npz (+ index.json). Cases:
  * the known-answer tests of proj/tests/test_pb_spgemm.cpp (identity,
    dense 2x2, 64-bit key widening at 2^21, empty, I*A = A);
  * random ER/RMAT pairs like acceptance.cpp:62-115 (seeded), A and B with
    U[0,1) values, multiplied by the reference pb_multiply (1 thread, so the
    values are bit-reproducible) with several nbins settings;
  * generator outputs gen_er / gen_rmat (generate.cpp:20-90) for the
    generator pins.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2002_11302_b200 import matrices as M  # noqa: E402


def coo_csc_csr(nrows, ncols, rows, cols, vals):
    """CSC and CSR of a COO through the REFERENCE conversion."""
    cp, ci, cv = oracle.ref_convert(False, nrows, ncols, rows, cols, vals)
    rp, ri, rv = oracle.ref_convert(True, nrows, ncols, rows, cols, vals)
    return (M.CscMatrix(nrows, ncols, cp, ci, cv), M.CsrMatrix(nrows, ncols, rp, ri, rv))


def with_values(rows, cols, vseed):
    return np.array([oracle.value(vseed, int(r), int(c)) for r, c in zip(rows, cols)],
                    dtype=np.float64)


def main():
    oracle.build(ref=True)
    store = {}
    index = []

    def add_case(name, a, b, nbins=0, balanced=False, l2=1 << 20):
        res = oracle.multiply(a, b, nbins=nbins, balanced=balanced, l2_bytes=l2,
                              impl="reference", nthreads=1)
        k = f"c{len(index)}"
        arrs = {
            "a_colptr": a.colptr, "a_rowids": a.rowids, "a_values": a.values,
            "b_rowptr": b.rowptr, "b_colids": b.colids, "b_values": b.values,
            "c_rowptr": res.rowptr, "c_colids": res.colids, "c_values": res.values,
            "per_column_flop": res.per_column_flop, "per_bin_flop": res.per_bin_flop,
            "bin_row_starts": res.bin_row_starts,
        }
        for kk, v in arrs.items():
            store[f"{k}_{kk}"] = v
        index.append({"key": k, "name": name, "a_dims": [a.nrows, a.ncols],
                      "b_dims": [b.nrows, b.ncols], "nbins": nbins, "balanced": balanced,
                      "l2_bytes": l2, "flop": res.flop, "nnz_c": int(res.colids.size),
                      "ref_nbins": res.nbins, "tuples_into_sort": res.tuples_into_sort,
                      "merged_total": res.merged_total})

    # --- known-answer tests (test_pb_spgemm.cpp) ---
    n = 4
    eye = coo_csc_csr(n, n, np.arange(n), np.arange(n), np.ones(n))
    add_case("identity4", eye[0], eye[1], nbins=1)
    d2 = coo_csc_csr(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [1.0, 2.0, 3.0, 4.0])
    add_case("dense2", d2[0], d2[1], nbins=1)
    big = 1 << 21
    wa = coo_csc_csr(big, big, [0, 5, big - 1], [0, big - 1, 5], [2.0, 3.0, 4.0])
    wb = coo_csc_csr(big, big, [0, big - 1, 5], [7, 0, 5], [5.0, 6.0, 7.0])
    add_case("widen_2^21", wa[0], wb[1])
    e = coo_csc_csr(16, 16, [], [], [])
    add_case("empty16", e[0], e[1])
    r, c, _ = oracle.ref_generate("rmat", 7, 5, 3)
    am = coo_csc_csr(128, 128, r, c, np.ones(r.size))
    ident = coo_csc_csr(128, 128, np.arange(128), np.arange(128), np.ones(128))
    add_case("I_times_rmat7", ident[0], am[1])
    # --- random pairs (acceptance.cpp:62-115 shape, U[0,1) values) ---
    rng = np.random.default_rng(20240901)
    for t in range(16):
        scale = int(rng.integers(4, 9))
        kinds = ["er" if rng.integers(2) else "rmat" for _ in range(2)]
        efs = [int(rng.integers(2, 17)) for _ in range(2)]
        seeds = [int(rng.integers(1, 1 << 30)) for _ in range(2)]
        mats = []
        for kind, ef, sd in zip(kinds, efs, seeds):
            ef = min(ef, 1 << scale)
            rr, cc, _ = oracle.ref_generate(kind, scale, ef, sd)
            vv = with_values(rr, cc, sd ^ M.VALUE_SEED_XOR)
            mats.append(coo_csc_csr(1 << scale, 1 << scale, rr, cc, vv))
        nbins = [0, 1, 4, 16][t % 4]
        add_case(f"rand{t}_{kinds[0]}{efs[0]}x{kinds[1]}{efs[1]}_s{scale}", mats[0][0],
                 mats[1][1], nbins=nbins)
    # balanced bins with a tiny l2 (test_pb_spgemm.cpp:361-379)
    r1, c1, _ = oracle.ref_generate("rmat", 9, 8, 5)
    r2, c2, _ = oracle.ref_generate("rmat", 9, 8, 6)
    a9 = coo_csc_csr(512, 512, r1, c1, with_values(r1, c1, 5))
    b9 = coo_csc_csr(512, 512, r2, c2, with_values(r2, c2, 6))
    add_case("balanced_rmat9", a9[0], b9[1], nbins=8, balanced=True, l2=1024)
    # --- generator pins ---
    gens = []
    for kind, scale, ef, seed in [("er", 8, 4, 1234), ("er", 10, 16, 7), ("rmat", 8, 6, 1234),
                                  ("rmat", 10, 8, 3)]:
        rr, cc, _ = oracle.ref_generate(kind, scale, ef, seed)
        g = f"g{len(gens)}"
        store[f"{g}_rows"] = rr
        store[f"{g}_cols"] = cc
        gens.append({"key": g, "kind": kind, "scale": scale, "ef": ef, "seed": seed})
    # value function pins: SplitMix64(split_seed(vseed, r<<32|c)).next_unit()
    vr = np.array([0, 1, 5, 1 << 20, (1 << 24) - 1], dtype=np.uint32)
    vc = np.array([0, 2, 7, 3, 9], dtype=np.uint32)
    store["values_rows"], store["values_cols"] = vr, vc
    store["values_seed99"] = with_values(vr, vc, 99)

    np.savez_compressed(HERE / "golden.npz", **store)
    (HERE / "index.json").write_text(json.dumps({"cases": index, "generators": gens}, indent=1))
    print(f"wrote {len(index)} cases, {len(gens)} generator pins")


if __name__ == "__main__":
    main()
