"""Column hash SpGEMM with RMAT hub columns (k_hash_hub) against PB-SpGEMM:
C = A·A for RMAT scale s, edge factor 16 (C3's generator at smaller scale;
C3 itself needs more flop scratch than the hash path's one-shot layout).
Device time of one multiply, median of 3 after a warm-up; one JSON line per scale."""
import json
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_11302_b200 import api, matrices as M  # noqa: E402

for s in [int(x) for x in (sys.argv[1:] or ["14", "16", "18"])]:
    a = M.make_matrix("rmat", s, 16, seed=1)
    a_csc = M.csr_to_csc(a)
    pc = api.PbConfig(device=0)
    th = [api.hash_multiply(a_csc, a_csc, pc) for _ in range(4)]
    tp = [api.pb_multiply(a_csc, a, pc, symbolic=False) for _ in range(4)]
    h, p = th[-1], tp[-1]
    hm = statistics.median(r.phases["t_total"] for r in th[1:])
    pm = statistics.median(r.phases["t_total"] for r in tp[1:])
    print(json.dumps({"rmat_scale": s, "ef": 16, "flop": p.sym.flop, "nnz_c": p.c.nnz,
                      "hash_ms": hm * 1e3, "pb_ms": pm * 1e3,
                      "hash_mult_per_s": p.sym.flop / hm, "pb_mult_per_s": p.sym.flop / pm,
                      "nnz_matches": h.c.nnz == p.c.nnz}), flush=True)
