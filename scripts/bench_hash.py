"""Column hash SpGEMM (api.hash_multiply) against the
PB-SpGEMM path on the same configs: device time of one multiply (CUDA events,
inputs already copied; median of 3 after a warm-up) and the compression
factor flop / nnz(C). Prints one JSON line per config."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2002_11302_b200 import api, matrices as M  # noqa: E402

for cfg in (sys.argv[1:] or ["C1", "C2", "C4", "C5a"]):
    a_csc, a_csr = M.make_config(cfg)
    pc = api.PbConfig(device=0)
    th, tp = [], []
    for i in range(4):
        try:
            r = api.hash_multiply(a_csc, a_csc, pc)
            th.append(r.phases["t_total"])
            hnnz, flop = r.c.nnz, r.flop
        except NotImplementedError as e:
            th, hnnz, flop = None, None, None
            print(json.dumps({"config": cfg, "hash": "unsupported", "why": str(e)}), flush=True)
            break
    for i in range(4):
        p = api.pb_multiply(a_csc, a_csr, pc, symbolic=False)
        tp.append(p.phases["t_total"])
    line = {"config": cfg, "flop": p.sym.flop, "nnz_c": p.c.nnz,
            "cf": p.sym.flop / max(p.c.nnz, 1),
            "pb_ms": statistics.median(tp[1:]) * 1e3,
            "pb_mult_per_s": p.sym.flop / statistics.median(tp[1:])}
    if th:
        line.update({"hash_ms": statistics.median(th[1:]) * 1e3,
                     "hash_mult_per_s": flop / statistics.median(th[1:]),
                     "hash_nnz_matches": hnnz == p.c.nnz})
    print(json.dumps(line), flush=True)
