"""COO -> CSR on the GPU (pbg_coo_convert_begin, the product path) against the
reference's coo_to_csr (oracle/_ref, convert.cpp:41-70, single thread) on a
config's COO entries (seeded generator draws + U[0,1) values). One JSON line.

    python scripts/bench_convert.py [--config C2] [--steps 5]
"""
import argparse, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
from paper_2002_11302_b200 import api, matrices as M

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--steps", type=int, default=5)
args = ap.parse_args()
kind, scale, ef = M.CONFIGS[args.config]
assert kind in ("er", "rmat")
rows, cols = (M.gen_er if kind == "er" else M.gen_rmat)(scale, ef, 1)
n = 1 << scale
vals = np.random.default_rng(1).random(rows.size)
res = api.coo_to_csr(n, n, rows, cols, vals)  # warm
ts = []
for _ in range(args.steps):
    t0 = time.perf_counter()
    res = api.coo_to_csr(n, n, rows, cols, vals)
    ts.append(time.perf_counter() - t0)
t_gpu = sorted(ts)[len(ts) // 2]
line = {"metric": "COO->CSR entries/sec", "config": f"{args.config} COO ({rows.size} entries)",
        "gpu_e2e_s": t_gpu, "gpu_entries_per_s": rows.size / t_gpu}
if oracle.ref_available():
    t0 = time.perf_counter()
    rp, ri, rv = oracle.ref_convert(True, n, n, rows, cols, vals)
    t_ref = time.perf_counter() - t0
    assert np.array_equal(rp, res.rowptr) and np.array_equal(ri, res.colids)
    line.update({"reference_s": t_ref, "reference_entries_per_s": rows.size / t_ref,
                 "speedup_e2e": t_ref / t_gpu, "reference": "oracle/_ref coo_to_csr, 1 thread"})
print(json.dumps(line))
