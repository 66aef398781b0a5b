"""Quick GPU parity + timing probe (development aid)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
from paper_2002_11302_b200 import api, matrices as M

def check(name, a, b, cfg=None, impl="port"):
    t = time.time(); res = api.pb_multiply(a, b, cfg); tg = time.time() - t
    t = time.time(); ref = oracle.multiply(a, b, impl=impl, nthreads=0 if impl == "reference" else 1); tc = time.time() - t
    ok_rp = np.array_equal(res.c.rowptr, ref.rowptr)
    ok_ci = np.array_equal(res.c.colids, ref.colids)
    ok_v = ok_ci and np.all(np.abs(res.c.values - ref.values) <= 1e-12 * np.maximum(np.maximum(abs(res.c.values), abs(ref.values)), 1e-300))
    print(f"{name}: flop={ref.flop} nnz={ref.colids.size} rowptr={ok_rp} colids={ok_ci} vals={ok_v} "
          f"gpu_wall={tg:.3f}s cpu={tc:.3f}s phases={ {k: round(v*1e3,3) for k,v in res.phases.items()} } bins={res.report["gpu_bins"]} fb={res.report["sort_fallbacks"]}", flush=True)
    return ok_rp and ok_ci and ok_v

ok = True
for scale, d in [(4, 2), (8, 3), (12, 4)]:
    csr = M.make_matrix("er", scale, d, 5); ok &= check(f"er{scale}d{d}", M.csr_to_csc(csr), csr)
for bc in (256, 1024):
    csr = M.make_matrix("er", 10, 6, 2); ok &= check(f"er10 cap{bc}", M.csr_to_csc(csr), csr, api.PbConfig(bin_cap=bc))
csr = M.make_matrix("rmat", 10, 4, 7); ok &= check("rmat10", M.csr_to_csc(csr), csr)
for sc in (13, 15):
    csr = M.make_matrix("rmat", sc, 16, 7); ok &= check(f"rmat{sc} (heavy rows)", M.csr_to_csc(csr), csr)
csr = M.make_matrix("er", 11, 8, 3); ok &= check("er11 cap64 (many heavy)", M.csr_to_csc(csr), csr, api.PbConfig(bin_cap=64))
import numpy as np
K, n = 6000, 512
a = M.coo_to_csr(4, K, np.r_[np.zeros(K, int), [1, 2]], np.r_[np.arange(K), [0, 1]], np.r_[np.linspace(0.5, 1.5, K), [2.0, 3.0]])
rows = np.r_[np.arange(K), np.arange(K)]; cols = np.r_[np.zeros(K, int), np.arange(K) % 100 + 1]
b = M.coo_to_csr(K, n, rows, cols, np.linspace(1.0, 2.0, 2 * K))
ok &= check("uniform-key column", M.csr_to_csc(a), b)
a, b = M.make_config("C1"); ok &= check("C1", a, b)
s = M.stencil27(16); ok &= check("stencil16", M.csr_to_csc(s), s)
if "--big" in sys.argv:
    a, b = M.make_config("C2"); ok &= check("C2", a, b, impl="reference")
print("ALL OK" if ok else "FAILURES")
