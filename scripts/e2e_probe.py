"""Breakdown of one host-API multiply (pinned host buffers): H2D, compute, D2H."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2002_11302_b200 import api, matrices as M
cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C2"
a, b = M.make_config(cfg_name)
pin = lambda x: torch.from_numpy(x).pin_memory().numpy()
ah = M.CscMatrix(a.nrows, a.ncols, pin(a.colptr), pin(a.rowids), pin(a.values))
bh = M.CsrMatrix(b.nrows, b.ncols, pin(b.rowptr), pin(b.colids), pin(b.values))
r0 = api.pb_multiply(ah, bh, api.PbConfig(), symbolic=False)
nnz = r0.c.nnz
out = (torch.empty(a.nrows + 1, dtype=torch.int64).pin_memory().numpy().view(np.uint64),
       torch.empty(nnz, dtype=torch.int32).pin_memory().numpy().view(np.uint32),
       torch.empty(nnz, dtype=torch.float64).pin_memory().numpy())
for i in range(4):
    t0 = time.perf_counter()
    r = api.pb_multiply(ah, bh, api.PbConfig(), symbolic=False, out=out)
    t = time.perf_counter() - t0
    ph = r.phases
    print(f"wall {t*1e3:.2f} ms", {k: round(v * 1e3, 2) if isinstance(v, float) else v for k, v in ph.items()})
# raw PCIe probe
x = torch.empty(int(3.2e9) // 8, dtype=torch.float64, device="cuda")
h = torch.empty_like(x, device="cpu").pin_memory()
torch.cuda.synchronize(); t0 = time.perf_counter(); h.copy_(x); torch.cuda.synchronize()
print("raw D2H GB/s", x.numel() * 8 / (time.perf_counter() - t0) / 1e9)
t0 = time.perf_counter(); x.copy_(h); torch.cuda.synchronize()
print("raw H2D GB/s", x.numel() * 8 / (time.perf_counter() - t0) / 1e9)
# begin / fetch split
import ctypes as C
from paper_2002_11302_b200 import _native
lib = _native.pbg()
for i in range(3):
    va = api._view(a.nrows, a.ncols, ah.colptr, ah.rowids, ah.values)
    vb = api._view(b.nrows, b.ncols, bh.rowptr, bh.colids, bh.values)
    cc = api.PbConfig().to_c(); h = C.c_void_p(); nz = C.c_uint64(0)
    t0 = time.perf_counter()
    rc = lib.pbg_multiply_begin(C.byref(va), C.byref(vb), C.byref(cc), C.byref(h), C.byref(nz))
    t1 = time.perf_counter()
    rep = _native.Report()
    rc2 = lib.pbg_multiply_fetch(h, out[0].ctypes.data, out[1].ctypes.data, out[2].ctypes.data, C.byref(rep))
    t2 = time.perf_counter()
    lib.pbg_release(h)
    t3 = time.perf_counter()
    print(f"begin {1e3*(t1-t0):.2f} ms fetch {1e3*(t2-t1):.2f} ms release {1e3*(t3-t2):.2f} ms  (h2d {rep.t_h2d*1e3:.2f} total {rep.t_total*1e3:.2f} d2h {rep.t_d2h*1e3:.2f})")
