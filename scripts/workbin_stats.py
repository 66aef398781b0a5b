"""Work-bin statistics of one device-resident multiply (development aid):
how the sort kernel's units of work split by kind, size, key range and
duplicate ratio. Usage as profile_step.py (--config / --rmat / --row-band)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2002_11302_b200 import api, matrices as M

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--rmat", type=int, nargs=2, default=None)
ap.add_argument("--row-from", type=float, default=0.0, help="first row of the band, as a fraction of the rows")
ap.add_argument("--row-band", type=float, default=1.0)
args = ap.parse_args()
if args.rmat:
    b = M.make_matrix("rmat", args.rmat[0], args.rmat[1], seed=1)
    a = M.csr_to_csc(b)
else:
    a, b = M.make_config(args.config)
if args.row_band < 1.0:
    r0 = int(a.nrows * args.row_from)
    a = M.row_band(a, r0, min(a.nrows, r0 + int(a.nrows * args.row_band)))
dev = torch.device("cuda", 0)
t = lambda x, dt: torch.from_numpy(x.view(dt)).to(dev)
A = (t(a.colptr, np.int64), t(a.rowids, np.int32), t(a.values, np.float64))
B = (t(b.rowptr, np.int64), t(b.colids, np.int32), t(b.values, np.float64))
ctx = api.DeviceContext(0)
va = ctx.view(a.nrows, a.ncols, *A); vb = ctx.view(b.nrows, b.ncols, *B)
nnz, rep = ctx.multiply(va, vb, api.PbConfig(device=0))
n, kb, fl, dz = ctx.workbins()
n = n.astype(np.int64); dz = dz.astype(np.int64)
print("work bins", len(n), "tuples", int(n.sum()), "distinct", int(dz.sum()), "flop", rep["flop"], "nnz", nnz)
merged = (fl & 2) != 0
heavy = (fl & 4) != 0
def show(name, sel):
    if not sel.any():
        print(name, "none"); return
    nn, dd, kk = n[sel], dz[sel], kb[sel]
    print(f"{name}: bins {sel.sum()} tuples {nn.sum()} ({nn.sum()/max(1,n.sum()):.3f}) distinct {dd.sum()} "
          f"cf {nn.sum()/max(1,dd.sum()):.2f} mean n {nn.mean():.0f}")
    print("   n quantiles", np.quantile(nn, [0, .1, .25, .5, .75, .9, 1]).astype(int).tolist())
    print("   keybits hist (tuple-weighted):", {int(k): round(float(nn[kk == k].sum() / nn.sum()), 3) for k in np.unique(kk)})
    r = dd / np.maximum(nn, 1)
    for lo, hi in [(0, .25), (.25, .5), (.5, .75), (.75, .999), (.999, 1.01)]:
        s2 = (r >= lo) & (r < hi)
        print(f"   distinct/n in [{lo},{hi}): bins {s2.sum()} tuples {nn[s2].sum()/nn.sum():.3f}")
show("merged (dense-reduced)", merged)
show("regular bins", ~heavy & ~merged)
show("heavy sub-bins (sorted)", heavy & ~merged)
hs = heavy & ~merged
for lo, hi in [(0, 256), (256, 1024), (1024, 2048), (2048, 3072), (3072, 4097)]:
    s2 = hs & (n >= lo) & (n < hi)
    print(f"   heavy sub-bins n in [{lo},{hi}): bins {s2.sum()} tuples {n[s2].sum()}")
s0 = hs & (kb <= 12)
print("   heavy sub-bins with keybits <= 12: bins", s0.sum(), "tuples", n[s0].sum())
