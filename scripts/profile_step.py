"""One warm-up + N multiplies of a config on cuda:0 (for ncu captures)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2002_11302_b200 import api, matrices as M

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--bin-cap", type=int, default=0)
ap.add_argument("--rmat", type=int, nargs=2, metavar=("SCALE", "EF"), default=None,
                help="C = A*A for a seeded RMAT matrix instead of a config (single pass)")
ap.add_argument("--row-from", type=float, default=0.0, help="first row of the band, as a fraction of the rows")
ap.add_argument("--row-band", type=float, default=1.0,
                help="multiply only the first fraction of A's rows (one bounded round)")
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
cfg = api.PbConfig(device=0, bin_cap=args.bin_cap)
for i in range(1 + args.steps):
    try:
        nnz, rep = ctx.multiply(va, vb, cfg)
    except Exception as e:  # diagnostic variants (PBG_DIAG_*) produce wrong output on purpose
        print("multiply failed:", e, flush=True)
        continue
    print({k: (round(v * 1e3, 4) if isinstance(v, float) else v) for k, v in rep.items()}, flush=True)
