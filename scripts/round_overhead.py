"""Per-round time of a bounded-memory round against its phase sum (development
aid): what the slab extraction, the symbolic pass and the host round trips add
to expand + count + sort. Usage: round_overhead.py CONFIG ROUNDS [q ...]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2002_11302_b200 import api, matrices as M

name, rounds = sys.argv[1], int(sys.argv[2])
qs = [int(x) for x in sys.argv[3:]] or [0, rounds // 2, rounds - 1]
a, b = M.make_config(name)
dev = torch.device("cuda", 0)
t = lambda x, dt: torch.from_numpy(x.view(dt)).to(dev)
A = (t(a.colptr, np.int64), t(a.rowids, np.int32), t(a.values, np.float64))
B = (t(b.rowptr, np.int64), t(b.colids, np.int32), t(b.values, np.float64))
ctx = api.DeviceContext(0)
va = ctx.view(a.nrows, a.ncols, *A); vb = ctx.view(b.nrows, b.ncols, *B)
cuts, _ = ctx.band_cuts(va, vb, rounds)
cfg = api.PbConfig(device=0)
for q in qs:
    for rep_i in range(2):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        _, rep = ctx.multiply_band(va, vb, int(cuts[q]), int(cuts[q + 1]), cfg, 0)
        e1.record(); torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    ph = {k: round(rep[k] * 1e3, 2) for k in ("t_symbolic", "t_expand", "t_count", "t_sortmerge_kernel", "t_total")}
    print(f"round {q}: rows [{cuts[q]},{cuts[q+1]}) flop {rep['flop']:.3e} wall(events) {tot:.2f} ms phases {ph} "
          f"untracked {tot - ph['t_total']:.2f} ms", flush=True)
