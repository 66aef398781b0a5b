"""Print the pbg_report counters (bins, heavy bins, LSD fallbacks, premerged
bins, tuples, merged) and phase times of one device-resident multiply
(development aid). Usage: report_config.py CONFIG | rmat SCALE EF."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2002_11302_b200 import api, matrices as M  # noqa: E402

if sys.argv[1] == "rmat":
    csr = M.make_matrix("rmat", int(sys.argv[2]), int(sys.argv[3]), seed=1)
    a, b = M.csr_to_csc(csr), csr
else:
    a, b = M.make_config(sys.argv[1])
dev = torch.device("cuda", 0)
t = lambda x, dt: torch.from_numpy(x.view(dt)).to(dev)  # noqa: E731
A = (t(a.colptr, np.int64), t(a.rowids, np.int32), t(a.values, np.float64))
B = (t(b.rowptr, np.int64), t(b.colids, np.int32), t(b.values, np.float64))
ctx = api.DeviceContext(0)
va = ctx.view(a.nrows, a.ncols, *A)
vb = ctx.view(b.nrows, b.ncols, *B)
for _ in range(2):
    nnz, rep = ctx.multiply(va, vb, api.PbConfig(device=0))
keep = ("gpu_bins", "heavy_bins", "sort_fallbacks", "premerged_bins", "tuples_into_sort",
        "merged_total", "flop", "nnz_c")
print({k: rep[k] for k in keep if k in rep})
print({k: round(v * 1e3, 3) for k, v in rep.items() if k.startswith("t_")})
