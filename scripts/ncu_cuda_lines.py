"""Per-CUDA-source-line totals (warp instructions executed, stall samples)
from `ncu -i REP --page source --csv --print-source cuda,sass -k K -c 1`."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None; hdr = None; line = None; src = {}
inst = defaultdict(int); samp = defaultdict(int)
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; ix = {h: i for i, h in enumerate(hdr)}; continue
    if hdr is None or r[0] == "Function Name": continue
    if r[0]:
        line = (fname, r[0]); src[line] = r[1].strip()[:90]
    if len(r) > ix["Instructions Executed"] and r[2]:
        try:
            inst[line] += int(r[ix["Instructions Executed"]] or 0)
            samp[line] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            pass
ti = sum(inst.values()) or 1; ts = sum(samp.values()) or 1
print(f"total warp inst {ti:.4e} samples {ts}")
keys = sorted(inst, key=lambda k: -(inst[k] / ti + samp[k] / ts))[:top]
for k in keys:
    print(f"{100*inst[k]/ti:5.1f}%i {100*samp[k]/ts:5.1f}%s {k[0]}:{k[1]} {src.get(k,'')}")
