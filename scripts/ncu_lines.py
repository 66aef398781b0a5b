"""Per-CUDA-source-line totals (instructions executed, stall samples) from
`ncu -i REP --page source --csv --print-source cuda,sass -k KERNEL`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None; hdr = None; out = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] in ("", "Function Name"): continue
    d = dict(zip(hdr[2:], r[4:])) if False else None
    try:
        samp = int(r[4] or 0); inst = int(r[7] or 0)
    except ValueError:
        continue
    out.append((inst, samp, fname, r[0], r[1][:90]))
ti = sum(o[0] for o in out) or 1; ts = sum(o[1] for o in out) or 1
print(f"total inst {ti:.3e} samples {ts}")
for o in sorted(out, key=lambda o: -(o[0] / ti + o[1] / ts))[:top]:
    print(f"{100*o[0]/ti:5.1f}%i {100*o[1]/ts:5.1f}%s {o[2]}:{o[3]} {o[4]}")
