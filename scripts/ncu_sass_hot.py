"""Hot SASS lines of one kernel from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.006
h = rows[1]; idx = {k: j for j, k in enumerate(h)}
body = []
for x in rows[2:]:
    if x and x[0] == "Kernel Name": break
    if len(x) == len(h): body.append(x)
S = 'Warp Stall Sampling (All Samples)'; I = 'Instructions Executed'
ts = sum(int(x[idx[S]] or 0) for x in body); ti = sum(int(x[idx[I]] or 0) for x in body)
print("total samples", ts, "inst", ti, "sass lines", len(body))
for j, x in enumerate(body):
    s = int(x[idx[S]] or 0); i = int(x[idx[I]] or 0)
    if s > ts * frac or i > ti * frac:
        print(j, str(s).rjust(7), str(i).rjust(11), x[idx['Source']][:95])
