"""Top SASS instructions of one kernel by executed warp instructions and by
stall samples, from `ncu -i REP --page source --csv --print-source sass -k K`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr): continue
    try:
        data.append((r[ix["Address"]][-5:], r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]] or 0),
                     int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
    except ValueError:
        pass
ti = sum(d[2] for d in data) or 1; ts = sum(d[3] for d in data) or 1
print(f"total warp inst {ti:.4e}  stall samples {ts}")
print("-- by samples")
for d in sorted(data, key=lambda d: -d[3])[:top]:
    print(f"{d[0]} {100*d[2]/ti:5.1f}%i {100*d[3]/ts:5.1f}%s {d[1][:80]}")
if "--inst" in sys.argv:
    print("-- by inst")
    for d in sorted(data, key=lambda d: -d[2])[:top]:
        print(f"{d[0]} {100*d[2]/ti:5.1f}%i {100*d[3]/ts:5.1f}%s {d[1][:80]}")
