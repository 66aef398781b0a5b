"""Per-kernel time totals of the last multiply in an ncu --csv launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5  # tail fraction = last multiply
hdr = None; ids = []
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x['Metric Name'] != 'gpu__time_duration.sum': continue
        ids.append((int(x['ID']), x['Kernel Name'].split('(')[0], float(x['Metric Value']), x['Metric Unit']))
ids = ids[int(len(ids) * (1 - frac)):]
agg = collections.defaultdict(float); cnt = collections.Counter()
sc = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}
for i, k, v, u in ids:
    agg[k] += v * sc[u]; cnt[k] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda t: -t[1])[:20]:
    print('%-32s %4d %10.1f us %5.1f%%' % (k, cnt[k], v, 100 * v / tot))
print('total %.1f us' % tot)
