"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
python scripts/ncu_launches.py file.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    v = float(d['Metric Value'].replace(',', ''))
    v *= {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6}.get(d.get('Metric Unit'), 1)
    k = d['Kernel Name'][:60]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(t for _, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print("%-60s %4d %10.1f us %5.1f%%" % (k, n, t / 1e3, 100 * t / tot))
print("total %.1f us" % (tot / 1e3))
