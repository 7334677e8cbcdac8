"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d['Metric Name'] == 'gpu__time_duration.sum':
            v = float(d['Metric Value']) * (1e-3 if d.get('Metric Unit') == 'nsecond' else 1.0)
            agg.setdefault(d['Kernel Name'][:70], []).append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in agg.items():
    print(f"{k:70s} n={len(v):4d} mean={sum(v)/len(v):9.2f}us tot={sum(v):10.1f}us {100*sum(v)/tot:5.1f}%")
