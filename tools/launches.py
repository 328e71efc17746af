"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[start]; idx = {k: i for i, k in enumerate(h)}
agg = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) < len(h):
        continue
    name = r[idx['Kernel Name']].split('(')[0][:48]
    v = float(r[idx['Metric Value']])
    unit = r[idx['Metric Unit']]
    if unit == 'msecond': v *= 1e6
    elif unit == 'usecond': v *= 1e3
    agg.setdefault(name, []).append(v)
for k, v in agg.items():
    print(f"{k:50s} n={len(v):3d} mean={sum(v)/len(v)/1e3:9.1f} us  total={sum(v)/1e3:9.1f} us")
