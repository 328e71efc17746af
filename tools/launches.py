"""Summarise an ncu --csv launch list (one or more --metrics): per kernel name,
launch count and the mean of every metric (durations in us, bytes in MB).
    python tools/launches.py gpurun_out/launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
h = rows[start]
idx = {k: i for i, k in enumerate(h)}
vals = collections.OrderedDict()   # name -> metric -> {launch id: value}
for r in rows[start + 1:]:
    if len(r) < len(h):
        continue
    name = r[idx['Kernel Name']].split('(')[0][:48]
    metric = r[idx['Metric Name']]
    unit = r[idx['Metric Unit']]
    v = float(r[idx['Metric Value']].replace(',', ''))
    if unit in ('msecond', 'ms'):
        v *= 1e3
    elif unit in ('nsecond', 'ns'):
        v *= 1e-3
    elif unit == 'byte':
        v /= 1e6
    elif unit == 'Kbyte':
        v /= 1e3
    elif unit == 'Gbyte':
        v *= 1e3
    vals.setdefault(name, collections.OrderedDict()).setdefault(metric, {})[r[idx['ID']]] = v
for name, ms in vals.items():
    n = max(len(d) for d in ms.values())
    parts = []
    for m, d in ms.items():
        short = {'gpu__time_duration.sum': 'us', 'dram__bytes_read.sum': 'MB rd',
                 'dram__bytes_write.sum': 'MB wr'}.get(m, m)
        parts.append(f"{sum(d.values()) / len(d):10.1f} {short}")
    print(f"{name:50s} n={n:3d} " + "  ".join(parts))
