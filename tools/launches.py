"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; out = []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            v = float(d['Metric Value'].replace(',', ''))
            u = d['Metric Unit']
            v = v * {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}.get(u, 1e-3)
            out.append((d['Kernel Name'].split('(')[0].replace('void ', '')[:60], v))
tot = sum(v for _, v in out)
agg = collections.OrderedDict()
for k, v in out:
    agg.setdefault(k, [0, 0.0]); agg[k][0] += 1; agg[k][1] += v
print(f"{len(out)} launches, total {tot/1e3:.3f} ms")
for k, (c, v) in agg.items():
    print(f"{v/1e3:9.3f} ms {100*v/tot:5.1f}%  x{c:<3d} {k}")
