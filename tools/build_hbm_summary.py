"""Per-kernel DRAM bytes and GB/s of the build phase from an ncu metrics CSV (tools/build_hbm.sh)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d['ID'], d['Kernel Name'].split('(')[0].replace('void ', '')[:55])
    v = float(d['Metric Value'].replace(',', ''))
    u = d['Metric Unit']
    per.setdefault(key, {})[d['Metric Name']] = v * {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-9,
                                                       'usecond': 1e-6, 'msecond': 1e-3, 'ns': 1e-9, 'us': 1e-6,
                                                       'ms': 1e-3}.get(u, 1)
print("one c4 substep (2x256^3), ncu --metrics dram__bytes_read/write, gpu__time_duration (cold, serialised)")
print(f"{'kernel':58s} {'ms':>8s} {'GB':>8s} {'GB/s':>8s}")
tot_t = tot_b = 0.0
for (i, k), m in per.items():
    if any(s in k for s in ("grav_", "pair_kernel", "list_kernel", "k_grav_finish", "k_gather_gas")):
        break  # the build ends where the force passes begin
    t = m.get('gpu__time_duration.sum', 0.0)
    b = m.get('dram__bytes_read.sum', 0.0) + m.get('dram__bytes_write.sum', 0.0)
    tot_t += t
    tot_b += b
    print(f"{k:58s} {t*1e3:8.3f} {b/1e9:8.3f} {b/t/1e9 if t else 0:8.0f}")
print(f"{'build total':58s} {tot_t*1e3:8.3f} {tot_b/1e9:8.3f} {tot_b/tot_t/1e9:8.0f}")
