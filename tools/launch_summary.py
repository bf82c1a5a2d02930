"""Summarise an ncu --metrics launch list (gpu__time_duration, dram bytes) per kernel."""
import csv, collections, json, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui, mi, ii = (h.index(x) for x in ('Kernel Name', 'Metric Value', 'Metric Unit', 'Metric Name', 'ID'))
per = collections.defaultdict(dict)
scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0, 'second': 1e3}
for r in data:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('void ', '').replace('sofg::dev::', '')
    per[r[ii]]['name'] = name
    per[r[ii]][r[mi]] = float(r[vi].replace(',', '')) * scale.get(r[ui], 1)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in per.values():
    a = agg[d['name']]
    a[0] += 1
    a[1] += d.get('gpu__time_duration.sum', 0.0)
    a[2] += d.get('dram__bytes_read.sum', 0.0) + d.get('dram__bytes_write.sum', 0.0)
tot = sum(v[1] for v in agg.values())
out = {}
print(f"{'ms':>9} {'share':>6} {'launches':>8} {'DRAM GB':>9} {'GB/s':>7}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:9.2f} {100 * v[1] / tot:5.1f}% {v[0]:8d} {v[2] / 1e9:9.2f} {v[2] / 1e6 / v[1] if v[1] else 0:7.0f}  {k}")
    out[k] = {"ms": round(v[1], 3), "launches": v[0], "dram_bytes": v[2], "dram_bytes_per_launch": v[2] / v[0]}
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], 'w'), indent=1)
