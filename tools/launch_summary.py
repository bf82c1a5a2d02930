"""Summarise an ncu --metrics launch list (gpu__time_duration, dram bytes) per kernel.

usage: launch_summary.py LIST.csv [OUT.json [--config JSON] [--exclude k1,k2]]
OUT.json = {"config": {...}, "kernels": {name: {ms, launches, dram_bytes, dram_bytes_per_launch}}}"""
import argparse, csv, collections, json

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("out", nargs="?")
ap.add_argument("--config", default=None)
ap.add_argument("--exclude", default="")
a = ap.parse_args()
excl = [x for x in a.exclude.split(",") if x]
rows = list(csv.reader(open(a.csv)))
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
    if any(d['name'].startswith(x) for x in excl):
        continue
    g = agg[d['name']]
    g[0] += 1
    g[1] += d.get('gpu__time_duration.sum', 0.0)
    g[2] += d.get('dram__bytes_read.sum', 0.0) + d.get('dram__bytes_write.sum', 0.0)
tot = sum(v[1] for v in agg.values())
out = {}
print(f"{'ms':>9} {'share':>6} {'launches':>8} {'DRAM GB':>9} {'GB/s':>7}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]:9.2f} {100 * v[1] / tot:5.1f}% {v[0]:8d} {v[2] / 1e9:9.2f} {v[2] / 1e6 / v[1] if v[1] else 0:7.0f}  {k}")
    out[k] = {"ms": round(v[1], 3), "launches": v[0], "dram_bytes": v[2], "dram_bytes_per_launch": v[2] / v[0]}
tb = sum(v[2] for v in agg.values())
print(f"total {tot:.1f} ms, {tb / 1e9:.1f} GB DRAM, {tb / 1e6 / tot if tot else 0:.0f} GB/s (serialised, cold-cache)")
if a.out:
    json.dump({"config": json.loads(a.config) if a.config else None, "kernels": out,
               "total_ms": tot, "total_dram_bytes": tb}, open(a.out, "w"), indent=1)
