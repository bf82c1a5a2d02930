"""Shared-memory wavefronts per SASS instruction of an ncu report (source page), top N."""
import csv, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
f = lambda d, k: float(d.get(k) or 0)
tot = sum(f(d, "L1 Wavefronts Shared") for d in data)
print("total shared wavefronts", tot)
for d in sorted(data, key=lambda d: -f(d, "L1 Wavefronts Shared"))[:n]:
    print(d["Address"][-5:], int(f(d, "L1 Wavefronts Shared")), "ideal", int(f(d, "L1 Wavefronts Shared Ideal")),
          "exec", int(f(d, "Instructions Executed")), d["Source"].strip()[:70])
import collections
agg = collections.defaultdict(lambda: [0, 0, 0])
for d in data:
    op = d["Source"].strip().split(" ")[0]
    if f(d, "L1 Wavefronts Shared") > 0:
        a = agg[op]
        a[0] += f(d, "L1 Wavefronts Shared"); a[1] += f(d, "L1 Wavefronts Shared Ideal"); a[2] += f(d, "Instructions Executed")
for op, (w, i, e) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{op:12s} wavefronts {w:.3e} ideal {i:.3e} instr {e:.3e}")
