"""Group an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel: launches, total
time and share. usage: python tools/launch_shares.py launches.csv [header-comment]"""
import csv
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]  # skip ncu notes and program output
rows = list(csv.reader(lines))
h = next(r for r in rows if "Kernel Name" in r)
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].split("<")[0].replace("void ", "").replace("nds::", "")
    v = float(r[iv].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[iu], 1e-6)
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:32s} launches {cnt[k]:5d} {v:10.3f} ms {100 * v / s:6.1f}%")
