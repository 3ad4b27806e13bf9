"""Summarise an ncu report's source page: stall reasons, hottest instructions, shared-memory
wavefronts vs ideal.  usage: python tools/ncu_source_summary.py report.ncu-rep [min_frac]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


tot = sum(num(r[si]) for r in data)
st = {c: sum(num(r[h.index(c)]) for r in data) for c in cols}
print("samples", int(tot), "stalls:", ", ".join(f"{c[6:]} {v / tot:.0%}" for c, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
wi, ii = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
print("smem wavefronts", int(sum(num(r[wi]) for r in data)), "ideal", int(sum(num(r[ii]) for r in data)))
ex = h.index("Instructions Executed")
print("instructions executed", int(sum(num(r[ex]) for r in data)))
for i, r in enumerate(data):
    if num(r[si]) > tot * min_frac:
        top = sorted(((num(r[h.index(c)]), c[6:]) for c in cols), reverse=True)[:2]
        print(f"{i:5d} {num(r[si]) / tot:5.1%} {r[1].strip()[:60]:60s} exec {r[ex]:>8s} wf {r[wi]:>8s}/{r[ii]:>8s} {top}")
