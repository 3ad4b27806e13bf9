"""Aggregate an ncu report's SASS-level samples, instructions and shared wavefronts by CUDA
source line.  usage: python tools/ncu_lines_by_source.py report.ncu-rep [min_frac]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
min_frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.006
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if r and r[0] == "Line No")
si, ie, iw = (h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"),
              h.index("L1 Wavefronts Shared"))


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


agg, cur, fname = {}, None, ""
for r in rows:
    if not r or r[0] in ("Function Name", "Line No"):
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0]:
        try:
            cur = (fname, int(r[0]), r[1][:90])
        except ValueError:
            continue
        agg.setdefault(cur, [0, 0, 0])
    elif cur and len(r) > si:
        agg[cur][0] += num(r[si])
        agg[cur][1] += num(r[ie])
        agg[cur][2] += num(r[iw])
tot = sum(v[0] for v in agg.values()) or 1
print(f"samples {int(tot)}, instructions {int(sum(v[1] for v in agg.values()))}, "
      f"shared wavefronts {int(sum(v[2] for v in agg.values()))}")
for k, v in sorted(agg.items()):
    if v[0] / tot > min_frac:
        print(f"{k[0][:14]:14s}{k[1]:5d} {v[0] / tot:6.1%} inst {int(v[1]):9d} wf {int(v[2]):8d}  {k[2]}")
