"""Summarise NDS_SOLVE_TRACE output (per-level far/near/diag event times of one solve).

usage: NDS_SOLVE_TRACE=1 python tools/profile_step.py --config c1 --reps 1 2> trace.txt
       python tools/solve_trace.py trace.txt
"""
import sys

rows = [l.split()[1:] for l in open(sys.argv[1]) if l.startswith("TRACE ")]
# keep the last solve only
last = []
for r in rows:
    if r[0] == "0":
        last = []
    last.append(r)
print(f"{'lv':>3} {'tiles':>5} {'nf':>5} {'nn':>5} {'far_s':>8} {'far_us':>7} {'near_us':>7} {'wait_us':>7} {'diag_us':>7} {'end':>8}")
tot = {"far": 0.0, "near": 0.0, "diag": 0.0, "wait": 0.0}
prev_end = 0.0
for r in last:
    lv, nt, nf, nn = map(int, r[:4])
    t = list(map(float, r[4:]))
    far = t[1] - t[0] if t[0] >= 0 else 0.0
    near = t[3] - t[2] if t[2] >= 0 else 0.0
    crit_ready = t[3] if t[2] >= 0 else prev_end
    wait = t[4] - crit_ready
    diag = t[5] - t[4]
    tot["far"] += far
    tot["near"] += near
    tot["diag"] += diag
    tot["wait"] += max(0.0, wait)
    print(f"{lv:>3} {nt:>5} {nf:>5} {nn:>5} {t[0]:>8.1f} {far:>7.1f} {near:>7.1f} {wait:>7.1f} {diag:>7.1f} {t[5]:>8.1f}")
    prev_end = t[5]
print("totals (us):", {k: round(v, 1) for k, v in tot.items()}, "end", prev_end)
