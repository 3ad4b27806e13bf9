"""Per-launch device times (CUDA events recorded by the library) for one solve of a config."""
import argparse
import json
import os
import sys
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_15840_b200 as nds  # noqa: E402
from paper_2412_15840_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--dims", default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=None)
args = ap.parse_args()
dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else None
ctx = nds.Context(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ctx.set_stream(s.cuda_stream)
a, b = configs.make_problem(args.config, seed=0, dims=dims)
us, ts = zip(*[ctx.schur(m) for m in a])
plan = ctx.plan(list(us), list(ts))
d_b = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).cuda()
d_x = torch.empty_like(d_b)
d_w = torch.empty_like(d_b)
for _ in range(2):
    plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
torch.cuda.synchronize()
plan.profile_begin(100000)
for _ in range(args.reps):
    plan.execute(d_b.data_ptr(), d_x.data_ptr(), d_w.data_ptr())
recs = plan.profile_end()
n = len(recs) // args.reps
agg = defaultdict(float)
rows = []
for i in range(n):
    ms = sum(recs[i + r * n][2] for r in range(args.reps)) / args.reps
    rows.append((recs[i][0], recs[i][1], ms))
    agg[recs[i][0]] += ms
total = sum(r[2] for r in rows)
print(json.dumps({"config": args.config, "dims": list(b.shape), "launches": n, "total_ms": total,
                  "by_kind_ms": dict(agg)}))
for k, m, ms in rows:
    print(f"{k:18s} {m:5d} {ms:8.4f}")
if args.out:
    with open(args.out, "w") as f:
        json.dump({"rows": rows, "by_kind_ms": dict(agg), "total_ms": total}, f)
