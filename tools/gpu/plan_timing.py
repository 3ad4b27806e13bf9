"""Host wall time of plan creation (factor upload, singular scan, diagonalisation) per config."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2412_15840_b200 as nds
from paper_2412_15840_b200 import configs
ctx = nds.Context(0)
for name in sys.argv[1:] or ["c1"]:
    a, b = configs.make_problem(name, seed=0)
    us, ts = zip(*[ctx.schur(m) for m in a])
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p = ctx.plan(list(us), list(ts))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(name, "plan create ms", round((t1 - t0) * 1e3, 3), p.diagonalised(), p.superblocks())
        p.close()
