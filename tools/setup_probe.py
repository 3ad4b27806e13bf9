import time, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2412_15840_b200 as nds
from paper_2412_15840_b200 import configs
ctx = nds.Context(0)
a, b = configs.make_problem("c1", seed=0)
us, ts = zip(*[ctx.schur(m) for m in a]); us=list(us); ts=list(ts)
pb = torch.from_numpy(np.ascontiguousarray(b.ravel(order="F"))).pin_memory()
px = torch.empty_like(pb).pin_memory()
for i in range(8):
    t0=time.perf_counter(); p = ctx.plan(us, ts); t1=time.perf_counter()
    rep = p.execute_host_ptr(pb.data_ptr(), px.data_ptr()); t2=time.perf_counter()
    p.close(); t3=time.perf_counter()
    print(f"plan_create {1e3*(t1-t0):.2f} ms, execute_host {1e3*(t2-t1):.2f} ms (h2d {rep['h2d_seconds']*1e3:.2f} fwd {rep['transform_seconds']*1e3:.2f} bs {rep['backsub_seconds']*1e3:.2f} inv {rep['inverse_seconds']*1e3:.2f} d2h {rep['d2h_seconds']*1e3:.2f}), destroy {1e3*(t3-t2):.2f} ms")
