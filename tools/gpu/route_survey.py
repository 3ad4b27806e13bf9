"""Guard survey: route taken, bound and X error of the block-diagonalised route against the
oracle on random spectra (tests/test_gpu_parity.py::_spectrum_factors)."""
import os, sys, zlib
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import oracle
import paper_2412_15840_b200 as nds
from test_gpu_parity import _spectrum_factors, rand_c, ROUTE_CASES
from conftest import rel_max
ctx = nds.Context(0); port = oracle.Port()
for seed in range(3):
    for dims, kind in ROUTE_CASES:
        rng = np.random.default_rng(zlib.crc32(f"{kind}{dims}{seed}".encode()))
        us, ts = _spectrum_factors(rng, dims, kind)
        b = rand_c(rng, dims)
        x_ref, _ = port.solve_schur(us, ts, b, flags=0)
        plan = ctx.plan(us, ts, allow_fast_path=False)
        taken, cond = plan.diagonalised()
        x = plan.execute_host(b).x
        print(f"{kind:9s} {'x'.join(map(str, dims)):12s} seed {seed} taken {taken!s:5s} bound {cond:9.3g} "
              f"D {plan.superblocks()[1]} err {rel_max(x, x_ref):.2e}")
        plan.close()
