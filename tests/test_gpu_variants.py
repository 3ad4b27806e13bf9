"""GPU parity of the solve paths that environment switches select (A/B experiments kept in the
library): plain per-target far items, grouped far items (G = 2 / 4 targets per slab read, with
remainder items that accumulate into their slot), k-split far items, the per-hyperplane diagonal
kernel, the separate near-update launches, no head / tail overlap, one far stream and the
dataflow (persistent-kernel) solve. The switches are read once per
process, so each variant runs in a subprocess against the C oracle on cubic-tile shapes with
several blocks per mode (far items, group remainders, truncated groups)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import oracle
import paper_2412_15840_b200 as nds
from paper_2412_15840_b200 import configs
ctx = nds.Context(0)
port = oracle.Port()
out = []
for name, dims in [("c1", (96, 80, 112)), ("c2", (40, 32, 48, 24)), ("c1", (64, 256, 32))]:
    a, b = configs.make_problem(name, seed=5, dims=dims)
    us, ts = zip(*[ctx.schur(m) for m in a])
    r = ctx.solve_schur(list(us), list(ts), b)
    x_ref, _ = port.solve_schur(list(us), list(ts), b)
    err = float(np.max(np.abs(r.x - x_ref)) / np.max(np.abs(x_ref)))
    res = ctx.apply_operator(a, r.x)
    out.append({"dims": dims, "err": err, "res": float(np.linalg.norm(res - b) / np.linalg.norm(b))})
print(json.dumps(out))
"""

VARIANTS = [
    {"NDS_FARGROUP": "plain"},
    {"NDS_FARGROUP": "2"},
    {"NDS_FARGROUP": "4"},
    {"NDS_KSPLIT": "296"},
    {"NDS_DIAG": "wave"},
    {"NDS_NEAR": "kernel"},
    {"NDS_HEAD": "0"},
    {"NDS_FAR2": "0"},
    {"NDS_TAIL": "0"},
    {"NDS_FARGROUP": "plain", "NDS_SOLVE": "split"},    # dataflow (persistent) solve, N = 3
    {"NDS_FARGROUP": "plain", "NDS_SOLVE": "unified"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=[",".join(f"{k}={v}" for k, v in e.items()) for e in VARIANTS])
def test_solve_variant_against_oracle(env):
    full_env = dict(os.environ, **env)
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=full_env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    for case in json.loads(p.stdout.strip().splitlines()[-1]):
        assert case["err"] <= 1e-9, case
        assert case["res"] <= 1e-10, case


def test_plan_graph_replay_in_subprocess():
    """The CUDA-graph replay path of nds_plan_execute (NDS_GRAPH=1) is bitwise-equal to eager."""
    env = dict(os.environ, NDS_GRAPH="1")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", os.path.join(ROOT, "tests", "test_gpu_fullsize.py"),
                        "-k", "graph"], env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]


def test_bench_sharded_mode_runs():
    """bench.py --sharded: the multi-GPU ShardedSolver path (single-member NCCL group here)."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--sharded", "--config", "c0", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["scaling"] == "strong" and line["value"] > 0 and line["config"]["parallelism"] == "sharded x1"
