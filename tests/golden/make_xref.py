"""Full-size X_ref fixtures for BASELINE configs c1-c4, produced by the REFERENCE itself.

Run here, where /root/reference exists (the reference build oracle/_ref is made by
oracle/Makefile from /root/reference/proj/src, unmodified):

    make -C oracle && python tests/golden/make_xref.py c1 c2 c3 c4

For each config the inputs come from generator v1 (paper_2412_15840_b200/configs.py) through the
bit-identical copy in the reference shim (``oracle.Ref().randn``; for c1/c3/c4 B is generated
inside the shim so an 8.6 GB host copy is avoided), so the product library is never loaded. The
reference ``ndsylv::solve`` (sylvester.cpp:167-227, its own Schur, all host threads) gives X_ref.
The fixture ``xref_<cfg>.npz`` (small enough to commit) holds:

* ``idx``/``x``: 65,536 seeded random flat (column-major) indices plus the first and last 512
  entries, and X_ref at them;
* ``xmax``: ||X_ref||_max;
* ``sum_first``/``sum_last``: X_ref summed over all modes but the first / the last (n_1 and n_N
  complex values — together they touch every entry, a checksum of checksums);
* the seed, generator version, reference build flags, thread count, stage seconds and min |den|.

tests/test_gpu_fullsize.py compares the GPU solve of the same inputs with it at the north_star
tolerance (relative max-norm 1e-9).
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2412_15840_b200 import configs  # noqa: E402

N_SAMPLES = 65536
EDGE = 512
SEED = 0
BUILD = "/usr/bin/g++ -std=c++20 -O3 -DNDEBUG -fopenmp (no -march), oracle/Makefile"


def sample_indices(total, seed=12345):
    rng = np.random.default_rng(seed)
    idx = rng.choice(total, size=min(N_SAMPLES, total), replace=False)
    edges = np.concatenate([np.arange(min(EDGE, total)), np.arange(max(total - EDGE, 0), total)])
    return np.unique(np.concatenate([idx, edges]).astype(np.int64))


def make(name):
    ref = oracle.Ref()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    dims = configs.CONFIGS[name]["dims"]
    kind = configs.CONFIGS[name]["kind"]
    if kind == "advdiff":
        a_list, b = configs.make_problem(name, SEED, randn=ref.randn)
    else:
        a_list = configs.gauss_coefficients(dims, SEED, configs.CONFIGS[name]["scaled"], randn=ref.randn)
        b = None  # generated inside the shim: identical to configs.gauss_rhs(dims, SEED)
    t0 = time.perf_counter()
    x, rep = ref.solve_gen(a_list, dims, SEED, b)
    wall = time.perf_counter() - t0
    del b
    flat = x.reshape(-1, order="F")
    idx = sample_indices(flat.size)
    out = {
        "dims": np.array(dims, dtype=np.int64), "idx": idx, "x": flat[idx].copy(),
        "xmax": np.abs(flat).max(),
        "sum_first": x.sum(axis=tuple(range(1, x.ndim))),
        "sum_last": x.sum(axis=tuple(range(0, x.ndim - 1))),
        "seed": SEED, "generator": configs.GENERATOR_VERSION,
        "meta": json.dumps({"config": name, "build": BUILD, "threads": threads, "wall_seconds": wall,
                            "report": rep}),
    }
    path = os.path.join(HERE, f"xref_{name}.npz")
    np.savez_compressed(path, **out)
    print(name, "done in", round(wall, 1), "s;", {k: rep[k] for k in ("transform_seconds", "backsub_seconds",
                                                                       "inverse_seconds", "min_abs_denominator")},
          flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c1", "c2", "c3", "c4"]:
        make(name)
