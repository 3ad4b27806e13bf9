"""Regenerate the golden fixtures from the REFERENCE itself (oracle/_ref, built from
/root/reference/proj/src by oracle/Makefile). Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Every instance is the reference's own: its xoshiro256++ `random_problem` seeds from
test_sylvester.cpp / acceptance.cpp, plus BASELINE config c0 from generator v1. Outputs are the
reference's Schur factors, forward transform, back-substitution and solution.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2412_15840_b200 import configs  # noqa: E402


def dump(name, a_list, b, ref, extra=None):
    us, ts = zip(*[ref.schur(a) for a in a_list])
    c = ref.forward_transform(us, b)
    y, st = ref.back_substitute(ts, c)
    x, rep = ref.solve(a_list, b)
    out = {"dims": np.array(b.shape, dtype=np.int64), "b": b, "c": c, "y": y, "x": x,
           "backsub_multiplies": st["multiplies"], "min_abs_denominator": st["min_abs_denominator"]}
    for j, (a, u, t) in enumerate(zip(a_list, us, ts)):
        out[f"a{j}"] = a
        out[f"u{j}"] = u
        out[f"t{j}"] = t
    out.update(extra or {})
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, b.shape, "multiplies", st["multiplies"])


def main():
    ref = oracle.Ref()
    for dims, seed in [((5, 4, 3), 905), ((3, 4, 2), 906), ((4, 4, 4), 908), ((2, 9, 33), 42), ((2,) * 8, 918),
                       ((7, 1, 5), 77)]:
        a, x_true, b = ref.random_problem(list(dims), seed)
        extra = {"x_true": x_true}
        if np.prod(dims) <= 4096:
            extra["x_kron"] = ref.oracle_solve(a, b)
        dump("ref_%s_s%d" % ("x".join(map(str, dims)), seed), a, b, ref, extra)
    a, b = configs.make_problem("c0", seed=0)
    dump("c0_seed0", a, b, ref, {"generator": np.array(configs.GENERATOR_VERSION)})
    a, b = configs.make_problem("c2", dims=(12, 12, 12, 12))
    dump("advdiff_n12_N4", a, b, ref)


if __name__ == "__main__":
    main()
