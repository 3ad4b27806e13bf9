"""Golden fixtures (tests/golden/*.npz, produced by the reference itself via make_golden.py):
the C oracle reproduces them bit for bit, and generator v1 reproduces the c0 inputs. CPU only;
needs no /root/reference, so it also runs on the GPU box."""
import glob
import os

import numpy as np
import pytest

from paper_2412_15840_b200 import configs

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def load(path):
    z = np.load(path)
    n = len(z["dims"])
    return z, [z[f"a{j}"] for j in range(n)], [z[f"u{j}"] for j in range(n)], [z[f"t{j}"] for j in range(n)]


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_oracle_reproduces_golden(port, path):
    z, a, us, ts = load(path)
    c = port.forward_transform(us, z["b"])
    assert np.array_equal(c, z["c"])
    y, st = port.back_substitute(ts, c)
    assert np.array_equal(y, z["y"])
    assert st["multiplies"] == int(z["backsub_multiplies"])
    assert st["min_abs_denominator"] == float(z["min_abs_denominator"])
    x, rep = port.solve_schur(us, ts, z["b"])
    assert np.array_equal(x, z["x"])
    if "x_true" in z:
        assert np.max(np.abs(x - z["x_true"])) <= 1e-9
    if "x_kron" in z:
        assert np.max(np.abs(x - z["x_kron"])) <= 1e-10


def test_generator_v1_pinned():
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "c0_seed0.npz"))
    a, b = configs.make_problem("c0", seed=0)
    assert np.array_equal(b, z["b"])
    for j in range(3):
        assert np.array_equal(a[j], z[f"a{j}"])
