"""Golden fixtures (tests/golden/*.npz, produced by the reference itself via make_golden.py):
the C oracle reproduces them bit for bit, and generator v1 reproduces the c0 inputs. CPU only;
needs no /root/reference, so it also runs on the GPU box."""
import glob
import os

import numpy as np
import pytest

from paper_2412_15840_b200 import configs

GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if not os.path.basename(p).startswith("xref_"))


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


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_xref_fixture_metadata(name):
    """The full-size X_ref fixtures (tests/golden/make_xref.py, the reference's own solve) carry
    the generator, seed, extents and enough samples for tests/test_gpu_fullsize.py."""
    import json
    from paper_2412_15840_b200 import configs
    fx = np.load(os.path.join(os.path.dirname(__file__), "golden", f"xref_{name}.npz"))
    assert tuple(fx["dims"]) == tuple(configs.CONFIGS[name]["dims"])
    assert str(fx["generator"]) == configs.GENERATOR_VERSION and int(fx["seed"]) == 0
    idx = fx["idx"]
    assert idx.size >= 65536 and np.all(np.diff(idx) > 0) and idx[0] == 0 and idx[-1] == np.prod(fx["dims"]) - 1
    assert np.all(np.isfinite(fx["x"])) and float(fx["xmax"]) >= np.abs(fx["x"]).max()
    assert fx["sum_first"].shape == (fx["dims"][0],) and fx["sum_last"].shape == (fx["dims"][-1],)
    meta = json.loads(str(fx["meta"]))
    assert meta["config"] == name and meta["report"]["backsub_entries"] == np.prod(fx["dims"])
