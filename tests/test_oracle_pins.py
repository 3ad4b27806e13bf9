"""Pin the plain-C oracle (oracle/ndsylv_oracle.c) to the reference library itself (oracle/_ref,
compiled from /root/reference/proj/src) — bit for bit — and restate the reference's own
known-answer tests (test_sylvester.cpp, test_kernels.cpp) against the oracle. CPU only."""
import numpy as np
import pytest

import oracle


def _factors(ref, a_list):
    us, ts = zip(*[ref.schur(a) for a in a_list])
    return list(us), list(ts)


@pytest.mark.parametrize("dims,seed", [((5, 4, 3), 905), ((3, 4, 2), 906), ((2, 9, 33), 42), ((2,) * 9, 919),
                                       ((6, 5, 4), 14), ((1, 3, 1, 2), 3), ((17, 3), 5)])
def test_port_matches_reference_bitwise(port, ref, dims, seed):
    a, x_true, b = ref.random_problem(list(dims), seed)
    us, ts = _factors(ref, a)
    for mode in range(1, len(dims) + 1):
        assert np.array_equal(port.mode_product(a[mode - 1], mode, x_true), ref.mode_product(a[mode - 1], mode, x_true))
        assert np.array_equal(ref.mode_product(a[mode - 1], mode, x_true),
                              ref.mode_product(a[mode - 1], mode, x_true, serial_twin=True))
    c = ref.forward_transform(us, b)
    assert np.array_equal(port.forward_transform(us, b), c)
    assert np.array_equal(port.inverse_transform(us, c), ref.inverse_transform(us, c))
    y_r, st_r = ref.back_substitute(ts, c)
    y_p, st_p = port.back_substitute(ts, c)
    assert np.array_equal(y_p, y_r)
    assert st_p == st_r
    assert np.array_equal(port.apply_operator(a, x_true), ref.apply_operator(a, x_true))
    if len(dims) >= 2:
        x_r, rep_r = ref.solve(a, b)
        x_p, rep_p = port.solve_schur(us, ts, b)
        assert np.array_equal(x_p, x_r)
        for k in ("backsub_multiplies", "backsub_entries", "min_abs_denominator", "used_normal_fast_path",
                  "flop_estimate", "schur_flop_estimate"):
            assert rep_p[k] == rep_r[k], k


def test_port_singular_matches_reference(port, ref):
    # test_sylvester.cpp:110-125: the first singular pair in descending order is (2, 2)
    ts = [np.diag([1.0, -1.0]).astype(complex), np.diag([-1.0, 1.0]).astype(complex)]
    c = np.ones((2, 2), dtype=complex)
    for impl in (port, ref):
        with pytest.raises(oracle.OracleError) as ei:
            impl.back_substitute(ts, c, 0.0)
        assert ei.value.code == 2
        assert ei.value.bad_index == [2, 2]
        assert abs(ei.value.bad_den) == 0.0


def test_known_answers_on_port(port):
    # test_sylvester.cpp:57-69 — diagonal factors divide by eigenvalue sums
    c = np.array([6.0, 8.0, 10.0, 12.0], dtype=complex).reshape((2, 2), order="F")
    ts = [np.diag([1.0, 2.0]).astype(complex), np.diag([10.0, 20.0]).astype(complex)]
    y, st = port.back_substitute(ts, c)
    assert np.allclose(y.ravel(order="F"), [6 / 11, 8 / 12, 10 / 21, 12 / 22], atol=1e-15, rtol=0)
    assert st["entries"] == 4 and st["min_abs_denominator"] == pytest.approx(11.0)
    # :71-85 — hand-worked 2x1
    c = np.array([5.0, 6.0], dtype=complex).reshape((2, 1), order="F")
    ts = [np.array([[1.0, 1.0], [0.0, 2.0]], dtype=complex), np.array([[3.0]], dtype=complex)]
    y, st = port.back_substitute(ts, c)
    y2 = 6.0 / 5.0
    assert abs(y[1, 0] - y2) <= 1e-15 and abs(y[0, 0] - (5.0 - y2) / 4.0) <= 1e-15
    assert st["multiplies"] == 1
    # :260-270 — flop estimates
    assert port.flop_estimate([2, 2]) == 76
    assert port.flop_estimate([3, 3, 3]) == 27 * (45 - 3 + 1)
    assert port.flop_estimate([1_000_000] * 4) == -1
    assert port.schur_flop_estimate([2, 9, 33]) == 25 * (8 + 729 + 35937)


def test_first_entry_and_multiply_count(port, ref):
    # test_sylvester.cpp:87-108 uses xoshiro draws for the strictly-upper part
    u = ref.xoshiro_uniform(903, 200)
    k = 0
    ts = []
    for n in (3, 4):
        t = np.zeros((n, n), dtype=complex)
        for j in range(n):
            for i in range(j):
                t[i, j] = complex(u[k], u[k + 1])
                k += 2
            t[j, j] = complex(3.0 + j, 1.0)
        ts.append(t)
    c = (u[k:k + 24:2] + 1j * u[k + 1:k + 24:2]).reshape((3, 4), order="F")
    y, st = port.back_substitute(ts, c)
    den = ts[0][2, 2] + ts[1][3, 3]
    assert abs(y[2, 3] - c[2, 3] / den) <= 1e-15
    assert st["entries"] == 12 and st["multiplies"] == 30


def test_identity_coefficients_bitwise(port):
    # test_sylvester.cpp:127-154 — N=2 identity: X = B/2 bitwise through the fast path
    rng = np.random.default_rng(904)
    b = rng.random((3, 4)) + 1j * rng.random((3, 4))
    eye = [np.eye(3, dtype=complex), np.eye(4, dtype=complex)]
    x, rep = port.solve_schur(eye, eye, b)
    assert rep["used_normal_fast_path"] == 1
    assert np.array_equal(x, b / 2.0)


def test_xoshiro_stream_matches_reference(port, ref):
    assert np.array_equal(port.xoshiro_uniform(12345, 1000), ref.xoshiro_uniform(12345, 1000))


def test_binary_ladder_multiplies(port, ref):
    # test_sylvester.cpp:181-190 — multiplies = 2^(N-1) N
    for n_modes in (2, 5, 8):
        dims = [2] * n_modes
        a, x_true, b = ref.random_problem(dims, 910 + n_modes)
        us, ts = _factors(ref, a)
        x, rep = port.solve_schur(us, ts, b)
        assert rep["backsub_multiplies"] == (1 << (n_modes - 1)) * n_modes
        assert np.max(np.abs(x - x_true)) <= 1e-12
