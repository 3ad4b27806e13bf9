"""SURVEY 8(f) rows 1-2 (ODE propagator, RK4): pin the plain-C restatement (oracle/ndsylv_oracle.c:
orc_triangular_exp, orc_ode_at_schur, orc_rk4) to the reference library itself (oracle/_ref) bit
for bit, and restate the reference's own known-answer tests (test_ode.cpp, test_schur.cpp:118-170)
on the port. CPU only."""
import numpy as np
import pytest

import oracle


def _system(rng, dims, shift=-2.0):
    a = [(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n) + shift * np.eye(n)
         for n in dims]
    b = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    x0 = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    return a, b, x0


@pytest.mark.parametrize("n,seed", [(1, 1), (2, 2), (7, 3), (24, 4)])
def test_triangular_exp_port_matches_reference(port, ref, n, seed):
    rng = np.random.default_rng(seed)
    t_mat = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    for t in (0.0, 0.3, -1.7, 2.5):
        assert np.array_equal(port.triangular_exp(t_mat, t), ref.triangular_exp(t_mat, t))
    if n >= 3:  # repeated eigenvalue -> the [6/6] Pade branch (schur.cpp:207-211)
        t2 = t_mat.copy()
        t2[n - 1, n - 1] = t2[0, 0]
        assert np.array_equal(port.triangular_exp(t2, 0.9), ref.triangular_exp(t2, 0.9))


def test_triangular_exp_known_answers(port):
    # test_schur.cpp:118-153: identity at t = 0, diagonal, 2x2 closed form, non-triangular rejected
    t = np.array([[1.0, 2.0], [0.0, 3.0]], dtype=complex)
    assert np.array_equal(port.triangular_exp(t, 0.0), np.eye(2))
    d = np.diag([0.5, -1.0 + 0.25j])
    f = port.triangular_exp(d, 0.5)
    assert np.allclose(np.diag(f), np.exp(0.5 * np.diag(d)), rtol=0, atol=1e-15)
    f = port.triangular_exp(t, 1.0)
    expect12 = 2.0 * (np.exp(3.0) - np.exp(1.0)) / (3.0 - 1.0)
    assert abs(f[0, 1] - expect12) <= 1e-12 * abs(expect12)
    with pytest.raises(oracle.OracleError) as ei:
        port.triangular_exp(np.array([[1.0, 0.0], [1.0, 1.0]], dtype=complex), 1.0)
    assert ei.value.code == 5


@pytest.mark.parametrize("dims,seed", [((3, 2, 2), 40), ((2, 3, 4), 42), ((3, 3), 43), ((2, 2, 2, 2), 44),
                                       ((5, 1, 3), 45)])
def test_ode_port_matches_reference(port, ref, dims, seed):
    rng = np.random.default_rng(seed)
    a, b, x0 = _system(rng, dims)
    us, ts = zip(*[ref.schur(m) for m in a])
    for t in (0.0, 0.4, -0.3, 1.3):
        assert np.array_equal(port.ode_at_schur(us, ts, b, x0, t), ref.propagate(a, b, x0, t))
    assert np.array_equal(port.ode_at_schur(us, ts, b, x0, 0.7, real_output=True),
                          ref.propagate(a, b, x0, 0.7, real_output=True))


@pytest.mark.parametrize("dims,seed,t,dt", [((2, 3), 46, 0.37, 0.1), ((2, 2, 3), 47, 0.5, 0.02),
                                            ((2, 2), 45, -0.3, 1e-2), ((3, 2, 2), 48, 0.05, 0.05)])
def test_rk4_port_matches_reference(port, ref, dims, seed, t, dt):
    rng = np.random.default_rng(seed)
    a, b, x0 = _system(rng, dims)
    assert np.array_equal(port.rk4(a, b, x0, t, dt), ref.rk4(a, b, x0, t, dt))


def test_ode_known_answers_on_port(port, ref):
    rng = np.random.default_rng(41)
    # test_ode.cpp:18-22: t = 0 returns the initial state
    a, b, x0 = _system(rng, (3, 2, 2))
    us, ts = zip(*[ref.schur(m) for m in a])
    x = port.ode_at_schur(us, ts, b, x0, 0.0)
    assert np.max(np.abs(x - x0)) <= 1e-13 * (1.0 + np.max(np.abs(x0)))
    # :24-36: scaled identities, zero forcing -> exp((s1 + s2) t) X0
    a2 = [-0.5 * np.eye(2, dtype=complex), (-1.0 + 0.3j) * np.eye(3, dtype=complex)]
    us2, ts2 = zip(*[ref.schur(m) for m in a2])
    x0b = rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))
    x = port.ode_at_schur(us2, ts2, np.zeros((2, 3), complex), x0b, 0.7)
    assert np.max(np.abs(x - np.exp((-1.5 + 0.3j) * 0.7) * x0b)) <= 1e-12
    # :38-44: closed form agrees with fine-step RK4
    a3, b3, x03 = _system(rng, (2, 3, 4))
    us3, ts3 = zip(*[ref.schur(m) for m in a3])
    exact = port.ode_at_schur(us3, ts3, b3, x03, 0.1)
    assert np.max(np.abs(exact - port.rk4(a3, b3, x03, 0.1, 2.5e-5))) <= 1e-10
    # :84-95: RK4 is exact for a constant derivative
    f = rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))
    x = port.rk4([np.zeros((2, 2), complex), np.zeros((3, 3), complex)], f, x0b, 0.37, 0.1)
    assert np.max(np.abs(x - (x0b + 0.37 * f))) <= 1e-13
    # :110-117: singular operator
    ts_s = [np.diag([1.0, -1.0]).astype(complex), np.diag([-1.0, 1.0]).astype(complex)]
    eye = [np.eye(2, dtype=complex)] * 2
    with pytest.raises(oracle.OracleError) as ei:
        port.ode_at_schur(eye, ts_s, np.eye(2, dtype=complex), np.zeros((2, 2), complex), 0.5)
    assert ei.value.code == 2 and ei.value.bad_index == [2, 2]
    # :119-125: step budget and argument validation
    for args in ((1.0, 0.0), (1.0, -0.1)):
        with pytest.raises(oracle.OracleError) as ei:
            port.rk4(a2, np.zeros((2, 3), complex), x0b, *args)
        assert ei.value.code == 5
    with pytest.raises(oracle.OracleError) as ei:
        port.rk4(a2, np.zeros((2, 3), complex), x0b, 1.0, 1e-9, 1000)
    assert ei.value.code == 5
    # :127-134: diverging integration
    big = [400.0 * np.eye(2, dtype=complex)] * 2
    with pytest.raises(oracle.OracleError) as ei:
        port.rk4(big, np.zeros((2, 2), complex), np.full((2, 2), 1e300, complex), 10.0, 0.5)
    assert ei.value.code == 9
