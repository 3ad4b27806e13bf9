"""SURVEY 8(f) rows 1-2 on the GPU: nds_ode_* (OdePropagator), nds_propagate, nds_rk4 and
nds_triangular_exp against the pinned oracle (tests/test_ode_oracle.py) and the reference."""
import numpy as np
import pytest

import paper_2412_15840_b200 as nds
from conftest import rel_max

pytestmark = pytest.mark.gpu


def _system(rng, dims, shift=-2.0):
    a = [(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n) + shift * np.eye(n)
         for n in dims]
    b = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    x0 = rng.standard_normal(dims) + 1j * rng.standard_normal(dims)
    return a, b, x0


def test_triangular_exp_matches_port(ctx, port):
    rng = np.random.default_rng(5)
    for n in (1, 3, 16, 64):
        t_mat = np.triu(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
        for t in (0.0, 0.25, -1.5):
            f = ctx.triangular_exp(t_mat, t)
            assert rel_max(f, port.triangular_exp(t_mat, t)) <= 1e-13
    t2 = np.triu(rng.standard_normal((6, 6)) + 0j)
    t2[5, 5] = t2[2, 2]  # Pade branch
    assert rel_max(ctx.triangular_exp(t2, 0.8), port.triangular_exp(t2, 0.8)) <= 1e-13
    with pytest.raises(ValueError):
        ctx.triangular_exp(np.array([[1.0, 0.0], [1.0, 1.0]], dtype=complex), 1.0)


@pytest.mark.parametrize("dims", [(5, 4, 3), (32, 32, 32), (16, 16, 16, 16), (2,) * 10, (48, 3, 20)],
                         ids=["5x4x3", "32^3", "16^4", "bin10", "48x3x20"])
def test_propagator_matches_port(ctx, port, ref, dims):
    rng = np.random.default_rng(sum(dims))
    a, b, x0 = _system(rng, dims)
    us, ts = zip(*[ctx.schur(m) for m in a])
    ode = ctx.ode(us, ts, b, x0)
    for t in (0.0, 0.35, -0.2):
        r = ode.at(t)
        assert rel_max(r.x, port.ode_at_schur(us, ts, b, x0, t)) <= 1e-11
    assert r.report["backsub_entries"] == int(np.prod(dims))
    ode.close()
    if int(np.prod(dims)) <= 4096:  # the reference (own Schur) on the small shapes: X(t) is unique
        assert rel_max(ctx.propagate(a, b, x0, 0.35).x, ref.propagate(a, b, x0, 0.35)) <= 1e-9


def test_propagator_semigroup_and_device_output(ctx):
    # test_ode.cpp:46-54 on the GPU: X(0.8) = propagate(restart from X(0.4), 0.4)
    import torch
    rng = np.random.default_rng(43)
    dims = (24, 20, 16)
    a, b, x0 = _system(rng, dims)
    half = ctx.propagate(a, b, x0, 0.4).x
    second = ctx.propagate(a, b, half, 0.4).x
    direct = ctx.propagate(a, b, x0, 0.8).x
    assert np.max(np.abs(second - direct)) <= 1e-9 * (1.0 + np.max(np.abs(direct)))
    us, ts = zip(*[ctx.schur(m) for m in a])
    ode = ctx.ode(us, ts, b, x0, real_output=True)
    d_x = torch.empty(int(np.prod(dims)), dtype=torch.complex128, device="cuda")
    torch.cuda.synchronize()
    ode.at_dev(0.8, d_x.data_ptr())
    torch.cuda.synchronize()
    x = d_x.cpu().numpy().reshape(dims, order="F")
    assert np.all(x.imag == 0) and rel_max(x.real, direct.real) <= 1e-11
    ode.close()


def test_propagator_scaled_identities(ctx):
    # test_ode.cpp:24-36 (repeated eigenvalues: the host Pade branch) on the GPU path
    rng = np.random.default_rng(41)
    a = [-0.5 * np.eye(2, dtype=complex), (-1.0 + 0.3j) * np.eye(3, dtype=complex)]
    x0 = rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))
    x = ctx.propagate(a, np.zeros((2, 3), complex), x0, 0.7).x
    assert np.max(np.abs(x - np.exp((-1.5 + 0.3j) * 0.7) * x0)) <= 1e-12


def test_propagator_errors(ctx):
    # test_ode.cpp:110-117 (singular at at(), not at construction), :124 (non-finite time), :136-141
    ts = [np.diag([1.0, -1.0]).astype(complex), np.diag([-1.0, 1.0]).astype(complex)]
    us = [np.eye(2, dtype=complex)] * 2
    f = np.zeros((2, 2), complex)
    f[0, 0] = 1.0
    ode = ctx.ode(us, ts, f, np.zeros((2, 2), complex))
    with pytest.raises(nds.SingularOperatorError) as ei:
        ode.at(0.5)
    assert ei.value.multi_index == [2, 2]
    ode.close()
    rng = np.random.default_rng(48)
    a, b, x0 = _system(rng, (2, 2))
    with pytest.raises(ValueError):
        ctx.propagate(a, b, x0, float("inf"))
    with pytest.raises(ValueError):
        ctx.ode([np.eye(2, dtype=complex)] * 2, [np.eye(2, dtype=complex)] * 2, b, np.zeros((2, 3), complex))


@pytest.mark.parametrize("dims,t,dt", [((2, 3), 0.37, 0.1), ((2, 2, 3), 0.5, 0.02), ((8, 6, 4), 0.26, 0.01),
                                       ((16, 16, 16), -0.05, 0.004)], ids=["2x3", "2x2x3", "8x6x4", "16^3"])
def test_rk4_matches_port(ctx, port, dims, t, dt):
    rng = np.random.default_rng(len(dims) * 7 + dims[0])
    a, b, x0 = _system(rng, dims)
    x = ctx.rk4(a, b, x0, t, dt)  # 8x6x4: 26 steps = 1 eager + 3 graph replays of 8 + 1
    assert rel_max(x, port.rk4(a, b, x0, t, dt)) <= 1e-11


def test_rk4_known_answers(ctx):
    rng = np.random.default_rng(46)
    f = rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))
    x0 = rng.standard_normal((2, 3)) + 1j * rng.standard_normal((2, 3))
    x = ctx.rk4([np.zeros((2, 2), complex), np.zeros((3, 3), complex)], f, x0, 0.37, 0.1)
    assert np.max(np.abs(x - (x0 + 0.37 * f))) <= 1e-13  # test_ode.cpp:84-95
    a, b, x1 = _system(rng, (2, 2, 3))
    exact = ctx.propagate(a, b, x1, 0.5).x  # :97-108 fourth-order convergence
    e1 = np.max(np.abs(ctx.rk4(a, b, x1, 0.5, 2e-2) - exact))
    e2 = np.max(np.abs(ctx.rk4(a, b, x1, 0.5, 1e-2) - exact))
    assert 12.0 <= e1 / e2 <= 20.0
    with pytest.raises(ValueError):
        ctx.rk4(a, b, x1, 1.0, 0.0)
    with pytest.raises(ValueError):
        ctx.rk4(a, b, x1, 1.0, 1e-9, 1000)
    big = [400.0 * np.eye(2, dtype=complex)] * 2  # :127-134
    with pytest.raises(nds.NonFiniteStateError):
        ctx.rk4(big, np.zeros((2, 2), complex), np.full((2, 2), 1e300, complex), 10.0, 0.5)
