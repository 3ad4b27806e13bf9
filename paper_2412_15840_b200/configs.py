"""BASELINE.json workloads (configs c0..c4) with seeded synthetic inputs — generator v1.

The reference has only a uniform sampler (rng.hpp:38-43), so the Gaussian inputs the configs ask
for come from :func:`paper_2412_15840_b200.randn` (counter-based splitmix64 + Box–Muller, order
independent). Draw layout, fixed for every config:

* A_j: G_j = randn(seed, 2j, n_j^2), H_j = randn(seed, 2j + 1, n_j^2), column-major, j = 0..N-1;
* B:   randn(seed, 1000, 2P) interleaved (re, im) per entry, column-major.

c2 is deterministic (finite-difference advection–diffusion, no randomness).
"""
from __future__ import annotations

import math

import numpy as np

GENERATOR_VERSION = "v1"

CONFIGS = {
    "c0": {"dims": (32, 32, 32), "kind": "gauss", "scaled": True},
    "c1": {"dims": (256, 256, 256), "kind": "gauss", "scaled": True},
    "c2": {"dims": (96, 96, 96, 96), "kind": "advdiff"},
    "c3": {"dims": (128, 128, 128, 128), "kind": "gauss", "scaled": True},
    "c4": {"dims": (2,) * 29, "kind": "gauss", "scaled": False},
}

DESCRIPTIONS = {
    "c0": "N=3 n=(32,32,32) A_j=(G+iH)/sqrt(n)+2I, B complex normal",
    "c1": "N=3 n=(256,256,256) A_j=(G+iH)/sqrt(n)+2I, B complex normal",
    "c2": "N=4 n=96 FD advection-diffusion backward-Euler step, B=exp(-|x|^2)",
    "c3": "N=4 n=(128,128,128,128) A_j=(G+iH)/sqrt(n)+2I, B complex normal",
    "c4": "N=29 n_j=2 A_j=G+iH+2I, B complex normal",
}


def _default_randn():
    from . import randn
    return randn


def gauss_coefficients(dims, seed, scaled=True, randn=None):
    randn = randn or _default_randn()
    out = []
    for j, n in enumerate(dims):
        g = randn(seed, 2 * j, n * n).reshape((n, n), order="F")
        h = randn(seed, 2 * j + 1, n * n).reshape((n, n), order="F")
        a = (g + 1j * h)
        if scaled:
            a = a / math.sqrt(n)
        a = a + 2.0 * np.eye(n)
        out.append(np.asfortranarray(a))
    return out


def gauss_rhs(dims, seed, randn=None):
    randn = randn or _default_randn()
    total = int(np.prod(dims))
    v = randn(seed, 1000, 2 * total).view(np.complex128)
    return v.reshape(dims, order="F")


def advdiff_coefficients(n=96, n_modes=4, nu=1.0, dt=1e-2):
    """A_j = I/N - dt L_j, L_j = nu tridiag(1,-2,1)/h^2 + c_j tridiag(-1,0,1)/(2h), c_j = 0.5 j."""
    h = 20.0 / (n + 1)
    out = []
    for j in range(1, n_modes + 1):
        cj = 0.5 * j
        lap = (np.diag(np.full(n - 1, 1.0), -1) + np.diag(np.full(n, -2.0)) + np.diag(np.full(n - 1, 1.0), 1)) / h**2
        adv = (np.diag(np.full(n - 1, -1.0), -1) + np.diag(np.full(n - 1, 1.0), 1)) / (2 * h)
        L = nu * lap + cj * adv
        a = np.eye(n) / n_modes - dt * L
        out.append(np.asfortranarray(a.astype(np.complex128)))
    return out


def advdiff_rhs(n=96, n_modes=4):
    h = 20.0 / (n + 1)
    x = -10.0 + h * np.arange(1, n + 1)
    g = np.exp(-x * x)
    b = g
    for _ in range(n_modes - 1):
        b = np.multiply.outer(b, g)
    # outer products give C-order (i1, i2, ...) indexing; value is symmetric in the modes
    return np.asfortranarray(b.astype(np.complex128))


def make_problem(name: str, seed: int = 0, dims=None, randn=None):
    """(coefficients, rhs) for a BASELINE config; `dims` overrides the shape (reduced sizes).

    `randn(seed, stream, count)` defaults to the product library's generator; the reference arm
    of bench.py and the X_ref fixture scripts pass the bit-identical copy in oracle/_ref
    (``oracle.Ref().randn``) so that they never load the product library."""
    cfg = CONFIGS[name]
    d = tuple(dims) if dims is not None else cfg["dims"]
    if cfg["kind"] == "advdiff":
        n = d[0]
        return advdiff_coefficients(n, len(d)), advdiff_rhs(n, len(d))
    return gauss_coefficients(d, seed, cfg["scaled"], randn), gauss_rhs(d, seed, randn)
