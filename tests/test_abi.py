"""The C-ABI library loads and exports every symbol include/ndsylv_b200.h declares; host-only
entry points (Schur, estimates, generator, validation) work without a GPU. CPU only."""
import os
import re

import numpy as np
import pytest

import paper_2412_15840_b200 as nds

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "ndsylv_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(nds_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_python_binding_list():
    assert declared_symbols() == sorted(nds.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = nds.load_library()
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym
    assert "sm_100a" in nds.version()


def test_flop_estimates_match_reference_closed_form():
    assert nds.flop_estimate([2, 2]) == 76
    for n_modes in (2, 3, 6):
        assert nds.flop_estimate([1] * n_modes) == 4 * n_modes + 1
    assert nds.flop_estimate([3, 3, 3]) == 27 * (45 - 3 + 1)
    with pytest.raises(OverflowError):
        nds.flop_estimate([1_000_000] * 4)
    assert nds.schur_flop_estimate([2, 9, 33]) == 25 * (8 + 729 + 35937)


def test_host_schur_quality():
    # acceptance.cpp criterion 4: residual, unitarity, exactly-zero strict lower triangle
    lib = nds.load_library()
    import ctypes as C
    for i in range(40):
        n = 2 + i % 19
        rng = np.random.default_rng(2000 + i)
        a = np.asfortranarray(rng.random((n, n)) + 1j * rng.random((n, n)))
        u = np.empty((n, n), dtype=complex, order="F")
        t = np.empty((n, n), dtype=complex, order="F")
        assert lib.nds_schur(None, n, a.ctypes.data, u.ctypes.data, t.ctypes.data) == 0
        assert np.linalg.norm(u @ t @ u.conj().T - a) / (1 + np.linalg.norm(a)) < 1e-13
        assert np.linalg.norm(u.conj().T @ u - np.eye(n)) / n < 1e-14
        assert np.all(np.tril(t, -1) == 0)
    bad = np.full((2, 2), np.nan, dtype=complex, order="F")
    assert lib.nds_schur(None, 2, bad.ctypes.data, u.ctypes.data, t.ctypes.data) == nds.ERR_INVALID


def test_host_schur_large_matches_eigenvalues():
    lib = nds.load_library()
    n = 96
    rng = np.random.default_rng(7)
    a = np.asfortranarray((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n) + 2 * np.eye(n))
    u = np.empty((n, n), dtype=complex, order="F")
    t = np.empty((n, n), dtype=complex, order="F")
    assert lib.nds_schur(None, n, a.ctypes.data, u.ctypes.data, t.ctypes.data) == 0
    ev = np.sort_complex(np.linalg.eigvals(a))
    assert np.max(np.abs(np.sort_complex(np.diag(t)) - ev)) < 1e-10
    assert np.linalg.norm(u @ t @ u.conj().T - a) / np.linalg.norm(a) < 1e-13


def test_randn_is_counter_based_and_normal():
    x = nds.randn(1, 2, 200001)
    assert np.array_equal(x[:1000], nds.randn(1, 2, 1000))
    assert not np.array_equal(x[:1000], nds.randn(1, 3, 1000))
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1.0) < 0.01


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(nds.NdsError):
        nds.Context(0)
