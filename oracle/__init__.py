"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front ends for the two CPU checkers of the hot path:

* :class:`Port` — ``liboracle.so``, the plain-C restatement (``ndsylv_oracle.c``).
* :class:`Ref`  — ``_ref/libndsylv_ref.so``, the unmodified reference library compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` (plus the ``ref_capi.cpp`` shim).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` leg and
``--impl reference``) may import this package, and only as the checker / CPU baseline.
The product package ``paper_2412_15840_b200`` never imports it.

Tensors are numpy complex128 arrays of shape ``dims`` (column-major flattening, the
reference's layout, tensor.hpp:23-39); matrices are ``(n, n)`` complex128 (column-major
storage, matrix.hpp:11-30).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libndsylv_ref.so")

ALLOW_FAST_PATH = 1
REAL_OUTPUT = 2

_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)
_dpp = C.POINTER(_dp)


class OracleError(RuntimeError):
    def __init__(self, code, msg="", bad_index=None, bad_den=None):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code
        self.bad_index = bad_index
        self.bad_den = bad_den


def fortran(x):
    return np.asfortranarray(np.asarray(x, dtype=np.complex128))


def _dims(shape):
    d = (C.c_int64 * len(shape))(*[int(v) for v in shape])
    return d


def _ptr(a):
    return a.ctypes.data_as(_dp)


def _ptrs(arrs):
    keep = [fortran(a) for a in arrs]
    p = (_dp * len(keep))(*[_ptr(a) for a in keep])
    return p, keep


class _ReportPort(C.Structure):
    _fields_ = [
        ("min_abs_denominator", C.c_double),
        ("used_normal_fast_path", C.c_int),
        ("flop_estimate", C.c_int64),
        ("schur_flop_estimate", C.c_int64),
        ("backsub_entries", C.c_int64),
        ("backsub_multiplies", C.c_int64),
        ("transform_seconds", C.c_double),
        ("backsub_seconds", C.c_double),
        ("inverse_seconds", C.c_double),
    ]


class _StatsPort(C.Structure):
    _fields_ = [("entries", C.c_int64), ("multiplies", C.c_int64), ("min_abs_denominator", C.c_double)]


class _ReportRef(C.Structure):
    _fields_ = [
        ("min_abs_denominator", C.c_double),
        ("used_normal_fast_path", C.c_int),
        ("flop_estimate", C.c_int64),
        ("schur_flop_estimate", C.c_int64),
        ("backsub_entries", C.c_int64),
        ("backsub_multiplies", C.c_int64),
        ("schur_seconds", C.c_double),
        ("transform_seconds", C.c_double),
        ("backsub_seconds", C.c_double),
        ("inverse_seconds", C.c_double),
        ("total_seconds", C.c_double),
    ]


def _as_dict(s):
    return {k: getattr(s, k) for k, _ in s._fields_}


class Port:
    """The plain-C restatement (scalar, single thread)."""

    def __init__(self, path=PORT_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = L = C.CDLL(path)
        L.orc_mode_product.argtypes = [C.c_int, _i64p, _dp, C.c_int, _dp, _dp]
        L.orc_forward_transform.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp]
        L.orc_inverse_transform.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp]
        L.orc_apply_operator.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp]
        L.orc_back_substitute.argtypes = [C.c_int, _i64p, _dpp, _dp, C.c_double, C.POINTER(_StatsPort), _i64p, _dp]
        L.orc_default_singular_tol.argtypes = [C.c_int, _i64p, _dpp]
        L.orc_default_singular_tol.restype = C.c_double
        L.orc_solve_schur.argtypes = [C.c_int, _i64p, _dpp, _dpp, _dp, _dp, C.c_double, C.c_uint,
                                      C.POINTER(_ReportPort), _i64p, _dp]
        L.orc_flop_estimate.argtypes = [C.c_int, _i64p]
        L.orc_flop_estimate.restype = C.c_int64
        L.orc_schur_flop_estimate.argtypes = [C.c_int, _i64p]
        L.orc_schur_flop_estimate.restype = C.c_int64
        L.orc_xoshiro_uniform.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.orc_numerically_diagonal.argtypes = [C.c_int, _dp]
        L.orc_triangular_exp.argtypes = [C.c_int, _dp, C.c_double, _dp]
        L.orc_ode_at_schur.argtypes = [C.c_int, _i64p, _dpp, _dpp, _dp, _dp, C.c_double, C.c_double, C.c_uint, _dp,
                                       _i64p, _dp]
        L.orc_rk4.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp, C.c_double, C.c_double, C.c_int64, _dp]

    def mode_product(self, m, mode, x):
        x = fortran(x)
        m = fortran(m)
        r = np.empty_like(x, order="F")
        rc = self.lib.orc_mode_product(x.ndim, _dims(x.shape), _ptr(m), mode, _ptr(x), _ptr(r))
        if rc:
            raise OracleError(rc)
        return r

    def _transform(self, fn, us, x):
        x = fortran(x)
        up, keep = _ptrs(us)
        r = np.empty_like(x, order="F")
        rc = fn(x.ndim, _dims(x.shape), up, _ptr(x), _ptr(r))
        if rc:
            raise OracleError(rc)
        return r

    def forward_transform(self, us, b):
        return self._transform(self.lib.orc_forward_transform, us, b)

    def inverse_transform(self, us, y):
        return self._transform(self.lib.orc_inverse_transform, us, y)

    def apply_operator(self, a_list, x):
        return self._transform(self.lib.orc_apply_operator, a_list, x)

    def default_singular_tol(self, ts):
        tp, keep = _ptrs(ts)
        dims = [t.shape[0] for t in ts]
        return self.lib.orc_default_singular_tol(len(ts), _dims(dims), tp)

    def back_substitute(self, ts, c, tol=0.0):
        """Returns (y, stats dict). Raises OracleError(2, bad_index, bad_den) when singular."""
        y = fortran(c).copy(order="F")
        tp, keep = _ptrs(ts)
        st = _StatsPort()
        bad = (C.c_int64 * y.ndim)()
        den = (C.c_double * 2)()
        rc = self.lib.orc_back_substitute(y.ndim, _dims(y.shape), tp, _ptr(y), tol, C.byref(st), bad, den)
        if rc:
            raise OracleError(rc, "singular" if rc == 2 else "", list(bad), complex(den[0], den[1]))
        return y, _as_dict(st)

    def solve_schur(self, us, ts, b, tol=0.0, flags=ALLOW_FAST_PATH):
        b = fortran(b)
        up, k1 = _ptrs(us)
        tp, k2 = _ptrs(ts)
        x = np.empty_like(b, order="F")
        rep = _ReportPort()
        bad = (C.c_int64 * b.ndim)()
        den = (C.c_double * 2)()
        rc = self.lib.orc_solve_schur(b.ndim, _dims(b.shape), up, tp, _ptr(b), _ptr(x), tol, flags, C.byref(rep),
                                      bad, den)
        if rc:
            raise OracleError(rc, "singular" if rc == 2 else "", list(bad), complex(den[0], den[1]))
        return x, _as_dict(rep)

    def flop_estimate(self, dims):
        return self.lib.orc_flop_estimate(len(dims), _dims(dims))

    def schur_flop_estimate(self, dims):
        return self.lib.orc_schur_flop_estimate(len(dims), _dims(dims))

    def xoshiro_uniform(self, seed, count):
        out = np.empty(count, dtype=np.float64)
        self.lib.orc_xoshiro_uniform(seed, count, _ptr(out))
        return out

    def numerically_diagonal(self, t):
        t = fortran(t)
        return bool(self.lib.orc_numerically_diagonal(t.shape[0], _ptr(t)))

    def triangular_exp(self, t_mat, t):
        tm = fortran(t_mat)
        f = np.empty_like(tm, order="F")
        rc = self.lib.orc_triangular_exp(tm.shape[0], _ptr(tm), float(t), _ptr(f))
        if rc:
            raise OracleError(rc)
        return f

    def ode_at_schur(self, us, ts, forcing, initial, t, tol=0.0, real_output=False):
        """OdePropagator(system).at(t) (ode.cpp:32-87) given the Schur factors."""
        f, x0 = fortran(forcing), fortran(initial)
        up, k1 = _ptrs(us)
        tp, k2 = _ptrs(ts)
        x = np.empty_like(f, order="F")
        bad = (C.c_int64 * f.ndim)()
        den = (C.c_double * 2)()
        rc = self.lib.orc_ode_at_schur(f.ndim, _dims(f.shape), up, tp, _ptr(f), _ptr(x0), float(t), tol,
                                       REAL_OUTPUT if real_output else 0, _ptr(x), bad, den)
        if rc:
            raise OracleError(rc, "singular" if rc == 2 else "", list(bad), complex(den[0], den[1]))
        return x

    def rk4(self, a_list, forcing, initial, t, dt, max_steps=50_000_000):
        f, x0 = fortran(forcing), fortran(initial)
        ap, keep = _ptrs(a_list)
        x = np.empty_like(f, order="F")
        rc = self.lib.orc_rk4(f.ndim, _dims(f.shape), ap, _ptr(f), _ptr(x0), float(t), float(dt), int(max_steps),
                              _ptr(x))
        if rc:
            raise OracleError(rc)
        return x


class Ref:
    """The reference library itself (oracle/_ref), OpenMP-parallel where the reference is."""

    def __init__(self, path=REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_get_max_threads.restype = C.c_int
        L.ref_solve.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp, C.c_double, C.c_uint, C.POINTER(_ReportRef),
                                _i64p, _dp]
        L.ref_schur.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_forward_transform.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp]
        L.ref_inverse_transform.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp]
        L.ref_back_substitute.argtypes = [C.c_int, _i64p, _dpp, _dp, C.c_double, _i64p, _i64p, _dp, _i64p, _dp]
        L.ref_mode_product.argtypes = [C.c_int, _i64p, _dp, C.c_int, _dp, _dp, C.c_int]
        L.ref_apply_operator.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp]
        L.ref_random_problem.argtypes = [C.c_int, _i64p, C.c_uint64, _dpp, _dp, _dp]
        L.ref_oracle_solve.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp]
        L.ref_flop_estimate.argtypes = [C.c_int, _i64p]
        L.ref_flop_estimate.restype = C.c_int64
        L.ref_schur_flop_estimate.argtypes = [C.c_int, _i64p]
        L.ref_schur_flop_estimate.restype = C.c_int64
        L.ref_xoshiro_uniform.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.ref_triangular_exp.argtypes = [C.c_int, _dp, C.c_double, _dp]
        L.ref_propagate.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp, C.c_double, C.c_int, _dp, C.POINTER(_ReportRef),
                                    _i64p, _dp]
        L.ref_rk4.argtypes = [C.c_int, _i64p, _dpp, _dp, _dp, C.c_double, C.c_double, C.c_int64, _dp]
        L.ref_write_tensor.argtypes = [C.c_char_p, C.c_int, _i64p, _dp]
        L.ref_read_tensor.argtypes = [C.c_char_p, C.POINTER(C.c_int), _i64p, _dp, C.c_int64]
        L.ref_random_ode_system.argtypes = [C.c_int, _i64p, C.c_uint64, _dpp, _dp, _dp]
        L.ref_harness_randn.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _dp]
        L.ref_solve_gen.argtypes = [C.c_int, _i64p, _dpp, _dp, C.c_uint64, _dp, C.POINTER(_ReportRef)]

    def _check(self, rc, bad=None, den=None):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode(), list(bad) if bad is not None else None,
                              complex(den[0], den[1]) if den is not None else None)

    def set_threads(self, n):
        self.lib.ref_set_threads(int(n))

    def max_threads(self):
        return self.lib.ref_get_max_threads()

    def solve(self, a_list, b, tol=0.0, flags=ALLOW_FAST_PATH):
        b = fortran(b)
        ap, keep = _ptrs(a_list)
        x = np.empty_like(b, order="F")
        rep = _ReportRef()
        bad = (C.c_int64 * b.ndim)()
        den = (C.c_double * 2)()
        rc = self.lib.ref_solve(b.ndim, _dims(b.shape), ap, _ptr(b), _ptr(x), tol, flags, C.byref(rep), bad, den)
        self._check(rc, bad, den)
        return x, _as_dict(rep)

    def schur(self, a):
        a = fortran(a)
        n = a.shape[0]
        u = np.empty((n, n), dtype=np.complex128, order="F")
        t = np.empty((n, n), dtype=np.complex128, order="F")
        self._check(self.lib.ref_schur(n, _ptr(a), _ptr(u), _ptr(t)))
        return u, t

    def _transform(self, fn, us, x):
        x = fortran(x)
        up, keep = _ptrs(us)
        r = np.empty_like(x, order="F")
        self._check(fn(x.ndim, _dims(x.shape), up, _ptr(x), _ptr(r)))
        return r

    def forward_transform(self, us, b):
        return self._transform(self.lib.ref_forward_transform, us, b)

    def inverse_transform(self, us, y):
        return self._transform(self.lib.ref_inverse_transform, us, y)

    def apply_operator(self, a_list, x):
        return self._transform(self.lib.ref_apply_operator, a_list, x)

    def oracle_solve(self, a_list, b):
        return self._transform(self.lib.ref_oracle_solve, a_list, b)

    def back_substitute(self, ts, c, tol=0.0):
        y = fortran(c).copy(order="F")
        tp, keep = _ptrs(ts)
        e = C.c_int64()
        m = C.c_int64()
        mad = C.c_double()
        bad = (C.c_int64 * y.ndim)()
        den = (C.c_double * 2)()
        rc = self.lib.ref_back_substitute(y.ndim, _dims(y.shape), tp, _ptr(y), tol, C.byref(e), C.byref(m),
                                          C.byref(mad), bad, den)
        self._check(rc, bad, den)
        return y, {"entries": e.value, "multiplies": m.value, "min_abs_denominator": mad.value}

    def mode_product(self, m, mode, x, serial_twin=False):
        x = fortran(x)
        m = fortran(m)
        r = np.empty_like(x, order="F")
        self._check(self.lib.ref_mode_product(x.ndim, _dims(x.shape), _ptr(m), mode, _ptr(x), _ptr(r),
                                              1 if serial_twin else 0))
        return r

    def random_problem(self, dims, seed):
        """rng.cpp:18-25: uniform A_j and X_true from one xoshiro stream, B = op(X_true)."""
        a = [np.empty((n, n), dtype=np.complex128, order="F") for n in dims]
        ap = (_dp * len(a))(*[_ptr(m) for m in a])
        x = np.empty(tuple(dims), dtype=np.complex128, order="F")
        b = np.empty_like(x, order="F")
        self._check(self.lib.ref_random_problem(len(dims), _dims(dims), seed, ap, _ptr(x), _ptr(b)))
        return a, x, b

    def flop_estimate(self, dims):
        return self.lib.ref_flop_estimate(len(dims), _dims(dims))

    def schur_flop_estimate(self, dims):
        return self.lib.ref_schur_flop_estimate(len(dims), _dims(dims))

    def xoshiro_uniform(self, seed, count):
        out = np.empty(count, dtype=np.float64)
        self.lib.ref_xoshiro_uniform(seed, count, _ptr(out))
        return out

    def triangular_exp(self, t_mat, t):
        tm = fortran(t_mat)
        f = np.empty_like(tm, order="F")
        self._check(self.lib.ref_triangular_exp(tm.shape[0], _ptr(tm), float(t), _ptr(f)))
        return f

    def propagate(self, a_list, forcing, initial, t, real_output=False, report=False):
        """ndsylv::propagate (ode.hpp:39): Schur + OdePropagator::at inside the reference."""
        f, x0 = fortran(forcing), fortran(initial)
        ap, keep = _ptrs(a_list)
        x = np.empty_like(f, order="F")
        rep = _ReportRef()
        bad = (C.c_int64 * f.ndim)()
        den = (C.c_double * 2)()
        rc = self.lib.ref_propagate(f.ndim, _dims(f.shape), ap, _ptr(f), _ptr(x0), float(t), 1 if real_output else 0,
                                    _ptr(x), C.byref(rep), bad, den)
        self._check(rc, bad, den)
        return (x, _as_dict(rep)) if report else x

    def rk4(self, a_list, forcing, initial, t, dt, max_steps=50_000_000):
        f, x0 = fortran(forcing), fortran(initial)
        ap, keep = _ptrs(a_list)
        x = np.empty_like(f, order="F")
        self._check(self.lib.ref_rk4(f.ndim, _dims(f.shape), ap, _ptr(f), _ptr(x0), float(t), float(dt),
                                     int(max_steps), _ptr(x)))
        return x

    def write_tensor(self, path, x):
        x = fortran(x)
        self._check(self.lib.ref_write_tensor(path.encode(), x.ndim, _dims(x.shape), _ptr(x)))

    def read_tensor(self, path):
        n = C.c_int()
        dims = (C.c_int64 * 64)()
        self._check(self.lib.ref_read_tensor(path.encode(), C.byref(n), dims, None, 0))
        shape = tuple(dims[j] for j in range(n.value))
        out = np.empty(shape, dtype=np.complex128, order="F")
        self._check(self.lib.ref_read_tensor(path.encode(), C.byref(n), dims, _ptr(out), out.size))
        return out

    def solve_gen(self, a_list, dims, seed, b=None):
        """ndsylv::solve with B = generator v1 (seed, stream 1000) built inside the library, or
        a copy of `b`; returns (X, report)."""
        ap, keep = _ptrs(a_list)
        x = np.empty(tuple(dims), dtype=np.complex128, order="F")
        bf = None if b is None else fortran(b)
        bp = None if bf is None else _ptr(bf)
        rep = _ReportRef()
        self._check(self.lib.ref_solve_gen(len(dims), _dims(dims), ap, bp, int(seed), _ptr(x), C.byref(rep)))
        return x, _as_dict(rep)

    def randn(self, seed, stream, count):
        """Harness generator v1 (same stream as the product's nds_randn) — inputs for the
        reference arm and the X_ref fixtures without loading the product library."""
        out = np.empty(int(count), dtype=np.float64)
        self.lib.ref_harness_randn(seed & (2**64 - 1), stream & (2**64 - 1), int(count), _ptr(out))
        return out

    def random_ode_system(self, dims, seed):
        a = [np.empty((n, n), dtype=np.complex128, order="F") for n in dims]
        ap = (_dp * len(a))(*[_ptr(m) for m in a])
        f = np.empty(tuple(dims), dtype=np.complex128, order="F")
        x0 = np.empty_like(f, order="F")
        self._check(self.lib.ref_random_ode_system(len(dims), _dims(dims), int(seed), ap, _ptr(f), _ptr(x0)))
        return a, f, x0
