"""ndsylv_b200 — B200-native (sm_100a) hot path of the N-D Bartels–Stewart Sylvester solver.

Python mirror of the reference C++ API (``/root/reference/proj/include/ndsylv``) over the C ABI
of ``libndsylv_b200.so`` (``include/ndsylv_b200.h``). Names, argument meaning and error
behaviour follow the reference:

========================  =====================================================
reference (C++)           here
========================  =====================================================
``solve`` (sylvester.hpp:79)           :meth:`Context.solve`
``schur`` (schur.hpp:19)               :meth:`Context.schur`
``forward_transform`` (:64)            :meth:`Context.forward_transform`
``inverse_transform`` (:67)            :meth:`Context.inverse_transform`
``back_substitute`` (:77)              :meth:`Context.back_substitute`
``mode_product`` (kernels.hpp:12)      :meth:`Context.mode_product`
``apply_operator`` (:61)               :meth:`Context.apply_operator`
``flop_estimate`` / ``schur_flop_estimate`` (:86-90)
``SingularOperatorError`` (types.hpp:31-47)   :class:`SingularOperatorError`
``std::invalid_argument``               ``ValueError``
``std::overflow_error``                 ``OverflowError``
``ConvergenceError``                    :class:`ConvergenceError`
========================  =====================================================

Tensors are numpy ``complex128`` arrays of shape ``dims`` interpreted in column-major
(Fortran) order, exactly the reference ``NDTensor`` storage; matrices are ``(n, n)``.
There is no CPU fallback: without the built library or an sm_100 GPU the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libndsylv_b200.so")

NDS_MAX_MODES = 64
ALLOW_FAST_PATH = 1
REAL_OUTPUT = 2
NO_DIAGONALISE = 4

(OK, ERR_OTHER, ERR_SINGULAR, ERR_FILE, ERR_NOMEM, ERR_INVALID, ERR_CONVERGENCE, ERR_OVERFLOW, ERR_CUDA,
 ERR_NONFINITE) = range(10)

# Symbols include/ndsylv_b200.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "nds_version", "nds_ctx_create", "nds_ctx_destroy", "nds_ctx_set_stream", "nds_ctx_stream", "nds_last_error",
    "nds_ctx_trim", "nds_solve", "nds_solve_schur", "nds_schur", "nds_forward_transform", "nds_inverse_transform",
    "nds_back_substitute", "nds_mode_product", "nds_apply_operator", "nds_flop_estimate", "nds_schur_flop_estimate",
    "nds_plan_create", "nds_plan_destroy", "nds_plan_report", "nds_plan_total", "nds_plan_execute",
    "nds_plan_forward", "nds_plan_backsub", "nds_plan_inverse", "nds_plan_execute_host", "nds_plan_execute_host_many", "nds_plan_launches", "nds_plan_solve_path",
    "nds_plan_diagonalised", "nds_plan_superblocks",
    "nds_plan_profile_begin", "nds_plan_profile_end",
    "nds_dev_mode_product", "nds_dev_mode_update", "nds_dev_mode_apply", "nds_dev_back_substitute", "nds_dev_residual",
    "nds_triangular_exp", "nds_ode_create", "nds_ode_destroy", "nds_ode_at", "nds_ode_at_dev", "nds_propagate",
    "nds_rk4", "nds_tensor_file_info", "nds_read_tensor", "nds_write_tensor", "nds_read_tensor_dev",
    "nds_write_tensor_dev", "nds_random_problem", "nds_random_ode_system", "nds_randn",
    "nds_comm_unique_id", "nds_comm_create_nccl", "nds_comm_create_loopback", "nds_comm_destroy", "nds_dist_create",
    "nds_dist_destroy", "nds_dist_slab", "nds_dist_info", "nds_dist_solve", "nds_solve_multi",
]


class NdsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class SingularOperatorError(NdsError):
    """types.hpp:31-47: 1-based multi-index of the first offender and its denominator."""

    def __init__(self, msg, multi_index, denominator):
        super().__init__(ERR_SINGULAR, msg)
        self.multi_index = list(multi_index)
        self.denominator = denominator


class ConvergenceError(NdsError):
    pass


class TensorFileError(NdsError):
    """TensorFileError (types.hpp): NDT1 I/O or format error."""


class NonFiniteStateError(NdsError):
    """NonFiniteStateError (types.hpp:62-66): an integration left finite range."""


class DeviceError(NdsError):
    pass


class _Report(C.Structure):
    _fields_ = [
        ("min_abs_denominator", C.c_double),
        ("used_normal_fast_path", C.c_int32),
        ("flop_estimate", C.c_int64),
        ("schur_flop_estimate", C.c_int64),
        ("backsub_entries", C.c_int64),
        ("backsub_multiplies", C.c_int64),
        ("schur_seconds", C.c_double),
        ("transform_seconds", C.c_double),
        ("backsub_seconds", C.c_double),
        ("inverse_seconds", C.c_double),
        ("total_seconds", C.c_double),
        ("h2d_seconds", C.c_double),
        ("d2h_seconds", C.c_double),
        ("kernel_launches", C.c_int32),
    ]


class _Singular(C.Structure):
    _fields_ = [("n_modes", C.c_int32), ("multi_index", C.c_int64 * NDS_MAX_MODES), ("den_re", C.c_double),
                ("den_im", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("entries", C.c_int64), ("multiplies", C.c_int64), ("min_abs_denominator", C.c_double)]


class _DistInfo(C.Structure):
    _fields_ = [("ranks", C.c_int32), ("rank", C.c_int32), ("head_modes", C.c_int32), ("tail_modes", C.c_int32),
                ("pipe_modes", C.c_int32), ("pipe_blocks", C.c_int32), ("local_solve_path", C.c_int32),
                ("launches", C.c_int32), ("alltoall_bytes", C.c_int64), ("pipeline_bytes", C.c_int64),
                ("min_abs_denominator", C.c_double)]


_vp = C.c_void_p
_i64p = C.POINTER(C.c_int64)
_lib = None


def load_library(path: str = LIB_PATH):
    """Load libndsylv_b200.so. Raises (loudly) when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -m paper_2412_15840_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(path)
    L.nds_version.restype = C.c_char_p
    L.nds_last_error.restype = C.c_char_p
    L.nds_last_error.argtypes = [_vp]
    L.nds_ctx_create.argtypes = [C.POINTER(_vp), C.c_int]
    L.nds_ctx_destroy.argtypes = [_vp]
    L.nds_ctx_set_stream.argtypes = [_vp, _vp]
    L.nds_ctx_stream.argtypes = [_vp]
    L.nds_ctx_stream.restype = _vp
    L.nds_ctx_trim.argtypes = [_vp]
    L.nds_solve.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp, C.c_double, C.c_uint, C.POINTER(_Report),
                            C.POINTER(_Singular)]
    L.nds_solve_schur.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp, _vp, C.c_double, C.c_uint,
                                  C.POINTER(_Report), C.POINTER(_Singular)]
    L.nds_schur.argtypes = [_vp, C.c_int, _vp, _vp, _vp]
    L.nds_forward_transform.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp]
    L.nds_inverse_transform.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp]
    L.nds_back_substitute.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, C.c_double, C.POINTER(_Stats),
                                      C.POINTER(_Singular)]
    L.nds_mode_product.argtypes = [_vp, C.c_int, _i64p, _vp, C.c_int, _vp, _vp]
    L.nds_apply_operator.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp]
    L.nds_flop_estimate.argtypes = [C.c_int, _i64p]
    L.nds_flop_estimate.restype = C.c_int64
    L.nds_schur_flop_estimate.argtypes = [C.c_int, _i64p]
    L.nds_schur_flop_estimate.restype = C.c_int64
    L.nds_plan_create.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, C.c_double, C.c_uint, C.POINTER(_vp),
                                  C.POINTER(_Singular)]
    L.nds_plan_destroy.argtypes = [_vp]
    L.nds_plan_report.argtypes = [_vp, C.POINTER(_Report)]
    L.nds_plan_total.argtypes = [_vp]
    L.nds_plan_total.restype = C.c_int64
    L.nds_plan_execute.argtypes = [_vp, _vp, _vp, _vp]
    L.nds_plan_forward.argtypes = [_vp, _vp, _vp, _vp]
    L.nds_plan_backsub.argtypes = [_vp, _vp]
    L.nds_plan_inverse.argtypes = [_vp, _vp, _vp, _vp]
    L.nds_plan_execute_host.argtypes = [_vp, _vp, _vp, C.POINTER(_Report)]
    L.nds_plan_execute_host_many.argtypes = [_vp, C.c_int, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_Report)]
    L.nds_plan_launches.argtypes = [_vp]
    L.nds_plan_solve_path.argtypes = [_vp]
    L.nds_plan_diagonalised.argtypes = [_vp, C.POINTER(C.c_double)]
    L.nds_plan_superblocks.argtypes = [_vp, C.POINTER(C.c_int64)]
    L.nds_plan_profile_begin.argtypes = [_vp, C.c_int]
    L.nds_plan_profile_end.argtypes = [_vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                       C.POINTER(C.c_float)]
    L.nds_dev_mode_product.argtypes = [_vp, C.c_int, _i64p, _vp, C.c_int, C.c_int, _vp, _vp, C.c_int]
    L.nds_dev_mode_update.argtypes = [_vp, C.c_int, _i64p, C.c_int, C.c_int64, _vp, _vp, _vp]
    L.nds_dev_mode_apply.argtypes = [_vp, C.c_int, _i64p, C.c_int, C.c_int64, _vp, _vp, _vp]
    L.nds_dev_back_substitute.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, C.c_double, C.POINTER(_Stats),
                                          C.POINTER(_Singular)]
    L.nds_dev_residual.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp, C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.nds_triangular_exp.argtypes = [_vp, C.c_int, _vp, C.c_double, _vp]
    L.nds_ode_create.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp, _vp, C.c_double, C.c_uint, C.POINTER(_vp)]
    L.nds_ode_destroy.argtypes = [_vp]
    L.nds_ode_at.argtypes = [_vp, C.c_double, _vp, C.POINTER(_Report), C.POINTER(_Singular)]
    L.nds_ode_at_dev.argtypes = [_vp, C.c_double, _vp]
    L.nds_propagate.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp, C.c_double, C.c_double, C.c_uint, _vp,
                                C.POINTER(_Report), C.POINTER(_Singular)]
    L.nds_rk4.argtypes = [_vp, C.c_int, _i64p, _vp, _vp, _vp, C.c_double, C.c_double, C.c_int64, _vp]
    L.nds_tensor_file_info.argtypes = [C.c_char_p, C.POINTER(C.c_int), _i64p]
    L.nds_read_tensor.argtypes = [C.c_char_p, C.c_int, _i64p, _vp]
    L.nds_write_tensor.argtypes = [C.c_char_p, C.c_int, _i64p, _vp]
    L.nds_read_tensor_dev.argtypes = [_vp, C.c_char_p, C.c_int, _i64p, _vp]
    L.nds_write_tensor_dev.argtypes = [_vp, C.c_char_p, C.c_int, _i64p, _vp]
    L.nds_random_problem.argtypes = [_vp, C.c_int, _i64p, C.c_uint64, _vp, _vp, _vp]
    L.nds_random_ode_system.argtypes = [C.c_int, _i64p, C.c_uint64, _vp, _vp, _vp]
    L.nds_randn.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _vp]
    L.nds_comm_unique_id.argtypes = [_vp]
    L.nds_comm_create_nccl.argtypes = [C.POINTER(_vp), C.c_int, C.c_int, C.c_int, _vp]
    L.nds_comm_create_loopback.argtypes = [C.c_int, C.POINTER(_vp)]
    L.nds_comm_destroy.argtypes = [_vp]
    L.nds_dist_create.argtypes = [_vp, _vp, C.c_int, _i64p, _vp, _vp, C.c_double, C.POINTER(_vp),
                                  C.POINTER(_Singular)]
    L.nds_dist_destroy.argtypes = [_vp]
    L.nds_dist_slab.argtypes = [_vp, C.c_int, _i64p, _i64p]
    L.nds_dist_info.argtypes = [_vp, C.POINTER(_DistInfo)]
    L.nds_dist_solve.argtypes = [_vp, _vp, _vp]
    L.nds_solve_multi.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, _i64p, _vp, _vp, _vp, _vp, C.c_double,
                                  C.POINTER(_Singular)]
    _lib = L
    return L


def solve_multi(devices, us, ts, rhs, singular_tol=0.0) -> np.ndarray:
    """nds_solve_multi: the solve after the Schur step, sharded over `devices` of this process
    (one host thread + NCCL communicator per device; host buffers)."""
    L = load_library()
    b = _f(rhs)
    x = np.empty_like(b, order="F")
    up, ku = _ptr_array(us)
    tp, kt = _ptr_array(ts)
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    sing = _Singular()
    rc = L.nds_solve_multi(len(devices), devs, b.ndim, _dims(b.shape), up, tp, b.ctypes.data, x.ctypes.data,
                           float(singular_tol), C.byref(sing))
    if rc == ERR_SINGULAR:
        raise SingularOperatorError(L.nds_last_error(None).decode(), sing.multi_index[:sing.n_modes],
                                    complex(sing.den_re, sing.den_im))
    if rc:
        raise NdsError(rc, L.nds_last_error(None).decode())
    return x


def version() -> str:
    return load_library().nds_version().decode()


# ---- marshalling -----------------------------------------------------------------------------

def _f(x):
    return np.asfortranarray(np.asarray(x, dtype=np.complex128))


def _dims(shape):
    return (C.c_int64 * len(shape))(*[int(v) for v in shape])


def _ptr_array(mats):
    keep = [_f(m) for m in mats]
    arr = (_vp * len(keep))(*[m.ctypes.data for m in keep])
    return arr, keep


def _dict(s):
    return {k: getattr(s, k) for k, _ in s._fields_}


def _raise(code, msg, sing=None):
    if code == ERR_SINGULAR:
        mi = [sing.multi_index[j] for j in range(sing.n_modes)] if sing is not None else []
        den = complex(sing.den_re, sing.den_im) if sing is not None else complex("nan")
        raise SingularOperatorError(msg, mi, den)
    if code == ERR_INVALID:
        raise ValueError(msg)
    if code == ERR_OVERFLOW:
        raise OverflowError(msg)
    if code == ERR_NOMEM:
        raise MemoryError(msg)
    if code == ERR_CONVERGENCE:
        raise ConvergenceError(code, msg)
    if code == ERR_CUDA:
        raise DeviceError(code, msg)
    if code == ERR_NONFINITE:
        raise NonFiniteStateError(code, msg)
    if code == ERR_FILE:
        raise TensorFileError(code, msg)
    raise NdsError(code, msg)


def flop_estimate(dims) -> int:
    v = load_library().nds_flop_estimate(len(dims), _dims(dims))
    if v < 0:
        raise OverflowError("flop estimate overflows int64")
    return v


def schur_flop_estimate(dims) -> int:
    v = load_library().nds_schur_flop_estimate(len(dims), _dims(dims))
    if v < 0:
        raise OverflowError("flop estimate overflows int64")
    return v


# ---- NDT1 files and the reference generator (tensor_file.hpp, rng.hpp) ------------------------

def _noctx_check(rc):
    if rc:
        _raise(rc, load_library().nds_last_error(None).decode())


def tensor_file_info(path: str):
    """Extents of an NDT1 file."""
    n = C.c_int()
    dims = (C.c_int64 * 64)()
    _noctx_check(load_library().nds_tensor_file_info(path.encode(), C.byref(n), dims))
    return tuple(dims[j] for j in range(n.value))


def read_tensor(path: str) -> np.ndarray:
    """ndsylv::read_tensor (tensor_file.cpp:67-96)."""
    dims = tensor_file_info(path)
    out = np.empty(dims, dtype=np.complex128, order="F")
    _noctx_check(load_library().nds_read_tensor(path.encode(), len(dims), _dims(dims), out.ctypes.data))
    return out


def write_tensor(path: str, x) -> None:
    """ndsylv::write_tensor (tensor_file.cpp:48-65)."""
    x = _f(x)
    _noctx_check(load_library().nds_write_tensor(path.encode(), x.ndim, _dims(x.shape), x.ctypes.data))


def random_ode_system(dims, seed: int):
    """ndsylv::random_ode_system (rng.cpp:27-33): (A_list, forcing, initial)."""
    dims = tuple(int(d) for d in dims)
    a = [np.empty((n, n), dtype=np.complex128, order="F") for n in dims]
    f = np.empty(dims, dtype=np.complex128, order="F")
    x0 = np.empty_like(f, order="F")
    ap = (_vp * len(a))(*[m.ctypes.data for m in a])
    _noctx_check(load_library().nds_random_ode_system(len(dims), _dims(dims), int(seed), ap, f.ctypes.data,
                                                      x0.ctypes.data))
    return a, f, x0


def randn(seed: int, stream: int, count: int) -> np.ndarray:
    """Seeded standard normals (harness generator v1)."""
    out = np.empty(int(count), dtype=np.float64)
    load_library().nds_randn(seed & (2**64 - 1), stream & (2**64 - 1), int(count), out.ctypes.data)
    return out


@dataclass
class SolveResult:
    """SolveResult (sylvester.hpp:44-47)."""
    x: np.ndarray
    report: dict = field(default_factory=dict)


class OdePropagator:
    """ndsylv::OdePropagator (ode.hpp:18-36) from Schur factors: C and G0 stay on the device;
    at(t) runs the exp(t T_j) mode passes, one triangular solve and the inverse transform."""

    def __init__(self, ctx: "Context", us, ts, forcing, initial, singular_tol=0.0, real_output=False):
        self.ctx = ctx
        f, x0 = _f(forcing), _f(initial)
        self.dims = tuple(int(v) for v in f.shape)
        if len(us) != f.ndim or len(ts) != f.ndim:
            raise ValueError("coefficient count does not match tensor order")
        if x0.shape != f.shape:
            raise ValueError("initial state shape mismatch")
        up, self._ku = _ptr_array(us)
        tp, self._kt = _ptr_array(ts)
        h = _vp()
        rc = ctx.lib.nds_ode_create(ctx.h, f.ndim, _dims(self.dims), up, tp, f.ctypes.data, x0.ctypes.data,
                                    float(singular_tol), REAL_OUTPUT if real_output else 0, C.byref(h))
        if rc:
            _raise(rc, ctx.last_error())
        self.h = h

    def at(self, t: float) -> SolveResult:
        x = np.empty(self.dims, dtype=np.complex128, order="F")
        rep = _Report()
        sing = _Singular()
        rc = self.ctx.lib.nds_ode_at(self.h, float(t), x.ctypes.data, C.byref(rep), C.byref(sing))
        if rc:
            _raise(rc, self.ctx.last_error(), sing)
        return SolveResult(x, _dict(rep))

    def at_ptr(self, t: float, h_x: int) -> dict:
        """at(t) into a caller-owned host buffer (e.g. pinned) of prod(dims) complex128."""
        rep = _Report()
        sing = _Singular()
        rc = self.ctx.lib.nds_ode_at(self.h, float(t), h_x, C.byref(rep), C.byref(sing))
        if rc:
            _raise(rc, self.ctx.last_error(), sing)
        return _dict(rep)

    def at_dev(self, t: float, d_x: int):
        rc = self.ctx.lib.nds_ode_at_dev(self.h, float(t), d_x)
        if rc:
            _raise(rc, self.ctx.last_error())

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.nds_ode_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """Device-resident solver for one coefficient set (factors uploaded once)."""

    def __init__(self, ctx: "Context", us, ts, singular_tol=0.0, allow_fast_path=True, real_output=False,
                 diagonalise=True):
        self.ctx = ctx
        self.dims = tuple(int(u.shape[0]) for u in us)
        up, self._ku = _ptr_array(us)
        tp, self._kt = _ptr_array(ts)
        flags = (ALLOW_FAST_PATH if allow_fast_path else 0) | (REAL_OUTPUT if real_output else 0) | (
            0 if diagonalise else NO_DIAGONALISE)
        h = _vp()
        sing = _Singular()
        rc = ctx.lib.nds_plan_create(ctx.h, len(us), _dims(self.dims), up, tp, float(singular_tol), flags,
                                     C.byref(h), C.byref(sing))
        if rc:
            _raise(rc, ctx.last_error(), sing)
        self.h = h
        self.total = int(np.prod(self.dims))

    def report(self) -> dict:
        r = _Report()
        self.ctx.lib.nds_plan_report(self.h, C.byref(r))
        return _dict(r)

    def _check(self, rc):
        if rc:
            _raise(rc, self.ctx.last_error())

    def execute(self, d_b: int, d_x: int, d_work: int = 0):
        """Device pointers (ints), async on the context stream."""
        self._check(self.ctx.lib.nds_plan_execute(self.h, d_b, d_x, d_work or None))

    def forward(self, d_in: int, d_out: int, d_work: int):
        self._check(self.ctx.lib.nds_plan_forward(self.h, d_in, d_out, d_work))

    def backsub(self, d_c: int):
        self._check(self.ctx.lib.nds_plan_backsub(self.h, d_c))

    def inverse(self, d_in: int, d_out: int, d_work: int):
        self._check(self.ctx.lib.nds_plan_inverse(self.h, d_in, d_out, d_work))

    def execute_host(self, b: np.ndarray, x: np.ndarray | None = None):
        """Host buffers (b, x column-major complex128 of shape dims; may be pinned)."""
        b = _f(b)
        if x is None:
            x = np.empty_like(b, order="F")
        rep = _Report()
        self._check(self.ctx.lib.nds_plan_execute_host(self.h, b.ctypes.data, x.ctypes.data, C.byref(rep)))
        return SolveResult(x, _dict(rep))

    def execute_host_ptr(self, h_b: int, h_x: int) -> dict:
        rep = _Report()
        self._check(self.ctx.lib.nds_plan_execute_host(self.h, h_b, h_x, C.byref(rep)))
        return _dict(rep)

    def execute_host_many(self, bs, xs=None):
        """Several right-hand sides through this plan (nds_plan_execute_host_many): pinned host
        buffers are pipelined (H2D of b[k+1] / D2H of x[k-1] under solve k). bs: list of
        column-major complex128 arrays of shape dims (or host pointers as ints, with xs given)."""
        if bs and isinstance(bs[0], int):
            hb, hx, keep = list(bs), list(xs), None
        else:
            bs = [_f(b) for b in bs]
            if xs is None:
                xs = [np.empty_like(b, order="F") for b in bs]
            hb = [b.ctypes.data for b in bs]
            hx = [x.ctypes.data for x in xs]
        n = len(hb)
        pb = (_vp * max(n, 1))(*hb)
        px = (_vp * max(n, 1))(*hx)
        rep = _Report()
        self._check(self.ctx.lib.nds_plan_execute_host_many(self.h, n, pb, px, C.byref(rep)))
        return xs, _dict(rep)

    def launches(self) -> int:
        return self.ctx.lib.nds_plan_launches(self.h)

    SOLVE_PATHS = {0: "fast", 1: "generic", 2: "cubic", 3: "binary"}

    def solve_path(self) -> str:
        """Triangular-solve route: 'fast', 'generic' (any shape), 'cubic' (16^3 / 8^4 DMMA tiles)
        or 'binary' (all n_j = 2)."""
        return self.SOLVE_PATHS[self.ctx.lib.nds_plan_solve_path(self.h)]

    def diagonalised(self):
        """(taken, cond): whether full solves run on diagonalised factors (cubic: T_j's diagonal
        blocks; binary: the outer modes) and the guard's prod_j cond_2 bound."""
        c = C.c_double(0.0)
        r = self.ctx.lib.nds_plan_diagonalised(self.h, C.byref(c))
        return bool(r == 1), float(c.value)

    def superblocks(self):
        """(levels, D) of the block-diagonalised cubic route (super-block extent per mode), or
        (0, None) when full solves do not take it."""
        d = (C.c_int64 * len(self.dims))()
        lv = self.ctx.lib.nds_plan_superblocks(self.h, d)
        return (lv, tuple(int(x) for x in d)) if lv > 0 else (0, None)

    def profile_begin(self, max_launches: int):
        self._check(self.ctx.lib.nds_plan_profile_begin(self.h, int(max_launches)))

    KINDS = {0: "transform_gemm", 1: "transform_direct", 2: "solve_level", 3: "elementwise", 4: "solve_persistent"}

    def profile_end(self, cap: int = 1 << 16):
        """[(kind, mode, ms)] for every launch recorded since profile_begin."""
        kinds = (C.c_int * cap)()
        modes = (C.c_int * cap)()
        ms = (C.c_float * cap)()
        n = self.ctx.lib.nds_plan_profile_end(self.h, cap, kinds, modes, ms)
        if n < 0:
            _raise(-n, self.ctx.last_error())
        return [(self.KINDS.get(kinds[i], str(kinds[i])), modes[i], ms[i]) for i in range(n)]

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.nds_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One CUDA device + stream + workspaces (nds_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = _vp()
        rc = self.lib.nds_ctx_create(C.byref(h), int(device))
        if rc:
            _raise(rc, self.lib.nds_last_error(None).decode())
        self.h = h

    def last_error(self) -> str:
        return self.lib.nds_last_error(self.h).decode()

    def _check(self, rc, sing=None):
        if rc:
            _raise(rc, self.last_error(), sing)

    # cudaStreamLegacy: the legacy default stream (torch's default stream reports handle 0)
    LEGACY_STREAM = 0x1

    def set_stream(self, stream_handle: int | None):
        """Run the context's device work on an external stream. None restores the context's own
        stream; 0 (torch's default stream) means the legacy default stream, which orders with
        every blocking stream of the process — NOT the context's own non-blocking stream."""
        if stream_handle is None:
            h = None
        elif int(stream_handle) == 0:
            h = self.LEGACY_STREAM
        else:
            h = int(stream_handle)
        self._check(self.lib.nds_ctx_set_stream(self.h, h))

    def stream(self) -> int:
        return self.lib.nds_ctx_stream(self.h) or 0

    def trim(self):
        self.lib.nds_ctx_trim(self.h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.nds_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- reference API ------------------------------------------------------------------
    @staticmethod
    def _flags(allow_fast_path, real_output):
        return (ALLOW_FAST_PATH if allow_fast_path else 0) | (REAL_OUTPUT if real_output else 0)

    def solve(self, coefficients, rhs, singular_tol=0.0, allow_fast_path=True, real_output=False) -> SolveResult:
        """ndsylv::solve (sylvester.cpp:167-227): host Schur + GPU transforms and solve."""
        b = _f(rhs)
        if len(coefficients) != b.ndim:
            raise ValueError("coefficient count does not match tensor order")
        for j, a in enumerate(coefficients):
            a = np.asarray(a)
            if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape[0] != b.shape[j]:
                raise ValueError(f"coefficient {j + 1} does not match mode extent")
        ap, keep = _ptr_array(coefficients)
        x = np.empty_like(b, order="F")
        rep = _Report()
        sing = _Singular()
        rc = self.lib.nds_solve(self.h, b.ndim, _dims(b.shape), ap, b.ctypes.data, x.ctypes.data,
                                float(singular_tol), self._flags(allow_fast_path, real_output), C.byref(rep),
                                C.byref(sing))
        self._check(rc, sing)
        return SolveResult(x, _dict(rep))

    def solve_schur(self, us, ts, rhs, singular_tol=0.0, allow_fast_path=True, real_output=False) -> SolveResult:
        b = _f(rhs)
        up, k1 = _ptr_array(us)
        tp, k2 = _ptr_array(ts)
        x = np.empty_like(b, order="F")
        rep = _Report()
        sing = _Singular()
        rc = self.lib.nds_solve_schur(self.h, b.ndim, _dims(b.shape), up, tp, b.ctypes.data, x.ctypes.data,
                                      float(singular_tol), self._flags(allow_fast_path, real_output), C.byref(rep),
                                      C.byref(sing))
        self._check(rc, sing)
        return SolveResult(x, _dict(rep))

    def schur(self, a):
        a = _f(a)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("schur requires a non-empty square matrix")
        n = a.shape[0]
        u = np.empty((n, n), dtype=np.complex128, order="F")
        t = np.empty((n, n), dtype=np.complex128, order="F")
        self._check(self.lib.nds_schur(self.h, n, a.ctypes.data, u.ctypes.data, t.ctypes.data))
        return u, t

    def forward_transform(self, us, b):
        b = _f(b)
        up, keep = _ptr_array(us)
        c = np.empty_like(b, order="F")
        self._check(self.lib.nds_forward_transform(self.h, b.ndim, _dims(b.shape), up, b.ctypes.data, c.ctypes.data))
        return c

    def inverse_transform(self, us, y):
        y = _f(y)
        up, keep = _ptr_array(us)
        x = np.empty_like(y, order="F")
        self._check(self.lib.nds_inverse_transform(self.h, y.ndim, _dims(y.shape), up, y.ctypes.data, x.ctypes.data))
        return x

    def back_substitute(self, ts, c, singular_tol=0.0):
        """Returns (y, stats). The reference overwrites c in place; here c is copied."""
        y = _f(c).copy(order="F")
        tp, keep = _ptr_array(ts)
        st = _Stats()
        sing = _Singular()
        rc = self.lib.nds_back_substitute(self.h, y.ndim, _dims(y.shape), tp, y.ctypes.data, float(singular_tol),
                                          C.byref(st), C.byref(sing))
        self._check(rc, sing)
        return y, _dict(st)

    def mode_product(self, m, mode, x):
        x = _f(x)
        m = _f(m)
        r = np.empty_like(x, order="F")
        self._check(self.lib.nds_mode_product(self.h, x.ndim, _dims(x.shape), m.ctypes.data, int(mode),
                                              x.ctypes.data, r.ctypes.data))
        return r

    def apply_operator(self, coefficients, x):
        x = _f(x)
        ap, keep = _ptr_array(coefficients)
        r = np.empty_like(x, order="F")
        self._check(self.lib.nds_apply_operator(self.h, x.ndim, _dims(x.shape), ap, x.ctypes.data, r.ctypes.data))
        return r

    # ---- ODE (ode.hpp) ------------------------------------------------------------------------
    def triangular_exp(self, t_mat, t: float):
        """ndsylv::triangular_exp (schur.cpp:203-228), host."""
        tm = _f(t_mat)
        if tm.ndim != 2 or tm.shape[0] != tm.shape[1]:
            raise ValueError("triangular_exp requires a square matrix")
        f = np.empty_like(tm, order="F")
        self._check(self.lib.nds_triangular_exp(self.h, tm.shape[0], tm.ctypes.data, float(t), f.ctypes.data))
        return f

    def ode(self, us, ts, forcing, initial, singular_tol=0.0, real_output=False) -> OdePropagator:
        return OdePropagator(self, us, ts, forcing, initial, singular_tol, real_output)

    def propagate(self, coefficients, forcing, initial, t: float, singular_tol=0.0, real_output=False) -> SolveResult:
        """ndsylv::propagate (ode.cpp:89-91): host Schur + OdePropagator(...).at(t)."""
        f, x0 = _f(forcing), _f(initial)
        ap, keep = _ptr_array(coefficients)
        x = np.empty_like(f, order="F")
        rep = _Report()
        sing = _Singular()
        rc = self.lib.nds_propagate(self.h, f.ndim, _dims(f.shape), ap, f.ctypes.data, x0.ctypes.data, float(t),
                                    float(singular_tol), REAL_OUTPUT if real_output else 0, x.ctypes.data,
                                    C.byref(rep), C.byref(sing))
        self._check(rc, sing)
        return SolveResult(x, _dict(rep))

    def rk4(self, coefficients, forcing, initial, t: float, dt: float, max_steps: int = 50_000_000):
        """ndsylv::rk4_reference (ode.cpp:93-129) on the device."""
        f, x0 = _f(forcing), _f(initial)
        ap, keep = _ptr_array(coefficients)
        x = np.empty_like(f, order="F")
        self._check(self.lib.nds_rk4(self.h, f.ndim, _dims(f.shape), ap, f.ctypes.data, x0.ctypes.data, float(t),
                                     float(dt), int(max_steps), x.ctypes.data))
        return x

    def random_problem(self, dims, seed: int):
        """ndsylv::random_problem (rng.cpp:18-25): (A_list, x_true, b), b computed on the GPU."""
        dims = tuple(int(d) for d in dims)
        a = [np.empty((n, n), dtype=np.complex128, order="F") for n in dims]
        x = np.empty(dims, dtype=np.complex128, order="F")
        b = np.empty_like(x, order="F")
        ap = (_vp * len(a))(*[m.ctypes.data for m in a])
        self._check(self.lib.nds_random_problem(self.h, len(dims), _dims(dims), int(seed), ap, x.ctypes.data,
                                                b.ctypes.data))
        return a, x, b

    def read_tensor_dev(self, path: str, dims, d_out: int):
        self._check(self.lib.nds_read_tensor_dev(self.h, path.encode(), len(dims), _dims(dims), d_out))

    def write_tensor_dev(self, path: str, dims, d_in: int):
        self._check(self.lib.nds_write_tensor_dev(self.h, path.encode(), len(dims), _dims(dims), d_in))

    # ---- device surfaces ------------------------------------------------------------------
    def plan(self, us, ts, singular_tol=0.0, allow_fast_path=True, real_output=False, diagonalise=True) -> Plan:
        return Plan(self, us, ts, singular_tol, allow_fast_path, real_output, diagonalise)

    def dev_mode_product(self, dims, d_m: int, mode: int, d_x: int, d_r: int, conj_transpose=False,
                         accumulate=False):
        self._check(self.lib.nds_dev_mode_product(self.h, len(dims), _dims(dims), d_m, int(mode),
                                                  1 if conj_transpose else 0, d_x, d_r, 1 if accumulate else 0))

    def dev_mode_update(self, dims_x, mode: int, m, d_x: int, d_r: int):
        """r += m x_mode x on device tensors; m is a host (rows_out, n_mode) matrix."""
        m = _f(m)
        self._check(self.lib.nds_dev_mode_update(self.h, len(dims_x), _dims(dims_x), int(mode), int(m.shape[0]),
                                                 m.ctypes.data, d_x, d_r))

    def dev_mode_apply(self, dims_x, mode: int, m, d_x: int, d_r: int):
        """r = m x_mode x on device tensors (no accumulation); m is a host (rows_out, n_mode) matrix."""
        m = _f(m)
        self._check(self.lib.nds_dev_mode_apply(self.h, len(dims_x), _dims(dims_x), int(mode), int(m.shape[0]),
                                                m.ctypes.data, d_x, d_r))

    def dev_back_substitute(self, ts, dims, d_c: int, singular_tol=0.0) -> dict:
        """In-place triangular solve of a device tensor (back_substitute on device memory)."""
        tp, keep = _ptr_array(ts)
        st = _Stats()
        sing = _Singular()
        rc = self.lib.nds_dev_back_substitute(self.h, len(dims), _dims(dims), tp, d_c, float(singular_tol),
                                              C.byref(st), C.byref(sing))
        self._check(rc, sing)
        return _dict(st)

    def dev_residual(self, coefficients, dims, d_x: int, d_b: int) -> dict:
        ap, keep = _ptr_array(coefficients)
        vals = [C.c_double() for _ in range(4)]
        self._check(self.lib.nds_dev_residual(self.h, len(dims), _dims(dims), ap, d_x, d_b, *[C.byref(v) for v in vals]))
        rm, r2, bm, b2 = (v.value for v in vals)
        return {"res_max": rm, "res_2": r2, "b_max": bm, "b_2": b2,
                "rel_res_max": rm / bm if bm else float("inf"), "rel_res_2": r2 / b2 if b2 else float("inf")}
