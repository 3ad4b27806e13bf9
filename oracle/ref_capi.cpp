// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj/src/*.cpp),
// compiled together with it by oracle/Makefile into oracle/_ref/libndsylv_ref.so.
// It exposes the reference's own public C++ API (proj/include/ndsylv/*.hpp) to ctypes so the
// tests can (1) pin the plain-C restatement in ndsylv_oracle.c and (2) generate golden
// fixtures, and so bench.py --impl reference can time the reference CPU solver.
// No reference source is copied; this file only marshals plain buffers to/from the
// reference types (NDTensor / Matrix / SchurFactors, column-major complex<double>).
#include <omp.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "ndsylv/kron.hpp"
#include "ndsylv/ode.hpp"
#include "ndsylv/schur.hpp"
#include "ndsylv/tensor_file.hpp"
#include "ndsylv/rng.hpp"
#include "ndsylv/sylvester.hpp"

using namespace ndsylv;

namespace {

thread_local std::string g_err;

std::vector<std::int64_t> dims_of(int n_modes, const std::int64_t* dims) {
  return std::vector<std::int64_t>(dims, dims + n_modes);
}

NDTensor tensor_from(int n_modes, const std::int64_t* dims, const double* data) {
  const auto d = dims_of(n_modes, dims);
  const std::int64_t total = checked_total(d);
  const cxd* p = reinterpret_cast<const cxd*>(data);
  return NDTensor::make(d, std::vector<cxd>(p, p + total));
}

void tensor_to(const NDTensor& t, double* out) { std::memcpy(out, t.data.data(), t.data.size() * sizeof(cxd)); }

Matrix matrix_from(int n, const double* data) {
  Matrix m(n, n);
  std::memcpy(m.data(), data, static_cast<std::size_t>(n) * n * sizeof(cxd));
  return m;
}

void matrix_to(const Matrix& m, double* out) {
  std::memcpy(out, m.data(), static_cast<std::size_t>(m.rows()) * m.cols() * sizeof(cxd));
}

// Exit-code mapping mirrors tools/ndsylv_main.cpp:366-381 plus finer codes for the tests.
template <class F>
int guarded(F&& f, std::int64_t* bad_index = nullptr, double* bad_den = nullptr) {
  try {
    f();
    return 0;
  } catch (const SingularOperatorError& e) {
    g_err = e.what();
    if (bad_index) std::copy(e.multi_index().begin(), e.multi_index().end(), bad_index);
    if (bad_den) {
      bad_den[0] = e.denominator().real();
      bad_den[1] = e.denominator().imag();
    }
    return 2;
  } catch (const TensorFileError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return 4;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 5;
  } catch (const ConvergenceError& e) {
    g_err = e.what();
    return 6;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return 7;
  } catch (const NonFiniteStateError& e) {
    g_err = e.what();
    return 9;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

std::vector<SchurFactors> factors_from(int n_modes, const std::int64_t* dims, const double* const* u,
                                       const double* const* t) {
  std::vector<SchurFactors> f;
  for (int j = 0; j < n_modes; ++j) {
    const int n = static_cast<int>(dims[j]);
    SchurFactors s{matrix_from(n, u[j]), t ? matrix_from(n, t[j]) : Matrix::identity(n)};
    f.push_back(std::move(s));
  }
  return f;
}

}  // namespace

extern "C" {

struct ref_report {
  double min_abs_denominator;
  int used_normal_fast_path;
  std::int64_t flop_estimate;
  std::int64_t schur_flop_estimate;
  std::int64_t backsub_entries;
  std::int64_t backsub_multiplies;
  double schur_seconds;
  double transform_seconds;
  double backsub_seconds;
  double inverse_seconds;
  double total_seconds;
};

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_get_max_threads() { return omp_get_max_threads(); }

// sylvester.hpp:79 — the reference drop-in surface, Schur included.
int ref_solve(int n_modes, const std::int64_t* dims, const double* const* a, const double* b, double* x,
              double singular_tol, unsigned flags, ref_report* rep, std::int64_t* bad_index, double* bad_den) {
  return guarded(
      [&] {
        SylvesterProblem p;
        for (int j = 0; j < n_modes; ++j) p.coefficients.push_back(matrix_from(static_cast<int>(dims[j]), a[j]));
        p.rhs = tensor_from(n_modes, dims, b);
        SolveOptions o;
        o.singular_tol = singular_tol;
        o.allow_fast_path = (flags & 1u) != 0;
        o.real_output = (flags & 2u) != 0;
        const SolveResult r = solve(p, o);
        tensor_to(r.x, x);
        if (rep) {
          rep->min_abs_denominator = r.report.min_abs_denominator;
          rep->used_normal_fast_path = r.report.used_normal_fast_path;
          rep->flop_estimate = r.report.flop_estimate;
          rep->schur_flop_estimate = r.report.schur_flop_estimate;
          rep->backsub_entries = r.report.backsub_entries;
          rep->backsub_multiplies = r.report.backsub_multiplies;
          rep->schur_seconds = r.report.schur_seconds;
          rep->transform_seconds = r.report.transform_seconds;
          rep->backsub_seconds = r.report.backsub_seconds;
          rep->inverse_seconds = r.report.inverse_seconds;
          rep->total_seconds = r.report.total_seconds;
        }
      },
      bad_index, bad_den);
}

// schur.hpp:19
int ref_schur(int n, const double* a, double* u, double* t) {
  return guarded([&] {
    const SchurFactors f = schur(matrix_from(n, a));
    matrix_to(f.u, u);
    matrix_to(f.t, t);
  });
}

// sylvester.hpp:64
int ref_forward_transform(int n_modes, const std::int64_t* dims, const double* const* u, const double* b, double* c) {
  return guarded([&] {
    const auto f = factors_from(n_modes, dims, u, nullptr);
    tensor_to(forward_transform(f, tensor_from(n_modes, dims, b)), c);
  });
}

// sylvester.hpp:67
int ref_inverse_transform(int n_modes, const std::int64_t* dims, const double* const* u, const double* y, double* x) {
  return guarded([&] {
    const auto f = factors_from(n_modes, dims, u, nullptr);
    tensor_to(inverse_transform(f, tensor_from(n_modes, dims, y)), x);
  });
}

// sylvester.hpp:77 — in place, like the reference.
int ref_back_substitute(int n_modes, const std::int64_t* dims, const double* const* t, double* c, double singular_tol,
                        std::int64_t* entries, std::int64_t* multiplies, double* min_abs_den, std::int64_t* bad_index,
                        double* bad_den) {
  return guarded(
      [&] {
        std::vector<Matrix> ts;
        for (int j = 0; j < n_modes; ++j) ts.push_back(matrix_from(static_cast<int>(dims[j]), t[j]));
        NDTensor ct = tensor_from(n_modes, dims, c);
        const BackSubstituteStats st = back_substitute(ts, ct, singular_tol);
        tensor_to(ct, c);
        if (entries) *entries = st.entries;
        if (multiplies) *multiplies = st.multiplies;
        if (min_abs_den) *min_abs_den = st.min_abs_denominator;
      },
      bad_index, bad_den);
}

// kernels.hpp:12 (OpenMP) and kernels.hpp:29 (serial twin)
int ref_mode_product(int n_modes, const std::int64_t* dims, const double* m, int mode, const double* x, double* r,
                     int serial_twin) {
  return guarded([&] {
    const Matrix mm = matrix_from(static_cast<int>(mode >= 1 && mode <= n_modes ? dims[mode - 1] : 0), m);
    const NDTensor xt = tensor_from(n_modes, dims, x);
    tensor_to(serial_twin ? serial::mode_product(mm, mode, xt) : mode_product(mm, mode, xt), r);
  });
}

// sylvester.hpp:61
int ref_apply_operator(int n_modes, const std::int64_t* dims, const double* const* a, const double* x, double* r) {
  return guarded([&] {
    std::vector<Matrix> as;
    for (int j = 0; j < n_modes; ++j) as.push_back(matrix_from(static_cast<int>(dims[j]), a[j]));
    tensor_to(apply_operator(as, tensor_from(n_modes, dims, x)), r);
  });
}

// rng.hpp:64 — A_1..A_N uniform, X_true uniform, B = op(X_true).
int ref_random_problem(int n_modes, const std::int64_t* dims, std::uint64_t seed, double* const* a, double* x_true,
                       double* b) {
  return guarded([&] {
    const GeneratedProblem g = random_problem(dims_of(n_modes, dims), seed);
    for (int j = 0; j < n_modes; ++j) matrix_to(g.problem.coefficients[static_cast<std::size_t>(j)], a[j]);
    tensor_to(g.x_true, x_true);
    tensor_to(g.problem.rhs, b);
  });
}

// kron.hpp:21 — dense Kronecker-sum LU oracle (order <= max_order).
int ref_oracle_solve(int n_modes, const std::int64_t* dims, const double* const* a, const double* b, double* x) {
  return guarded([&] {
    SylvesterProblem p;
    for (int j = 0; j < n_modes; ++j) p.coefficients.push_back(matrix_from(static_cast<int>(dims[j]), a[j]));
    p.rhs = tensor_from(n_modes, dims, b);
    tensor_to(oracle_solve(p), x);
  });
}

std::int64_t ref_flop_estimate(int n_modes, const std::int64_t* dims) {
  std::int64_t v = -1;
  guarded([&] { v = flop_estimate(dims_of(n_modes, dims)); });
  return v;
}

std::int64_t ref_schur_flop_estimate(int n_modes, const std::int64_t* dims) {
  std::int64_t v = -1;
  guarded([&] { v = schur_flop_estimate(dims_of(n_modes, dims)); });
  return v;
}

// ndsylv::triangular_exp (schur.hpp:24)
int ref_triangular_exp(int n, const double* t_mat, double t, double* f) {
  return guarded([&] { matrix_to(triangular_exp(matrix_from(n, t_mat), t), f); });
}

OdeSystem system_from(int n_modes, const std::int64_t* dims, const double* const* a, const double* forcing,
                      const double* initial) {
  OdeSystem sys;
  for (int j = 0; j < n_modes; ++j) sys.coefficients.push_back(matrix_from(static_cast<int>(dims[j]), a[j]));
  sys.forcing = tensor_from(n_modes, dims, forcing);
  sys.initial = tensor_from(n_modes, dims, initial);
  return sys;
}

// ndsylv::propagate (ode.hpp:39): Schur inside the OdePropagator constructor.
int ref_propagate(int n_modes, const std::int64_t* dims, const double* const* a, const double* forcing,
                  const double* initial, double time, int real_output, double* x, ref_report* rep,
                  std::int64_t* bad_index, double* bad_den) {
  return guarded(
      [&] {
        SolveOptions opt;
        opt.real_output = real_output != 0;
        const SolveResult r = propagate(system_from(n_modes, dims, a, forcing, initial), time, opt);
        tensor_to(r.x, x);
        if (rep) {
          rep->min_abs_denominator = r.report.min_abs_denominator;
          rep->used_normal_fast_path = r.report.used_normal_fast_path ? 1 : 0;
          rep->flop_estimate = r.report.flop_estimate;
          rep->schur_flop_estimate = r.report.schur_flop_estimate;
          rep->backsub_entries = r.report.backsub_entries;
          rep->backsub_multiplies = r.report.backsub_multiplies;
          rep->schur_seconds = r.report.schur_seconds;
          rep->transform_seconds = r.report.transform_seconds;
          rep->backsub_seconds = r.report.backsub_seconds;
          rep->inverse_seconds = r.report.inverse_seconds;
          rep->total_seconds = r.report.total_seconds;
        }
      },
      bad_index, bad_den);
}

// ndsylv::rk4_reference (ode.hpp:44)
int ref_rk4(int n_modes, const std::int64_t* dims, const double* const* a, const double* forcing,
            const double* initial, double time, double dt, std::int64_t max_steps, double* x) {
  return guarded([&] {
    tensor_to(rk4_reference(system_from(n_modes, dims, a, forcing, initial), time, dt, max_steps), x);
  });
}

// ndsylv::write_tensor / read_tensor (tensor_file.hpp)
int ref_write_tensor(const char* path, int n_modes, const std::int64_t* dims, const double* data) {
  return guarded([&] { write_tensor(path, tensor_from(n_modes, dims, data)); });
}
int ref_read_tensor(const char* path, int* n_modes, std::int64_t* dims, double* out, std::int64_t cap) {
  return guarded([&] {
    const NDTensor t = read_tensor(path);
    *n_modes = t.order();
    for (int j = 0; j < t.order(); ++j) dims[j] = t.dims[j];
    if (out && t.size() <= cap) tensor_to(t, out);
  });
}

// ndsylv::random_ode_system (rng.hpp:70)
int ref_random_ode_system(int n_modes, const std::int64_t* dims, std::uint64_t seed, double* const* a, double* forcing,
                          double* initial) {
  return guarded([&] {
    const OdeSystem s = random_ode_system(dims_of(n_modes, dims), seed);
    for (int j = 0; j < n_modes; ++j) matrix_to(s.coefficients[j], a[j]);
    tensor_to(s.forcing, forcing);
    tensor_to(s.initial, initial);
  });
}

void ref_xoshiro_uniform(std::uint64_t seed, std::int64_t count, double* out) {
  Xoshiro256pp rng(seed);
  for (std::int64_t i = 0; i < count; ++i) out[i] = rng.uniform();
}

// Harness input generator v1 (NOT reference code): counter-based splitmix64 +
// Box-Muller, the same stream as the product's nds_randn (csrc/randn.cpp), so that the reference
// arm of bench.py and the X_ref fixture scripts build their inputs without loading the product
// library. Value pair m of (seed, stream) uses counters 2m and 2m+1.
void ref_harness_randn(std::uint64_t seed, std::uint64_t stream, std::int64_t count, double* out) {
  auto mix = [](std::uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  };
  const std::uint64_t key = mix(mix(seed) ^ (stream * 0xd1342543de82ef95ULL + 0x632be59bd9b4e019ULL));
  const std::int64_t pairs = (count + 1) / 2;
  const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static)
  for (std::int64_t m = 0; m < pairs; ++m) {
    const std::uint64_t b1 = mix(key + (2 * static_cast<std::uint64_t>(m) + 1) * 0x9e3779b97f4a7c15ULL);
    const std::uint64_t b2 = mix(key + (2 * static_cast<std::uint64_t>(m) + 2) * 0x9e3779b97f4a7c15ULL);
    const double u1 = static_cast<double>((b1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(b2 >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = two_pi * u2;
    out[2 * m] = r * std::cos(th);
    if (2 * m + 1 < count) out[2 * m + 1] = r * std::sin(th);
  }
}

// ndsylv::solve on a harness-generated right-hand side: B = ref_harness_randn(seed, 1000, 2P)
// (generator v1) written straight into the reference's NDTensor, or copied from
// `b` when it is non-null. Used by tests/golden/make_xref.py for the full-size X_ref fixtures of
// c1-c4, where a separate host copy of an 8.6 GB B would not fit next to the solve.
int ref_solve_gen(int n_modes, const std::int64_t* dims, const double* const* a, const double* b,
                  std::uint64_t seed, double* x, ref_report* rep) {
  return guarded([&] {
    SylvesterProblem p;
    for (int j = 0; j < n_modes; ++j) p.coefficients.push_back(matrix_from(static_cast<int>(dims[j]), a[j]));
    if (b) {
      p.rhs = tensor_from(n_modes, dims, b);
    } else {
      const auto d = dims_of(n_modes, dims);
      const std::int64_t total = checked_total(d);
      std::vector<cxd> v(static_cast<std::size_t>(total));
      ref_harness_randn(seed, 1000, 2 * total, reinterpret_cast<double*>(v.data()));
      p.rhs = NDTensor::make(d, std::move(v));
    }
    const SolveResult r = solve(p, SolveOptions{});
    tensor_to(r.x, x);
    if (rep) {
      rep->min_abs_denominator = r.report.min_abs_denominator;
      rep->used_normal_fast_path = r.report.used_normal_fast_path;
      rep->flop_estimate = r.report.flop_estimate;
      rep->schur_flop_estimate = r.report.schur_flop_estimate;
      rep->backsub_entries = r.report.backsub_entries;
      rep->backsub_multiplies = r.report.backsub_multiplies;
      rep->schur_seconds = r.report.schur_seconds;
      rep->transform_seconds = r.report.transform_seconds;
      rep->backsub_seconds = r.report.backsub_seconds;
      rep->inverse_seconds = r.report.inverse_seconds;
      rep->total_seconds = r.report.total_seconds;
    }
  });
}

}  // extern "C"
