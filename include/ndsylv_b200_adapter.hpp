// ndsylv_b200_adapter.hpp — B200 back end for ndsylv::solve with the reference's own types and
// exceptions (include together with the reference headers, link libndsylv_b200.so).
#pragma once
#include <chrono>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>
#include "ndsylv/ode.hpp"
#include "ndsylv/sylvester.hpp"
#include "ndsylv_b200.h"

namespace ndsylv::gpu {

inline nds_ctx* context() {  // one context per host thread (sylvester.hpp: solve is reentrant)
  thread_local std::unique_ptr<nds_ctx, void (*)(nds_ctx*)> c{nullptr, nds_ctx_destroy};
  if (!c) {
    nds_ctx* raw = nullptr;
    if (nds_ctx_create(&raw, 0) != NDS_OK) throw std::runtime_error(nds_last_error(nullptr));
    c.reset(raw);
  }
  return c.get();
}

inline void rethrow(int rc, const nds_singular& s) {
  const char* msg = nds_last_error(context());
  switch (rc) {
    case NDS_OK: return;
    case NDS_ERR_SINGULAR:
      throw SingularOperatorError(std::vector<std::int64_t>(s.multi_index, s.multi_index + s.n_modes),
                                  cxd(s.den_re, s.den_im));
    case NDS_ERR_INVALID: throw std::invalid_argument(msg);
    case NDS_ERR_OVERFLOW: throw std::overflow_error(msg);
    case NDS_ERR_CONVERGENCE: throw ConvergenceError(msg);
    case NDS_ERR_NOMEM: throw std::bad_alloc();
    case NDS_ERR_NONFINITE: throw NonFiniteStateError(msg);
    default: throw std::runtime_error(msg);
  }
}

// The reference's shape checks (sylvester.cpp:17-27 validate_problem, ode.cpp:17-28) with its
// messages, run before any Schur step or C-ABI call reads the coefficient storage.
inline void validate_coefficients(const std::vector<Matrix>& coefficients, const std::vector<std::int64_t>& dims,
                                  const char* what) {
  const int n_modes = static_cast<int>(dims.size());
  if (n_modes < 2) throw std::invalid_argument(std::string(what) + " order must be at least 2");
  if (static_cast<int>(coefficients.size()) != n_modes)
    throw std::invalid_argument("coefficient count does not match tensor order");
  for (int j = 0; j < n_modes; ++j) {
    const Matrix& a = coefficients[static_cast<std::size_t>(j)];
    if (!a.square() || a.rows() != dims[static_cast<std::size_t>(j)])
      throw std::invalid_argument("coefficient " + std::to_string(j + 1) + " does not match mode extent");
  }
}

// Same contract as ndsylv::solve (sylvester.cpp:167-227): Schur on the host with the
// reference's own ndsylv::schur, transforms + triangular solve on the GPU.
inline SolveResult solve(const SylvesterProblem& p, const SolveOptions& o = {}) {
  validate_coefficients(p.coefficients, p.rhs.dims, "problem");
  const int n = p.rhs.order();
  std::vector<SchurFactors> f;
  SolveResult r;
  auto t0 = std::chrono::steady_clock::now();
  for (const Matrix& a : p.coefficients) f.push_back(schur(a));
  const double schur_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<const nds_z*> u, t;
  for (auto& s : f) {
    u.push_back(reinterpret_cast<const nds_z*>(s.u.data()));
    t.push_back(reinterpret_cast<const nds_z*>(s.t.data()));
  }
  r.x = NDTensor::zeros(p.rhs.dims);
  nds_report rep{};
  nds_singular sing{};
  const unsigned flags = (o.allow_fast_path ? NDS_ALLOW_FAST_PATH : 0u) | (o.real_output ? NDS_REAL_OUTPUT : 0u);
  rethrow(nds_solve_schur(context(), n, p.rhs.dims.data(), u.data(), t.data(),
                          reinterpret_cast<const nds_z*>(p.rhs.data.data()),
                          reinterpret_cast<nds_z*>(r.x.data.data()), o.singular_tol, flags, &rep, &sing),
          sing);
  r.report.min_abs_denominator = rep.min_abs_denominator;
  r.report.used_normal_fast_path = rep.used_normal_fast_path != 0;
  r.report.flop_estimate = rep.flop_estimate;
  r.report.schur_flop_estimate = rep.schur_flop_estimate;
  r.report.backsub_entries = rep.backsub_entries;
  r.report.backsub_multiplies = rep.backsub_multiplies;
  r.report.schur_seconds = schur_s;
  r.report.transform_seconds = rep.transform_seconds;
  r.report.backsub_seconds = rep.backsub_seconds;
  r.report.inverse_seconds = rep.inverse_seconds;
  r.report.total_seconds = schur_s + rep.total_seconds;
  return r;
}

// Several right-hand sides with the same coefficients: what a loop of ndsylv::solve over
// problems that share A_1..A_N computes (sylvester.cpp:167-227 per call), with the Schur step and
// the device plan done once (nds_plan_create) and the right-hand sides streamed through
// nds_plan_execute_host_many (pipelined when the tensors' storage is pinned).
inline std::vector<NDTensor> solve_many(const std::vector<Matrix>& coefficients, const std::vector<NDTensor>& rhs,
                                        const SolveOptions& o = {}) {
  std::vector<NDTensor> xs;
  if (rhs.empty()) return xs;
  validate_coefficients(coefficients, rhs[0].dims, "problem");
  for (const NDTensor& b : rhs)
    if (b.dims != rhs[0].dims) throw std::invalid_argument("right-hand side shape mismatch");
  std::vector<SchurFactors> f;
  for (const Matrix& a : coefficients) f.push_back(schur(a));
  std::vector<const nds_z*> u, t;
  for (auto& s : f) {
    u.push_back(reinterpret_cast<const nds_z*>(s.u.data()));
    t.push_back(reinterpret_cast<const nds_z*>(s.t.data()));
  }
  const unsigned flags = (o.allow_fast_path ? NDS_ALLOW_FAST_PATH : 0u) | (o.real_output ? NDS_REAL_OUTPUT : 0u);
  nds_plan* plan = nullptr;
  nds_singular sing{};
  rethrow(nds_plan_create(context(), rhs[0].order(), rhs[0].dims.data(), u.data(), t.data(), o.singular_tol, flags,
                          &plan, &sing),
          sing);
  std::vector<const nds_z*> hb;
  std::vector<nds_z*> hx;
  for (const NDTensor& b : rhs) {
    xs.push_back(NDTensor::zeros(b.dims));
    hb.push_back(reinterpret_cast<const nds_z*>(b.data.data()));
    hx.push_back(reinterpret_cast<nds_z*>(xs.back().data.data()));
  }
  const int rc = nds_plan_execute_host_many(plan, static_cast<int>(rhs.size()), hb.data(), hx.data(), nullptr);
  nds_plan_destroy(plan);
  rethrow(rc, sing);
  return xs;
}

// The same solve sharded over several GPUs of this process (nds_solve_multi: one host thread,
// context and NCCL communicator per device). Report: Schur time only (the per-device stage times
// stay inside the library).
inline SolveResult solve_multi(const SylvesterProblem& p, const std::vector<int>& devices, const SolveOptions& o = {}) {
  validate_coefficients(p.coefficients, p.rhs.dims, "problem");
  std::vector<SchurFactors> f;
  SolveResult r;
  const auto t0 = std::chrono::steady_clock::now();
  for (const Matrix& a : p.coefficients) f.push_back(schur(a));
  r.report.schur_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<const nds_z*> u, t;
  for (auto& s : f) {
    u.push_back(reinterpret_cast<const nds_z*>(s.u.data()));
    t.push_back(reinterpret_cast<const nds_z*>(s.t.data()));
  }
  r.x = NDTensor::zeros(p.rhs.dims);
  nds_singular sing{};
  const int rc = nds_solve_multi(static_cast<int>(devices.size()), devices.data(), p.rhs.order(), p.rhs.dims.data(),
                                 u.data(), t.data(), reinterpret_cast<const nds_z*>(p.rhs.data.data()),
                                 reinterpret_cast<nds_z*>(r.x.data.data()), o.singular_tol, &sing);
  if (rc == NDS_ERR_SINGULAR)
    throw SingularOperatorError(std::vector<std::int64_t>(sing.multi_index, sing.multi_index + sing.n_modes),
                                cxd(sing.den_re, sing.den_im));
  if (rc != NDS_OK) throw std::runtime_error(nds_last_error(nullptr));
  r.report.backsub_entries = static_cast<std::int64_t>(p.rhs.data.size());
  r.report.total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

// Stage functions (sylvester.hpp:64-77) map 1:1: nds_forward_transform, nds_inverse_transform,
// nds_back_substitute (in place, like the reference), nds_mode_product, nds_apply_operator.

// ---- ODE (ode.hpp): same contracts as ndsylv::OdePropagator / propagate / rk4_reference -----
class OdePropagator {
 public:
  explicit OdePropagator(OdeSystem system, SolveOptions options = {})
      : system_(std::move(system)), options_(options) {
    const int n = system_.forcing.order();
    validate_coefficients(system_.coefficients, system_.forcing.dims, "system");
    if (system_.initial.dims != system_.forcing.dims) throw std::invalid_argument("initial state shape mismatch");
    const auto t0 = std::chrono::steady_clock::now();
    for (const Matrix& a : system_.coefficients) factors_.push_back(schur(a));
    schur_seconds_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<const nds_z*> u, t;
    for (auto& f : factors_) {
      u.push_back(reinterpret_cast<const nds_z*>(f.u.data()));
      t.push_back(reinterpret_cast<const nds_z*>(f.t.data()));
    }
    nds_ode* raw = nullptr;
    rethrow(nds_ode_create(context(), n, system_.forcing.dims.data(), u.data(), t.data(),
                           reinterpret_cast<const nds_z*>(system_.forcing.data.data()),
                           reinterpret_cast<const nds_z*>(system_.initial.data.data()), options_.singular_tol,
                           options_.real_output ? NDS_REAL_OUTPUT : 0u, &raw),
            nds_singular{});
    ode_.reset(raw);
  }

  SolveResult at(double t) const {
    SolveResult r;
    r.x = NDTensor::zeros(system_.forcing.dims);
    nds_report rep{};
    nds_singular sing{};
    rethrow(nds_ode_at(ode_.get(), t, reinterpret_cast<nds_z*>(r.x.data.data()), &rep, &sing), sing);
    r.report.min_abs_denominator = rep.min_abs_denominator;
    r.report.flop_estimate = rep.flop_estimate;
    r.report.schur_flop_estimate = rep.schur_flop_estimate;
    r.report.backsub_entries = rep.backsub_entries;
    r.report.backsub_multiplies = rep.backsub_multiplies;
    r.report.schur_seconds = schur_seconds_;
    r.report.transform_seconds = rep.transform_seconds;
    r.report.backsub_seconds = rep.backsub_seconds;
    r.report.inverse_seconds = rep.inverse_seconds;
    r.report.total_seconds = schur_seconds_ + rep.total_seconds;
    return r;
  }

  const OdeSystem& system() const noexcept { return system_; }

 private:
  OdeSystem system_;
  SolveOptions options_;
  std::vector<SchurFactors> factors_;
  double schur_seconds_ = 0.0;
  std::unique_ptr<nds_ode, void (*)(nds_ode*)> ode_{nullptr, nds_ode_destroy};
};

inline SolveResult propagate(const OdeSystem& system, double t, const SolveOptions& options = {}) {
  return OdePropagator(system, options).at(t);
}

inline NDTensor rk4_reference(const OdeSystem& system, double t, double dt, std::int64_t max_steps = 50'000'000) {
  const int n = system.forcing.order();
  validate_coefficients(system.coefficients, system.forcing.dims, "system");
  if (system.initial.dims != system.forcing.dims) throw std::invalid_argument("initial state shape mismatch");
  std::vector<const nds_z*> a;
  for (const Matrix& m : system.coefficients) a.push_back(reinterpret_cast<const nds_z*>(m.data()));
  NDTensor x = NDTensor::zeros(system.forcing.dims);
  rethrow(nds_rk4(context(), n, system.forcing.dims.data(), a.data(),
                  reinterpret_cast<const nds_z*>(system.forcing.data.data()),
                  reinterpret_cast<const nds_z*>(system.initial.data.data()), t, dt, max_steps,
                  reinterpret_cast<nds_z*>(x.data.data())),
          nds_singular{});
  return x;
}
}  // namespace ndsylv::gpu
