// Drop-in check: the reference's own problem generator and CPU solver against
// ndsylv::gpu::solve (include/ndsylv_b200_adapter.hpp) on the same SylvesterProblem.
// Built by __graft_entry__.build() where the reference headers exist; run by
// tests/test_integration.py on a GPU box. Prints "max_rel_diff <x> singular_ok <0|1>" and, for
// the ODE surface (ode.hpp: propagate, OdePropagator::at, rk4_reference), "ode_rel_diff <x>
// rk4_rel_diff <x> nonfinite_ok <0|1>".
#include <cstdio>

#include "ndsylv/ode.hpp"
#include "ndsylv/rng.hpp"
#include "ndsylv/sylvester.hpp"
#include "ndsylv_b200_adapter.hpp"

int main() {
  using namespace ndsylv;
  double worst = 0.0;
  for (auto [dims, seed] : std::vector<std::pair<std::vector<std::int64_t>, std::uint64_t>>{
           {{5, 4, 3}, 905}, {{2, 9, 33}, 42}, {{32, 32, 32}, 7}, {{2, 2, 2, 2, 2, 2}, 4206}}) {
    const GeneratedProblem g = random_problem(dims, seed);
    const SolveResult cpu = solve(g.problem);
    const SolveResult gpu = ndsylv::gpu::solve(g.problem);
    const double d = max_abs_diff(cpu.x, gpu.x) / max_abs(cpu.x);
    worst = std::max(worst, d);
    if (cpu.report.backsub_multiplies != gpu.report.backsub_multiplies) {
      std::printf("multiply count mismatch\n");
      return 1;
    }
  }
  int singular_ok = 0;
  try {
    SylvesterProblem p;
    p.coefficients = {Matrix::diagonal(std::vector<cxd>{1.0, -1.0}), Matrix::diagonal(std::vector<cxd>{-1.0, 1.0})};
    p.rhs = NDTensor::zeros({2, 2});
    ndsylv::gpu::solve(p);
  } catch (const SingularOperatorError& e) {
    singular_ok = e.multi_index() == std::vector<std::int64_t>{2, 2};
  }
  // validate_problem (sylvester.cpp:17-27): too few coefficients / wrong extent -> invalid_argument
  int shape_ok = 0;
  for (int variant = 0; variant < 2; ++variant) {
    SylvesterProblem p;
    p.rhs = NDTensor::zeros({3, 4});
    p.coefficients = {Matrix::identity(3)};
    if (variant == 1) p.coefficients.push_back(Matrix::identity(2));
    try {
      ndsylv::gpu::solve(p);
    } catch (const std::invalid_argument&) {
      ++shape_ok;
    }
  }
  singular_ok = singular_ok && shape_ok == 2;
  {  // the sharded entry on this process's device(s): one device here
    const GeneratedProblem g = random_problem({12, 10, 16}, 77);
    const SolveResult cpu = solve(g.problem);
    const SolveResult gpu = ndsylv::gpu::solve_multi(g.problem, {0});
    worst = std::max(worst, max_abs_diff(cpu.x, gpu.x) / max_abs(cpu.x));
  }
  {  // several right-hand sides through one plan: each against the reference's own solve
    const GeneratedProblem g = random_problem({32, 24, 16}, 501);
    std::vector<NDTensor> rhs;
    for (std::uint64_t s : {502u, 503u, 504u}) rhs.push_back(random_problem({32, 24, 16}, s).problem.rhs);
    const std::vector<NDTensor> xs = ndsylv::gpu::solve_many(g.problem.coefficients, rhs);
    for (size_t k = 0; k < rhs.size(); ++k) {
      SylvesterProblem p = g.problem;
      p.rhs = rhs[k];
      const SolveResult cpu = solve(p);
      worst = std::max(worst, max_abs_diff(cpu.x, xs[k]) / max_abs(cpu.x));
    }
  }
  std::printf("max_rel_diff %.3e singular_ok %d\n", worst, singular_ok);

  // ODE: the reference's own random systems (rng.hpp random_ode_system), CPU vs GPU
  double ode_worst = 0.0, rk_worst = 0.0;
  for (auto [dims, seed] : std::vector<std::pair<std::vector<std::int64_t>, std::uint64_t>>{
           {{3, 2, 2}, 40}, {{2, 3, 4}, 42}, {{16, 12, 8}, 43}}) {
    const OdeSystem sys = random_ode_system(dims, seed);
    const OdePropagator cpu(sys);
    const ndsylv::gpu::OdePropagator gpu(sys);
    for (double t : {0.0, 0.1, -0.05}) {
      const NDTensor a = cpu.at(t).x, b = gpu.at(t).x;
      ode_worst = std::max(ode_worst, max_abs_diff(a, b) / std::max(1e-300, max_abs(a)));
    }
    const NDTensor r1 = rk4_reference(sys, 0.02, 1e-3), r2 = ndsylv::gpu::rk4_reference(sys, 0.02, 1e-3);
    rk_worst = std::max(rk_worst, max_abs_diff(r1, r2) / max_abs(r1));
  }
  int nonfinite_ok = 0;
  try {
    OdeSystem sys;
    sys.coefficients = {cxd(400.0, 0.0) * Matrix::identity(2), cxd(400.0, 0.0) * Matrix::identity(2)};
    sys.forcing = NDTensor::zeros({2, 2});
    sys.initial = NDTensor::zeros({2, 2});
    for (cxd& v : sys.initial.data) v = 1e300;
    ndsylv::gpu::rk4_reference(sys, 10.0, 0.5);
  } catch (const NonFiniteStateError&) {
    nonfinite_ok = 1;
  }
  std::printf("ode_rel_diff %.3e rk4_rel_diff %.3e nonfinite_ok %d\n", ode_worst, rk_worst, nonfinite_ok);
  return worst <= 1e-9 && singular_ok && ode_worst <= 1e-9 && rk_worst <= 1e-9 && nonfinite_ok ? 0 : 1;
}
