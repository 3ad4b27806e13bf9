// Drop-in check: the reference's own problem generator and CPU solver against
// ndsylv::gpu::solve (include/ndsylv_b200_adapter.hpp) on the same SylvesterProblem.
// Built by __graft_entry__.build() where the reference headers exist; run by
// tests/test_integration.py on a GPU box. Prints "max_rel_diff <x> singular_ok <0|1>".
#include <cstdio>

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
  std::printf("max_rel_diff %.3e singular_ok %d\n", worst, singular_ok);
  return worst <= 1e-9 && singular_ok ? 0 : 1;
}
