// ndsylv_gpu — the reference batch front end's solve | ode | bench | selftest subcommands
// (reference tools/ndsylv_main.cpp) on the B200 path, over the C ABI only (include/ndsylv_b200.h).
// Same options, the same output lines and the same bench CSV schema
// ("# ndsylv bench csv 1" / N,total_size,schur_s,transform_s,backsub_s,inverse_s,total_s,max_error),
// the same exit codes: 0 success, 2 singular operator, 3 file I/O or format error, 4 memory
// budget exceeded, 1 anything else. Instances drawn with --random come from the reference's own
// generator (nds_random_problem / nds_random_ode_system: same xoshiro256++ stream), tensors are
// NDT1 files (nds_read_tensor / nds_write_tensor). Own argument parser (the reference's CLI11 is
// not vendored). Build: __graft_entry__.build() -> tools/cli/ndsylv_gpu.
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ndsylv_b200.h"

namespace {

using cxd = std::complex<double>;
using Clock = std::chrono::steady_clock;
double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

struct Failure : std::runtime_error {  // carries the exit code
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

nds_ctx* g_ctx = nullptr;

int exit_code_of(int status) {  // ndsylv_main.cpp:366-381
  switch (status) {
    case NDS_ERR_SINGULAR: return 2;
    case NDS_ERR_FILE: return 3;
    case NDS_ERR_NOMEM: return 4;
    default: return 1;
  }
}

void check(int status) {
  if (status != NDS_OK) throw Failure(exit_code_of(status), nds_last_error(g_ctx));
}
void check_file(int status) {  // context-free calls keep their message per thread
  if (status != NDS_OK) throw Failure(exit_code_of(status), nds_last_error(nullptr));
}

struct Tensor {
  std::vector<int64_t> dims;
  std::vector<nds_z> data;
  int64_t size() const { return (int64_t)data.size(); }
};

int64_t total_of(const std::vector<int64_t>& d) {
  int64_t t = 1;
  for (int64_t n : d) t *= n;
  return t;
}

Tensor read_file(const std::string& path) {
  int n = 0;
  int64_t dims[NDS_MAX_MODES];
  check_file(nds_tensor_file_info(path.c_str(), &n, dims));
  Tensor t{std::vector<int64_t>(dims, dims + n), {}};
  t.data.resize((size_t)total_of(t.dims));
  check_file(nds_read_tensor(path.c_str(), n, dims, t.data.data()));
  return t;
}

void write_file(const std::string& path, const Tensor& t) {
  check_file(nds_write_tensor(path.c_str(), (int)t.dims.size(), t.dims.data(), t.data.data()));
}

std::string dims_string(const std::vector<int64_t>& d) {
  std::string s;
  for (size_t j = 0; j < d.size(); ++j) s += (j ? "," : "") + std::to_string(d[j]);
  return s;
}

double max_abs_diff(const std::vector<nds_z>& a, const std::vector<nds_z>& b) {
  double m = 0.0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(cxd(a[i].re - b[i].re, a[i].im - b[i].im)));
  return m;
}

// ndsylv_main.cpp:61-74
void check_budget(const std::vector<int64_t>& dims, int live, uint64_t max_bytes) {
  uint64_t need = 16ull * (uint64_t)live;
  for (int64_t n : dims) {
    if (n <= 0) throw Failure(1, "extents must be positive");
    if (__builtin_mul_overflow(need, (uint64_t)n, &need)) throw Failure(4, "projected allocation overflows the address space");
  }
  if (need > max_bytes)
    throw Failure(4, "projected " + std::to_string(need) + " bytes for " + std::to_string(live) +
                         " buffers of shape (" + dims_string(dims) + ") exceeds the budget of " +
                         std::to_string(max_bytes) + " bytes");
}

struct Args {
  std::vector<int64_t> dims;
  uint64_t seed = 1;
  bool random = false;
  std::vector<std::string> coeffs;
  std::string rhs, x0, out, csv, n_range = "2:16";
  double tol = 0.0, t = 0.0, dt = 2.5e-5;
  bool have_t = false;
  uint64_t max_mem = 8589934592ULL;
};

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> v;
  size_t a = 0;
  for (;;) {
    const size_t b = s.find(',', a);
    v.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
    if (b == std::string::npos) break;
    a = b + 1;
  }
  return v;
}

Args parse(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw Failure(1, k + " needs a value");
      return argv[++i];
    };
    if (k == "--random") a.random = true;
    else if (k == "--dims") for (auto& x : split(val())) a.dims.push_back(std::stoll(x));
    else if (k == "--seed") a.seed = std::stoull(val());
    else if (k == "--coeffs") for (auto& x : split(val())) a.coeffs.push_back(x);
    else if (k == "--rhs") a.rhs = val();
    else if (k == "--x0") a.x0 = val();
    else if (k == "--out") a.out = val();
    else if (k == "--tol") a.tol = std::stod(val());
    else if (k == "--max-mem") a.max_mem = std::stoull(val());
    else if (k == "--t") { a.t = std::stod(val()); a.have_t = true; }
    else if (k == "--dt") a.dt = std::stod(val());
    else if (k == "--n-range") a.n_range = val();
    else if (k == "--csv") a.csv = val();
    else throw Failure(1, "unknown option " + k);
  }
  return a;
}

std::vector<const nds_z*> cptrs(const std::vector<std::vector<nds_z>>& m) {
  std::vector<const nds_z*> p;
  for (auto& x : m) p.push_back(x.data());
  return p;
}

std::vector<std::vector<nds_z>> read_coeffs(const std::vector<std::string>& paths) {
  std::vector<std::vector<nds_z>> m;
  for (auto& p : paths) {
    Tensor t = read_file(p);
    if (t.dims.size() != 2)
      throw Failure(3, "'" + p + "': expected an order-2 tensor, got order " + std::to_string(t.dims.size()));
    m.push_back(std::move(t.data));
  }
  return m;
}

void print_report(const nds_report& r) {  // ndsylv_main.cpp:76-83
  std::printf("min |denominator|: %.6e%s\n", r.min_abs_denominator, r.used_normal_fast_path ? "  (diagonal fast path)" : "");
  std::printf("flops: transform+backsub %lld, schur bound %lld\n", (long long)r.flop_estimate,
              (long long)r.schur_flop_estimate);
  std::printf("timings: schur %.6f s, transform %.6f s, backsub %.6f s, inverse %.6f s, total %.6f s\n",
              r.schur_seconds, r.transform_seconds, r.backsub_seconds, r.inverse_seconds, r.total_seconds);
}

struct Problem {
  std::vector<std::vector<nds_z>> a;
  Tensor rhs, x_true;
};

Problem random_problem(const std::vector<int64_t>& dims, uint64_t seed) {
  Problem p;
  for (int64_t n : dims) p.a.emplace_back((size_t)(n * n));
  p.rhs.dims = p.x_true.dims = dims;
  p.rhs.data.resize((size_t)total_of(dims));
  p.x_true.data.resize(p.rhs.data.size());
  std::vector<nds_z*> ap;
  for (auto& m : p.a) ap.push_back(m.data());
  check(nds_random_problem(g_ctx, (int)dims.size(), dims.data(), seed, ap.data(), p.x_true.data.data(),
                           p.rhs.data.data()));
  return p;
}

int run_solve(const Args& a) {  // ndsylv_main.cpp:85-124
  Problem p;
  bool truth = false;
  if (a.random) {
    if (a.dims.empty()) throw Failure(1, "--random needs --dims");
    check_budget(a.dims, 3, a.max_mem);
    p = random_problem(a.dims, a.seed);
    truth = true;
  } else {
    if (a.coeffs.empty() || a.rhs.empty()) throw Failure(1, "need --coeffs and --rhs, or --random");
    p.a = read_coeffs(a.coeffs);
    p.rhs = read_file(a.rhs);
    check_budget(p.rhs.dims, 3, a.max_mem);
  }
  const int N = (int)p.rhs.dims.size();
  Tensor x{p.rhs.dims, std::vector<nds_z>(p.rhs.data.size())};
  nds_report rep{};
  nds_singular sing{};
  auto ap = cptrs(p.a);
  check(nds_solve(g_ctx, N, p.rhs.dims.data(), ap.data(), p.rhs.data.data(), x.data.data(), a.tol,
                  NDS_ALLOW_FAST_PATH, &rep, &sing));
  std::printf("dims: %s  (total %lld)\n", dims_string(p.rhs.dims).c_str(), (long long)p.rhs.size());
  if (truth) std::printf("max error vs known solution: %.3e\n", max_abs_diff(x.data, p.x_true.data));
  std::vector<nds_z> rec(x.data.size());
  check(nds_apply_operator(g_ctx, N, p.rhs.dims.data(), ap.data(), x.data.data(), rec.data()));
  std::printf("residual: %.3e\n", max_abs_diff(rec, p.rhs.data));
  print_report(rep);
  if (!a.out.empty()) {
    write_file(a.out, x);
    std::printf("wrote %s\n", a.out.c_str());
  }
  return 0;
}

int run_ode(const Args& a) {  // ndsylv_main.cpp:126-159
  if (!a.have_t) throw Failure(1, "--t is required");
  std::vector<std::vector<nds_z>> coef;
  Tensor forcing, initial;
  if (a.random) {
    if (a.dims.empty()) throw Failure(1, "--random needs --dims");
    check_budget(a.dims, 3, a.max_mem);
    for (int64_t n : a.dims) coef.emplace_back((size_t)(n * n));
    forcing.dims = initial.dims = a.dims;
    forcing.data.resize((size_t)total_of(a.dims));
    initial.data.resize(forcing.data.size());
    std::vector<nds_z*> ap;
    for (auto& m : coef) ap.push_back(m.data());
    check_file(nds_random_ode_system((int)a.dims.size(), a.dims.data(), a.seed, ap.data(), forcing.data.data(),
                                     initial.data.data()));
  } else {
    if (a.coeffs.empty() || a.rhs.empty() || a.x0.empty()) throw Failure(1, "need --coeffs, --rhs and --x0, or --random");
    coef = read_coeffs(a.coeffs);
    forcing = read_file(a.rhs);
    initial = read_file(a.x0);
    check_budget(initial.dims, 3, a.max_mem);
  }
  const int N = (int)initial.dims.size();
  auto ap = cptrs(coef);
  Tensor closed{initial.dims, std::vector<nds_z>(initial.data.size())};
  std::vector<nds_z> rk(initial.data.size());
  nds_report rep{};
  nds_singular sing{};
  auto t0 = Clock::now();
  check(nds_propagate(g_ctx, N, initial.dims.data(), ap.data(), forcing.data.data(), initial.data.data(), a.t, a.tol,
                      0, closed.data.data(), &rep, &sing));
  const double closed_s = seconds_since(t0);
  t0 = Clock::now();
  check(nds_rk4(g_ctx, N, initial.dims.data(), ap.data(), forcing.data.data(), initial.data.data(), a.t, a.dt,
                50000000, rk.data()));
  const double rk_s = seconds_since(t0);
  std::printf("dims: %s  t=%g  dt=%g\n", dims_string(initial.dims).c_str(), a.t, a.dt);
  std::printf("closed form: %.6f s\n", closed_s);
  std::printf("rk4: %.6f s  (%lld steps)\n", rk_s, (long long)std::ceil(std::abs(a.t) / a.dt));
  std::printf("max discrepancy: %.3e\n", max_abs_diff(closed.data, rk));
  if (!a.out.empty()) {
    write_file(a.out, closed);
    std::printf("wrote %s\n", a.out.c_str());
  }
  return 0;
}

int run_bench(const Args& a) {  // ndsylv_main.cpp:208-236: Fig. 1 sweep, all n_j = 2
  const std::string& r = a.n_range;
  size_t c = r.find(':'), len = 1;
  if (c == std::string::npos) {
    c = r.find("..");
    len = 2;
  }
  const int lo = std::stoi(c == std::string::npos ? r : r.substr(0, c));
  const int hi = std::stoi(c == std::string::npos ? r : r.substr(c + len));
  if (lo < 1 || hi < lo) throw Failure(1, "--n-range wants LO:HI with 1 <= LO <= HI");
  std::FILE* out = stdout;
  if (!a.csv.empty() && !(out = std::fopen(a.csv.c_str(), "w"))) throw Failure(3, "cannot open '" + a.csv + "' for writing");
  std::fprintf(out, "# ndsylv bench csv 1\n");
  std::fprintf(out, "N,total_size,schur_s,transform_s,backsub_s,inverse_s,total_s,max_error\n");
  for (int n = lo; n <= hi; ++n) {
    const std::vector<int64_t> dims((size_t)n, 2);
    check_budget(dims, 3, a.max_mem);
    Problem p = random_problem(dims, a.seed + (uint64_t)n);
    Tensor x{dims, std::vector<nds_z>(p.rhs.data.size())};
    nds_report rep{};
    nds_singular sing{};
    auto ap = cptrs(p.a);
    check(nds_solve(g_ctx, n, dims.data(), ap.data(), p.rhs.data.data(), x.data.data(), 0.0, NDS_ALLOW_FAST_PATH,
                    &rep, &sing));
    std::fprintf(out, "%d,%lld,%.6e,%.6e,%.6e,%.6e,%.6e,%.3e\n", n, (long long)p.rhs.size(), rep.schur_seconds,
                 rep.transform_seconds, rep.backsub_seconds, rep.inverse_seconds, rep.total_seconds,
                 max_abs_diff(x.data, p.x_true.data));
  }
  if (out != stdout && std::fclose(out) != 0) throw Failure(3, "writing benchmark output failed");
  return 0;
}

int run_selftest() {  // the solve / Schur / ODE parts of ndsylv_main.cpp:238-300
  int failures = 0;
  auto report = [&](const char* name, bool ok, double value, double bound) {
    std::printf("%-28s %s  (%.3e, bound %.1e)\n", name, ok ? "ok" : "FAIL", value, bound);
    if (!ok) ++failures;
  };
  {
    const std::vector<std::vector<int64_t>> shapes = {{2, 3, 4}, {3, 3, 3}, {2, 2, 2, 2}, {5, 4}, {4, 4, 3}};
    double worst = 0.0;
    for (size_t k = 0; k < shapes.size(); ++k) {
      Problem p = random_problem(shapes[k], 201 + k);
      std::vector<nds_z> x(p.rhs.data.size());
      nds_report rep{};
      nds_singular sing{};
      auto ap = cptrs(p.a);
      check(nds_solve(g_ctx, (int)shapes[k].size(), shapes[k].data(), ap.data(), p.rhs.data.data(), x.data(), 0.0,
                      NDS_ALLOW_FAST_PATH, &rep, &sing));
      worst = std::max(worst, max_abs_diff(x, p.x_true.data));
    }
    report("solve vs known solution", worst <= 1e-9, worst, 1e-9);
  }
  {
    std::vector<std::vector<nds_z>> coef;
    const std::vector<int64_t> dims = {2, 3};
    for (int64_t n : dims) coef.emplace_back((size_t)(n * n));
    std::vector<nds_z> f(6), x0(6), closed(6), rk(6);
    std::vector<nds_z*> ap;
    for (auto& m : coef) ap.push_back(m.data());
    check_file(nds_random_ode_system(2, dims.data(), 401, ap.data(), f.data(), x0.data()));
    auto cp = cptrs(coef);
    nds_report rep{};
    nds_singular sing{};
    check(nds_propagate(g_ctx, 2, dims.data(), cp.data(), f.data(), x0.data(), 0.2, 0.0, 0, closed.data(), &rep, &sing));
    check(nds_rk4(g_ctx, 2, dims.data(), cp.data(), f.data(), x0.data(), 0.2, 1e-3, 50000000, rk.data()));
    const double diff = max_abs_diff(closed, rk);
    report("closed form vs rk4", diff <= 1e-8, diff, 1e-8);
  }
  std::printf("selftest: %s\n", failures == 0 ? "all ok" : "FAILURES");
  return failures == 0 ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ndsylv_gpu {solve|ode|bench|selftest} [options]\n");
    return 1;
  }
  const std::string cmd = argv[1];
  try {
    const Args a = parse(argc, argv, 2);
    check(nds_ctx_create(&g_ctx, 0));
    int rc = 1;
    if (cmd == "solve") rc = run_solve(a);
    else if (cmd == "ode") rc = run_ode(a);
    else if (cmd == "bench") rc = run_bench(a);
    else if (cmd == "selftest") rc = run_selftest();
    else throw Failure(1, "unknown subcommand " + cmd);
    nds_ctx_destroy(g_ctx);
    return rc;
  } catch (const Failure& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return e.code;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
