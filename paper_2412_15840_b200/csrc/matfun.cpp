// exp(t T) of an upper-triangular T on the host — setup of the closed-form ODE propagator
// (reference ode.cpp:59-87 calls its triangular_exp per mode), timed with the call.
//
// Two routes, both exploiting that T (and so exp(tT) and every power of tT) is upper triangular:
//
// * Parlett recurrence (Golub & Van Loan, Matrix Computations, 4th ed., Alg. 9.1.1) when the
//   diagonal is well separated (exp_diagonal_separated): F_jj = exp(S_jj) and, column by
//   column, bottom to top,
//     F_ij = [ S_ij (F_jj - F_ii) + sum_{i<k<j} (S_ik F_kj - F_ik S_kj) ] / (S_jj - S_ii),  S = tT.
//   The device kernel (matfun.cu) evaluates the same recurrence superdiagonal by superdiagonal.
// * Otherwise scaling and squaring with a truncated Taylor series (Moler & Van Loan, "Nineteen
//   dubious ways", method 3) and Higham's exact re-computation of the diagonal and first
//   superdiagonal after every squaring (Higham, SIAM J. Matrix Anal. Appl. 31 (2009), sec. 3):
//   A = S / 2^s with ||A||_1 <= 1/4, exp(A) by a degree-14 Horner scheme (truncation error
//   below 1e-19 relative), then s squarings; no linear solve is needed.
#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

#include "error.h"
#include "ndsylv_b200.h"
#include "schur.h"

namespace nds {

using cxd = std::complex<double>;

namespace {

struct Tri {  // upper-triangular n x n, column-major, strict lower part kept at zero
  int n;
  std::vector<cxd> a;
  explicit Tri(int n_) : n(n_), a((size_t)n_ * n_) {}
  cxd& operator()(int i, int j) { return a[(size_t)i + (size_t)j * n]; }
  cxd operator()(int i, int j) const { return a[(size_t)i + (size_t)j * n]; }
};

// r = x y for upper-triangular x, y: r_ij = sum_{i<=k<=j} x_ik y_kj
Tri tri_mul(const Tri& x, const Tri& y) {
  const int n = x.n;
  Tri r(n);
#pragma omp parallel for schedule(dynamic, 8) if (n >= 96)
  for (int j = 0; j < n; ++j)
    for (int k = 0; k <= j; ++k) {
      const cxd ykj = y(k, j);
      if (ykj == cxd{}) continue;
      for (int i = 0; i <= k; ++i) r(i, j) += x(i, k) * ykj;
    }
  return r;
}

double norm1(const Tri& m) {
  double best = 0.0;
  for (int j = 0; j < m.n; ++j) {
    double s = 0.0;
    for (int i = 0; i <= j; ++i) s += std::abs(m(i, j));
    best = std::max(best, s);
  }
  return best;
}

// (e^b - e^a) / (b - a) without cancellation: e^{(a+b)/2} sinh(d) / d, d = (b - a) / 2
cxd exp_divided_difference(cxd a, cxd b) {
  const cxd d = 0.5 * (b - a);
  cxd shc;  // sinh(d) / d
  if (std::abs(d) < 1e-3) {
    const cxd d2 = d * d;
    shc = 1.0 + d2 / 6.0 * (1.0 + d2 / 20.0 * (1.0 + d2 / 42.0));
  } else {
    shc = std::sinh(d) / d;
  }
  return std::exp(0.5 * (a + b)) * shc;
}

// diagonal and first superdiagonal of exp(A) for upper-triangular A, computed exactly
void set_exact_band(Tri& f, const Tri& a) {
  for (int i = 0; i < a.n; ++i) f(i, i) = std::exp(a(i, i));
  for (int i = 0; i + 1 < a.n; ++i) f(i, i + 1) = a(i, i + 1) * exp_divided_difference(a(i, i), a(i + 1, i + 1));
}

Tri exp_scaling_squaring(const Tri& s_mat) {
  const int n = s_mat.n;
  const double nrm = norm1(s_mat);
  int sq = 0;
  if (nrm > 0.25) sq = (int)std::ceil(std::log2(nrm / 0.25));
  const double scale = std::ldexp(1.0, -sq);
  Tri a(n);
  for (size_t i = 0; i < a.a.size(); ++i) a.a[i] = s_mat.a[i] * scale;
  // Horner: exp(A) ~ I + A (I + A/2 (I + A/3 (... (I + A/14))))
  constexpr int kDegree = 14;
  Tri p(n);
  for (int i = 0; i < n; ++i) p(i, i) = 1.0;
  for (int k = kDegree; k >= 1; --k) {
    Tri q = tri_mul(a, p);
    const double inv = 1.0 / k;
    for (size_t i = 0; i < q.a.size(); ++i) q.a[i] *= inv;
    for (int i = 0; i < n; ++i) q(i, i) += 1.0;
    p = std::move(q);
  }
  set_exact_band(p, a);
  for (int r = 1; r <= sq; ++r) {
    p = tri_mul(p, p);
    const double sc = std::ldexp(1.0, r - sq);  // p now approximates exp(S 2^{r - sq})
    Tri ar(n);
    for (int i = 0; i < n; ++i) {
      ar(i, i) = s_mat(i, i) * sc;
      if (i + 1 < n) ar(i, i + 1) = s_mat(i, i + 1) * sc;
    }
    set_exact_band(p, ar);
  }
  return p;
}

Tri exp_parlett(const Tri& s) {
  const int n = s.n;
  Tri f(n);
  for (int j = 0; j < n; ++j) {
    f(j, j) = std::exp(s(j, j));
    for (int i = j - 1; i >= 0; --i) {
      cxd acc = s(i, j) * (f(j, j) - f(i, i));
      for (int k = i + 1; k < j; ++k) acc += s(i, k) * f(k, j) - f(i, k) * s(k, j);
      f(i, j) = acc / (s(j, j) - s(i, i));
    }
  }
  return f;
}

}  // namespace

bool exp_diagonal_separated(int n, const nds_z* t) {
  double dmax = 0.0;
  for (int i = 0; i < n; ++i) dmax = std::max(dmax, std::hypot(t[(size_t)i * (n + 1)].re, t[(size_t)i * (n + 1)].im));
  // Parlett divides by T_jj - T_ii: require every gap to exceed 1e-8 of the diagonal's scale
  const double gap = 1e-8 * std::max(1.0, dmax);
  for (int i = 0; i < n; ++i)
    for (int k = i + 1; k < n; ++k) {
      const nds_z a = t[(size_t)i * (n + 1)], b = t[(size_t)k * (n + 1)];
      if (std::hypot(a.re - b.re, a.im - b.im) < gap) return false;
    }
  return true;
}

void triangular_exp_host(int n, const nds_z* t_in, double t, nds_z* f_out) {
  Tri s(n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const nds_z z = t_in[(size_t)i + (size_t)j * n];
      if (i > j) {
        if (z.re != 0.0 || z.im != 0.0) throw Error(NDS_ERR_INVALID, "triangular_exp requires an upper triangular matrix");
        continue;
      }
      s(i, j) = cxd(z.re, z.im) * t;
    }
  Tri f(n);
  if (t == 0.0) {
    for (int i = 0; i < n; ++i) f(i, i) = 1.0;
  } else if (exp_diagonal_separated(n, t_in)) {
    f = exp_parlett(s);
  } else {
    f = exp_scaling_squaring(s);
  }
  for (size_t i = 0; i < f.a.size(); ++i) f_out[i] = nds_z{f.a[i].real(), f.a[i].imag()};
}

}  // namespace nds
