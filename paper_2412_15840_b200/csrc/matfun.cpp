// Host matrix functions for the closed-form ODE propagator: exp(t T) of an upper triangular T.
//
// Restates the reference's triangular_exp (schur.cpp:203-228): the Parlett recurrence
//   F_ii = exp(t T_ii),  F_ij = [ S_ij (F_jj - F_ii) + sum_{i<k<j} (S_ik F_kj - F_ik S_kj) ] / (S_jj - S_ii)
// with S = t T, used when every pair of diagonal entries is separated by >= 1e-8 (1 + max|T_ii|)
// (schur.cpp:164-174); otherwise the [6/6] Pade approximant with scaling and squaring
// (schur.cpp:230-255) and a partial-pivoting LU solve (matrix.cpp:143-201), strict lower part
// zeroed. Arithmetic is std::complex<double> in the reference's operation order, so the
// compiled code uses the same libgcc complex multiply / divide and glibc cexp.
// The superdiagonal sweep is OpenMP-parallel over the entries of one superdiagonal (they are
// independent); this is host setup like the Schur factorisation, timed separately.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <stdexcept>
#include <string>
#include <vector>

#include "error.h"
#include "ndsylv_b200.h"

namespace nds {

using cxd = std::complex<double>;

namespace {

struct Mat {  // column-major n x n
  int n;
  std::vector<cxd> a;
  explicit Mat(int n_) : n(n_), a((size_t)n_ * n_) {}
  cxd& operator()(int i, int j) { return a[(size_t)i + (size_t)j * n]; }
  const cxd& operator()(int i, int j) const { return a[(size_t)i + (size_t)j * n]; }
  static Mat identity(int n) {
    Mat m(n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

// r = a b with the reference's loop order (matrix.cpp:48-58: j, k, skip zero b(k, j), i)
Mat mul(const Mat& a, const Mat& b) {
  const int n = a.n;
  Mat r(n);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const cxd bk = b(k, j);
      if (bk == cxd{}) continue;
      for (int i = 0; i < n; ++i) r(i, j) += a(i, k) * bk;
    }
  return r;
}

Mat scaled(cxd s, const Mat& m) {  // matrix.cpp:94-97, 127-133
  Mat r = m;
  for (auto& v : r.a) v *= s;
  return r;
}

void add_to(Mat& r, const Mat& m) {
  for (size_t i = 0; i < r.a.size(); ++i) r.a[i] += m.a[i];
}

double norm_inf(const Mat& m) {  // matrix.cpp:105-113
  double best = 0.0;
  for (int i = 0; i < m.n; ++i) {
    double s = 0.0;
    for (int j = 0; j < m.n; ++j) s += std::abs(m(i, j));
    best = std::max(best, s);
  }
  return best;
}

// LU with partial pivoting, rows exchanged in full (matrix.cpp:143-170), then column-by-column
// forward / back substitution (matrix.cpp:172-201).
Mat lu_solve(Mat lu, Mat rhs) {
  const int n = lu.n;
  const double tol = std::numeric_limits<double>::epsilon() * norm_inf(lu);
  std::vector<int> perm(n);
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = std::abs(lu(k, k));
    for (int i = k + 1; i < n; ++i) {
      const double cand = std::abs(lu(i, k));
      if (cand > best) {
        best = cand;
        piv = i;
      }
    }
    if (best <= tol) throw Error(NDS_ERR_OTHER, "pivot below threshold at column " + std::to_string(k));
    perm[k] = piv;
    if (piv != k)
      for (int j = 0; j < n; ++j) std::swap(lu(k, j), lu(piv, j));
    const cxd inv_piv = 1.0 / lu(k, k);
    for (int i = k + 1; i < n; ++i) {
      const cxd f = lu(i, k) * inv_piv;
      lu(i, k) = f;
      if (f == cxd{}) continue;
      for (int j = k + 1; j < n; ++j) lu(i, j) -= f * lu(k, j);
    }
  }
  std::vector<cxd> col(n);
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < n; ++i) col[i] = rhs(i, j);
    for (int k = 0; k < n; ++k)
      if (perm[k] != k) std::swap(col[k], col[perm[k]]);
    for (int k = 0; k < n; ++k)
      for (int i = k + 1; i < n; ++i) col[i] -= lu(i, k) * col[k];
    for (int i = n - 1; i >= 0; --i) {
      cxd s = col[i];
      for (int k = i + 1; k < n; ++k) s -= lu(i, k) * col[k];
      col[i] = s / lu(i, i);
    }
    for (int i = 0; i < n; ++i) rhs(i, j) = col[i];
  }
  return rhs;
}

// [6/6] Pade with scaling and squaring (schur.cpp:230-255).
Mat pade_exp(const Mat& a) {
  const int n = a.n;
  const double norm = norm_inf(a);
  int squarings = 0;
  Mat a1 = a;
  if (norm > 0.5) {
    squarings = (int)std::ceil(std::log2(norm)) + 1;
    for (auto& v : a1.a) v *= cxd(std::ldexp(1.0, -squarings), 0.0);
  }
  constexpr int q = 6;
  double coeff[q + 1];
  coeff[0] = 1.0;
  for (int k = 1; k <= q; ++k) coeff[k] = coeff[k - 1] * (double)(q - k + 1) / (k * (2.0 * q - k + 1));
  const Mat a2 = mul(a1, a1);
  Mat even = scaled(cxd(coeff[0], 0.0), Mat::identity(n));
  Mat odd_inner = scaled(cxd(coeff[1], 0.0), Mat::identity(n));
  Mat power = a2;
  for (int k = 2; k <= q; k += 2) {
    add_to(even, scaled(cxd(coeff[k], 0.0), power));
    if (k + 1 <= q) add_to(odd_inner, scaled(cxd(coeff[k + 1], 0.0), power));
    if (k + 2 <= q) power = mul(power, a2);
  }
  const Mat odd = mul(a1, odd_inner);
  Mat num = even, den = even;
  for (size_t i = 0; i < num.a.size(); ++i) {
    num.a[i] += odd.a[i];
    den.a[i] -= odd.a[i];
  }
  Mat f = lu_solve(den, num);
  for (int i = 0; i < squarings; ++i) f = mul(f, f);
  return f;
}

bool diagonal_well_separated(const Mat& t) {  // schur.cpp:164-174
  const int n = t.n;
  double dmax = 0.0;
  for (int i = 0; i < n; ++i) dmax = std::max(dmax, std::abs(t(i, i)));
  const double threshold = 1e-8 * (1.0 + dmax);
  for (int i = 0; i < n; ++i)
    for (int k = i + 1; k < n; ++k)
      if (std::abs(t(i, i) - t(k, k)) < threshold) return false;
  return true;
}

}  // namespace

void triangular_exp_host(int n, const nds_z* t_in, double t, nds_z* f_out) {
  Mat tm(n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const nds_z z = t_in[(size_t)i + (size_t)j * n];
      tm(i, j) = cxd(z.re, z.im);
      if (i > j && tm(i, j) != cxd{}) throw Error(NDS_ERR_INVALID, "triangular_exp requires an upper triangular matrix");
    }
  Mat f(n);
  if (t == 0.0) {
    f = Mat::identity(n);
  } else if (!diagonal_well_separated(tm)) {
    f = pade_exp(scaled(cxd(t, 0.0), tm));
    for (int j = 0; j < n; ++j)
      for (int i = j + 1; i < n; ++i) f(i, j) = cxd{};
  } else {
    const Mat s = scaled(cxd(t, 0.0), tm);
    for (int i = 0; i < n; ++i) f(i, i) = std::exp(s(i, i));
    for (int p = 1; p < n; ++p) {
      const int cnt = n - p;
#pragma omp parallel for schedule(static) if (cnt * p > 4096)
      for (int i = 0; i < cnt; ++i) {
        const int j = i + p;
        cxd num = s(i, j) * (f(j, j) - f(i, i));
        for (int k = i + 1; k < j; ++k) num += s(i, k) * f(k, j) - f(i, k) * s(k, j);
        f(i, j) = num / (s(j, j) - s(i, i));
      }
    }
  }
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const cxd v = f(i, j);
      f_out[(size_t)i + (size_t)j * n] = nds_z{v.real(), v.imag()};
    }
}

}  // namespace nds
