// Host complex Schur factorisation A = U T U^H — setup of the solve, timed separately
// (BASELINE.json north_star: "the Schur factorisations stay host setup").
//
// Contract of the reference's ndsylv::schur (schur.hpp:7-19): unitary U, upper-triangular T with
// an exactly-zero strict lower triangle, NDS_ERR_INVALID for empty / non-finite input,
// NDS_ERR_CONVERGENCE when the iteration budget runs out. X = U-transformed solve is unique, so
// parity with the reference is on X, not on these factors.
//
// Algorithm: the LAPACK pair ZGEHD2 + ZLAHQR (Anderson et al., LAPACK Users' Guide, 3rd ed.;
// deflation test of Ahues & Tisseur, LAPACK Working Note 122), restated here in column-major
// storage with generic complex 2-element reflectors:
//   1. Householder reduction to upper Hessenberg form, reflectors from ZLARFG;
//   2. single-shift implicit QR on the active window [l, i]: Ahues-Tisseur deflation test,
//      Wilkinson-type shift from the trailing 2x2 (ZLAHQR's formulation), exceptional shifts
//      after 10 / 20 iterations without deflation, the bulge started at the lowest of two
//      consecutive small subdiagonals, chased with 2x2 reflectors applied to the full rows /
//      columns (so T is the complete Schur form) and accumulated into U;
//   3. a budget of 30 max(10, n) iterations per eigenvalue.
#include <algorithm>
#include <cmath>
#include <complex>
#include <limits>
#include <vector>

#include "ndsylv_b200.h"
#include "schur.h"

namespace nds {

namespace {

using cx = std::complex<double>;

inline double cabs1(cx z) { return std::fabs(z.real()) + std::fabs(z.imag()); }

struct ColMajor {
  int n;
  std::vector<cx> v;
  explicit ColMajor(int n_) : n(n_), v((size_t)n_ * n_) {}
  cx& operator()(int r, int c) { return v[(size_t)r + (size_t)c * n]; }
  cx operator()(int r, int c) const { return v[(size_t)r + (size_t)c * n]; }
  cx* col(int c) { return &v[(size_t)c * n]; }
};

// ZLARFG: reflector H = I - tau v v^H, v = (1, x'), with H^H (alpha; x) = (beta; 0), beta real.
// On return alpha = beta and x holds v(2:).
cx make_reflector(cx& alpha, cx* x, int len) {
  double xnorm = 0.0;
  for (int i = 0; i < len; ++i) xnorm = std::hypot(xnorm, std::abs(x[i]));
  const double ar = alpha.real(), ai = alpha.imag();
  if (xnorm == 0.0 && ai == 0.0) return cx(0.0);
  const double beta = -std::copysign(std::hypot(std::hypot(ar, ai), xnorm), ar);
  const cx tau((beta - ar) / beta, -ai / beta);
  const cx scale = 1.0 / (alpha - beta);
  for (int i = 0; i < len; ++i) x[i] *= scale;
  alpha = beta;
  return tau;
}

// ZGEHD2: A <- Q^H A Q upper Hessenberg, Z <- Z Q.
void hessenberg(ColMajor& a, ColMajor& z) {
  const int n = a.n;
  std::vector<cx> v(n), w(n);
  for (int k = 0; k + 2 < n; ++k) {
    const int len = n - k - 1;  // rows k+1 .. n-1 of column k
    cx* colk = a.col(k);
    cx alpha = colk[k + 1];
    const cx tau = make_reflector(alpha, colk + k + 2, len - 1);
    v[0] = 1.0;
    for (int i = 1; i < len; ++i) v[i] = colk[k + 1 + i];
    colk[k + 1] = alpha;
    for (int i = k + 2; i < n; ++i) colk[i] = 0.0;
    if (tau == cx(0.0)) continue;
    // right: A(:, k+1:) <- A(:, k+1:) (I - tau v v^H), all rows; Z likewise
    for (ColMajor* m : {&a, &z}) {
      std::fill(w.begin(), w.end(), cx(0.0));
      for (int i = 0; i < len; ++i) {
        const cx* c = m->col(k + 1 + i);
        for (int r = 0; r < n; ++r) w[r] += c[r] * v[i];
      }
      for (int i = 0; i < len; ++i) {
        cx* c = m->col(k + 1 + i);
        const cx f = tau * std::conj(v[i]);
        for (int r = 0; r < n; ++r) c[r] -= w[r] * f;
      }
    }
    // left: A(k+1:, k+1:) <- (I - conj(tau) v v^H) A(k+1:, k+1:)
    for (int c = k + 1; c < n; ++c) {
      cx* cc = a.col(c) + k + 1;
      cx s = 0.0;
      for (int i = 0; i < len; ++i) s += std::conj(v[i]) * cc[i];
      s *= std::conj(tau);
      for (int i = 0; i < len; ++i) cc[i] -= s * v[i];
    }
  }
}

// ZLAHQR on the whole matrix (ilo = 0, ihi = n - 1, wantt = wantz = true).
void hessenberg_qr(ColMajor& h, ColMajor& z) {
  const int n = h.n;
  const double ulp = std::numeric_limits<double>::epsilon();
  const double safmin = std::numeric_limits<double>::min();
  const double smlnum = safmin * ((double)n / ulp);
  const int itmax = 30 * std::max(10, n);
  int kdefl = 0;  // iterations since the last deflation
  for (int i = n - 1; i >= 0;) {
    int l = 0;
    bool converged = false;
    for (int its = 0; its <= itmax; ++its) {
      // small subdiagonal (Ahues-Tisseur)
      int k = i;
      for (; k > l; --k) {
        if (cabs1(h(k, k - 1)) <= smlnum) break;
        double tst = cabs1(h(k - 1, k - 1)) + cabs1(h(k, k));
        if (tst == 0.0) {
          if (k - 2 >= 0) tst += std::fabs(h(k - 1, k - 2).real());
          if (k + 1 <= n - 1) tst += std::fabs(h(k + 1, k).real());
        }
        if (cabs1(h(k, k - 1)) <= ulp * tst) {
          const double ab = std::max(cabs1(h(k, k - 1)), cabs1(h(k - 1, k)));
          const double ba = std::min(cabs1(h(k, k - 1)), cabs1(h(k - 1, k)));
          const double aa = std::max(cabs1(h(k, k)), cabs1(h(k - 1, k - 1) - h(k, k)));
          const double bb = std::min(cabs1(h(k, k)), cabs1(h(k - 1, k - 1) - h(k, k)));
          const double s = aa + ab;
          if (ba * (ab / s) <= std::max(smlnum, ulp * (bb * (aa / s)))) break;
        }
      }
      l = k;
      if (l > 0) h(l, l - 1) = 0.0;
      if (l >= i) {
        converged = true;
        break;
      }
      ++kdefl;
      // shift
      cx t;
      if (kdefl % 20 == 0) {
        t = 0.75 * cabs1(h(i, i - 1)) + h(i, i);
      } else if (kdefl % 10 == 0) {
        t = 0.75 * cabs1(h(l + 1, l)) + h(l, l);
      } else {
        t = h(i, i);
        const cx u = std::sqrt(h(i - 1, i)) * std::sqrt(h(i, i - 1));
        double s = cabs1(u);
        if (s != 0.0) {
          const cx x = 0.5 * (h(i - 1, i - 1) - t);
          const double sx = cabs1(x);
          s = std::max(s, sx);
          cx y = s * std::sqrt((x / s) * (x / s) + (u / s) * (u / s));
          if (sx > 0.0 && (x / sx).real() * y.real() + (x / sx).imag() * y.imag() < 0.0) y = -y;
          t -= u * (u / (x + y));
        }
      }
      // start of the bulge: two consecutive small subdiagonals, else l
      int m = i - 1;
      cx v0, v1;
      for (;; --m) {
        const cx h11 = h(m, m), h22 = h(m + 1, m + 1);
        cx h11s = h11 - t;
        cx h21 = h(m + 1, m);
        const double s = cabs1(h11s) + cabs1(h21);
        h11s /= s;
        h21 /= s;
        v0 = h11s;
        v1 = h21;
        if (m == l) break;
        const double h10 = cabs1(h(m, m - 1));
        if (h10 * cabs1(h21) <= ulp * (cabs1(h11s) * (cabs1(h11) + cabs1(h22)))) break;
      }
      // chase: reflectors on rows / columns (k, k+1), k = m .. i-1
      for (int k2 = m; k2 < i; ++k2) {
        if (k2 > m) {
          v0 = h(k2, k2 - 1);
          v1 = h(k2 + 1, k2 - 1);
        }
        const cx tau = make_reflector(v0, &v1, 1);
        if (k2 > m) {
          h(k2, k2 - 1) = v0;
          h(k2 + 1, k2 - 1) = 0.0;
        }
        if (tau == cx(0.0)) continue;
        const cx v2 = v1, tc = std::conj(tau), v2c = std::conj(v2);
        // left, rows k2, k2+1. A step started at m > l also rotates H(m, m-1) (by 1 - conj(tau));
        // the fill-in it creates at H(m+1, m-1) is below the two-small-subdiagonals threshold
        // and is dropped (ZLAHQR's argument).
        const int j0 = (k2 == m && m > l) ? m - 1 : k2;
        for (int j = j0; j < n; ++j) {
          const cx s = tc * (h(k2, j) + v2c * h(k2 + 1, j));
          h(k2, j) -= s;
          h(k2 + 1, j) -= s * v2;
        }
        if (j0 < k2) h(k2 + 1, k2 - 1) = 0.0;
        const int rmax = std::min(k2 + 2, i);
        for (int r = 0; r <= rmax; ++r) {  // right, columns k2, k2+1
          const cx s = tau * (h(r, k2) + h(r, k2 + 1) * v2);
          h(r, k2) -= s;
          h(r, k2 + 1) -= s * v2c;
        }
        cx* z0 = z.col(k2);
        cx* z1 = z.col(k2 + 1);
        for (int r = 0; r < n; ++r) {
          const cx s = tau * (z0[r] + z1[r] * v2);
          z0[r] -= s;
          z1[r] -= s * v2c;
        }
      }
    }
    if (!converged) throw Error(NDS_ERR_CONVERGENCE, "QR iteration did not deflate within the iteration budget");
    kdefl = 0;
    i = l - 1;
  }
}

}  // namespace

void schur_host(int n, const nds_z* a, nds_z* u_out, nds_z* t_out) {
  if (n <= 0) throw Error(NDS_ERR_INVALID, "schur requires a non-empty square matrix");
  for (size_t i = 0; i < (size_t)n * n; ++i)
    if (!std::isfinite(a[i].re) || !std::isfinite(a[i].im)) throw Error(NDS_ERR_INVALID, "schur requires finite entries");
  ColMajor h(n), z(n);
  for (size_t i = 0; i < (size_t)n * n; ++i) h.v[i] = cx(a[i].re, a[i].im);
  for (int i = 0; i < n; ++i) z(i, i) = 1.0;
  if (n > 1) {
    hessenberg(h, z);
    hessenberg_qr(h, z);
  }
  for (int c = 0; c < n; ++c)
    for (int r = 0; r < n; ++r) {
      const cx tv = r > c ? cx(0.0) : h(r, c);
      t_out[r + (size_t)c * n] = {tv.real(), tv.imag()};
      const cx uv = z(r, c);
      u_out[r + (size_t)c * n] = {uv.real(), uv.imag()};
    }
}

}  // namespace nds
