// Host complex Schur factorisation A = U T U^H (setup of the solve, timed separately).
//
// Same contract as the reference's ndsylv::schur (schur.hpp:7-19, schur.cpp:190-201): unitary U,
// upper-triangular T with an exactly-zero strict lower triangle, invalid_argument on empty /
// non-square / non-finite input, ConvergenceError when the sweep budget (30 per eigenvalue) runs
// out. The algorithm is the textbook one (Golub & Van Loan, 7.4-7.5): Householder reduction to
// Hessenberg form, then implicitly shifted single-shift QR with Wilkinson shifts and an
// exceptional shift every tenth sweep on a stalled eigenvalue. The transformations are applied to
// the full rows/columns so T is the complete Schur form, and accumulated into U.
// Working storage is row-major (row rotations touch contiguous memory).
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

struct Dense {
  int n;
  std::vector<cx> v;  // row-major
  explicit Dense(int n_) : n(n_), v((size_t)n_ * n_) {}
  cx& at(int r, int c) { return v[(size_t)r * n + c]; }
  cx at(int r, int c) const { return v[(size_t)r * n + c]; }
};

// Rotation G = [[c, s], [-conj(s), c]] with G [f; g] = [r; 0].
struct Rot {
  double c;
  cx s;
};

Rot make_rot(cx f, cx g) {
  const double af = std::abs(f), ag = std::abs(g);
  if (ag == 0.0) return {1.0, cx(0.0)};
  if (af == 0.0) return {0.0, std::conj(g) / ag};
  const double h = std::hypot(af, ag);
  return {af / h, (f / af) * std::conj(g) / h};
}

void householder_hessenberg(Dense& h, Dense& u) {
  const int n = h.n;
  std::vector<cx> v(n), w(n);
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;  // length of the reflected column part
    double s2 = 0.0;
    for (int i = 0; i < m; ++i) s2 += std::norm(h.at(k + 1 + i, k));
    if (s2 == 0.0) continue;
    const double alpha = std::sqrt(s2);
    const cx x0 = h.at(k + 1, k);
    const cx phase = std::abs(x0) > 0.0 ? x0 / std::abs(x0) : cx(1.0);
    for (int i = 0; i < m; ++i) v[i] = h.at(k + 1 + i, k);
    v[0] += phase * alpha;
    double vn2 = 0.0;
    for (int i = 0; i < m; ++i) vn2 += std::norm(v[i]);
    if (vn2 == 0.0) continue;
    const double tau = 2.0 / vn2;
    // H <- (I - tau v v^H) H   on rows k+1.., columns k..
    for (int c = k; c < n; ++c) w[c] = 0.0;
    for (int i = 0; i < m; ++i) {
      const cx cv = std::conj(v[i]);
      const cx* row = &h.v[(size_t)(k + 1 + i) * n];
      for (int c = k; c < n; ++c) w[c] += cv * row[c];
    }
    for (int i = 0; i < m; ++i) {
      const cx f = tau * v[i];
      cx* row = &h.v[(size_t)(k + 1 + i) * n];
      for (int c = k; c < n; ++c) row[c] -= f * w[c];
    }
    // H <- H (I - tau v v^H) on columns k+1.. ; U likewise
    for (Dense* mat : {&h, &u}) {
      for (int r = 0; r < n; ++r) {
        cx* row = &mat->v[(size_t)r * n + k + 1];
        cx dot = 0.0;
        for (int i = 0; i < m; ++i) dot += row[i] * v[i];
        dot *= tau;
        for (int i = 0; i < m; ++i) row[i] -= dot * std::conj(v[i]);
      }
    }
    h.at(k + 1, k) = -phase * alpha;
    for (int i = k + 2; i < n; ++i) h.at(i, k) = 0.0;
  }
}

// Eigenvalue of [[a, b], [c, d]] nearest d.
cx wilkinson(cx a, cx b, cx c, cx d) {
  const cx p = 0.5 * (a - d);
  const cx bc = b * c;
  if (bc == cx(0.0)) return d;
  cx disc = std::sqrt(p * p + bc);
  cx q = p + disc;
  const cx q2 = p - disc;
  if (std::abs(q2) > std::abs(q)) q = q2;
  if (q == cx(0.0)) return d;
  return d - bc / q;
}

void shifted_qr(Dense& h, Dense& u) {
  const int n = h.n;
  const double eps = std::numeric_limits<double>::epsilon();
  double hnorm = 0.0;
  for (const cx& z : h.v) hnorm += std::norm(z);
  hnorm = std::sqrt(hnorm);
  int hi = n - 1;
  int stall = 0;
  long sweeps = 0;
  const long budget = 30L * n + 10;
  while (hi > 0) {
    // Find the active window [lo, hi]: deflate negligible subdiagonals.
    int lo = hi;
    while (lo > 0) {
      double scale = std::abs(h.at(lo - 1, lo - 1)) + std::abs(h.at(lo, lo));
      if (scale == 0.0) scale = hnorm;
      if (std::abs(h.at(lo, lo - 1)) <= eps * scale) {
        h.at(lo, lo - 1) = 0.0;
        break;
      }
      --lo;
    }
    if (lo == hi) {
      --hi;
      stall = 0;
      continue;
    }
    if (stall >= 30 || sweeps >= budget) throw Error(NDS_ERR_CONVERGENCE, "QR iteration did not deflate within the sweep budget");
    ++stall;
    ++sweeps;
    cx mu;
    if (stall % 10 == 0) {
      double s = std::abs(h.at(hi, hi - 1));
      if (hi >= 2) s += std::abs(h.at(hi - 1, hi - 2));
      mu = h.at(hi, hi) + 0.75 * s;
    } else {
      mu = wilkinson(h.at(hi - 1, hi - 1), h.at(hi - 1, hi), h.at(hi, hi - 1), h.at(hi, hi));
    }
    // Bulge chase over [lo, hi].
    cx f = h.at(lo, lo) - mu, g = h.at(lo + 1, lo);
    for (int k = lo; k < hi; ++k) {
      const Rot q = make_rot(f, g);
      const cx sc = std::conj(q.s);
      // rows k, k+1 (left): G
      {
        cx* r0 = &h.v[(size_t)k * n];
        cx* r1 = &h.v[(size_t)(k + 1) * n];
        for (int c = (k > lo ? k - 1 : lo); c < n; ++c) {
          const cx x = r0[c], y = r1[c];
          r0[c] = q.c * x + q.s * y;
          r1[c] = q.c * y - sc * x;
        }
      }
      // columns k, k+1 (right): G^H, rows up to min(k + 2, hi)
      const int rmax = std::min(k + 2, hi);
      for (int r = 0; r <= rmax; ++r) {
        cx* row = &h.v[(size_t)r * n];
        const cx x = row[k], y = row[k + 1];
        row[k] = q.c * x + sc * y;
        row[k + 1] = q.c * y - q.s * x;
      }
      for (int r = 0; r < n; ++r) {
        cx* row = &u.v[(size_t)r * n];
        const cx x = row[k], y = row[k + 1];
        row[k] = q.c * x + sc * y;
        row[k + 1] = q.c * y - q.s * x;
      }
      if (k + 1 < hi) {
        f = h.at(k + 1, k);
        g = h.at(k + 2, k);
      }
    }
  }
}

}  // namespace

void schur_host(int n, const nds_z* a, nds_z* u_out, nds_z* t_out) {
  if (n <= 0) throw Error(NDS_ERR_INVALID, "schur requires a non-empty square matrix");
  for (size_t i = 0; i < (size_t)n * n; ++i)
    if (!std::isfinite(a[i].re) || !std::isfinite(a[i].im)) throw Error(NDS_ERR_INVALID, "schur requires finite entries");
  Dense h(n), u(n);
  for (int c = 0; c < n; ++c)
    for (int r = 0; r < n; ++r) h.at(r, c) = cx(a[r + (size_t)c * n].re, a[r + (size_t)c * n].im);
  for (int i = 0; i < n; ++i) u.at(i, i) = 1.0;
  if (n > 1) {
    householder_hessenberg(h, u);
    shifted_qr(h, u);
  }
  for (int c = 0; c < n; ++c)
    for (int r = 0; r < n; ++r) {
      const cx tv = r > c ? cx(0.0) : h.at(r, c);
      t_out[r + (size_t)c * n] = {tv.real(), tv.imag()};
      const cx uv = u.at(r, c);
      u_out[r + (size_t)c * n] = {uv.real(), uv.imag()};
    }
}

}  // namespace nds
