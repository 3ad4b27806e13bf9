/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see ndsylv_oracle.h). Never linked by the product.
 *
 * Scalar C11 restatement of the reference hot path. Arithmetic uses C99 `double _Complex`,
 * which GCC lowers exactly as it lowers std::complex<double> in the reference (inline
 * multiply with the __muldc3 NaN-recovery fallback, __divdc3 for division, cabs for
 * std::abs), and loops keep the reference's summation order, so results are bitwise
 * identical to the reference build in oracle/_ref (pinned by tests/test_oracle_pins.py).
 */
#define _POSIX_C_SOURCE 199309L
#include "ndsylv_oracle.h"

#include <complex.h>
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef double _Complex cxd;

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* tensor.cpp:8-16 */
int64_t orc_checked_total(int n_modes, const int64_t* dims) {
  if (n_modes < 1) return -1;
  int64_t total = 1;
  for (int j = 0; j < n_modes; ++j) {
    if (dims[j] < 1) return -1;
    if (__builtin_mul_overflow(total, dims[j], &total)) return -2;
  }
  return total;
}

/* kernels.cpp:9-21 — the (inner, n, outer) view of mode `mode` (1-based). */
static void slab(int n_modes, const int64_t* dims, int mode, int64_t* inner, int64_t* n, int64_t* outer) {
  *inner = 1;
  *outer = 1;
  *n = dims[mode - 1];
  for (int j = 0; j < mode - 1; ++j) *inner *= dims[j];
  for (int j = mode; j < n_modes; ++j) *outer *= dims[j];
}

/* kernels.cpp:24-44 — serial twin (kernels.cpp:92); same loop nest and summation order. */
int orc_mode_product(int n_modes, const int64_t* dims, const double* m_raw, int mode, const double* x_raw,
                     double* r_raw) {
  if (mode < 1 || mode > n_modes) return ORC_ERR_INVALID;
  int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  int64_t inner, n, outer;
  slab(n_modes, dims, mode, &inner, &n, &outer);
  const cxd* m = (const cxd*)m_raw;
  const cxd* x = (const cxd*)x_raw;
  cxd* r = (cxd*)r_raw;
  memset(r, 0, (size_t)total * sizeof(cxd)); /* NDTensor::zeros, kernels.cpp:28 */
  const int64_t block = inner * n;
  for (int64_t b = 0; b < outer; ++b) {
    for (int64_t i = 0; i < n; ++i) {
      cxd* out = r + b * block + i * inner;
      for (int64_t k = 0; k < n; ++k) {
        const cxd mik = m[i + k * n]; /* Matrix::operator() column-major, matrix.hpp:29-30 */
        const cxd* in = x + b * block + k * inner;
        for (int64_t a = 0; a < inner; ++a) out[a] += mik * in[a];
      }
    }
  }
  return ORC_OK;
}

/* matrix.cpp:34-39 */
static void adjoint(int64_t n, const cxd* u, cxd* uh) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) uh[j + i * n] = conj(u[i + j * n]);
}

/* sylvester.cpp:55-69 — modes applied 1..N, a fresh tensor per mode. */
static int transform(int n_modes, const int64_t* dims, const double* const* u, const double* in, double* out,
                     int use_adjoint) {
  int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  cxd* cur = (cxd*)malloc((size_t)total * sizeof(cxd));
  cxd* nxt = (cxd*)malloc((size_t)total * sizeof(cxd));
  if (!cur || !nxt) {
    free(cur);
    free(nxt);
    return ORC_ERR_OTHER;
  }
  memcpy(cur, in, (size_t)total * sizeof(cxd));
  for (int j = 1; j <= n_modes; ++j) {
    const int64_t n = dims[j - 1];
    const double* m = u[j - 1];
    cxd* tmp = NULL;
    if (use_adjoint) {
      tmp = (cxd*)malloc((size_t)(n * n) * sizeof(cxd));
      adjoint(n, (const cxd*)u[j - 1], tmp);
      m = (const double*)tmp;
    }
    orc_mode_product(n_modes, dims, m, j, (const double*)cur, (double*)nxt);
    free(tmp);
    cxd* s = cur;
    cur = nxt;
    nxt = s;
  }
  memcpy(out, cur, (size_t)total * sizeof(cxd));
  free(cur);
  free(nxt);
  return ORC_OK;
}

int orc_forward_transform(int n_modes, const int64_t* dims, const double* const* u, const double* b, double* c) {
  return transform(n_modes, dims, u, b, c, 1);
}

int orc_inverse_transform(int n_modes, const int64_t* dims, const double* const* u, const double* y, double* x) {
  return transform(n_modes, dims, u, y, x, 0);
}

/* sylvester.cpp:44-53 — r = 0; r += 1.0 * (A_j x_j x) per mode (add_scaled, kernels.cpp:81-88). */
int orc_apply_operator(int n_modes, const int64_t* dims, const double* const* a, const double* x, double* r_raw) {
  int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  cxd* term = (cxd*)malloc((size_t)total * sizeof(cxd));
  if (!term) return ORC_ERR_OTHER;
  cxd* r = (cxd*)r_raw;
  memset(r, 0, (size_t)total * sizeof(cxd));
  for (int j = 1; j <= n_modes; ++j) {
    orc_mode_product(n_modes, dims, a[j - 1], j, x, (double*)term);
    const cxd alpha = 1.0;
    for (int64_t i = 0; i < total; ++i) r[i] += alpha * term[i];
  }
  free(term);
  return ORC_OK;
}

/* matrix.cpp:99-103 */
static double norm_frobenius(int64_t n, const cxd* t) {
  double s = 0.0;
  for (int64_t i = 0; i < n * n; ++i) {
    const double re = creal(t[i]), im = cimag(t[i]);
    s += re * re + im * im; /* std::norm for double: x*x + y*y */
  }
  return sqrt(s);
}

/* sylvester.cpp:29-33 */
double orc_default_singular_tol(int n_modes, const int64_t* dims, const double* const* t) {
  double s = 0.0;
  for (int j = 0; j < n_modes; ++j) s += norm_frobenius(dims[j], (const cxd*)t[j]);
  return DBL_EPSILON * s;
}

/* sylvester.cpp:35-40 */
int orc_numerically_diagonal(int n, const double* t_raw) {
  const cxd* t = (const cxd*)t_raw;
  double off2 = 0.0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < j; ++i) {
      const double re = creal(t[i + (int64_t)j * n]), im = cimag(t[i + (int64_t)j * n]);
      off2 += re * re + im * im;
    }
  return sqrt(off2) <= 1e-12 * (1.0 + norm_frobenius(n, t));
}

/* Decode a 0-based flat index into the 1-based multi-index (tensor.cpp:29-41 inverted). */
static void decode(int n_modes, const int64_t* dims, int64_t flat, int64_t* multi) {
  for (int j = 0; j < n_modes; ++j) {
    multi[j] = flat % dims[j] + 1;
    flat /= dims[j];
  }
}

/* sylvester.cpp:71-108. The MultiIndexCursor (tensor.cpp:68-93, paper Alg. 2) visits flat
 * positions total..1 with i_1 fastest; we keep the decoded multi-index in `cur` and step it
 * the same way (odometer decrement). */
int orc_back_substitute(int n_modes, const int64_t* dims, const double* const* t_raw, double* c_raw,
                        double singular_tol, orc_backsub_stats* stats, int64_t* bad_index, double* bad_den) {
  int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  int64_t strides[64];
  int64_t cur[64];
  if (n_modes > 64) return ORC_ERR_INVALID;
  int64_t acc = 1;
  for (int j = 0; j < n_modes; ++j) {
    strides[j] = acc;
    acc *= dims[j];
    cur[j] = dims[j];
  }
  cxd* data = (cxd*)c_raw;
  orc_backsub_stats st = {0, 0, INFINITY};
  for (int64_t index = total; index >= 1; --index) {
    const int64_t flat = index - 1;
    cxd num = data[flat];
    cxd den = 0.0;
    for (int j = 0; j < n_modes; ++j) {
      const cxd* t = (const cxd*)t_raw[j];
      const int64_t ij = cur[j], nj = dims[j];
      den += t[(ij - 1) + (ij - 1) * nj];
      const int64_t stride = strides[j];
      for (int64_t k = ij + 1; k <= nj; ++k) num -= t[(ij - 1) + (k - 1) * nj] * data[flat + (k - ij) * stride];
      st.multiplies += nj - ij;
    }
    const double aden = cabs(den);
    st.min_abs_denominator = fmin(st.min_abs_denominator, aden);
    if (aden <= singular_tol) {
      if (bad_index) memcpy(bad_index, cur, (size_t)n_modes * sizeof(int64_t));
      if (bad_den) {
        bad_den[0] = creal(den);
        bad_den[1] = cimag(den);
      }
      if (stats) *stats = st;
      return ORC_ERR_SINGULAR;
    }
    data[flat] = num / den;
    ++st.entries;
    /* MultiIndexCursor::next, tensor.cpp:77-93 */
    if (cur[0] >= 2) {
      --cur[0];
    } else {
      int k = 1;
      while (k < n_modes && cur[k] == 1) ++k;
      if (k < n_modes) {
        --cur[k];
        for (int j = 0; j < k; ++j) cur[j] = dims[j];
      }
    }
  }
  if (stats) *stats = st;
  return ORC_OK;
}

/* sylvester.cpp:119-141 — eigenvalue sums in cursor order; first offender (descending) wins. */
static int eigenvalue_sums(int n_modes, const int64_t* dims, const double* const* t_raw, double tol, cxd* sums,
                           double* min_abs, int64_t* bad_index, double* bad_den) {
  const int64_t total = orc_checked_total(n_modes, dims);
  double best = INFINITY;
  int64_t multi[64];
  for (int64_t index = total; index >= 1; --index) {
    decode(n_modes, dims, index - 1, multi);
    cxd den = 0.0;
    for (int j = 0; j < n_modes; ++j) {
      const cxd* t = (const cxd*)t_raw[j];
      den += t[(multi[j] - 1) + (multi[j] - 1) * dims[j]];
    }
    const double aden = cabs(den);
    best = fmin(best, aden);
    if (aden <= tol) {
      if (bad_index) memcpy(bad_index, multi, (size_t)n_modes * sizeof(int64_t));
      if (bad_den) {
        bad_den[0] = creal(den);
        bad_den[1] = cimag(den);
      }
      return ORC_ERR_SINGULAR;
    }
    sums[index - 1] = den;
  }
  *min_abs = best;
  return ORC_OK;
}

/* sylvester.cpp:17-27 validation is the caller's (shapes are implied by dims here);
 * sylvester.cpp:167-227 minus the Schur step. */
int orc_solve_schur(int n_modes, const int64_t* dims, const double* const* u, const double* const* t,
                    const double* b, double* x, double singular_tol, unsigned flags, orc_report* rep,
                    int64_t* bad_index, double* bad_den) {
  if (n_modes < 2) return ORC_ERR_INVALID;
  const int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  orc_report r;
  memset(&r, 0, sizeof r);
  r.flop_estimate = orc_flop_estimate(n_modes, dims);
  r.schur_flop_estimate = orc_schur_flop_estimate(n_modes, dims);
  const double tol = singular_tol > 0.0 ? singular_tol : orc_default_singular_tol(n_modes, dims, t);
  int diagonal_route = (flags & 1u) != 0;
  for (int j = 0; diagonal_route && j < n_modes; ++j)
    if (!orc_numerically_diagonal((int)dims[j], t[j])) diagonal_route = 0;
  cxd* c = (cxd*)malloc((size_t)total * sizeof(cxd));
  if (!c) return ORC_ERR_OTHER;
  int rc = ORC_OK;
  if (diagonal_route) {
    cxd* sums = (cxd*)malloc((size_t)total * sizeof(cxd));
    if (!sums) {
      free(c);
      return ORC_ERR_OTHER;
    }
    rc = eigenvalue_sums(n_modes, dims, t, tol, sums, &r.min_abs_denominator, bad_index, bad_den);
    if (rc == ORC_OK) {
      double t0 = now_seconds();
      orc_forward_transform(n_modes, dims, u, b, (double*)c);
      r.transform_seconds = now_seconds() - t0;
      t0 = now_seconds();
      for (int64_t i = 0; i < total; ++i) c[i] /= sums[i];
      r.backsub_seconds = now_seconds() - t0;
      t0 = now_seconds();
      orc_inverse_transform(n_modes, dims, u, (const double*)c, x);
      r.inverse_seconds = now_seconds() - t0;
      r.used_normal_fast_path = 1;
    }
    free(sums);
  } else {
    double t0 = now_seconds();
    orc_forward_transform(n_modes, dims, u, b, (double*)c);
    r.transform_seconds = now_seconds() - t0;
    t0 = now_seconds();
    orc_backsub_stats st;
    rc = orc_back_substitute(n_modes, dims, t, (double*)c, tol, &st, bad_index, bad_den);
    r.backsub_seconds = now_seconds() - t0;
    r.backsub_entries = st.entries;
    r.backsub_multiplies = st.multiplies;
    r.min_abs_denominator = st.min_abs_denominator;
    if (rc == ORC_OK) {
      t0 = now_seconds();
      orc_inverse_transform(n_modes, dims, u, (const double*)c, x);
      r.inverse_seconds = now_seconds() - t0;
    }
  }
  free(c);
  if (rc == ORC_OK && (flags & 2u)) /* real_output, sylvester.cpp:223-224 */
    for (int64_t i = 0; i < total; ++i) x[2 * i + 1] = 0.0;
  if (rep) *rep = r;
  return rc;
}

/* sylvester.cpp:229-241 */
int64_t orc_flop_estimate(int n_modes, const int64_t* dims) {
  const int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return -1;
  int64_t sum = 0, factor = 0, flops = 0;
  for (int j = 0; j < n_modes; ++j)
    if (__builtin_add_overflow(sum, dims[j], &sum)) return -1;
  if (__builtin_mul_overflow(sum, (int64_t)5, &factor) || __builtin_add_overflow(factor, (int64_t)1 - n_modes, &factor))
    return -1;
  if (__builtin_mul_overflow(total, factor, &flops)) return -1;
  return flops;
}

/* sylvester.cpp:243-257 */
int64_t orc_schur_flop_estimate(int n_modes, const int64_t* dims) {
  if (orc_checked_total(n_modes, dims) < 0) return -1;
  int64_t sum_cubes = 0, flops = 0;
  for (int j = 0; j < n_modes; ++j) {
    int64_t sq = 0, cube = 0;
    if (__builtin_mul_overflow(dims[j], dims[j], &sq) || __builtin_mul_overflow(sq, dims[j], &cube) ||
        __builtin_add_overflow(sum_cubes, cube, &sum_cubes))
      return -1;
  }
  if (__builtin_mul_overflow(sum_cubes, (int64_t)25, &flops)) return -1;
  return flops;
}

/* rng.hpp:12-43 */
static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void orc_xoshiro_uniform(uint64_t seed, int64_t count, double* out) {
  uint64_t s[4];
  uint64_t sm = seed;
  for (int w = 0; w < 4; ++w) {
    sm += 0x9e3779b97f4a7c15ULL;
    uint64_t z = sm;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    s[w] = z ^ (z >> 31);
  }
  for (int64_t i = 0; i < count; ++i) {
    const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    out[i] = (double)(result >> 11) * 0x1.0p-53;
  }
}

/* ---- ODE propagator and RK4 (ode.cpp) ------------------------------------ */

/* matrix.cpp:48-58: r = a b, loops j, k (skipping zero b(k, j)), i. n x n column-major. */
static void mat_mul(int n, const cxd* a, const cxd* b, cxd* r) {
  memset(r, 0, (size_t)n * n * sizeof(cxd));
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const cxd bk = b[k + (size_t)j * n];
      if (bk == 0.0) continue;
      for (int i = 0; i < n; ++i) r[i + (size_t)j * n] += a[i + (size_t)k * n] * bk;
    }
}

/* matrix.cpp:105-113 */
static double mat_norm_inf(int n, const cxd* a) {
  double best = 0.0;
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += cabs(a[i + (size_t)j * n]);
    if (s > best) best = s;
  }
  return best;
}

/* matrix.cpp:143-201: PartialPivLU(lu).solve(rhs), rhs overwritten column by column. */
static int lu_solve(int n, cxd* lu, cxd* rhs) {
  const double tol = DBL_EPSILON * mat_norm_inf(n, lu);
  int* perm = (int*)malloc((size_t)n * sizeof(int));
  cxd* col = (cxd*)malloc((size_t)n * sizeof(cxd));
  if (!perm || !col) {
    free(perm);
    free(col);
    return ORC_ERR_OTHER;
  }
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = cabs(lu[k + (size_t)k * n]);
    for (int i = k + 1; i < n; ++i) {
      const double cand = cabs(lu[i + (size_t)k * n]);
      if (cand > best) {
        best = cand;
        piv = i;
      }
    }
    if (best <= tol) {
      free(perm);
      free(col);
      return ORC_ERR_OTHER;
    }
    perm[k] = piv;
    if (piv != k)
      for (int j = 0; j < n; ++j) {
        const cxd tmp = lu[k + (size_t)j * n];
        lu[k + (size_t)j * n] = lu[piv + (size_t)j * n];
        lu[piv + (size_t)j * n] = tmp;
      }
    const cxd inv_piv = 1.0 / lu[k + (size_t)k * n];
    for (int i = k + 1; i < n; ++i) {
      const cxd f = lu[i + (size_t)k * n] * inv_piv;
      lu[i + (size_t)k * n] = f;
      if (f == 0.0) continue;
      for (int j = k + 1; j < n; ++j) lu[i + (size_t)j * n] -= f * lu[k + (size_t)j * n];
    }
  }
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < n; ++i) col[i] = rhs[i + (size_t)j * n];
    for (int k = 0; k < n; ++k)
      if (perm[k] != k) {
        const cxd tmp = col[k];
        col[k] = col[perm[k]];
        col[perm[k]] = tmp;
      }
    for (int k = 0; k < n; ++k)
      for (int i = k + 1; i < n; ++i) col[i] -= lu[i + (size_t)k * n] * col[k];
    for (int i = n - 1; i >= 0; --i) {
      cxd acc = col[i];
      for (int k = i + 1; k < n; ++k) acc -= lu[i + (size_t)k * n] * col[k];
      col[i] = acc / lu[i + (size_t)i * n];
    }
    for (int i = 0; i < n; ++i) rhs[i + (size_t)j * n] = col[i];
  }
  free(perm);
  free(col);
  return ORC_OK;
}

/* schur.cpp:230-255: [6/6] Pade with scaling and squaring; a is overwritten, result in f. */
static int pade_exp(int n, cxd* a1, cxd* f) {
  const size_t nn = (size_t)n * n;
  const double norm = mat_norm_inf(n, a1);
  int squarings = 0;
  if (norm > 0.5) {
    squarings = (int)ceil(log2(norm)) + 1;
    const cxd sc = ldexp(1.0, -squarings);
    for (size_t i = 0; i < nn; ++i) a1[i] *= sc;
  }
  enum { Q = 6 };
  double coeff[Q + 1];
  coeff[0] = 1.0;
  for (int k = 1; k <= Q; ++k) coeff[k] = coeff[k - 1] * (double)(Q - k + 1) / (k * (2.0 * Q - k + 1));
  cxd* a2 = (cxd*)malloc(nn * sizeof(cxd));
  cxd* even = (cxd*)calloc(nn, sizeof(cxd));
  cxd* odd_inner = (cxd*)calloc(nn, sizeof(cxd));
  cxd* power = (cxd*)malloc(nn * sizeof(cxd));
  cxd* tmp = (cxd*)malloc(nn * sizeof(cxd));
  cxd* num = (cxd*)malloc(nn * sizeof(cxd));
  if (!a2 || !even || !odd_inner || !power || !tmp || !num) {
    free(a2), free(even), free(odd_inner), free(power), free(tmp), free(num);
    return ORC_ERR_OTHER;
  }
  mat_mul(n, a1, a1, a2);
  for (int i = 0; i < n; ++i) {  /* coeff * identity: every entry multiplied (zeros included) */
    even[i + (size_t)i * n] = 1.0;
    odd_inner[i + (size_t)i * n] = 1.0;
  }
  {
    const cxd c0 = coeff[0], c1 = coeff[1];
    for (size_t i = 0; i < nn; ++i) {
      even[i] *= c0;
      odd_inner[i] *= c1;
    }
  }
  memcpy(power, a2, nn * sizeof(cxd));
  for (int k = 2; k <= Q; k += 2) {
    const cxd ck = coeff[k];
    for (size_t i = 0; i < nn; ++i) even[i] += ck * power[i];
    if (k + 1 <= Q) {
      const cxd ck1 = coeff[k + 1];
      for (size_t i = 0; i < nn; ++i) odd_inner[i] += ck1 * power[i];
    }
    if (k + 2 <= Q) {
      mat_mul(n, power, a2, tmp);
      memcpy(power, tmp, nn * sizeof(cxd));
    }
  }
  mat_mul(n, a1, odd_inner, tmp); /* odd */
  for (size_t i = 0; i < nn; ++i) {
    num[i] = even[i] + tmp[i];
    even[i] = even[i] - tmp[i]; /* den */
  }
  int rc = lu_solve(n, even, num);
  if (rc == ORC_OK) {
    memcpy(f, num, nn * sizeof(cxd));
    for (int i = 0; i < squarings; ++i) {
      mat_mul(n, f, f, tmp);
      memcpy(f, tmp, nn * sizeof(cxd));
    }
  }
  free(a2), free(even), free(odd_inner), free(power), free(tmp), free(num);
  return rc;
}

int orc_triangular_exp(int n, const double* t_raw, double t, double* f_raw) {
  const cxd* tm = (const cxd*)t_raw;
  cxd* f = (cxd*)f_raw;
  const size_t nn = (size_t)n * n;
  for (int j = 0; j < n; ++j)
    for (int i = j + 1; i < n; ++i)
      if (tm[i + (size_t)j * n] != 0.0) return ORC_ERR_INVALID;
  memset(f, 0, nn * sizeof(cxd));
  if (t == 0.0) {
    for (int i = 0; i < n; ++i) f[i + (size_t)i * n] = 1.0;
    return ORC_OK;
  }
  /* schur.cpp:164-174 diagonal_well_separated */
  double dmax = 0.0;
  for (int i = 0; i < n; ++i) dmax = fmax(dmax, cabs(tm[i + (size_t)i * n]));
  const double threshold = 1e-8 * (1.0 + dmax);
  int separated = 1;
  for (int i = 0; i < n && separated; ++i)
    for (int k = i + 1; k < n; ++k)
      if (cabs(tm[i + (size_t)i * n] - tm[k + (size_t)k * n]) < threshold) {
        separated = 0;
        break;
      }
  cxd* s = (cxd*)malloc(nn * sizeof(cxd));
  if (!s) return ORC_ERR_OTHER;
  const cxd ct = t; /* cxd(t, 0.0) * t_mat */
  for (size_t i = 0; i < nn; ++i) s[i] = tm[i] * ct;
  int rc = ORC_OK;
  if (!separated) {
    rc = pade_exp(n, s, f);
    for (int j = 0; j < n; ++j)
      for (int i = j + 1; i < n; ++i) f[i + (size_t)j * n] = 0.0;
  } else {
    for (int i = 0; i < n; ++i) f[i + (size_t)i * n] = cexp(s[i + (size_t)i * n]);
    for (int p = 1; p < n; ++p)
      for (int i = 0; i + p < n; ++i) {
        const int j = i + p;
#define S_(a, b) s[(a) + (size_t)(b) * n]
#define F_(a, b) f[(a) + (size_t)(b) * n]
        cxd num = S_(i, j) * (F_(j, j) - F_(i, i));
        for (int k = i + 1; k < j; ++k) num += S_(i, k) * F_(k, j) - F_(i, k) * S_(k, j);
        F_(i, j) = num / (S_(j, j) - S_(i, i));
#undef S_
#undef F_
      }
  }
  free(s);
  return rc;
}

/* kernels.cpp:81-88 add_scaled: y += alpha x */
static void add_scaled(int64_t total, cxd* y, cxd alpha, const cxd* x) {
  for (int64_t i = 0; i < total; ++i) y[i] += alpha * x[i];
}

int orc_ode_at_schur(int n_modes, const int64_t* dims, const double* const* u, const double* const* t,
                     const double* forcing, const double* initial, double time, double singular_tol, unsigned flags,
                     double* x, int64_t* bad_index, double* bad_den) {
  if (n_modes < 2) return ORC_ERR_INVALID;
  if (!isfinite(time)) return ORC_ERR_INVALID;
  const int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  const double tol = singular_tol > 0.0 ? singular_tol : orc_default_singular_tol(n_modes, dims, t);
  cxd* c = (cxd*)malloc((size_t)total * sizeof(cxd));
  cxd* y0 = (cxd*)malloc((size_t)total * sizeof(cxd));
  cxd* g = (cxd*)malloc((size_t)total * sizeof(cxd));
  cxd* h = (cxd*)malloc((size_t)total * sizeof(cxd));
  int64_t fmax_n = 0;
  for (int j = 0; j < n_modes; ++j) fmax_n = dims[j] > fmax_n ? dims[j] : fmax_n;
  cxd* fe = (cxd*)malloc((size_t)(fmax_n * fmax_n) * sizeof(cxd));
  int rc = ORC_OK;
  if (!c || !y0 || !g || !h || !fe) rc = ORC_ERR_OTHER;
  if (rc == ORC_OK) {
    /* constructor (ode.cpp:53-56): C, Y0, operator image G0 = sum_j T_j x_j Y0 + C */
    orc_forward_transform(n_modes, dims, u, forcing, (double*)c);
    orc_forward_transform(n_modes, dims, u, initial, (double*)y0);
    orc_apply_operator(n_modes, dims, t, (const double*)y0, (double*)g);
    add_scaled(total, g, 1.0, c);
    /* at() (ode.cpp:71-73) */
    for (int j = 1; j <= n_modes && rc == ORC_OK; ++j) {
      rc = orc_triangular_exp((int)dims[j - 1], t[j - 1], time, (double*)fe);
      if (rc != ORC_OK) break;
      orc_mode_product(n_modes, dims, (const double*)fe, j, (const double*)g, (double*)h);
      cxd* sw = g;
      g = h;
      h = sw;
    }
  }
  if (rc == ORC_OK) {
    add_scaled(total, g, -1.0, c);
    orc_backsub_stats st;
    rc = orc_back_substitute(n_modes, dims, t, (double*)g, tol, &st, bad_index, bad_den);
  }
  if (rc == ORC_OK) {
    orc_inverse_transform(n_modes, dims, u, (const double*)g, x);
    if (flags & 2u) {
      cxd* xc = (cxd*)x;
      for (int64_t i = 0; i < total; ++i) xc[i] = creal(xc[i]);
    }
  }
  free(c), free(y0), free(g), free(h), free(fe);
  return rc;
}

int orc_rk4(int n_modes, const int64_t* dims, const double* const* a, const double* forcing, const double* initial,
            double time, double dt, int64_t max_steps, double* x_raw) {
  if (n_modes < 2) return ORC_ERR_INVALID;
  const int64_t total = orc_checked_total(n_modes, dims);
  if (total < 0) return total == -2 ? ORC_ERR_OVERFLOW : ORC_ERR_INVALID;
  if (!isfinite(time)) return ORC_ERR_INVALID;
  if (!(dt > 0.0) || !isfinite(dt)) return ORC_ERR_INVALID;
  cxd* x = (cxd*)x_raw;
  memcpy(x, initial, (size_t)total * sizeof(cxd));
  if (time == 0.0) return ORC_OK;
  const double direction = time > 0.0 ? 1.0 : -1.0;
  const double span = fabs(time);
  const int64_t full_steps = (int64_t)floor(span / dt);
  if (full_steps + 1 > max_steps) return ORC_ERR_INVALID;
  const cxd* b = (const cxd*)forcing;
  cxd* k[4];
  cxd* stage = (cxd*)malloc((size_t)total * sizeof(cxd));
  int rc = stage ? ORC_OK : ORC_ERR_OTHER;
  for (int i = 0; i < 4; ++i) {
    k[i] = (cxd*)malloc((size_t)total * sizeof(cxd));
    if (!k[i]) rc = ORC_ERR_OTHER;
  }
  /* rhs(state) = apply_operator(A, state) + B (ode.cpp:101-105) */
#define RHS(state, out)                                                         \
  do {                                                                          \
    orc_apply_operator(n_modes, dims, a, (const double*)(state), (double*)(out)); \
    add_scaled(total, (out), 1.0, b);                                           \
  } while (0)
  for (int64_t step = 0; rc == ORC_OK && step <= full_steps; ++step) {
    double hh;
    if (step < full_steps) {
      hh = direction * dt;
    } else {
      const double remainder = span - (double)full_steps * dt;
      if (!(remainder > 0.0)) break;
      hh = direction * remainder;
    }
    const cxd ch = hh; /* advance (ode.cpp:107-123) */
    RHS(x, k[0]);
    memcpy(stage, x, (size_t)total * sizeof(cxd));
    add_scaled(total, stage, 0.5 * ch, k[0]);
    RHS(stage, k[1]);
    memcpy(stage, x, (size_t)total * sizeof(cxd));
    add_scaled(total, stage, 0.5 * ch, k[1]);
    RHS(stage, k[2]);
    memcpy(stage, x, (size_t)total * sizeof(cxd));
    add_scaled(total, stage, ch, k[2]);
    RHS(stage, k[3]);
    add_scaled(total, x, ch / 6.0, k[0]);
    add_scaled(total, x, ch / 3.0, k[1]);
    add_scaled(total, x, ch / 3.0, k[2]);
    add_scaled(total, x, ch / 6.0, k[3]);
    for (int64_t i = 0; i < total; ++i)
      if (!isfinite(creal(x[i])) || !isfinite(cimag(x[i]))) {
        rc = ORC_ERR_NONFINITE;
        break;
      }
  }
#undef RHS
  free(stage);
  for (int i = 0; i < 4; ++i) free(k[i]);
  return rc;
}
