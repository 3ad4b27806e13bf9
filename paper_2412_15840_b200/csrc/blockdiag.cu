// Device side of the block-diagonalised cubic route's plan (capi.cu plan_cubic_diag): the
// eigenvector matrices of the D x D diagonal blocks of every T_j for every candidate D, their
// inverses and condition numbers (one launch), and the merged factors U W, U W^{-H} and
// T' = W^{-1} T W of the chosen D (block-diagonal matrix products).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace nds {

// One CTA (128 threads) per job: block q of a candidate (mode j, extent d <= 128). Both
// triangular recurrences run ROW by row (row i from the bottom up, all columns k > i at once,
// thread k <-> column k), so every step's operands are shared-memory reads: the unknown matrix
// is kept packed (upper triangle, row i holding columns i..d-1 at i d - i (i - 1) / 2; 132 KB at
// d = 128) and the known row streams in from global memory one step ahead.
//  1. V: T V = V diag(T), V(k, k) = 1, V(i, k) = sum_{l = i+1..k} T(i, l) V(l, k) / (T(k, k) -
//     T(i, i)); then every column scaled to unit 2-norm;
//  2. W = V^{-1}: W(c, c) = 1 / V(c, c), W(i, c) = -sum_{l = i+1..c} V(i, l) W(l, c) / V(i, i);
//  3. cond_2(V) = ||V||_2 ||W||_2, both by 12 power iterations on M^H M (shared vectors).
// A zero eigenvalue gap (repeated eigenvalue) or a non-finite entry makes cond infinite.
constexpr int kEigThreads = 128;
__host__ __device__ constexpr int tri_off(int i, int d) { return i * d - i * (i - 1) / 2; }
size_t block_eig_smem(int dmax) { return (size_t)tri_off(dmax, dmax) * sizeof(double2); }
// sum_{l = l0..k} r[l] * U(l, k) for the packed upper triangle U in shared memory (row l at
// tri_off(l, d)): consecutive rows of column k are d - l - 1 apart; four independent accumulators
__device__ __forceinline__ double2 tri_dot_impl(const double2* __restrict__ r, const double2* __restrict__ tri, int l0,
                                                int k, int d) {
  double2 a[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  int p = tri_off(l0, d) + (k - l0);
  int l = l0;
  for (; l + 3 <= k; l += 4) {
    const int p1 = p + (d - l - 1), p2 = p1 + (d - l - 2), p3 = p2 + (d - l - 3);
    a[0] = cfma(a[0], r[l], tri[p]);
    a[1] = cfma(a[1], r[l + 1], tri[p1]);
    a[2] = cfma(a[2], r[l + 2], tri[p2]);
    a[3] = cfma(a[3], r[l + 3], tri[p3]);
    p = p3 + (d - l - 4);
  }
  for (; l <= k; ++l) {
    a[0] = cfma(a[0], r[l], tri[p]);
    p += d - l - 1;
  }
  return cadd(cadd(a[0], a[1]), cadd(a[2], a[3]));
}

__global__ void __launch_bounds__(kEigThreads) block_eig_kernel(const double2* __restrict__ t_pool, const EigCands cs,
                                                               double2* __restrict__ vpool, double2* __restrict__ wpool,
                                                               double* __restrict__ cond) {
  extern __shared__ __align__(16) double2 tri[];  // the packed unknown upper triangle (V, then W)
  int ci = 0;
  while (ci + 1 < cs.count && (int)blockIdx.x >= cs.first[ci + 1]) ++ci;
  const int q = blockIdx.x - cs.first[ci];
  const int d = cs.d[ci];
  if (d > 128) return;  // block_eig_big_kernel's job
  const int k = threadIdx.x, lane = k & 31, warp = k >> 5;
  const int64_t n = cs.n[ci], o = (int64_t)q * d;
  const double2* T = t_pool + cs.toff[ci];
  double2* V = vpool + cs.voff[ci] + (int64_t)q * d * d;  // column-major d x d
  double2* W = wpool + cs.voff[ci] + (int64_t)q * d * d;
  auto P = [d](int r, int c) { return tri_off(r, d) + (c - r); };
  auto tri_dot = [&](const double2* r, int l0, int kk, int dd) { return tri_dot_impl(r, tri, l0, kk, dd); };
  __shared__ int bad;
  __shared__ double2 row[2][128];  // the known row of this step (double-buffered)
  __shared__ double2 x[128], y[128];
  __shared__ double red[4];
  if (k == 0) bad = 0;
  // ---- 1. V, rows d-1 .. 0 ----
  if (k < d) row[(d - 1) & 1][k] = T[(o + d - 1) + (o + k) * n];
  double2 lk = k < d ? T[(o + k) + (o + k) * n] : make_double2(0.0, 0.0);
  __syncthreads();
  for (int i = d - 1; i >= 0; --i) {
    const double2* ti = row[i & 1];  // ti[c] = T(i, c)
    if (i > 0 && k < d) row[(i - 1) & 1][k] = T[(o + i - 1) + (o + k) * n];  // next row, one step ahead
    if (k == i) tri[P(i, i)] = make_double2(1.0, 0.0);
    else if (k > i && k < d) {
      const double2 acc = tri_dot(ti, i + 1, k, d);
      const double2 gap = csub(lk, ti[i]);
      if (gap.x == 0.0 && gap.y == 0.0) {
        bad = 1;
        tri[P(i, k)] = make_double2(0.0, 0.0);
      } else {
        tri[P(i, k)] = cdiv(acc, gap);
      }
    }
    __syncthreads();
  }
  // ||M||_2 of the packed upper triangle in shared memory: 12 power iterations on M^H M
  auto norm2 = [&]() {
    if (k < d) x[k] = make_double2(1.0 + 0.37 * k, 0.11 * (k % 5));
    __syncthreads();
    double lam = 0.0;
    for (int it = 0; it < 12; ++it) {
      if (k < d) {  // y = M x (row k)
        double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
        const double2* mk = tri + tri_off(k, d) - k;
        int c = k;
        for (; c + 1 < d; c += 2) {
          s0 = cfma(s0, mk[c], x[c]);
          s1 = cfma(s1, mk[c + 1], x[c + 1]);
        }
        if (c < d) s0 = cfma(s0, mk[c], x[c]);
        y[k] = cadd(s0, s1);
      }
      __syncthreads();
      double part = 0.0;
      double2 xn = make_double2(0.0, 0.0);
      if (k < d) {  // x = M^H y (column k)
        double2 x1 = make_double2(0.0, 0.0);
        int p = k, r = 0;  // P(r, k) = p, rows r -> r + 1 step by d - r - 1
        for (; r + 1 <= k; r += 2) {
          const double2 m0 = tri[p], m1 = tri[p + (d - r - 1)];
          xn = cfma(xn, make_double2(m0.x, -m0.y), y[r]);
          x1 = cfma(x1, make_double2(m1.x, -m1.y), y[r + 1]);
          p += (d - r - 1) + (d - r - 2);
        }
        if (r <= k) xn = cfma(xn, make_double2(tri[p].x, -tri[p].y), y[r]);
        xn = cadd(xn, x1);
        part = xn.x * xn.x + xn.y * xn.y;
      }
      for (int sh = 16; sh > 0; sh >>= 1) part += __shfl_xor_sync(0xffffffffu, part, sh);
      if (lane == 0) red[warp] = part;
      __syncthreads();
      const double tot = sqrt(red[0] + red[1] + red[2] + red[3]);
      lam = tot;
      if (k < d) x[k] = make_double2(xn.x / tot, xn.y / tot);
      __syncthreads();
    }
    return sqrt(lam);
  };
  if (k < d) {  // unit columns (in place), stored column-major
    double nn = 0.0;
    for (int i = 0; i <= k; ++i) {
      const double2 v = tri[P(i, k)];
      nn += v.x * v.x + v.y * v.y;
    }
    nn = sqrt(nn);
    if (!isfinite(nn) || nn == 0.0) {
      bad = 1;
      nn = 1.0;
    }
    const double sc = 1.0 / nn;
    for (int i = 0; i < d; ++i) {
      double2 v = make_double2(0.0, 0.0);
      if (i <= k) {
        v = tri[P(i, k)];
        v = make_double2(v.x * sc, v.y * sc);
        tri[P(i, k)] = v;
      }
      V[i + (int64_t)k * d] = v;
    }
  }
  __syncthreads();
  const double nv = norm2();
  // ---- 2. W = V^{-1}, rows d-1 .. 0 (V rows from global, just written) ----
  if (k < d) row[(d - 1) & 1][k] = V[(d - 1) + (int64_t)k * d];
  __syncthreads();
  for (int i = d - 1; i >= 0; --i) {
    const double2* vi = row[i & 1];  // vi[c] = V(i, c)
    if (i > 0 && k < d) row[(i - 1) & 1][k] = V[(i - 1) + (int64_t)k * d];
    if (k == i) tri[P(i, i)] = cdiv(make_double2(1.0, 0.0), vi[i]);
    else if (k > i && k < d) {
      const double2 acc = tri_dot(vi, i + 1, k, d);
      tri[P(i, k)] = cdiv(make_double2(-acc.x, -acc.y), vi[i]);
    }
    __syncthreads();
  }
  if (k < d)
    for (int i = 0; i < d; ++i) W[i + (int64_t)k * d] = i <= k ? tri[P(i, k)] : make_double2(0.0, 0.0);
  const double nw = norm2();
  if (k == 0) {
    const double c = nv * nw;
    cond[blockIdx.x] = (bad || !isfinite(c)) ? INFINITY : c;
  }
}

// The same for one block of 128 < d <= 256 (a whole mode: D = n), one CTA of 256 threads: the
// unknown triangles (V, then W) live row-major in global scratch (2 d^2 entries per job, L2
// resident) so a step's reads are coalesced across the columns, then are written column-major.
constexpr int kEigBigThreads = 256;
__global__ void __launch_bounds__(kEigBigThreads) block_eig_big_kernel(const double2* __restrict__ t_pool,
                                                                      const EigCands cs, double2* __restrict__ vpool,
                                                                      double2* __restrict__ wpool,
                                                                      double* __restrict__ cond,
                                                                      double2* __restrict__ scratch) {
  int ci = 0;
  while (ci + 1 < cs.count && (int)blockIdx.x >= cs.first[ci + 1]) ++ci;
  const int d = cs.d[ci];
  if (d <= 128) return;  // block_eig_kernel's job
  const int q = blockIdx.x - cs.first[ci];
  const int k = threadIdx.x, lane = k & 31, warp = k >> 5;
  const int64_t n = cs.n[ci], o = (int64_t)q * d;
  const double2* T = t_pool + cs.toff[ci];
  double2* V = vpool + cs.voff[ci] + (int64_t)q * d * d;
  double2* W = wpool + cs.voff[ci] + (int64_t)q * d * d;
  double2* R = scratch + cs.soff[ci] + (int64_t)q * 2 * d * d;  // V row-major
  double2* Q = R + (int64_t)d * d;                              // W row-major
  __shared__ int bad;
  __shared__ double2 row[2][kEigBigThreads];
  __shared__ double2 x[kEigBigThreads], y[kEigBigThreads];
  __shared__ double red[kEigBigThreads / 32];
  __shared__ double colscale[kEigBigThreads];
  if (k == 0) bad = 0;
  // ---- 1. V (row-major in R), rows d-1 .. 0 ----
  if (k < d) row[(d - 1) & 1][k] = T[(o + d - 1) + (o + k) * n];
  const double2 lk = k < d ? T[(o + k) + (o + k) * n] : make_double2(0.0, 0.0);
  __syncthreads();
  for (int i = d - 1; i >= 0; --i) {
    const double2* ti = row[i & 1];
    if (i > 0 && k < d) row[(i - 1) & 1][k] = T[(o + i - 1) + (o + k) * n];
    if (k < d) {
      double2 v = make_double2(k == i ? 1.0 : 0.0, 0.0);
      if (k > i) {
        double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
        int l = i + 1;
        for (; l + 1 <= k; l += 2) {
          a0 = cfma(a0, ti[l], R[(int64_t)l * d + k]);
          a1 = cfma(a1, ti[l + 1], R[(int64_t)(l + 1) * d + k]);
        }
        if (l <= k) a0 = cfma(a0, ti[l], R[(int64_t)l * d + k]);
        const double2 gap = csub(lk, ti[i]);
        if (gap.x == 0.0 && gap.y == 0.0) {
          bad = 1;
        } else {
          v = cdiv(cadd(a0, a1), gap);
        }
      }
      R[(int64_t)i * d + k] = v;
    }
    __syncthreads();
  }
  if (k < d) {  // unit columns
    double nn = 0.0;
    for (int i = 0; i <= k; ++i) {
      const double2 v = R[(int64_t)i * d + k];
      nn += v.x * v.x + v.y * v.y;
    }
    nn = sqrt(nn);
    if (!isfinite(nn) || nn == 0.0) {
      bad = 1;
      nn = 1.0;
    }
    colscale[k] = 1.0 / nn;
  }
  __syncthreads();
  for (int64_t e = k; e < (int64_t)d * d; e += kEigBigThreads) {  // scale R in place; V column-major
    const int i = (int)(e / d), c = (int)(e % d);
    double2 v = R[e];
    v = make_double2(v.x * colscale[c], v.y * colscale[c]);
    R[e] = v;
    V[i + (int64_t)c * d] = v;
  }
  __syncthreads();
  // ||M||_2 of a row-major upper triangular M in global memory: 12 power iterations on M^H M
  auto norm2 = [&](const double2* M) {
    if (k < d) x[k] = make_double2(1.0 + 0.37 * k, 0.11 * (k % 5));
    __syncthreads();
    double lam = 0.0;
    for (int it = 0; it < 12; ++it) {
      if (k < d) {
        double2 sacc = make_double2(0.0, 0.0);
        for (int c = k; c < d; ++c) sacc = cfma(sacc, M[(int64_t)k * d + c], x[c]);
        y[k] = sacc;
      }
      __syncthreads();
      double part = 0.0;
      double2 xn = make_double2(0.0, 0.0);
      if (k < d) {
        for (int r = 0; r <= k; ++r) {
          const double2 m = M[(int64_t)r * d + k];
          xn = cfma(xn, make_double2(m.x, -m.y), y[r]);
        }
        part = xn.x * xn.x + xn.y * xn.y;
      }
      for (int sh = 16; sh > 0; sh >>= 1) part += __shfl_xor_sync(0xffffffffu, part, sh);
      if (lane == 0) red[warp] = part;
      __syncthreads();
      double tot = 0.0;
      for (int w2 = 0; w2 < kEigBigThreads / 32; ++w2) tot += red[w2];
      tot = sqrt(tot);
      lam = tot;
      if (k < d) x[k] = make_double2(xn.x / tot, xn.y / tot);
      __syncthreads();
    }
    return sqrt(lam);
  };
  const double nv = norm2(R);
  // ---- 2. W = V^{-1} (row-major in Q), rows d-1 .. 0 ----
  if (k < d) row[(d - 1) & 1][k] = R[(int64_t)(d - 1) * d + k];
  __syncthreads();
  for (int i = d - 1; i >= 0; --i) {
    const double2* vi = row[i & 1];
    if (i > 0 && k < d) row[(i - 1) & 1][k] = R[(int64_t)(i - 1) * d + k];
    if (k < d) {
      double2 w = make_double2(0.0, 0.0);
      if (k == i) {
        w = cdiv(make_double2(1.0, 0.0), vi[i]);
      } else if (k > i) {
        double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
        int l = i + 1;
        for (; l + 1 <= k; l += 2) {
          a0 = cfma(a0, vi[l], Q[(int64_t)l * d + k]);
          a1 = cfma(a1, vi[l + 1], Q[(int64_t)(l + 1) * d + k]);
        }
        if (l <= k) a0 = cfma(a0, vi[l], Q[(int64_t)l * d + k]);
        const double2 acc = cadd(a0, a1);
        w = cdiv(make_double2(-acc.x, -acc.y), vi[i]);
      }
      Q[(int64_t)i * d + k] = w;
    }
    __syncthreads();
  }
  for (int64_t e = k; e < (int64_t)d * d; e += kEigBigThreads) W[(e / d) + (e % d) * d] = Q[e];
  __syncthreads();
  const double nw = norm2(Q);
  if (k == 0) {
    const double c = nv * nw;
    cond[blockIdx.x] = (bad || !isfinite(c)) ? INFINITY : c;
  }
}

void block_eig_launch(const double2* t_pool, const EigCands& cands, double2* vpool, double2* wpool, double* cond,
                      double2* scratch, cudaStream_t stream) {
  const int njobs = cands.count > 0 ? cands.first[cands.count] : 0;
  if (njobs <= 0) return;
  int dmax = 0;
  for (int c = 0; c < cands.count; ++c) dmax = std::max(dmax, std::min(cands.d[c], 128));
  const size_t smem = block_eig_smem(dmax);
  smem_optin(block_eig_kernel, smem);
  block_eig_kernel<<<(unsigned)njobs, kEigThreads, smem, stream>>>(t_pool, cands, vpool, wpool, cond);
  NDS_LAUNCH_CHECK();
  bool big = false;
  for (int c = 0; c < cands.count; ++c) big = big || cands.d[c] > 128;
  if (big) {
    block_eig_big_kernel<<<(unsigned)njobs, kEigBigThreads, 0, stream>>>(t_pool, cands, vpool, wpool, cond, scratch);
    NDS_LAUNCH_CHECK();
  }
}

// ---- Schur reordering (ZTREXC by adjacent swaps, all pairs of a round at once) -----------------
// Reorders the diagonal of every upper triangular T_j (n x n column-major, in place) by unitary
// adjacent swaps, accumulating the rotations into U_j (T_j = U_j^H A_j U_j stays a Schur form).
// Target: position P holds the eigenvalue whose rank by real part (ties by imaginary part, then
// position) is R(P) = the digits of P read in reverse over the mixed radix (B, 2, 2, .., rest):
// then every aligned block of B 2^k positions holds eigenvalues spread evenly over the spectrum
// instead of the neighbours the QR iteration deflates together, which is what keeps the
// eigenvector matrices of the diagonal blocks well conditioned (c2: prod cond at D = 16 from 1e19
// to 7e2). Odd-even transposition sort: n rounds; in a round the pairs (k, k+1) of one parity whose
// keys are out of order swap — per pair a ZLARTG rotation of (T(k,k+1), T(k+1,k+1) - T(k,k)),
// applied to rows k, k+1 (columns > k+1), then to columns k, k+1 (rows < k) of T and of U, and
// T(k,k) <-> T(k+1,k+1) (T(k,k+1) is unchanged). Disjoint pairs commute (left vs right
// multiplications), so a round is three barrier-separated phases. One CTA per mode.
__device__ __forceinline__ void zlartg_dev(double2 f, double2 g, double& cs, double2& sn) {
  const double af = hypot(f.x, f.y), ag = hypot(g.x, g.y);
  if (ag == 0.0) {
    cs = 1.0;
    sn = make_double2(0.0, 0.0);
  } else if (af == 0.0) {
    cs = 0.0;
    sn = make_double2(g.x / ag, -g.y / ag);  // conj(g) / |g|
  } else {
    const double nrm = hypot(af, ag);
    cs = af / nrm;
    const double2 fu = make_double2(f.x / af, f.y / af);                 // f / |f|
    const double2 gc = make_double2(g.x / nrm, -g.y / nrm);              // conj(g) / norm
    sn = cmul(fu, gc);
  }
}
__global__ void __launch_bounds__(1024) schur_reorder_kernel(const ReorderArgs ra, double2* __restrict__ tpool,
                                                             double2* __restrict__ upool) {
  __shared__ int key[kReorderMaxN];
  __shared__ int act[kReorderMaxN / 2];
  __shared__ double rc[kReorderMaxN / 2];
  __shared__ double2 rs[kReorderMaxN / 2];
  const int m = blockIdx.x;
  const int n = ra.n[m];
  double2* T = tpool + ra.off[m];
  double2* U = upool + ra.off[m];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (n > kReorderMaxN || ra.nrad[m] <= 0) return;
  // target position of the eigenvalue now at position p: its rank s, digits of s over the reversed
  // radices (most significant = the within-block digit), recomposed over the radices
  for (int p = tid; p < n; p += nt) {
    const double2 lp = T[p + (int64_t)p * n];
    int srank = 0;
    for (int q = 0; q < n; ++q) {
      const double2 lq = T[q + (int64_t)q * n];
      srank += (lq.x < lp.x) || (lq.x == lp.x && (lq.y < lp.y || (lq.y == lp.y && q < p)));
    }
    int rem = srank, pos = 0, place = 1;
    // weights of R: digit i has weight prod_{k > i} r_k; peel from the most significant (i = 0)
    int wt = 1;
    for (int i = 1; i < ra.nrad[m]; ++i) wt *= ra.rad[m][i];
    for (int i = 0; i < ra.nrad[m]; ++i) {
      const int d = rem / wt;
      rem -= d * wt;
      pos += d * place;
      place *= ra.rad[m][i];
      if (i + 1 < ra.nrad[m]) wt /= ra.rad[m][i + 1];
    }
    key[p] = pos;
  }
  __syncthreads();
  for (int round = 0; round < n; ++round) {
    const int par = round & 1, np = (n - par) / 2;
    for (int i = tid; i < np; i += nt) {  // 1. rotations of the out-of-order pairs
      const int k = par + 2 * i;
      const bool sw = key[k] > key[k + 1];
      act[i] = sw;
      if (sw) {
        const double2 t11 = T[k + (int64_t)k * n], t22 = T[(k + 1) + (int64_t)(k + 1) * n];
        double cs;
        double2 sn;
        zlartg_dev(T[k + (int64_t)(k + 1) * n], csub(t22, t11), cs, sn);
        rc[i] = cs;
        rs[i] = sn;
      }
    }
    __syncthreads();
    // 2. rows k, k+1, columns > k+1: (x, y) <- (c x + s y, c y - conj(s) x)
    for (int64_t e = tid; e < (int64_t)np * n; e += nt) {
      const int i = (int)(e / n), j = (int)(e % n), k = par + 2 * i;
      if (!act[i] || j <= k + 1) continue;
      const double c = rc[i];
      const double2 sv = rs[i];
      const double2 x = T[k + (int64_t)j * n], y = T[(k + 1) + (int64_t)j * n];
      T[k + (int64_t)j * n] = cadd(make_double2(c * x.x, c * x.y), cmul(sv, y));
      T[(k + 1) + (int64_t)j * n] = csub(make_double2(c * y.x, c * y.y), cmul(make_double2(sv.x, -sv.y), x));
    }
    __syncthreads();
    // 3. columns k, k+1 of T (rows < k) and of U (all rows) with (c, conj(s)); the diagonal swap
    for (int64_t e = tid; e < (int64_t)np * n; e += nt) {
      const int i = (int)(e / n), r = (int)(e % n), k = par + 2 * i;
      if (!act[i]) continue;
      const double c = rc[i];
      const double2 sc = make_double2(rs[i].x, -rs[i].y);  // conj(s)
      if (r < k) {
        const double2 x = T[r + (int64_t)k * n], y = T[r + (int64_t)(k + 1) * n];
        T[r + (int64_t)k * n] = cadd(make_double2(c * x.x, c * x.y), cmul(sc, y));
        T[r + (int64_t)(k + 1) * n] = csub(make_double2(c * y.x, c * y.y), cmul(make_double2(sc.x, -sc.y), x));
      }
      {
        const double2 x = U[r + (int64_t)k * n], y = U[r + (int64_t)(k + 1) * n];
        U[r + (int64_t)k * n] = cadd(make_double2(c * x.x, c * x.y), cmul(sc, y));
        U[r + (int64_t)(k + 1) * n] = csub(make_double2(c * y.x, c * y.y), cmul(make_double2(sc.x, -sc.y), x));
      }
      if (r == 0) {
        const double2 t11 = T[k + (int64_t)k * n];
        T[k + (int64_t)k * n] = T[(k + 1) + (int64_t)(k + 1) * n];
        T[(k + 1) + (int64_t)(k + 1) * n] = t11;
        const int kk = key[k];
        key[k] = key[k + 1];
        key[k + 1] = kk;
      }
    }
    __syncthreads();
  }
}

// The same sort spread over C CTAs per mode (one cooperative launch, every mode's CTAs in
// lockstep): each CTA keeps the keys and computes every pair's rotation itself (redundantly, from
// T's diagonal and superdiagonal), applies the row rotations to its own slice of columns and,
// after a grid barrier, the column rotations to its own slice of rows of T and U. Two grid
// barriers per round instead of one CTA sweeping the whole n x n per phase (c1, n = 256: 13.5 ms
// on one CTA per mode).
__device__ __forceinline__ void reorder_grid_barrier(unsigned int* bar, unsigned int& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}
__global__ void __launch_bounds__(256) schur_reorder_coop_kernel(const ReorderArgs ra, int C, int nmax,
                                                                 double2* __restrict__ tpool,
                                                                 double2* __restrict__ upool,
                                                                 unsigned int* __restrict__ bar) {
  __shared__ int key[kReorderMaxN];
  __shared__ int act[kReorderMaxN / 2];
  __shared__ double rc[kReorderMaxN / 2];
  __shared__ double2 rs[kReorderMaxN / 2];
  const int m = blockIdx.x / C, c = blockIdx.x % C;
  const int n = ra.n[m];
  const bool live = n <= kReorderMaxN && ra.nrad[m] > 0;
  double2* T = tpool + ra.off[m];
  double2* U = upool + ra.off[m];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int s0 = (int)((int64_t)n * c / C), s1 = (int)((int64_t)n * (c + 1) / C);  // this CTA's slice
  unsigned int target = 0;
  if (live)
    for (int p = tid; p < n; p += nt) {
      const double2 lp = T[p + (int64_t)p * n];
      int srank = 0;
      for (int q = 0; q < n; ++q) {
        const double2 lq = T[q + (int64_t)q * n];
        srank += (lq.x < lp.x) || (lq.x == lp.x && (lq.y < lp.y || (lq.y == lp.y && q < p)));
      }
      int rem = srank, pos = 0, place = 1, wt = 1;
      for (int i = 1; i < ra.nrad[m]; ++i) wt *= ra.rad[m][i];
      for (int i = 0; i < ra.nrad[m]; ++i) {
        const int d = rem / wt;
        rem -= d * wt;
        pos += d * place;
        place *= ra.rad[m][i];
        if (i + 1 < ra.nrad[m]) wt /= ra.rad[m][i + 1];
      }
      key[p] = pos;
    }
  __syncthreads();
  for (int round = 0; round < nmax; ++round) {
    const int par = round & 1;
    const int np = live && round < n ? (n - par) / 2 : 0;
    for (int i = tid; i < np; i += nt) {  // every pair's rotation (T's diagonal: final since the last barrier)
      const int k = par + 2 * i;
      const bool sw = key[k] > key[k + 1];
      act[i] = sw;
      if (sw) {
        const double2 t11 = T[k + (int64_t)k * n], t22 = T[(k + 1) + (int64_t)(k + 1) * n];
        double cs;
        double2 sn;
        zlartg_dev(T[k + (int64_t)(k + 1) * n], csub(t22, t11), cs, sn);
        rc[i] = cs;
        rs[i] = sn;
      }
    }
    __syncthreads();
    // rows k, k+1 over this CTA's columns j in [s0, s1), j > k+1
    const int w = s1 - s0;
    for (int64_t e = tid; e < (int64_t)np * w; e += nt) {
      const int i = (int)(e / w), j = s0 + (int)(e % w), k = par + 2 * i;
      if (!act[i] || j <= k + 1) continue;
      const double cc = rc[i];
      const double2 sv = rs[i];
      const double2 x = T[k + (int64_t)j * n], y = T[(k + 1) + (int64_t)j * n];
      T[k + (int64_t)j * n] = cadd(make_double2(cc * x.x, cc * x.y), cmul(sv, y));
      T[(k + 1) + (int64_t)j * n] = csub(make_double2(cc * y.x, cc * y.y), cmul(make_double2(sv.x, -sv.y), x));
    }
    reorder_grid_barrier(bar, target);
    // columns k, k+1 over this CTA's rows r in [s0, s1): T (r < k) and U; the diagonal swap by the
    // owner of row k
    for (int64_t e = tid; e < (int64_t)np * w; e += nt) {
      const int i = (int)(e / w), r = s0 + (int)(e % w), k = par + 2 * i;
      if (!act[i]) continue;
      const double cc = rc[i];
      const double2 sc = make_double2(rs[i].x, -rs[i].y);  // conj(s)
      if (r < k) {
        const double2 x = T[r + (int64_t)k * n], y = T[r + (int64_t)(k + 1) * n];
        T[r + (int64_t)k * n] = cadd(make_double2(cc * x.x, cc * x.y), cmul(sc, y));
        T[r + (int64_t)(k + 1) * n] = csub(make_double2(cc * y.x, cc * y.y), cmul(make_double2(sc.x, -sc.y), x));
      }
      {
        const double2 x = U[r + (int64_t)k * n], y = U[r + (int64_t)(k + 1) * n];
        U[r + (int64_t)k * n] = cadd(make_double2(cc * x.x, cc * x.y), cmul(sc, y));
        U[r + (int64_t)(k + 1) * n] = csub(make_double2(cc * y.x, cc * y.y), cmul(make_double2(sc.x, -sc.y), x));
      }
      if (r == k) {
        const double2 t11 = T[k + (int64_t)k * n];
        T[k + (int64_t)k * n] = T[(k + 1) + (int64_t)(k + 1) * n];
        T[(k + 1) + (int64_t)(k + 1) * n] = t11;
      }
    }
    for (int i = tid; i < np; i += nt)  // every CTA tracks the keys itself
      if (act[i]) {
        const int k = par + 2 * i;
        const int kk = key[k];
        key[k] = key[k + 1];
        key[k + 1] = kk;
      }
    reorder_grid_barrier(bar, target);
  }
}

void schur_reorder_launch(const ReorderArgs& ra, int n_modes, double2* tpool, double2* upool, unsigned int* bar,
                          cudaStream_t stream) {
  int nmax = 0;
  for (int m = 0; m < n_modes; ++m)
    if (ra.nrad[m] > 0) nmax = std::max(nmax, ra.n[m]);
  if (nmax == 0) return;
  // slices of >= 16 rows / columns, at most 16 CTAs per mode; all CTAs co-resident (cooperative)
  int C = std::max(1, std::min(16, nmax / 16));
  int dev = 0, sms = 0;
  NDS_CUDA(cudaGetDevice(&dev));
  NDS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  while (C > 1 && n_modes * C > sms) --C;
  if (n_modes * C > sms) {  // more modes than SMs: one CTA per mode, no grid barrier
    schur_reorder_kernel<<<(unsigned)n_modes, 1024, 0, stream>>>(ra, tpool, upool);
    NDS_LAUNCH_CHECK();
    return;
  }
  NDS_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned int), stream));
  ReorderArgs a = ra;
  void* args[] = {&a, &C, &nmax, &tpool, &upool, &bar};
  NDS_CUDA(cudaLaunchCooperativeKernel((const void*)schur_reorder_coop_kernel, n_modes * C, 256, args, 0, stream));
}

__global__ void diag_extract_kernel(const Geom g, const double2* __restrict__ t, double2* __restrict__ diag) {
  const int m = blockIdx.y;
  const int64_t n = g.dims[m];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    diag[g.doff[m] + i] = t[g.toff[m] + i * (n + 1)];
}

void diag_extract_launch(const Geom& g, const double2* t_pool, double2* diag, cudaStream_t stream) {
  diag_extract_kernel<<<dim3(4, (unsigned)g.n_modes), 256, 0, stream>>>(g, t_pool, diag);
  NDS_LAUNCH_CHECK();
}

__global__ void param_blob_kernel(const ParamBlob b, double2* __restrict__ dst) {
  for (int i = threadIdx.x; i < b.count; i += blockDim.x) dst[i] = b.v[i];
}

void param_blob_launch(const ParamBlob& blob, double2* dst, cudaStream_t stream) {
  if (blob.count <= 0) return;
  param_blob_kernel<<<1, 256, 0, stream>>>(blob, dst);
  NDS_LAUNCH_CHECK();
}

// out_y = A_y blockdiag(B_y) for y = blockIdx.y (up to three products of one mode per launch):
// out(r, c) = sum_{k in block(c)} A(r, o + k) B_q(k, c - o), B_q or B_q^H (conj).
struct BdRight {
  int count;
  const double2* a[3];
  const double2* blk[3];
  int conj[3];
  double2* out[3];
};
__global__ void blockdiag_right_kernel(int64_t n, int d, const BdRight j) {
  const int y = blockIdx.y;
  const double2* __restrict__ a = j.a[y];
  const double2* __restrict__ blk = j.blk[y];
  const bool conj_t = j.conj[y] != 0;
  double2* __restrict__ out = j.out[y];
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % n, c = e / n;
    const int64_t q = c / d, o = q * d, cc = c - o;
    const double2* bq = blk + q * (int64_t)d * d;
    double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
    for (int k = 0; k < d; k += 2) {  // d even
      double2 b0 = conj_t ? bq[cc + k * d] : bq[k + cc * d];
      double2 b1 = conj_t ? bq[cc + (k + 1) * d] : bq[k + 1 + cc * d];
      if (conj_t) {
        b0.y = -b0.y;
        b1.y = -b1.y;
      }
      s0 = cfma(s0, a[r + (o + k) * n], b0);
      s1 = cfma(s1, a[r + (o + k + 1) * n], b1);
    }
    out[e] = cadd(s0, s1);
  }
}

// T' = blockdiag(W_q) TV with the route's structure imposed: entries of a diagonal d-block are
// diag(T) exactly (off-diagonal 0), entries below the block diagonal 0.
__global__ void blockdiag_left_fix_kernel(int64_t n, int d, const double2* __restrict__ w, const double2* __restrict__ tv,
                                          const double2* __restrict__ t, double2* __restrict__ out) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % n, c = e / n;
    const int64_t qr = r / d, qc = c / d;
    if (qr == qc) {
      out[e] = r == c ? t[e] : make_double2(0.0, 0.0);
      continue;
    }
    if (qr > qc) {
      out[e] = make_double2(0.0, 0.0);
      continue;
    }
    const int64_t o = qr * d;
    const double2* wq = w + qr * (int64_t)d * d;
    double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
    for (int k = (int)(r - o); k < d; k += 2) {  // W_q upper triangular: columns k >= r - o
      s0 = cfma(s0, wq[(r - o) + k * d], tv[(o + k) + c * n]);
      if (k + 1 < d) s1 = cfma(s1, wq[(r - o) + (k + 1) * d], tv[(o + k + 1) + c * n]);
    }
    out[e] = cadd(s0, s1);
  }
}

void blockdiag_factors_launch(int64_t n, int d, const double2* u, const double2* t, const double2* v, const double2* w,
                              double2* minv, double2* mfh, double2* tv, double2* tprime, cudaStream_t stream) {
  const int64_t total = n * n;
  const unsigned gx = (unsigned)std::min<int64_t>((total + 255) / 256, 2048);
  BdRight j{3, {u, u, t}, {v, w, v}, {0, 1, 0}, {minv, mfh, tv}};
  blockdiag_right_kernel<<<dim3(gx, 3), 256, 0, stream>>>(n, d, j);
  NDS_LAUNCH_CHECK();
  blockdiag_left_fix_kernel<<<gx, 256, 0, stream>>>(n, d, w, tv, t, tprime);
  NDS_LAUNCH_CHECK();
}

}  // namespace nds
