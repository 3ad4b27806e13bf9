// Device side of the block-diagonalised cubic route's plan (capi.cu plan_cubic_diag): the
// eigenvector matrices of the D x D diagonal blocks of every T_j for every candidate D, their
// inverses and condition numbers (one launch), and the merged factors U W, U W^{-H} and
// T' = W^{-1} T W of the chosen D (block-diagonal matrix products).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace nds {

// One CTA per job (block q of mode j at candidate extent d, d <= blockDim.x), thread k <-> column k.
//  1. V(:, k): the eigenvector of the upper triangular block T_q for T_q(k, k), V(k, k) = 1,
//     V(i, k) = sum_{l = i+1..k} T(i, l) V(l, k) / (T(k, k) - T(i, i)), then unit 2-norm;
//  2. W = V^{-1} (upper triangular): column c by back substitution;
//  3. cond_2(V) = ||V||_2 ||W||_2, both by 12 power iterations on M^H M (shared vectors).
// A zero eigenvalue gap (repeated eigenvalue) or a non-finite entry makes cond infinite.
__global__ void __launch_bounds__(128) block_eig_kernel(const double2* __restrict__ t_pool,
                                                        const EigJob* __restrict__ jobs, double2* __restrict__ vpool,
                                                        double2* __restrict__ wpool, double* __restrict__ cond) {
  const EigJob jb = jobs[blockIdx.x];
  const int d = jb.d, k = threadIdx.x;
  const int64_t n = jb.n, o = jb.o;
  const double2* T = t_pool + jb.toff;
  auto Tq = [&](int r, int c) { return T[(o + r) + (o + c) * n]; };
  double2* V = vpool + jb.voff;  // column-major d x d
  double2* W = wpool + jb.voff;
  __shared__ int bad;
  __shared__ double2 x[128], y[128];
  __shared__ double red[4];
  if (k == 0) bad = 0;
  __syncthreads();
  if (k < d) {
    double2* vk = V + (int64_t)k * d;
    for (int i = k + 1; i < d; ++i) vk[i] = make_double2(0.0, 0.0);
    vk[k] = make_double2(1.0, 0.0);
    const double2 lk = Tq(k, k);
    double nn = 1.0;
    for (int i = k - 1; i >= 0; --i) {
      double2 acc = make_double2(0.0, 0.0);
      for (int l = i + 1; l <= k; ++l) acc = cfma(acc, Tq(i, l), vk[l]);
      const double2 gap = csub(lk, Tq(i, i));
      if (gap.x == 0.0 && gap.y == 0.0) {
        bad = 1;
        break;
      }
      const double2 vi = cdiv(acc, gap);
      vk[i] = vi;
      nn += vi.x * vi.x + vi.y * vi.y;
    }
    nn = sqrt(nn);
    if (!isfinite(nn)) bad = 1;
    const double s = 1.0 / nn;
    for (int i = 0; i <= k; ++i) vk[i] = make_double2(vk[i].x * s, vk[i].y * s);
  }
  __syncthreads();
  if (k < d) {  // W(:, c), c = k: W(c, c) = 1 / V(c, c); W(i, c) = -sum_{l=i+1..c} V(i, l) W(l, c) / V(i, i)
    double2* wc = W + (int64_t)k * d;
    for (int i = k + 1; i < d; ++i) wc[i] = make_double2(0.0, 0.0);
    for (int i = k; i >= 0; --i) {
      double2 acc = make_double2(i == k ? 1.0 : 0.0, 0.0);
      for (int l = i + 1; l <= k; ++l) acc = csub(acc, cmul(V[i + (int64_t)l * d], wc[l]));
      wc[i] = cdiv(acc, V[i + (int64_t)i * d]);
    }
  }
  __syncthreads();
  double nrm[2];
  for (int which = 0; which < 2; ++which) {
    const double2* M = which ? W : V;
    if (k < d) x[k] = make_double2(1.0 + 0.37 * k, 0.11 * (k % 5));
    __syncthreads();
    double lam = 0.0;
    for (int it = 0; it < 12; ++it) {
      if (k < d) {  // y = M x (row k)
        double2 s = make_double2(0.0, 0.0);
        for (int c = k; c < d; ++c) s = cfma(s, M[k + (int64_t)c * d], x[c]);
        y[k] = s;
      }
      __syncthreads();
      double part = 0.0;
      double2 xn = make_double2(0.0, 0.0);
      if (k < d) {  // x = M^H y (column k)
        for (int r = 0; r <= k; ++r) {
          const double2 m = M[r + (int64_t)k * d];
          xn = cfma(xn, make_double2(m.x, -m.y), y[r]);
        }
        part = xn.x * xn.x + xn.y * xn.y;
      }
      for (int sh = 16; sh > 0; sh >>= 1) part += __shfl_xor_sync(0xffffffffu, part, sh);
      if ((k & 31) == 0) red[k >> 5] = part;
      __syncthreads();
      const double tot = sqrt(red[0] + red[1] + red[2] + red[3]);
      lam = tot;
      if (k < d) x[k] = make_double2(xn.x / tot, xn.y / tot);
      __syncthreads();
    }
    nrm[which] = sqrt(lam);
  }
  if (k == 0) {
    const double c = nrm[0] * nrm[1];
    cond[blockIdx.x] = (bad || !isfinite(c)) ? INFINITY : c;
  }
}

void block_eig_launch(const double2* t_pool, const EigJob* jobs, int njobs, double2* vpool, double2* wpool,
                      double* cond, cudaStream_t stream) {
  if (njobs <= 0) return;
  block_eig_kernel<<<(unsigned)njobs, 128, 0, stream>>>(t_pool, jobs, vpool, wpool, cond);
  NDS_LAUNCH_CHECK();
}

__global__ void blockdiag_mul_kernel(int64_t n, int d, const double2* __restrict__ a, const double2* __restrict__ blk,
                                     int right, int conj_t, double2* __restrict__ out) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % n, c = e / n;
    const int64_t q = (right ? c : r) / d, o = q * d;
    const double2* bq = blk + q * (int64_t)d * d;
    auto bel = [&](int64_t i, int64_t k) {  // Bq(i, k) or Bq^H(i, k)
      if (!conj_t) return bq[i + k * d];
      const double2 v = bq[k + i * d];
      return make_double2(v.x, -v.y);
    };
    double2 s = make_double2(0.0, 0.0);
    if (right)
      for (int k = 0; k < d; ++k) s = cfma(s, a[r + (o + k) * n], bel(k, c - o));
    else
      for (int k = 0; k < d; ++k) s = cfma(s, bel(r - o, k), a[(o + k) + c * n]);
    out[e] = s;
  }
}

__global__ void blockdiag_fix_kernel(int64_t n, int d, const double2* __restrict__ diag_src, double2* __restrict__ t) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % n, c = e / n;
    if (r / d == c / d)
      t[e] = r == c ? diag_src[e] : make_double2(0.0, 0.0);
    else if (r / d > c / d)
      t[e] = make_double2(0.0, 0.0);
  }
}

void blockdiag_mul_launch(int64_t n, int d, const double2* a, const double2* blk, bool right, bool conj_t,
                          double2* out, cudaStream_t stream) {
  const int64_t total = n * n;
  blockdiag_mul_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, stream>>>(
      n, d, a, blk, right ? 1 : 0, conj_t ? 1 : 0, out);
  NDS_LAUNCH_CHECK();
}

void blockdiag_fix_launch(int64_t n, int d, const double2* diag_src, double2* t, cudaStream_t stream) {
  const int64_t total = n * n;
  blockdiag_fix_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, stream>>>(n, d, diag_src, t);
  NDS_LAUNCH_CHECK();
}

}  // namespace nds
