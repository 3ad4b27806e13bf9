// exp(t T_j) for the ODE propagator on the device: the Parlett recurrence of triangular_exp
// (reference schur.cpp:212-226) for every mode with a well-separated diagonal, one thread-block
// cluster per mode.
//
// Superdiagonal p of F depends only on superdiagonals < p, so the cluster sweeps p = 1 .. n-1 with
// a barrier per step; within a step every entry (i, i + p) is a group of lanes that split
// sum_{i<k<j} S_ik F_kj - F_ik S_kj, a shuffle tree combines them, lane 0 forms
//   F_ij = [S_ij (F_jj - F_ii) + sum] / (S_jj - S_ii)
// with the reference's complex division (cdiv). S = t T is formed on the fly. F is written
// straight into the two layouts the mode-product GEMM reads (row-major | column-major); the
// column-major copy doubles as the working storage. Summation order differs from the
// reference's sequential k loop (round-off only; the host restatement in matfun.cpp keeps it).
#include "common.cuh"
#include "kernels.h"

namespace nds {

namespace {

__device__ __forceinline__ double2 cexp_dev(double2 z) {
  double s, c;
  sincos(z.y, &s, &c);
  const double e = exp(z.x);
  return make_double2(e * c, e * s);
}

// One thread-block CLUSTER of kParlettCta CTAs per mode (grid = modes x kParlettCta): the
// entries of a superdiagonal are spread over the cluster's CTAs and the per-step barrier is the
// cluster barrier (release / acquire at cluster scope orders the F stores in global memory);
// F written by other CTAs is read through L2 (__ldcg).
constexpr int kParlettCta = 8;  // 16 (non-portable) measured no faster: latency-bound per step

__global__ void __cluster_dims__(kParlettCta, 1, 1) __launch_bounds__(1024) parlett_kernel(const ExpArgs a) {
  const int rank = blockIdx.x % kParlettCta;
  const int m = a.mode[blockIdx.x / kParlettCta];
  const int n = (int)a.n[blockIdx.x / kParlettCta];
  const double2* T = a.t_pool + a.toff[m];     // column-major
  const double2* Tr = a.t_row + a.foff[m] / 2;  // row-major copy
  double2* Frow = a.f + a.foff[m];
  double2* F = Frow + (int64_t)n * n;  // column-major
  const double2 tc = make_double2(a.t, 0.0);
  const int tid = threadIdx.x, nt = blockDim.x;
  auto cluster_sync = [] {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  };
  for (int64_t e = (int64_t)rank * nt + tid; e < (int64_t)n * n; e += (int64_t)nt * kParlettCta) {
    const int i = (int)(e % n), k = (int)(e / n);  // strict lower part 0, diagonal exp(S_ii)
    double2 v = make_double2(0.0, 0.0);
    if (i == k) v = cexp_dev(cmul(__ldg(T + e), tc));
    F[e] = v;
    Frow[(int64_t)i * n + k] = v;
  }
  cluster_sync();
  for (int p = 1; p < n; ++p) {
    // lanes per entry: a power of two giving each lane ~4 of the p - 1 terms (all reads coalesced:
    // S_ik, F_ik from the row-major copies, F_kj, S_kj from the column-major ones)
    int lpe = 1;
    while (lpe < 32 && lpe * 4 < p - 1) lpe <<= 1;
    const int sub = tid & (lpe - 1), grp = tid / lpe, ngrp = nt / lpe;
    const int per_pass = ngrp * kParlettCta;
    for (int base = 0; base < n - p; base += per_pass) {  // warp-uniform trip count (shuffles below)
      const int i = base + grp * kParlettCta + rank, j = i + p;
      const bool active = j < n;
      double2 tail_sij{}, tail_sii{}, tail_sjj{}, tail_fii{}, tail_fjj{};
      if (active && sub == 0) {  // the lane-0 operands, issued before the dot product
        tail_sij = __ldg(T + i + (int64_t)j * n);
        tail_sii = __ldg(T + i + (int64_t)i * n);
        tail_sjj = __ldg(T + j + (int64_t)j * n);
        tail_fii = __ldcg(F + i + (int64_t)i * n);
        tail_fjj = __ldcg(F + j + (int64_t)j * n);
      }
      double2 acc = make_double2(0.0, 0.0);
      if (active) {
        const double2* tri = Tr + (int64_t)i * n;
        const double2* fri = Frow + (int64_t)i * n;
        const double2* fcj = F + (int64_t)j * n;
        const double2* tcj = T + (int64_t)j * n;
        for (int k = i + 1 + sub; k < j; k += lpe)
          acc = cadd(acc, csub(cmul(cmul(__ldg(tri + k), tc), __ldcg(fcj + k)),
                               cmul(__ldcg(fri + k), cmul(__ldg(tcj + k), tc))));
      }
      for (int o = lpe >> 1; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (active && sub == 0) {
        const double2 sij = cmul(tail_sij, tc), sii = cmul(tail_sii, tc), sjj = cmul(tail_sjj, tc);
        const double2 v = cdiv(cadd(cmul(sij, csub(tail_fjj, tail_fii)), acc), csub(sjj, sii));
        F[i + (int64_t)j * n] = v;
        Frow[(int64_t)i * n + j] = v;
      }
    }
    cluster_sync();
  }
}

}  // namespace

int parlett_launch(const ExpArgs& a, int count, cudaStream_t stream) {
  if (count <= 0) return 0;
  parlett_kernel<<<count * kParlettCta, 1024, 0, stream>>>(a);
  NDS_LAUNCH_CHECK();
  return 1;
}

}  // namespace nds
