// Mode-j tensor-times-matrix (TTM) kernels for the forward / inverse transforms
// (reference: kernels.cpp:24-44 mode_product_impl, driven by sylvester.cpp:55-69).
//
// On the column-major (inner, n, outer) view of mode j (kernels.cpp:9-21) the product
//   R[a, i, b] = sum_k M[i, k] X[a, k, b]
// is a strided-batched complex GEMM with no permutation pass:
//   * inner >= 8  ("ROWM"): C(i, c) = M(i, :) . X(:, c), columns c = (a, b) read straight from the
//     tensor's native strides, a contiguous;
//   * inner == 1  ("COLM", mode 1): C(b, i) = X(b, :) . M^T(:, i), rows of X contiguous in k;
//   * otherwise (tiny inner, e.g. n_1 < 8): a direct kernel.
// The GEMM runs on the FP64 tensor pipe (DMMA, mma.sync.m8n8k4.f64): measured 37.1 TF on B200
// vs 34.1 TF for DFMA (tools/microbench/fp64_peaks.cu, profiles/). Complex products use the
// 3-multiplication form: per 8x8x4 block three real DMMAs Ar Br, Ai Bi, (Ar + Ai)(Br + Bi), with
// Re = p1 - p2 and Im = p3 - p1 - p2 (6 of the 8 real flops of a complex MAC); tiles are staged
// global->shared with a multi-stage cp.async pipeline into bank-conflict-free padded layouts
// (row strides = 4 resp. 2 mod 8 complex for the DMMA fragment pattern).
#include <cstdlib>

#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace nds {

// ------------------------------------------------------------------------------------------
// Direct kernel: one output entry per thread. Used for 1 < inner < 8 or tiny n.
// ------------------------------------------------------------------------------------------
// r (extent m along the mode) = M (m x n, column-major) x_mode x (extent n).
__global__ void mode_product_direct_kernel(const double2* __restrict__ mcol, int64_t inner, int n, int m,
                                           int64_t outer, const double2* __restrict__ x, double2* __restrict__ r,
                                           int accumulate) {
  const int64_t total = inner * m * outer;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = idx % inner;
    const int64_t t = idx / inner;
    const int i = (int)(t % m);
    const int64_t b = t / m;
    const double2* xp = x + b * n * inner + a;
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < n; ++k) s = cfma(s, __ldg(mcol + i + (int64_t)k * m), __ldg(xp + (int64_t)k * inner));
    if (accumulate) s = cadd(r[idx], s);
    r[idx] = s;
  }
}

// ------------------------------------------------------------------------------------------
// DMMA complex GEMM
// ------------------------------------------------------------------------------------------
struct GemmArgs {
  const double2* A;  // A(r, k) = A[r * lda + k]
  int64_t lda;
  int64_t rows;      // rows of A and C
  const double2* B;  // B(k, a, b) = B[k * ldbk + a + b * ldbb]
  int64_t ldbk, ldbb;
  double2* C;        // C(r, a, b) = C[r * ldcr + a + b * ldcb]
  int64_t ldcr, ldcb;
  int K;
  int wshift;        // tile column c = a' + (b' << wshift)
  int64_t alim, blim;
  int64_t ntile_rows, ntile_a;
  int accumulate;
  // bulk-copy (TMA) path: stage-blocked image of the constant operand (ROWM: A, COLM: B) for the
  // chosen CTA shape, or null; colm = the mode-1 form (A = the tensor, B = M^T)
  const double2* blk;
  const double2* blk_shape[2];
  int colm;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct GemmCfg {
  static constexpr int kThreads = WM * WN * 32;
  static constexpr int kLdA = BK + 4;  // complex; = 4 mod 8 -> conflict-free A fragments
  static constexpr int kLdB = BN + 2;  // complex; = 2 mod 8 -> conflict-free B fragments
  static constexpr int kStageA = BM * kLdA;
  static constexpr int kStageB = BK * kLdB;
  static constexpr size_t kSmem = (size_t)STAGES * (kStageA + kStageB) * sizeof(double2);
  static constexpr int MI = BM / WM / 8;
  static constexpr int NI = BN / WN / 8;
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool M3, int MINB = 1>
__global__ void __launch_bounds__(WM* WN * 32, MINB) zgemm_dmma_kernel(const GemmArgs g) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  constexpr int NT = Cfg::kThreads;
  constexpr int MI = Cfg::MI, NI = Cfg::NI;
  extern __shared__ __align__(16) double2 smem[];
  double2* sA = smem;
  double2* sB = smem + STAGES * Cfg::kStageA;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wy = warp / WN, wx = warp % WN;

  const int64_t tile = blockIdx.x;
  const int64_t row_tile = tile % g.ntile_rows;
  const int64_t col_tile = tile / g.ntile_rows;
  const int64_t row0 = row_tile * BM;
  const int64_t a0 = (col_tile % g.ntile_a) << g.wshift;
  const int64_t b0 = (col_tile / g.ntile_a) * (BN >> g.wshift);
  const int wmask = (1 << g.wshift) - 1;

  auto load_stage = [&](int stage, int k0) {
    double2* dA = sA + stage * Cfg::kStageA;
    double2* dB = sB + stage * Cfg::kStageB;
#pragma unroll
    for (int e = tid; e < BM * BK; e += NT) {
      const int r = e / BK, k = e % BK;
      const int64_t gr = row0 + r;
      const int gk = k0 + k;
      const bool ok = gr < g.rows && gk < g.K;
      const double2* src = ok ? g.A + gr * g.lda + gk : g.A;
      cp_async16(dA + r * Cfg::kLdA + k, src, ok ? 16 : 0);
    }
#pragma unroll
    for (int e = tid; e < BK * BN; e += NT) {
      const int c = e % BN, k = e / BN;
      const int64_t ga = a0 + (c & wmask);
      const int64_t gb = b0 + (c >> g.wshift);
      const int gk = k0 + k;
      const bool ok = gk < g.K && ga < g.alim && gb < g.blim;
      const double2* src = ok ? g.B + (int64_t)gk * g.ldbk + ga + gb * g.ldbb : g.B;
      cp_async16(dB + k * Cfg::kLdB + c, src, ok ? 16 : 0);
    }
  };

  // 4M: cre, cim. 3M (Karatsuba): cre = Ar Br, cim = Ai Bi, c3 = (Ar + Ai)(Br + Bi);
  // Re = cre - cim, Im = c3 - cre - cim (3 real DMMAs per complex 8x8x4 block instead of 4).
  double cre[MI][NI][2], cim[MI][NI][2], c3[M3 ? MI : 1][M3 ? NI : 1][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) cre[mi][ni][0] = cre[mi][ni][1] = cim[mi][ni][0] = cim[mi][ni][1] = 0.0;
  if constexpr (M3) {
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) c3[mi][ni][0] = c3[mi][ni][1] = 0.0;
  }

  const int nk = (g.K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s * BK);
    cp_async_commit();
  }

  const int arow = wy * (BM / WM) + (lane >> 2);
  const int bcol = wx * (BN / WN) + (lane >> 2);
  const int kq = lane & 3;

  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt % STAGES, nxt * BK);
      cp_async_commit();
    }
    const double2* cA = sA + (kt % STAGES) * Cfg::kStageA;
    const double2* cB = sB + (kt % STAGES) * Cfg::kStageB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[MI], ai[MI], an[MI], br[NI], bi[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const double2 v = cA[(arow + mi * 8) * Cfg::kLdA + kk + kq];
        ar[mi] = v.x;
        ai[mi] = v.y;
        an[mi] = M3 ? v.x + v.y : -v.y;  // 3M: Ar + Ai; 4M: -Ai
      }
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const double2 v = cB[(kk + kq) * Cfg::kLdB + bcol + ni * 8];
        br[ni] = v.x;
        bi[ni] = v.y;
      }
      if constexpr (M3) {
        double bs[NI];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) bs[ni] = br[ni] + bi[ni];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            dmma(cre[mi][ni][0], cre[mi][ni][1], ar[mi], br[ni]);
            dmma(cim[mi][ni][0], cim[mi][ni][1], ai[mi], bi[ni]);
            dmma(c3[mi][ni][0], c3[mi][ni][1], an[mi], bs[ni]);
          }
      } else {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            dmma(cre[mi][ni][0], cre[mi][ni][1], ar[mi], br[ni]);
            dmma(cim[mi][ni][0], cim[mi][ni][1], ar[mi], bi[ni]);
            dmma(cre[mi][ni][0], cre[mi][ni][1], an[mi], bi[ni]);
            dmma(cim[mi][ni][0], cim[mi][ni][1], ai[mi], br[ni]);
          }
      }
    }
  }
  cp_async_wait<0>();

  // Epilogue: lane holds C[r][2q], C[r][2q+1] of each 8x8 fragment.
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int64_t r = row0 + wy * (BM / WM) + mi * 8 + (lane >> 2);
    if (r >= g.rows) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int c = wx * (BN / WN) + ni * 8 + 2 * kq;
      const int64_t ga = a0 + (c & wmask);
      const int64_t gb = b0 + (c >> g.wshift);
      if (gb >= g.blim) continue;
      double2* dst = g.C + r * g.ldcr + ga + gb * g.ldcb;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (ga + h < g.alim) {
          double2 v;
          if constexpr (M3)
            v = make_double2(cre[mi][ni][h] - cim[mi][ni][h], c3[mi][ni][h] - cre[mi][ni][h] - cim[mi][ni][h]);
          else
            v = make_double2(cre[mi][ni][h], cim[mi][ni][h]);
          if (g.accumulate) v = cadd(dst[h], v);
          dst[h] = v;
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// The same GEMM fed by bulk asynchronous copies (TMA engine, cp.async.bulk) into an mbarrier
// ring: per stage ONE copy of the constant operand's stage image (FactorSet::ablk / bblk: the
// padded, bank-conflict-free layout precomputed per factor) plus one copy per contiguous run of
// the tensor operand (ROWM: BK rows of W entries per column group; COLM: BM rows of BK entries).
// Warp 0 is also the producer: at the top of k-tile kt its lanes refill the stage k-tile kt - 1
// used (after every warp released it on the stage's empty barrier), so each stage is in flight
// for STAGES - 1 k-tiles; consumers wait on the stage's full barrier (expect-tx byte count) —
// no per-thread cp.async address work and no CTA-wide barrier per stage. Needs K % BK == 0 and
// whole column groups (inner % W == 0); other GEMMs take zgemm_dmma_kernel.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB, bool DF = false>
__global__ void __launch_bounds__(WM* WN * 32, MINB) zgemm_tma_kernel(const GemmArgs g, int colm) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  constexpr int NW = WM * WN;
  constexpr int MI = Cfg::MI, NI = Cfg::NI;
  extern __shared__ __align__(16) double2 smem[];
  double2* sA = smem;
  double2* sB = smem + STAGES * Cfg::kStageA;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wy = warp / WN, wx = warp % WN;
  const int64_t tile = blockIdx.x;
  const int64_t row_tile = tile % g.ntile_rows;
  const int64_t col_tile = tile / g.ntile_rows;
  const int64_t row0 = row_tile * BM;
  const int64_t a0 = (col_tile % g.ntile_a) << g.wshift;
  const int64_t b0 = (col_tile / g.ntile_a) * (BN >> g.wshift);
  const int W = 1 << g.wshift;
  const int groups = BN >> g.wshift;
  const int gshift = __popc(BN - 1) - g.wshift;  // log2(groups)
  const int nk = g.K / BK;
  // valid rows (COLM A) / column groups (ROWM B) of this tile; the rest stays zero in every stage
  const int vrows = colm ? (int)(g.rows - row0 < BM ? g.rows - row0 : BM) : BM;
  const int vgroups = colm ? groups : (int)(g.blim - b0 < groups ? g.blim - b0 : groups);
  if (colm) {
    for (int e = tid; e < STAGES * (BM - vrows) * Cfg::kLdA; e += blockDim.x) {
      const int st = e / ((BM - vrows) * Cfg::kLdA), rem = e % ((BM - vrows) * Cfg::kLdA);
      sA[st * Cfg::kStageA + vrows * Cfg::kLdA + rem] = make_double2(0.0, 0.0);
    }
  } else if (vgroups < groups) {
    for (int e = tid; e < STAGES * BK * BN; e += blockDim.x) {
      const int st = e / (BK * BN), k = (e / BN) % BK, c = e % BN;
      if ((c >> g.wshift) >= vgroups) sB[st * Cfg::kStageB + k * Cfg::kLdB + c] = make_double2(0.0, 0.0);
    }
  }
  if (tid == 0) {
    for (int s2 = 0; s2 < STAGES; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const unsigned stage_bytes =
      colm ? (unsigned)(vrows * BK * 16 + Cfg::kStageB * 16) : (unsigned)(Cfg::kStageA * 16 + vgroups * BK * W * 16);
  const int64_t ct = col_tile % g.ntile_a;  // COLM: column tile of B
  // warp 0: fill stage st with k-tile kt (lane 0 arms the barrier, the lanes issue the copies)
  auto produce = [&](int st, int kt) {
    if (lane == 0) mbar_expect_tx(&full[st], stage_bytes);
    __syncwarp();
    double2* dA = sA + st * Cfg::kStageA;
    double2* dB = sB + st * Cfg::kStageB;
    const int k0 = kt * BK;
    if (colm) {
      if (lane == 0) bulk_g2s(dB, g.blk + ((ct * nk + kt) * BK) * Cfg::kLdB, Cfg::kStageB * 16, &full[st]);
      for (int r = lane; r < vrows; r += 32)
        bulk_g2s(dA + r * Cfg::kLdA, g.A + (row0 + r) * g.lda + k0, BK * 16, &full[st]);
    } else {
      if (lane == 0) bulk_g2s(dA, g.blk + ((row_tile * nk + kt) * BM) * Cfg::kLdA, Cfg::kStageA * 16, &full[st]);
      if (DF) {  // short K: index by the power-of-two group count, no divisions (c2 1.79 -> 1.66 ms per
                 // pass; on c1's 16 k-tiles the same change measured 0.877 -> 0.914, so long K keeps
                 // the plain form — a compile-time choice: a run-time one slowed both)
        for (int e = lane; e < BK * groups; e += 32) {
          const int k = e >> gshift, q = e & (groups - 1);
          if (q < vgroups)
            bulk_g2s(dB + k * Cfg::kLdB + q * W, g.B + (int64_t)(k0 + k) * g.ldbk + a0 + (b0 + q) * g.ldbb, W * 16,
                     &full[st]);
        }
      } else {
        for (int e = lane; e < BK * vgroups; e += 32) {
          const int k = e / vgroups, q = e % vgroups;
          bulk_g2s(dB + k * Cfg::kLdB + q * W, g.B + (int64_t)(k0 + k) * g.ldbk + a0 + (b0 + q) * g.ldbb, W * 16,
                   &full[st]);
        }
      }
    }
  };
  if (warp == 0)
    for (int s2 = 0; s2 < STAGES && s2 < nk; ++s2) produce(s2, s2);

  double cre[MI][NI][2], cim[MI][NI][2], c3[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
      cre[mi][ni][0] = cre[mi][ni][1] = cim[mi][ni][0] = cim[mi][ni][1] = c3[mi][ni][0] = c3[mi][ni][1] = 0.0;
  const int arow = wy * (BM / WM) + (lane >> 2);
  const int bcol = wx * (BN / WN) + (lane >> 2);
  const int kq = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    if (warp == 0 && kt >= 1 && kt - 1 + STAGES < nk) {  // refill the stage k-tile kt - 1 used
      const int st = (kt - 1) % STAGES;
      if (lane == 0) mbar_wait(&empty[st], ((kt - 1) / STAGES) & 1);
      __syncwarp();
      produce(st, kt - 1 + STAGES);
    }
    const int st = kt % STAGES;
    mbar_wait(&full[st], (kt / STAGES) & 1);
    const double2* cA = sA + st * Cfg::kStageA;
    const double2* cB = sB + st * Cfg::kStageB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[MI], ai[MI], an[MI], br[NI], bi[NI], bs[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const double2 v = cA[(arow + mi * 8) * Cfg::kLdA + kk + kq];
        ar[mi] = v.x;
        ai[mi] = v.y;
        an[mi] = v.x + v.y;
      }
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const double2 v = cB[(kk + kq) * Cfg::kLdB + bcol + ni * 8];
        br[ni] = v.x;
        bi[ni] = v.y;
        bs[ni] = v.x + v.y;
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          dmma(cre[mi][ni][0], cre[mi][ni][1], ar[mi], br[ni]);
          dmma(cim[mi][ni][0], cim[mi][ni][1], ai[mi], bi[ni]);
          dmma(c3[mi][ni][0], c3[mi][ni][1], an[mi], bs[ni]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int64_t r = row0 + wy * (BM / WM) + mi * 8 + (lane >> 2);
    if (r >= g.rows) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int c = wx * (BN / WN) + ni * 8 + 2 * kq;
      const int64_t ga = a0 + (c & (W - 1));
      const int64_t gb = b0 + (c >> g.wshift);
      if (gb >= g.blim) continue;
      double2* dst = g.C + r * g.ldcr + ga + gb * g.ldcb;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (ga + h < g.alim) {
          double2 v = make_double2(cre[mi][ni][h] - cim[mi][ni][h], c3[mi][ni][h] - cre[mi][ni][h] - cim[mi][ni][h]);
          if (g.accumulate) v = cadd(dst[h], v);
          dst[h] = v;
        }
      }
    }
  }
}

// ---- mode-1 form fed by tensor-map TMA ---------------------------------------------------------
// The mode-1 product (inner = 1) is C(b, i) = sum_k X(b, k) M^T(k, i): the tensor is the A operand,
// one contiguous n-entry fibre per row b. A 2-D tensor map over (k as doubles, b) lets ONE
// cp.async.bulk.tensor per group of four k's fetch the BM x 4 box of a stage (64 bytes per row,
// rows n * 16 bytes apart) straight from the tensor's own strides — the per-row bulk copies of the
// plain bulk-copy form (BM of them per stage) were slower than cp.async. The box lands as
// [row][4 k], so a stage is [k group][row][4]: the A fragment of a quarter-warp (2 rows x 4 k) is
// 128 contiguous bytes, conflict-free without padding. Rows beyond the tensor are zero-filled by
// the copy engine. B = the factor's stage-blocked image (FactorSet::bblk), one bulk copy per stage.
static bool encode_colm_tmap(CUtensorMap* out, const double2* a, int64_t rows, int64_t lda, int K, int bm) {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (EncodeFn)f;
  }();
  if (!fn || ((uintptr_t)a & 15) || rows > 0x7fffffffll) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)2 * K, (cuuint64_t)rows};  // doubles along k, fibres
  const cuuint64_t strides[1] = {(cuuint64_t)lda * 16};
  const cuuint32_t box[2] = {8, (cuuint32_t)bm};
  const cuuint32_t estr[2] = {1, 1};
  return fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)a, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
__device__ __forceinline__ void tmap_g2s_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB>
__global__ void __launch_bounds__(WM* WN * 32, MINB)
    zgemm_tmap_colm_kernel(const GemmArgs g, const __grid_constant__ CUtensorMap amap) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, STAGES>;
  constexpr int NW = WM * WN;
  constexpr int MI = Cfg::MI, NI = Cfg::NI;
  constexpr int kStageA = BM * BK;  // [BK / 4][BM][4], unpadded
  extern __shared__ __align__(16) double2 smem[];
  // the tensor copies need 128-byte aligned destinations: align the stage area by hand (the launch
  // allocates 128 spare bytes)
  double2* sA = smem + ((128u - (smem_u32(smem) & 127u)) & 127u) / 16;
  double2* sB = sA + STAGES * kStageA;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wy = warp / WN, wx = warp % WN;
  const int64_t tile = blockIdx.x;
  // column tiles fastest: the CTAs sharing a row tile of the tensor run together (tensor read once)
  const int64_t row_tile = tile / g.ntile_a;
  const int64_t ct = tile % g.ntile_a;  // column tile of M^T (blim = 1)
  const int64_t row0 = row_tile * BM;
  const int64_t a0 = ct * BN;
  const int nk = g.K / BK;
  if (tid == 0) {
    for (int s2 = 0; s2 < STAGES; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  constexpr unsigned stage_bytes = (unsigned)((kStageA + Cfg::kStageB) * 16);
  auto produce = [&](int st, int kt) {  // one lane: the B image and BK / 4 boxes of the tensor
    mbar_expect_tx(&full[st], stage_bytes);
    bulk_g2s(sB + st * Cfg::kStageB, g.blk + ((ct * nk + kt) * BK) * Cfg::kLdB, Cfg::kStageB * 16, &full[st]);
#pragma unroll
    for (int kg = 0; kg < BK / 4; ++kg)
      tmap_g2s_2d(sA + st * kStageA + kg * BM * 4, &amap, 2 * (kt * BK + kg * 4), (int)row0, &full[st]);
  };
  if (tid == 0)
    for (int s2 = 0; s2 < STAGES && s2 < nk; ++s2) produce(s2, s2);

  double cre[MI][NI][2], cim[MI][NI][2], c3[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
      cre[mi][ni][0] = cre[mi][ni][1] = cim[mi][ni][0] = cim[mi][ni][1] = c3[mi][ni][0] = c3[mi][ni][1] = 0.0;
  const int arow = wy * (BM / WM) + (lane >> 2);
  const int bcol = wx * (BN / WN) + (lane >> 2);
  const int kq = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    if (warp == 0 && kt >= 1 && kt - 1 + STAGES < nk) {  // refill the stage k-tile kt - 1 used
      const int st = (kt - 1) % STAGES;
      if (lane == 0) {
        mbar_wait(&empty[st], ((kt - 1) / STAGES) & 1);
        produce(st, kt - 1 + STAGES);
      }
      __syncwarp();
    }
    const int st = kt % STAGES;
    mbar_wait(&full[st], (kt / STAGES) & 1);
    const double2* cA = sA + st * kStageA;
    const double2* cB = sB + st * Cfg::kStageB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[MI], ai[MI], an[MI], br[NI], bi[NI], bs[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const double2 v = cA[((kk >> 2) * BM + arow + mi * 8) * 4 + kq];
        ar[mi] = v.x;
        ai[mi] = v.y;
        an[mi] = v.x + v.y;
      }
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const double2 v = cB[(kk + kq) * Cfg::kLdB + bcol + ni * 8];
        br[ni] = v.x;
        bi[ni] = v.y;
        bs[ni] = v.x + v.y;
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          dmma(cre[mi][ni][0], cre[mi][ni][1], ar[mi], br[ni]);
          dmma(cim[mi][ni][0], cim[mi][ni][1], ai[mi], bi[ni]);
          dmma(c3[mi][ni][0], c3[mi][ni][1], an[mi], bs[ni]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int64_t r = row0 + wy * (BM / WM) + mi * 8 + (lane >> 2);
    if (r >= g.rows) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int64_t ga = a0 + wx * (BN / WN) + ni * 8 + 2 * kq;
      double2* dst = g.C + r * g.ldcr + ga;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (ga + h < g.alim) {
          double2 v = make_double2(cre[mi][ni][h] - cim[mi][ni][h], c3[mi][ni][h] - cre[mi][ni][h] - cim[mi][ni][h]);
          if (g.accumulate) v = cadd(dst[h], v);
          dst[h] = v;
        }
      }
    }
  }
}

// Stage geometry of the short-K bulk-copy GEMM: the constant operand's stage image is UNPADDED
// (BM x BK, 16-byte chunks XOR-swizzled by row parity: entry (r, k) at r BK + (k ^ 4 (r & 1)),
// the same banks as the padded rows), which leaves room for a 4-stage ring at 2 CTAs / SM.
// Measured (per pass): n = 128 (c3) 7.26 ms vs 7.36 with zgemm_tma_kernel's padded 3-stage ring;
// n = 256 (c1) 0.917 vs 0.886 — so factors with n >= 256 keep the padded images and that kernel.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool PAD = false>
struct TmaCfg {
  static constexpr int kThreads = WM * WN * 32;
  static constexpr int kLdA = PAD ? BK + 4 : BK;
  static constexpr int kLdB = BN + 2;  // complex; = 2 mod 8 -> conflict-free B fragments
  static constexpr int kStageA = BM * kLdA;
  static constexpr int kStageB = BK * kLdB;
  static constexpr size_t kSmem = (size_t)STAGES * (kStageA + kStageB) * sizeof(double2);
  static constexpr int MI = BM / WM / 8;
  static constexpr int NI = BN / WN / 8;
};
__host__ __device__ __forceinline__ int ablk_swz(int r, int k) { return k ^ ((r & 1) << 2); }
// Operand images of an n x n factor: padded rows for long K (n >= 256: 16 or more k-tiles, where
// the 3-stage padded ring is faster) and for extents that take the 32 x 64 CTA shape (n = 96, c2:
// 13.30 vs 13.10 ms with the deeper ring), swizzled unpadded rows with a 4-stage ring otherwise.
__host__ __device__ __forceinline__ bool tma_padded(int64_t n) { return n >= 256 || n % 64 != 0; }

// The short-K variant of zgemm_tma_kernel (row-major form only): unpadded, swizzled constant-
// operand stages and a deeper ring.
template <int BM, int BN, int BK, int WM, int WN, int STAGES, int MINB>
__global__ void __launch_bounds__(WM* WN * 32, MINB) zgemm_tma_swz_kernel(const GemmArgs g) {
  constexpr bool PAD = false;
  using Cfg = TmaCfg<BM, BN, BK, WM, WN, STAGES, PAD>;
  constexpr int NW = WM * WN;
  constexpr int MI = Cfg::MI, NI = Cfg::NI;
  static_assert(BK == 16, "the stage images are 16 deep");
  extern __shared__ __align__(16) double2 smem[];
  double2* sA = smem;
  double2* sB = smem + STAGES * Cfg::kStageA;
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wy = warp / WN, wx = warp % WN;
  const int64_t tile = blockIdx.x;
  const int64_t row_tile = tile % g.ntile_rows;
  const int64_t col_tile = tile / g.ntile_rows;
  const int64_t row0 = row_tile * BM;
  const int64_t a0 = (col_tile % g.ntile_a) << g.wshift;
  const int64_t b0 = (col_tile / g.ntile_a) * (BN >> g.wshift);
  const int W = 1 << g.wshift;
  const int groups = BN >> g.wshift;
  const int gshift = __popc(BN - 1) - g.wshift;  // log2(groups)
  const int nk = g.K / BK;
  // valid column groups of this tile; the rest of B stays zero in every stage
  const int vgroups = (int)(g.blim - b0 < groups ? g.blim - b0 : groups);
  if (vgroups < groups) {
    for (int e = tid; e < STAGES * BK * BN; e += blockDim.x) {
      const int st = e / (BK * BN), k = (e / BN) % BK, c = e % BN;
      if ((c >> g.wshift) >= vgroups) sB[st * Cfg::kStageB + k * Cfg::kLdB + c] = make_double2(0.0, 0.0);
    }
  }
  if (tid == 0) {
    for (int s2 = 0; s2 < STAGES; ++s2) {
      mbar_init(&full[s2], 1);
      mbar_init(&empty[s2], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const unsigned stage_bytes = (unsigned)(Cfg::kStageA * 16 + vgroups * BK * W * 16);
  // warp 0: fill stage st with k-tile kt (lane 0 arms the barrier, the lanes issue the copies)
  auto produce = [&](int st, int kt) {
    if (lane == 0) mbar_expect_tx(&full[st], stage_bytes);
    __syncwarp();
    double2* dA = sA + st * Cfg::kStageA;
    double2* dB = sB + st * Cfg::kStageB;
    const int k0 = kt * BK;
    if (lane == 0) bulk_g2s(dA, g.blk + ((row_tile * nk + kt) * BM) * Cfg::kLdA, Cfg::kStageA * 16, &full[st]);
    for (int e = lane; e < BK * groups; e += 32) {  // groups is a power of two: no divisions
      const int k = e >> gshift, q = e & (groups - 1);
      if (q < vgroups)
        bulk_g2s(dB + k * Cfg::kLdB + q * W, g.B + (int64_t)(k0 + k) * g.ldbk + a0 + (b0 + q) * g.ldbb, W * 16,
                 &full[st]);
    }
  };
  if (warp == 0)
    for (int s2 = 0; s2 < STAGES && s2 < nk; ++s2) produce(s2, s2);

  double cre[MI][NI][2], cim[MI][NI][2], c3[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
      cre[mi][ni][0] = cre[mi][ni][1] = cim[mi][ni][0] = cim[mi][ni][1] = c3[mi][ni][0] = c3[mi][ni][1] = 0.0;
  const int arow = wy * (BM / WM) + (lane >> 2);
  const int bcol = wx * (BN / WN) + (lane >> 2);
  const int kq = lane & 3;
  const int asw = PAD ? 0 : (arow & 1) << 2;  // rows arow + 8 mi share the parity
  for (int kt = 0; kt < nk; ++kt) {
    if (warp == 0 && kt >= 1 && kt - 1 + STAGES < nk) {  // refill the stage k-tile kt - 1 used
      const int st = (kt - 1) % STAGES;
      if (lane == 0) mbar_wait(&empty[st], ((kt - 1) / STAGES) & 1);
      __syncwarp();
      produce(st, kt - 1 + STAGES);
    }
    const int st = kt % STAGES;
    mbar_wait(&full[st], (kt / STAGES) & 1);
    const double2* cA = sA + st * Cfg::kStageA;
    const double2* cB = sB + st * Cfg::kStageB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[MI], ai[MI], an[MI], br[NI], bi[NI], bs[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const double2 v = cA[(arow + mi * 8) * Cfg::kLdA + ((kk + kq) ^ asw)];
        ar[mi] = v.x;
        ai[mi] = v.y;
        an[mi] = v.x + v.y;
      }
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const double2 v = cB[(kk + kq) * Cfg::kLdB + bcol + ni * 8];
        br[ni] = v.x;
        bi[ni] = v.y;
        bs[ni] = v.x + v.y;
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          dmma(cre[mi][ni][0], cre[mi][ni][1], ar[mi], br[ni]);
          dmma(cim[mi][ni][0], cim[mi][ni][1], ai[mi], bi[ni]);
          dmma(c3[mi][ni][0], c3[mi][ni][1], an[mi], bs[ni]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }

#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int64_t r = row0 + wy * (BM / WM) + mi * 8 + (lane >> 2);
    if (r >= g.rows) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int c = wx * (BN / WN) + ni * 8 + 2 * kq;
      const int64_t ga = a0 + (c & (W - 1));
      const int64_t gb = b0 + (c >> g.wshift);
      if (gb >= g.blim) continue;
      double2* dst = g.C + r * g.ldcr + ga + gb * g.ldcb;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (ga + h < g.alim) {
          double2 v = make_double2(cre[mi][ni][h] - cim[mi][ni][h], c3[mi][ni][h] - cre[mi][ni][h] - cim[mi][ni][h]);
          if (g.accumulate) v = cadd(dst[h], v);
          dst[h] = v;
        }
      }
    }
  }
}

// Tile configurations. 3M kernels, 2 CTAs / SM, 8 warps, BK = 16, 3 stages:
//   kWide: 64 x 32 per CTA;  kTall: 32 x 64 per CTA; warps of 16 x 16.
// The shape with the least padded output is chosen per GEMM (ties: kWide).
// Algorithmic flops are counted as 8 per complex MAC in every roofline figure regardless.
template <int BM, int BN, int BK, int WM, int WN, int ST, bool M3, int MINB = 1, int TST = ST>
static void launch_gemm_t(GemmArgs g, cudaStream_t stream) {
  using Cfg = GemmCfg<BM, BN, BK, WM, WN, ST>;
  using PCfg = GemmCfg<BM, BN, BK, WM, WN, TST>;  // the padded bulk-copy kernel's ring
  using SCfg = TmaCfg<BM, BN, BK, WM, WN, 4>;
  auto kern = zgemm_dmma_kernel<BM, BN, BK, WM, WN, ST, M3, MINB>;
  auto tkern = zgemm_tma_kernel<BM, BN, BK, WM, WN, TST, MINB>;
  auto tkern_df = zgemm_tma_kernel<BM, BN, BK, WM, WN, TST, MINB, true>;  // short K (< 256)
  smem_optin(tkern_df, PCfg::kSmem);
  auto skern = zgemm_tma_swz_kernel<BM, BN, BK, WM, WN, 4, MINB>;
  smem_optin(kern, Cfg::kSmem);
  smem_optin(tkern, PCfg::kSmem);
  smem_optin(skern, SCfg::kSmem);
  const bool colm = g.colm != 0;
  g.ntile_rows = (g.rows + BM - 1) / BM;
  const int64_t W = 1ll << g.wshift;
  g.ntile_a = (g.alim + W - 1) / W;
  const int64_t bb = BN / W;
  const int64_t ntile_b = (g.blim + bb - 1) / bb;
  const int64_t tiles = g.ntile_rows * g.ntile_a * ntile_b;
  // bulk-copy feed for the row-major form only: the mode-1 form would need one copy per 256-byte
  // row of the tensor operand (64 per stage) and measured 1.32 ms per c1 pass vs 0.94 with cp.async
  const bool tma = M3 && g.blk && !colm && g.K % BK == 0 && g.alim % W == 0;
  if (M3 && g.blk && colm && g.K % BK == 0 && g.ldbb == 0 && g.blim == 1 && g.wshift == __builtin_ctz(BN)) {
    // mode-1 form: the tensor through a 2-D tensor map (falls through to cp.async if the driver
    // cannot encode one)
    CUtensorMap amap;
    if (encode_colm_tmap(&amap, g.A, g.rows, g.lda, g.K, BM)) {
      auto ckern = zgemm_tmap_colm_kernel<BM, BN, BK, WM, WN, TST, MINB>;
      constexpr size_t csmem = (size_t)TST * (BM * BK + PCfg::kStageB) * sizeof(double2) + 128;
      smem_optin(ckern, csmem);
      ckern<<<(unsigned)tiles, PCfg::kThreads, csmem, stream>>>(g, amap);
      NDS_LAUNCH_CHECK();
      return;
    }
  }
  if (tma && !tma_padded(g.K))  // short K: the swizzled images of that factor, 4-stage ring
    skern<<<(unsigned)tiles, SCfg::kThreads, SCfg::kSmem, stream>>>(g);
  else if (tma && g.K < 256)
    tkern_df<<<(unsigned)tiles, PCfg::kThreads, PCfg::kSmem, stream>>>(g, colm ? 1 : 0);
  else if (tma)
    tkern<<<(unsigned)tiles, PCfg::kThreads, PCfg::kSmem, stream>>>(g, colm ? 1 : 0);
  else
    kern<<<(unsigned)tiles, Cfg::kThreads, Cfg::kSmem, stream>>>(g);
  NDS_LAUNCH_CHECK();
}

// Two CTA shapes (64 x 32 and 32 x 64, 8 warps of 16 x 16, 2 CTAs / SM, BK = 16, 3-stage ring);
// per GEMM the one with the least padded output wins (n = 96 pads 64-row tiles by a third).
// Warp tiles of 16 x 16 (2 x 2 fragments) need 4 operand sums and 4 fragment loads per 12 DMMAs
// (32 x 8 warps: 5 and 5) — the 3M sums share the FP64 pipe with the DMMAs (c1 transforms
// 4.74 -> 4.63 ms). Measured and removed: 4M 64 x 128, 3M 64 x 64 at 4 stages, 32 x 8 warps.
enum GemmShape { kWide = 0, kTall = 1 };
struct ShapeDims {
  int bm, bn;
};
static ShapeDims shape_dims(GemmShape s) { return s == kTall ? ShapeDims{32, 64} : ShapeDims{64, 32}; }

// The 32 x 64 shape's smaller padded A stage leaves room for a 4-stage bulk-copy ring at 2 CTAs /
// SM (c1 mode-2 pass 0.883 -> 0.877 ms, c2 2.04 -> 2.00).
static void launch_gemm(GemmShape shape, GemmArgs g, cudaStream_t stream) {
  if (shape == kTall) launch_gemm_t<32, 64, 16, 2, 4, 3, true, 2, 4>(g, stream);
  else launch_gemm_t<64, 32, 16, 4, 2, 3, true, 2>(g, stream);
}

// Column split for ROWM: power of two W in [8, bn] minimising padded columns (ties -> wider).
static int pick_wshift(int64_t inner, int bn) {
  int best = 3;
  double best_waste = 1e30;
  for (int s = 3; (1 << s) <= bn; ++s) {
    const int64_t w = 1ll << s;
    const double waste = (double)(((inner + w - 1) / w) * w) / (double)inner;
    if (waste <= best_waste + 1e-12) {
      best_waste = waste;
      best = s;
    }
  }
  return best;
}

// Fill the shape-dependent fields (wshift) and return the padded output volume of the grid.
static double shape_cost(GemmArgs& g, bool colm, int64_t inner, GemmShape s) {
  const ShapeDims sd = shape_dims(s);
  g.wshift = colm ? __builtin_ctz(sd.bn) : pick_wshift(inner, sd.bn);
  const int64_t W = 1ll << g.wshift, bb = sd.bn / W;
  const double rows = (double)((g.rows + sd.bm - 1) / sd.bm) * sd.bm;
  const double cols = (double)((g.alim + W - 1) / W) * W * (double)((g.blim + bb - 1) / bb) * bb;
  return rows * cols;
}

static void launch_gemm_auto(GemmArgs g, bool colm, int64_t inner, cudaStream_t stream) {
  GemmArgs gt = g;
  const double cw = shape_cost(gt, colm, inner, kWide);
  const double ct = shape_cost(gt, colm, inner, kTall);
  // ties (same padded volume): the 32 x 64 shape for long K (n >= 256: c1 mode 1 (cp.async) 0.932
  // vs 0.939 ms, mode 2 (padded bulk copy, 4 stages) 0.877 vs 0.886), 64 x 32 below (c3: 58.5 vs
  // 58.0 ms of transforms with the 32 x 64 shape on ties)
  const GemmShape best = ct < cw * (1.0 - 1e-9) || (ct <= cw * (1.0 + 1e-9) && g.K >= 256) ? kTall : kWide;
  shape_cost(g, colm, inner, best);
  g.blk = g.blk_shape[best];
  launch_gemm(best, g, stream);
}

// ---- stage-blocked operand images for the bulk-copy GEMM (FactorSet::ablk / bblk) ---------------
// shape 0 = kWide (BM 64, BN 32), 1 = kTall (BM 32, BN 64); BK = 16, row pads BK + 4 / BN + 2.
static int64_t ablk_entries(int64_t n, int bm) { return (n + bm - 1) / bm * bm * (n / 16) * (tma_padded(n) ? 20 : 16); }
static int64_t bblk_entries(int64_t n, int bn) { return (n + bn - 1) / bn * (n / 16) * 16 * (bn + 2); }

int64_t blocked_entries(int64_t n) {
  if (n < 16 || n % 16) return 0;
  return 2 * (ablk_entries(n, 64) + ablk_entries(n, 32) + bblk_entries(n, 32) + bblk_entries(n, 64));
}

// A image: [row tile][k tile][BM][ld]: (row, k) of M row-major, zero beyond n rows; ld = 20
// (padded, k at slot k, zero pad) when tma_padded(n), else 16 with k at slot ablk_swz(r, k).
__global__ void ablk_kernel(const double2* __restrict__ mrow, int n, int bm, double2* __restrict__ out, int64_t total) {
  const int nkt = n / 16;
  const bool pad = tma_padded(n);
  const int ld = pad ? 20 : 16;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int slot = (int)(e % ld);
    const int64_t q = e / ld;
    const int r = (int)(q % bm);
    const int64_t q2 = q / bm;
    const int kt = (int)(q2 % nkt);
    const int64_t rt = q2 / nkt;
    const int64_t row = rt * bm + r;
    const int c = pad ? slot : ablk_swz(r, slot);  // the swizzle is an involution
    out[e] = (row < n && c < 16) ? mrow[row * n + kt * 16 + c] : make_double2(0.0, 0.0);
  }
}
// B image of the mode-1 GEMM: [col tile][k tile][16][BN + 2]: B(k, i) = mcol[i + k n].
__global__ void bblk_kernel(const double2* __restrict__ mcol, int n, int bn, double2* __restrict__ out, int64_t total) {
  const int nkt = n / 16, ld = bn + 2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % ld);
    const int64_t q = e / ld;
    const int k = (int)(q % 16);
    const int64_t q2 = q / 16;
    const int kt = (int)(q2 % nkt);
    const int64_t ct = q2 / nkt;
    const int64_t col = ct * bn + c;
    out[e] = (col < n && c < bn) ? mcol[col + (int64_t)(kt * 16 + k) * n] : make_double2(0.0, 0.0);
  }
}

void blocked_layouts_launch(FactorSet& f, double2* base, cudaStream_t stream, int op_mask) {
  double2* p = base;
  for (int j = 0; j < f.n_modes; ++j) {
    const int n = (int)f.dims[j];
    if (!blocked_entries(n)) continue;
    for (int op = 0; op < 2; ++op) {
      if (!((op_mask >> op) & 1)) {  // not needed: keep the slot layout, skip the build
        for (int sh = 0; sh < 2; ++sh) p += ablk_entries(n, sh ? 32 : 64) + bblk_entries(n, sh ? 64 : 32);
        continue;
      }
      const double2* mrow = op ? f.uh_row[j] : f.u_row[j];
      const double2* mcol = op ? f.uh_col[j] : f.u_col[j];
      for (int sh = 0; sh < 2; ++sh) {
        const int bm = sh ? 32 : 64, bn = sh ? 64 : 32;
        const int64_t na = ablk_entries(n, bm), nb = bblk_entries(n, bn);
        f.ablk[j][op][sh] = p;
        ablk_kernel<<<(unsigned)std::min<int64_t>((na + 255) / 256, 1024), 256, 0, stream>>>(mrow, n, bm, p, na);
        NDS_LAUNCH_CHECK();
        p += na;
        // the mode-1 (column-major) form exists for the first mode only
        f.bblk[j][op][sh] = nullptr;
        if (j == 0) {
          f.bblk[j][op][sh] = p;
          bblk_kernel<<<(unsigned)std::min<int64_t>((nb + 255) / 256, 1024), 256, 0, stream>>>(mcol, n, bn, p, nb);
          NDS_LAUNCH_CHECK();
        }
        p += nb;
      }
    }
  }
}

int mode_product_launch(const FactorSet& f, int mode, bool adjoint, const ModeView& v, const double2* x, double2* r,
                        bool accumulate, cudaStream_t stream) {
  const double2* mrow = adjoint ? f.uh_row[mode - 1] : f.u_row[mode - 1];
  const double2* mcol = adjoint ? f.uh_col[mode - 1] : f.u_col[mode - 1];
  const int op = adjoint ? 1 : 0;
  const bool colm = v.inner == 1;
  const double2* blk[2] = {colm ? f.bblk[mode - 1][op][0] : f.ablk[mode - 1][op][0],
                           colm ? f.bblk[mode - 1][op][1] : f.ablk[mode - 1][op][1]};
  return mode_product_matrix_launch(mrow, mcol, v, x, r, accumulate, stream, -1, -1, blk);
}

int mode_product_matrix_launch(const double2* mrow, const double2* mcol, const ModeView& v, const double2* x,
                               double2* r, bool accumulate, cudaStream_t stream, int64_t rows_out, int64_t lda_row,
                               const double2* const* blk) {
  const int n = (int)v.n;
  const int64_t m = rows_out > 0 ? rows_out : v.n;  // rows of M (output extent along the mode)
  // DMMA GEMM from 16 rows of K up (K is zero-padded to the 16-deep stage; rectangular updates
  // with many output rows already pay from K = 8); tiny inner extents use the direct kernel
  const bool gemm = (n >= 16 || (n >= 8 && m >= 32)) && (v.inner == 1 || v.inner >= 8);
  if (!gemm) {
    const int64_t total = v.inner * m * v.outer;
    const int threads = 256;
    const int64_t blocks = std::min<int64_t>((total + threads - 1) / threads, 148 * 16);
    mode_product_direct_kernel<<<(unsigned)blocks, threads, 0, stream>>>(mcol, v.inner, n, (int)m, v.outer, x, r,
                                                                        accumulate ? 1 : 0);
    NDS_LAUNCH_CHECK();
    return kXformDirect;
  }
  GemmArgs g{};
  g.K = n;
  g.accumulate = accumulate ? 1 : 0;
  g.colm = v.inner == 1 ? 1 : 0;
  if (blk && rows_out <= 0 && lda_row <= 0) {
    g.blk_shape[0] = blk[0];
    g.blk_shape[1] = blk[1];
  }
  if (v.inner == 1) {  // COLM: C(b, i) = X(b, :) . M^T(:, i)
    g.A = x;
    g.lda = n;
    g.rows = v.outer;
    g.B = mcol;  // B(k, i) = M[i][k] = mcol[i + k m]
    g.ldbk = m;
    g.ldbb = 0;
    g.alim = m;
    g.blim = 1;
    g.C = r;
    g.ldcr = m;
    g.ldcb = 0;
  } else {  // ROWM: C(i, (a, b)) = M(i, :) . X(:, (a, b))
    g.A = mrow;  // A(i, k) = M[i][k] = mrow[i lda + k] (lda = n unless M is a column block)
    g.lda = lda_row > 0 ? lda_row : n;
    g.rows = m;
    g.B = x;
    g.ldbk = v.inner;
    g.ldbb = v.inner * n;
    g.alim = v.inner;
    g.blim = v.outer;
    g.C = r;
    g.ldcr = v.inner;
    g.ldcb = v.inner * m;
  }
  launch_gemm_auto(g, v.inner == 1, v.inner, stream);
  return kXformGemm;
}

}  // namespace nds
