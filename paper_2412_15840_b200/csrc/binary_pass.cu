// Fused mode-product passes for runs of binary modes (n_j = 2), the tiny-mode regime of
// BASELINE config c4 (N = 29, n_j = 2): reference kernels.cpp:24-44 applied to one mode at a
// time costs a full read+write of the tensor per mode (29 passes per transform); here k
// consecutive binary modes are applied in ONE pass.
//
// A pass covers modes [a, a+k) of the column-major tensor viewed as (inner I, 2^k, outer O).
// Each CTA owns a 4096-entry tile: a run of R consecutive inner positions (R >= 8 entries =
// 128 B when I > 1, so global access stays coalesced) x all 2^k group positions, at one outer
// index; tile bit b < log2 R is a run bit, bit log2 R + q is group mode q. The tile is staged in
// shared memory (XOR-swizzled in 8-entry groups), then processed in rounds of up to 4 group
// modes: each thread gathers the 2^4 entries spanning the round's modes into registers, applies
// the 2x2 matrices as butterflies, and scatters back. Modes commute (test_kernels.cpp:91-99), so
// the grouping changes rounding only.
#include <algorithm>
#include <complex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace nds {

constexpr int kBinThreads = 256;

struct BinPass {
  int64_t I;       // inner extent (product of modes before the group)
  int64_t O;       // outer extent
  int64_t n_runs;  // I / R
  int logR, k;     // run bits, group bits (logR + k = 12)
  int rounds;
  int nrb[3];      // group bits per round (<= 4)
  int rb[3][4];    // tile bit of each round bit
  int tb[3][12];   // tile bits carried by the thread index (and slot index) in each round
  int rsw[3][16];  // swz(round bits of entry e): swz is linear over XOR, so swz(p0 | bits_e) =
                   // swz(p0) ^ rsw[e] — one XOR per access instead of the full swizzle
  int lane_mode;   // >= 0: round 0 also applies this group mode across lanes l, l ^ 16 by shuffles (its
                   // tile bit is thread bit 4 of round 0), so 9 modes take two rounds
  int64_t gbit[12];      // global offset of tile bit b (run bits: 2^b; group bit q: I 2^q)
  const double2* M[12];  // 2x2 column-major op(U_j) per group mode
};

__host__ __device__ __forceinline__ constexpr int swz(int p) { return p ^ (((p >> 3) ^ (p >> 6) ^ (p >> 9)) & 7); }

// Where a round reads / writes the tile: the first round of a pass gathers straight from global
// memory (its thread bits are the lowest tile bits, so a warp reads whole 128-byte runs) and the
// last one scatters straight to it — the tile crosses shared memory only between rounds.
enum : int { kIoShared = 0, kSrcGlobal = 1, kDstGlobal = 2 };

template <int NB, bool UNIT>
__device__ __forceinline__ void bin_butterflies(const int (&rbit)[NB], int logR, const double2 (*Mq)[4],
                                                double2 (&v)[1 << NB]) {
  constexpr int V = 1 << NB;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int mode = rbit[q] - logR;
    const double2 m00 = Mq[mode][0], m10 = Mq[mode][1], m01 = Mq[mode][2], m11 = Mq[mode][3];
#pragma unroll
    for (int e = 0; e < V; ++e) {
      if (!((e >> q) & 1)) {
        const double2 a = v[e], b = v[e | (1 << q)];
        if (UNIT) {
          v[e] = cfma(a, m01, b);
          v[e | (1 << q)] = cfma(b, m10, a);
        } else {
          v[e] = cfma(cmul(m00, a), m01, b);
          v[e | (1 << q)] = cfma(cmul(m10, a), m11, b);
        }
      }
    }
  }
}

// One round: each thread slot gathers the 2^NB entries spanning the round's NB group modes,
// applies the NB 2x2 matrices as butterflies in registers, and scatters them back.
// UNIT: the matrices are unit-diagonal ([[1, p], [q, 1]], the normalised factors of the fused
// route — four FMAs per output instead of eight). SYNC: a CTA barrier between the first slot's
// loads and its butterflies (publishes Mq written just before the call).
template <int NB, bool UNIT, int IO, bool SYNC = false, bool LANE = false>
__device__ __forceinline__ void bin_round(const BinPass& bp, int rd, double2* S, const double2 (*Mq)[4], int tid,
                                          const double2* __restrict__ gin = nullptr, double2* __restrict__ gout = nullptr) {
  constexpr int V = 1 << NB;
  int rbit[NB];
#pragma unroll
  for (int q = 0; q < NB; ++q) rbit[q] = bp.rb[rd][q];
  // slot s = tid + 256 j: its tile position p0(s) = p0(tid) ^ p0(256 j) (disjoint bits), and
  // swz is linear, so swz(p0(s)) = swz(p0(tid)) ^ swz(p0(256 j)) — the thread part once per round
  int p0t = 0;
  int64_t g0t = 0;
#pragma unroll
  for (int i = 0; i < 8 && i < 12 - NB; ++i) {
    const int bit = (tid >> i) & 1;
    p0t |= bit << bp.tb[rd][i];
    if (IO != kIoShared && bit) g0t += bp.gbit[bp.tb[rd][i]];
  }
  const int spt = swz(p0t);
  int64_t ge[V];
  if (IO != kIoShared) {
#pragma unroll
    for (int e = 0; e < V; ++e) {
      ge[e] = 0;
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if ((e >> q) & 1) ge[e] += bp.gbit[rbit[q]];
    }
  }
  for (int s = tid; s < (4096 >> NB); s += kBinThreads) {
    int p0j = 0;
    int64_t g0 = g0t;
#pragma unroll
    for (int i = 8; i < 12 - NB; ++i) {
      const int bit = (s >> i) & 1;
      p0j |= bit << bp.tb[rd][i];
      if (IO != kIoShared && bit) g0 += bp.gbit[bp.tb[rd][i]];
    }
    const int sp0 = spt ^ swz(p0j);
    double2 v[V];
#pragma unroll
    for (int e = 0; e < V; ++e) v[e] = (IO & kSrcGlobal) ? gin[g0 + ge[e]] : S[sp0 ^ bp.rsw[rd][e]];
    if (SYNC && s == tid) __syncthreads();
    bin_butterflies<NB, UNIT>(rbit, bp.logR, Mq, v);
    if (LANE) {
      // one more mode across the lane pair (l, l ^ 16): every lane computes its own output
      const bool hi = (tid & 16) != 0;
      const double2 cs = Mq[bp.lane_mode][hi ? 3 : 0], co = Mq[bp.lane_mode][hi ? 1 : 2];
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const double2 o = make_double2(__shfl_xor_sync(0xffffffffu, v[e].x, 16), __shfl_xor_sync(0xffffffffu, v[e].y, 16));
        v[e] = UNIT ? cfma(v[e], co, o) : cfma(cmul(cs, v[e]), co, o);
      }
    }
#pragma unroll
    for (int e = 0; e < V; ++e) {
      if (IO & kDstGlobal)
        gout[g0 + ge[e]] = v[e];
      else
        S[sp0 ^ bp.rsw[rd][e]] = v[e];
    }
  }
}

template <bool UNIT, int IO, bool SYNC = false>
__device__ __forceinline__ void bin_round_any(const BinPass& bp, int rd, double2* S, const double2 (*Mq)[4], int tid,
                                              const double2* __restrict__ gin = nullptr,
                                              double2* __restrict__ gout = nullptr) {
  if (IO == kSrcGlobal && bp.lane_mode >= 0) {  // (a four-bit first round by construction)
    bin_round<4, UNIT, IO, SYNC, true>(bp, rd, S, Mq, tid, gin, gout);
    return;
  }
  switch (bp.nrb[rd]) {
    case 4: bin_round<4, UNIT, IO, SYNC>(bp, rd, S, Mq, tid, gin, gout); break;
    case 3: bin_round<3, UNIT, IO, SYNC>(bp, rd, S, Mq, tid, gin, gout); break;
    case 2: bin_round<2, UNIT, IO, SYNC>(bp, rd, S, Mq, tid, gin, gout); break;
    default: bin_round<1, UNIT, IO, SYNC>(bp, rd, S, Mq, tid, gin, gout); break;
  }
}

// All rounds of a tile staged in shared memory (the coupled fused kernel below).
template <bool UNIT>
__device__ __forceinline__ void bin_rounds(const BinPass& bp, double2* S, const double2 (*Mq)[4], int tid) {
  for (int rd = 0; rd < bp.rounds; ++rd) {
    bin_round_any<UNIT, kIoShared>(bp, rd, S, Mq, tid);
    __syncthreads();
  }
}

// A pass: round 0 global -> shared, middle rounds in shared memory, the last one shared -> global
// (a single round: global -> global, no shared memory at all).
template <bool UNIT>
__global__ void __launch_bounds__(kBinThreads, 2) binary_pass_kernel(const BinPass bp, const double2* __restrict__ x,
                                                                  double2* __restrict__ r) {
  extern __shared__ __align__(16) double2 S[];  // 4096 entries (64 KB, dynamic)
  __shared__ double2 Mq[12][4];
  const int tid = threadIdx.x;
  if (tid < 4 * bp.k) Mq[tid >> 2][tid & 3] = bp.M[tid >> 2][tid & 3];
  const int64_t tile = blockIdx.x;
  const int64_t run = tile % bp.n_runs;
  const int64_t o = tile / bp.n_runs;
  const int64_t base = (run << bp.logR) + bp.I * ((int64_t)1 << bp.k) * o;
  if (bp.rounds == 1) {
    bin_round_any<UNIT, kSrcGlobal | kDstGlobal, true>(bp, 0, S, Mq, tid, x + base, r + base);
    return;
  }
  bin_round_any<UNIT, kSrcGlobal, true>(bp, 0, S, Mq, tid, x + base, nullptr);
  __syncthreads();
  for (int rd = 1; rd + 1 < bp.rounds; ++rd) {
    bin_round_any<UNIT, kIoShared>(bp, rd, S, Mq, tid);
    __syncthreads();
  }
  bin_round_any<UNIT, kDstGlobal>(bp, bp.rounds - 1, S, Mq, tid, nullptr, r + base);
}

// ---- fused pass: forward modes 1-12, decoupled tile solve, inverse modes 1-12 -------------------
// The all-binary route with diagonalised outer modes (capi.cu plan_binary_diag) leaves 2^(N-12)
// independent 12-mode tile solves, and a tile is exactly the 4096-entry contiguous tile of the
// modes-1-12 pass. Modes commute, so a full solve applies the outer modes' passes first; then
// ONE kernel loads each tile, applies U_j^H of modes 1-12 (butterfly rounds), solves the tile
// (popcount wavefront; den = sum over all N modes of T_j(i_j, i_j), the outer part from the
// tile's outer index), applies U_j of modes 1-12 and stores — two passes and the separate solve
// pass fused into one read and one write of the tensor.
struct BinTileSolve {
  const double2* t;    // T_j (2x2 column-major) at t + 4 j, all N modes
  const double2* e;    // normalised route (UNIT): the deferred diagonal scale e_j[bit] of every mode at
                       // e + 2 j (forward row scale x inverse column scale); nullptr otherwise
  int n_outer;         // N - 12
  const uint16_t* wf;  // the 4096 tile entries by popcount over the coupled modes, highest first
                       // (bank-interleaved)
  const int* wf_off;   // levels + 1 offsets
  int levels;          // coupled inner modes + 1
};

// UNIT (normalised factors): every forward factor is diag(f_j) [[1, p], [q, 1]] and every inverse
// factor [[1, p'], [q', 1]] diag(g_j) — here and in the outer modes' passes. The diagonal parts
// commute with all the other modes' butterflies and with the division by den, so all of them
// meet in this kernel as one separable scale E[l] = prod_j (f_j g_j)[bit_j(l)] applied where the
// tile solve reads its right-hand side: with c = D_f c^ (c^ = the tile after the unit butterflies)
// and w = D_g y the tile the unit inverse butterflies expect,
//   w[l] = (E[l] c^[l] - sum_j t01_j (g_j[0] / g_j[1]) w[l | e_j]) / den[l]
// (the ratio folded into ts.t on the host).
template <bool UNIT>
__global__ void __launch_bounds__(kBinThreads, 2)
    binary_fused_solve_kernel(const BinPass fw, const BinPass iv, const BinTileSolve ts, const double2* __restrict__ x,
                              double2* __restrict__ r) {
  extern __shared__ __align__(16) double2 S[];  // 4096 entries, swizzled (swz)
  __shared__ double2 Mq[12][4];
  __shared__ double2 t01[12], dlo[64], dhi[64];
  __shared__ double2 dout, eout;
  __shared__ double2 elo[UNIT ? 64 : 1], ehi[UNIT ? 64 : 1];
  const int tid = threadIdx.x;
  const int64_t tile = blockIdx.x;  // outer index (modes 13..N)
  const int64_t base = tile << 12;
  if (tid < 48) Mq[tid >> 2][tid & 3] = fw.M[tid >> 2][tid & 3];
  if (tid < 12) t01[tid] = ts.t[4 * tid + 2];
  if (tid == 0) {
    double2 d = make_double2(0.0, 0.0);
    for (int q = 0; q < ts.n_outer; ++q) d = cadd(d, ts.t[4 * (12 + q) + (((tile >> q) & 1) ? 3 : 0)]);
    dout = d;
    if (UNIT) {
      double2 e = make_double2(1.0, 0.0);
      for (int q = 0; q < ts.n_outer; ++q) e = cmul(e, ts.e[2 * (12 + q) + ((tile >> q) & 1)]);
      eout = e;
    }
  }
  const int stid = swz(tid);
  // tile load: contiguous 4096 entries (run R = 4096 / ... : pass geometry inner = 1)
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    double2 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = x[base + tid + (h * 8 + i) * kBinThreads];
#pragma unroll
    for (int i = 0; i < 8; ++i) S[stid ^ swz((h * 8 + i) * kBinThreads)] = v[i];
  }
  __syncthreads();
  bin_rounds<UNIT>(fw, S, Mq, tid);
  // den tables (modes 1-6 | modes 7-12 + the outer part), then the inverse factors
  if (tid < 64) {
    double2 d = make_double2(0.0, 0.0);
    for (int j = 0; j < 6; ++j) d = cadd(d, ts.t[4 * j + (((tid >> j) & 1) ? 3 : 0)]);
    dlo[tid] = d;
    if (UNIT) {
      double2 e = make_double2(1.0, 0.0);
      for (int j = 0; j < 6; ++j) e = cmul(e, ts.e[2 * j + ((tid >> j) & 1)]);
      elo[tid] = e;
    }
  } else if (tid < 128) {
    const int xh = tid - 64;
    double2 d = make_double2(0.0, 0.0);
    for (int j = 0; j < 6; ++j) d = cadd(d, ts.t[4 * (6 + j) + (((xh >> j) & 1) ? 3 : 0)]);
    dhi[xh] = cadd(d, dout);
    if (UNIT) {
      double2 e = eout;
      for (int j = 0; j < 6; ++j) e = cmul(e, ts.e[2 * (6 + j) + ((xh >> j) & 1)]);
      ehi[xh] = e;
    }
  } else if (tid < 128 + 48) {
    const int e = tid - 128;
    Mq[e >> 2][e & 3] = iv.M[e >> 2][e & 3];
  }
  __syncthreads();
  // popcount wavefront on the swizzled tile: swz is XOR-linear, so the slot of l | e_j (bit j of
  // l clear) is swz(l) ^ swz(e_j); terms split over two accumulators (even / odd modes)
  for (int lv = 0; lv < ts.levels; ++lv) {
    const int p1 = ts.wf_off[lv + 1];
    for (int p = ts.wf_off[lv] + tid; p < p1; p += kBinThreads) {
      const int l = ts.wf[p];
      const int sl = swz(l);
      double2 n0 = S[sl], n1 = make_double2(0.0, 0.0);
      if (UNIT) n0 = cmul(cmul(elo[l & 63], ehi[l >> 6]), n0);
#pragma unroll
      for (int j = 0; j < 12; j += 2) {
        if (!((l >> j) & 1)) n0 = cfms(n0, t01[j], S[sl ^ swz(1 << j)]);
        if (!((l >> (j + 1)) & 1)) n1 = cfms(n1, t01[j + 1], S[sl ^ swz(2 << j)]);
      }
      S[sl] = cmul(cadd(n0, n1), crecip_fast(cadd(dlo[l & 63], dhi[l >> 6])));
    }
    __syncthreads();
  }
  bin_rounds<UNIT>(iv, S, Mq, tid);
#pragma unroll
  for (int i = 0; i < 4096 / kBinThreads; ++i) r[base + tid + i * kBinThreads] = S[stid ^ swz(i * kBinThreads)];
}

// ---- the same with at most four coupled inner modes: the tile solve is a round -----------------
// When the modes left coupled fit one round (<= 4: c4 keeps 2), the round that holds them (C)
// does forward butterflies, the triangular solve of its 16 entries (descending, all couplings
// are inside the thread's registers) and the inverse butterflies in one visit; round A (the
// highest remaining bits) gathers from / scatters to global memory, so the tile crosses shared
// memory four times in all (A -> B -> C -> B -> A) instead of once per round and once per
// wavefront level. Rounds: 0 = A, 1 = B, 2 = C in fw and iv (same bits, different matrices).
struct BinRoundSolve {
  const double2* t;  // T'_j (2 x 2 column-major) at t + 4 j, all N modes (couplings pre-scaled if UNIT)
  const double2* e;  // UNIT: the deferred scales e_j[0], e_j[1] at e + 2 j
  int n_outer;       // N - 12
  int cpl;           // bit q: round-C bit q is a coupled mode
  // By value, so every coefficient is a constant-bank operand of its DFMA (no shared-memory
  // table reads in the inner loops): the 2 x 2 matrices by [round][round bit] (column-major:
  // m00, m10, m01, m11), forward and inverse; round C's coupling t01 per bit and its part of den
  // and of the scale per entry e.
  double2 mf[3][4][4], mi[3][4][4];
  double2 t01[4], dround[16], eround[16];
};

template <bool UNIT>
__device__ __forceinline__ void const_butterflies(const double2 (&m)[4][4], double2 (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      if (!((e >> q) & 1)) {
        const double2 a = v[e], b = v[e | (1 << q)];
        if (UNIT) {
          v[e] = cfma(a, m[q][2], b);
          v[e | (1 << q)] = cfma(b, m[q][1], a);
        } else {
          v[e] = cfma(cmul(m[q][0], a), m[q][2], b);
          v[e | (1 << q)] = cfma(cmul(m[q][1], a), m[q][3], b);
        }
      }
    }
  }
}

// One round of the persistent kernel below on a contiguous tile: the thread's slot (one per
// thread: 256 threads x 16 entries) is fixed per round for the whole launch, so its tile offset
// p0 comes precomputed.
template <bool UNIT, int IO>
__device__ __forceinline__ void fused_round(const BinPass& bp, int rd, const double2 (&m)[4][4], double2* S, int p0,
                                            const double2* __restrict__ gin, double2* __restrict__ gout) {
  const int sp0 = swz(p0);
  double2 v[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    if (IO & kSrcGlobal) {
      int eb = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) eb |= ((e >> q) & 1) << bp.rb[rd][q];
      v[e] = gin[p0 | eb];
    } else {
      v[e] = S[sp0 ^ bp.rsw[rd][e]];
    }
  }
  const_butterflies<UNIT>(m, v);
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    if (IO & kDstGlobal) {
      int eb = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) eb |= ((e >> q) & 1) << bp.rb[rd][q];
      gout[p0 | eb] = v[e];
    } else {
      S[sp0 ^ bp.rsw[rd][e]] = v[e];
    }
  }
}

// Persistent: a CTA walks tiles blockIdx.x, + gridDim.x, ... (two CTAs per SM), so the per-thread
// slot positions and the thread's tile-independent part of den / scale are set up once per CTA;
// per tile only the outer modes' part (one warp, lanes over modes, shuffle tree) is new.
template <bool UNIT>
__global__ void __launch_bounds__(kBinThreads, 2)
    binary_fused_round_kernel(const __grid_constant__ BinPass fw, const __grid_constant__ BinRoundSolve ts,
                              int64_t n_tiles, const double2* __restrict__ x, double2* __restrict__ r) {
  extern __shared__ __align__(16) double2 S[];  // 4096 entries, swizzled (swz)
  __shared__ double2 dout, eout;
  const int tid = threadIdx.x;
  // slot positions per round (A, B, C) and the tile-independent part of den / scale (the 8 tile
  // bits outside round C): per-thread constants of the launch, parked in shared memory
  __shared__ int slot_p0[3][kBinThreads];
  __shared__ double2 slot_d[kBinThreads], slot_e[kBinThreads];
  {
#pragma unroll
    for (int rd = 0; rd < 3; ++rd) {
      int p = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) p |= ((tid >> i) & 1) << fw.tb[rd][i];
      slot_p0[rd][tid] = p;
    }
    double2 d = make_double2(0.0, 0.0), sc = make_double2(1.0, 0.0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = fw.tb[2][i], bit = (tid >> i) & 1;
      d = cadd(d, ts.t[4 * j + (bit ? 3 : 0)]);
      if (UNIT) sc = cmul(sc, ts.e[2 * j + bit]);
    }
    slot_d[tid] = d;
    slot_e[tid] = sc;
  }
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {  // tile = outer index (modes 13..N)
    const double2* xt = x + (tile << 12);
    double2* rt = r + (tile << 12);
    if (tid < 32) {
      // the outer modes' part of den and of the scale: lane q takes modes 12 + q, 12 + q + 32
      double2 d = make_double2(0.0, 0.0), sc = make_double2(1.0, 0.0);
      for (int q = tid; q < ts.n_outer; q += 32) {
        const int bit = (int)((tile >> q) & 1);
        d = cadd(d, ts.t[4 * (12 + q) + (bit ? 3 : 0)]);
        if (UNIT) sc = cmul(sc, ts.e[2 * (12 + q) + bit]);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        d.x += __shfl_xor_sync(0xffffffffu, d.x, o);
        d.y += __shfl_xor_sync(0xffffffffu, d.y, o);
        if (UNIT) {
          const double2 w = make_double2(__shfl_xor_sync(0xffffffffu, sc.x, o), __shfl_xor_sync(0xffffffffu, sc.y, o));
          sc = cmul(sc, w);
        }
      }
      if (tid == 0) {
        dout = d;
        eout = sc;
      }
    }
    fused_round<UNIT, kSrcGlobal>(fw, 0, ts.mf[0], S, slot_p0[0][tid], xt, nullptr);
    __syncthreads();
    fused_round<UNIT, kIoShared>(fw, 1, ts.mf[1], S, slot_p0[1][tid], nullptr, nullptr);
    __syncthreads();
    {
      const double2 dfix = cadd(slot_d[tid], dout);
      const double2 efix = UNIT ? cmul(slot_e[tid], eout) : make_double2(1.0, 0.0);
      const int sp0c = swz(slot_p0[2][tid]);
      double2 v[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = S[sp0c ^ fw.rsw[2][e]];
      const_butterflies<UNIT>(ts.mf[2], v);
#pragma unroll
      for (int e = 15; e >= 0; --e) {
        double2 n = v[e];
        if (UNIT) n = cmul(cmul(efix, ts.eround[e]), n);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (!((e >> q) & 1) && ((ts.cpl >> q) & 1)) n = cfms(n, ts.t01[q], v[e | (1 << q)]);
        v[e] = cmul(n, crecip_fast(cadd(dfix, ts.dround[e])));
      }
      const_butterflies<UNIT>(ts.mi[2], v);
#pragma unroll
      for (int e = 0; e < 16; ++e) S[sp0c ^ fw.rsw[2][e]] = v[e];
    }
    __syncthreads();
    fused_round<UNIT, kIoShared>(fw, 1, ts.mi[1], S, slot_p0[1][tid], nullptr, nullptr);
    __syncthreads();
    fused_round<UNIT, kDstGlobal>(fw, 0, ts.mi[0], S, slot_p0[0][tid], nullptr, rt);
    __syncthreads();  // the tile buffer and dout / eout are reused
  }
}

// Plan the passes over [mode0, mode1) (1-based, all n_j = 2): greedily take as many binary modes
// as fit a 4096-entry tile with runs of min(I, 8..4096) entries.
std::vector<BinGroup> plan_binary_groups(int n_modes, const int64_t* dims, int lo, int hi) {
  std::vector<BinGroup> out;
  if (hi < 0) hi = n_modes;
  int64_t inner = 1;
  int j = 0;
  while (j < n_modes) {
    int avail = 0;
    while (j >= lo && j + avail < hi && dims[j + avail] == 2) ++avail;
    if (avail == 0) {
      inner *= dims[j];
      ++j;
      continue;
    }
    // runs of R = 2^logR inner entries: at least min(I, 8) (128 B), the rest of the 12 tile bits
    // go to group modes
    int logI = 0;
    while (((int64_t)1 << logI) < inner) ++logI;
    const int k = std::min(avail, 12 - std::min(logI, 3));
    const int logR = 12 - k;
    int64_t outer = 1;
    for (int m = j + k; m < n_modes; ++m) outer *= dims[m];
    if (logR <= logI && inner % ((int64_t)1 << logR) == 0) {
      BinGroup gr;
      gr.first = j + 1;
      gr.count = k;
      gr.inner = inner;
      gr.outer = outer;
      gr.logR = logR;
      out.push_back(gr);
    }
    for (int m = 0; m < k; ++m) inner *= 2;
    j += k;
  }
  return out;
}

// rounds: the tile bits of each round (<= 4 each, all group bits exactly once); ascending[rd]:
// thread bits in ascending tile-bit order (rounds that touch global memory: a warp covers the
// lowest tile bits, i.e. whole runs), otherwise the first three with distinct residues mod 3
// where possible (conflict-free shared-memory phases under swz).
static BinPass make_bin_pass(const FactorSet& f, const BinGroup& gr, bool adjoint,
                             const std::vector<std::vector<int>>& rounds, const std::vector<bool>& ascending,
                             int lane_bit = -1) {
  BinPass bp{};
  bp.lane_mode = lane_bit >= 0 ? lane_bit - gr.logR : -1;
  bp.I = gr.inner;
  bp.O = gr.outer;
  bp.logR = gr.logR;
  bp.k = gr.count;
  bp.n_runs = gr.inner >> gr.logR;
  for (int q = 0; q < gr.count; ++q) bp.M[q] = adjoint ? f.uh_col[gr.first - 1 + q] : f.u_col[gr.first - 1 + q];
  for (int b = 0; b < 12; ++b) bp.gbit[b] = b < gr.logR ? (int64_t)1 << b : gr.inner << (b - gr.logR);
  bp.rounds = (int)rounds.size();
  for (int rd = 0; rd < bp.rounds; ++rd) {
    const int nb = (int)rounds[rd].size();
    bp.nrb[rd] = nb;
    bool used[12] = {};
    for (int q = 0; q < nb; ++q) {
      bp.rb[rd][q] = rounds[rd][q];
      used[bp.rb[rd][q]] = true;
    }
    std::vector<int> rest;
    for (int b = 0; b < 12; ++b)
      if (!used[b]) rest.push_back(b);
    std::vector<int> order;
    if (!ascending[rd])
      for (int want = 0; want < 3; ++want)
        for (size_t i = 0; i < rest.size(); ++i)
          if (rest[i] >= 0 && rest[i] % 3 == want) {
            order.push_back(rest[i]);
            rest[i] = -1;
            break;
          }
    for (int b : rest)
      if (b >= 0) order.push_back(b);
    if (rd == 0 && lane_bit >= 0) {  // the lane-pair mode's tile bit becomes thread bit 4
      order.erase(std::find(order.begin(), order.end(), lane_bit));
      order.insert(order.begin() + 4, lane_bit);
    }
    for (size_t i = 0; i < order.size(); ++i) bp.tb[rd][i] = order[i];
    for (int e = 0; e < (1 << nb); ++e) {
      int bits = 0;
      for (int q = 0; q < nb; ++q) bits |= ((e >> q) & 1) << bp.rb[rd][q];
      bp.rsw[rd][e] = swz(bits);
    }
  }
  return bp;
}

// Rounds of consecutive group bits, all staged in shared memory.
static BinPass make_bin_pass_staged(const FactorSet& f, const BinGroup& gr, bool adjoint) {
  std::vector<std::vector<int>> rounds;
  for (int b = 0; b < gr.count; b += 4) {
    rounds.emplace_back();
    for (int q = b; q < std::min(b + 4, gr.count); ++q) rounds.back().push_back(gr.logR + q);
  }
  return make_bin_pass(f, gr, adjoint, rounds, std::vector<bool>(rounds.size(), false));
}

// A pass of its own: the first round (global -> shared) takes the highest group bits, the last
// (shared -> global) the lowest, a middle one the rest.
static BinPass make_bin_pass_streamed(const FactorSet& f, const BinGroup& gr, bool adjoint) {
  const int k = gr.count, lo = gr.logR;
  std::vector<std::vector<int>> rounds;
  auto range = [&](int a, int b) {  // group bits [a, b)
    rounds.emplace_back();
    for (int q = a; q < b; ++q) rounds.back().push_back(lo + q);
  };
  if (k <= 4) {
    range(0, k);
  } else if (k <= 8) {
    range(k - 4, k);
    range(0, k - 4);
  } else if (k == 9) {  // 4 register bits + 1 lane bit in the first round, 4 in the last
    range(5, 9);
    range(0, 4);
    return make_bin_pass(f, gr, adjoint, rounds, {true, true}, lo + 4);
  } else {
    range(k - 4, k);
    range(4, k - 4);
    range(0, 4);
  }
  std::vector<bool> asc(rounds.size(), false);
  asc.front() = asc.back() = true;
  return make_bin_pass(f, gr, adjoint, rounds, asc);
}

int binary_pass_launch(const FactorSet& f, const BinGroup& gr, bool adjoint, const double2* x, double2* r,
                       cudaStream_t stream, bool unit) {
  const BinPass bp = make_bin_pass_streamed(f, gr, adjoint);
  const int64_t tiles = bp.n_runs * bp.O;
  if (unit) {
    smem_optin(binary_pass_kernel<true>, 4096 * 16);
    binary_pass_kernel<true><<<(unsigned)tiles, kBinThreads, 4096 * 16, stream>>>(bp, x, r);
  } else {
    smem_optin(binary_pass_kernel<false>, 4096 * 16);
    binary_pass_kernel<false><<<(unsigned)tiles, kBinThreads, 4096 * 16, stream>>>(bp, x, r);
  }
  NDS_LAUNCH_CHECK();
  return kXformDirect;
}

int binary_fused_solve_launch(const FactorSet& fwd, const FactorSet& inv, const BinGroup& gr, const double2* t_pool,
                              int n_outer, const uint16_t* wf, const int* wf_off, int levels, int cmask,
                              const BinHostFactors& host, const double2* x, double2* r, cudaStream_t stream,
                              const double2* unit_scales) {
  if (gr.first != 1 || gr.count != 12 || gr.logR != 0 || gr.inner != 1) throw Error(NDS_ERR_OTHER, "fused pass: not a modes-1-12 tile pass");
  if (__builtin_popcount(cmask) <= 4 && host.fwd) {
    // round C = the coupled bits, filled up with the lowest other bits; A = the highest four of
    // the rest (global side), B = the other four
    std::vector<int> c, rest;
    for (int b = 0; b < 12; ++b)
      if ((cmask >> b) & 1) c.push_back(b);
    for (int b = 0; b < 12 && c.size() < 4; ++b)
      if (!((cmask >> b) & 1)) c.push_back(b);
    std::sort(c.begin(), c.end());
    for (int b = 0; b < 12; ++b)
      if (std::find(c.begin(), c.end(), b) == c.end()) rest.push_back(b);
    const std::vector<std::vector<int>> rounds = {{rest[4], rest[5], rest[6], rest[7]},
                                                  {rest[0], rest[1], rest[2], rest[3]},
                                                  c};
    const std::vector<bool> asc = {true, false, false};
    const BinPass fw = make_bin_pass(fwd, gr, true, rounds, asc);
    int cpl = 0;
    for (int q = 0; q < 4; ++q)
      if ((cmask >> c[q]) & 1) cpl |= 1 << q;
    BinRoundSolve ts{};
    ts.t = t_pool;
    ts.e = unit_scales;
    ts.n_outer = n_outer;
    ts.cpl = cpl;
    auto cx = [](double2 a) { return std::complex<double>(a.x, a.y); };
    auto d2 = [](std::complex<double> a) { return make_double2(a.real(), a.imag()); };
    for (int rd = 0; rd < 3; ++rd)
      for (int q = 0; q < 4; ++q)
        for (int e = 0; e < 4; ++e) {
          ts.mf[rd][q][e] = host.fwd[4 * rounds[rd][q] + e];
          ts.mi[rd][q][e] = host.inv[4 * rounds[rd][q] + e];
        }
    for (int q = 0; q < 4; ++q) ts.t01[q] = host.t[4 * c[q] + 2];
    for (int e = 0; e < 16; ++e) {
      std::complex<double> d(0.0, 0.0), sc(1.0, 0.0);
      for (int q = 0; q < 4; ++q) {
        const int bit = (e >> q) & 1;
        d += cx(host.t[4 * c[q] + (bit ? 3 : 0)]);
        if (host.e) sc *= cx(host.e[2 * c[q] + bit]);
      }
      ts.dround[e] = d2(d);
      ts.eround[e] = d2(sc);
    }
    // persistent: the resident CTAs (two per SM) walk the tiles
    int dev = 0, sms = 0, per_sm = 0;
    NDS_CUDA(cudaGetDevice(&dev));
    NDS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (unit_scales) {
      smem_optin(binary_fused_round_kernel<true>, 4096 * 16);
      NDS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, binary_fused_round_kernel<true>, kBinThreads,
                                                             4096 * 16));
    } else {
      smem_optin(binary_fused_round_kernel<false>, 4096 * 16);
      NDS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, binary_fused_round_kernel<false>, kBinThreads,
                                                             4096 * 16));
    }
    const unsigned grid = (unsigned)std::min<int64_t>(gr.outer, (int64_t)sms * std::max(per_sm, 1));
    if (unit_scales)
      binary_fused_round_kernel<true><<<grid, kBinThreads, 4096 * 16, stream>>>(fw, ts, gr.outer, x, r);
    else
      binary_fused_round_kernel<false><<<grid, kBinThreads, 4096 * 16, stream>>>(fw, ts, gr.outer, x, r);
    NDS_LAUNCH_CHECK();
    return kBacksubLevel;
  }
  const BinPass fw = make_bin_pass_staged(fwd, gr, true);
  const BinPass iv = make_bin_pass_staged(inv, gr, false);
  BinTileSolve ts{t_pool, unit_scales, n_outer, wf, wf_off, levels};
  if (unit_scales) {
    smem_optin(binary_fused_solve_kernel<true>, 4096 * 16);
    binary_fused_solve_kernel<true><<<(unsigned)gr.outer, kBinThreads, 4096 * 16, stream>>>(fw, iv, ts, x, r);
  } else {
    smem_optin(binary_fused_solve_kernel<false>, 4096 * 16);
    binary_fused_solve_kernel<false><<<(unsigned)gr.outer, kBinThreads, 4096 * 16, stream>>>(fw, iv, ts, x, r);
  }
  NDS_LAUNCH_CHECK();
  return kBacksubLevel;
}

}  // namespace nds
