// v2 of the blocked triangular solve — GEMM regime: cubic tiles of B^N = 4096 entries with B a
// in {8, 16} dividing every n_j (c0, c1: N=3 B=16; c2, c3: N=4 B=8).
// Included by backsub.cu.

#ifdef NDS_LINES_PROBE  // phase probes for tools/microbench/lines_bench.cu only
#define NDS_LPROBE(k) \
  if (threadIdx.x == 0 && blockIdx.x == 0) nds_lines_probe[k] = clock64()
#else
#define NDS_LPROBE(k)
#endif
constexpr int kUpdThreads = 256;


__device__ __forceinline__ void cp_async16_bs(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit_bs() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1_bs() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_wait0_bs() { asm volatile("cp.async.wait_group 0;\n" ::); }

__device__ __forceinline__ void dmma_bs(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// Grouped far update (SolvePlan::fgroup = G > 1). One item covers up to G target tiles that are
// consecutive along its mode j (same other block coordinates, so the same columns), rows
// [rb0 b, (rb0 + G) b) of T_j, and one k-range of the neighbour slab (source rows) that every
// one of those targets still needs:
//   out_q(l_j, c) (+)= sum_{k in [kb, ke)} T_j(rb0 b + q b + l_j, k) * Y(k along j, c),  q < nrb,
// q = row block (target block rb0 + q), out_q a slot of the far-partial ring (its target's
// level region). acc = 1 accumulates into an existing slot (the remainder item of a target whose
// group item ran at an earlier level). Raising the rows from b to G b divides the slab traffic
// per flop by G and gives every B fragment G times the DMMA work. Row blocks q >= nrb (a
// truncated group at the bottom of a line) are computed but not stored.
template <int BT, int G, int CB, bool M3, int KM, int ST, int H>
__device__ __forceinline__ void far_group_body(const TileGeom& g, const double2* __restrict__ T,
                                               const int64_t* __restrict__ tiles, const FarGroupItem& it,
                                               const int half, double2* __restrict__ ring,
                                               const double2* __restrict__ Y, double2* __restrict__ sm) {
  constexpr int RB = G * BT / 8;         // row fragments
  constexpr int BJ = G * BT;             // rows
  constexpr int TCOLS = 4096 / BT;       // columns of a tile
  constexpr int COLS = TCOLS / H;        // columns of this CTA
  constexpr int BK = KM * 2048 / TCOLS;
  constexpr int LDB = COLS + 2;
  constexpr int ALD = BK <= 8 ? 12 : BK + 4;
  constexpr int SL = 8 * KM / H;
  static_assert(CB * 8 * (kUpdThreads / 32) == COLS && BK % 4 == 0 && BJ * BK <= kUpdThreads, "tile shape");
  __shared__ int64_t s_base;
  const int j = it.j, kb = it.kb, ke = it.ke;
  const int N = g.n_modes;
  int64_t* colg = (int64_t*)sm;
  int* coll = (int*)(colg + COLS);
  double2* sA = (double2*)(coll + COLS);  // [ST][BJ][ALD]
  double2* sB = sA + ST * BJ * ALD;       // [ST][BK][LDB]
  const int tid = threadIdx.x;
  if (tid == 0) {
    int64_t t = tiles[it.tile];
    int64_t base = 0;
    for (int m = 0; m < N; ++m) {
      const int64_t I = t % g.nb[m];
      t /= g.nb[m];
      if (m != j) base += I * g.b[m] * g.strides[m];
    }
    s_base = base;
  }
  for (int c = tid; c < COLS; c += kUpdThreads) {
    int rem = c + half * COLS;
    int64_t og = 0;
    int ol = 0;
    for (int m = 0; m < N; ++m) {
      if (m == j) continue;
      const int lm = rem % BT;
      rem /= BT;
      og += lm * g.strides[m];
      ol += lm * g.bstride[m];
    }
    colg[c] = og;
    coll[c] = ol;
  }
  __syncthreads();
  const int64_t sj = g.strides[j];
  const double2* Yb = Y + s_base;
  const double2* Tj = T + g.toff[j] + (int64_t)it.rb0 * BT;
  const int64_t nj = g.dims[j];
  const bool kfast = j == 0;
  int gofs[SL];
  int sofs[SL];
#pragma unroll
  for (int i = 0; i < SL; ++i) {
    const int e = tid + i * kUpdThreads;
    int k, c;
    if (kfast) {
      k = e % BK;
      c = e / BK;
      sofs[i] = c * BK + (k ^ (BK >= 8 ? (c & 1) << 2 : 0));
    } else {
      c = e % COLS;
      k = e / COLS;
      sofs[i] = k * LDB + c;
    }
    gofs[i] = (int)((int64_t)k * sj + colg[c]);
  }
  const bool a_loader = tid < BJ * BK;
  const int a_r = tid % BJ, a_k = tid / BJ;
  auto load_stage = [&](int stage, int k0) {
    double2* dB = sB + stage * BK * LDB;
    const double2* src = Yb + (int64_t)k0 * sj;
#pragma unroll
    for (int i = 0; i < SL; ++i) cp_async16_bs(dB + sofs[i], src + gofs[i]);
    if (a_loader) cp_async16_bs(sA + stage * BJ * ALD + a_r * ALD + a_k, Tj + a_r + (int64_t)(k0 + a_k) * nj);
  };
  const int lane = tid & 31, warp = tid >> 5;
  double cre[RB][CB][2], cim[RB][CB][2], c3[M3 ? RB : 1][M3 ? CB : 1][2];
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int q = 0; q < CB; ++q) {
      cre[r][q][0] = cre[r][q][1] = cim[r][q][0] = cim[r][q][1] = 0.0;
      if constexpr (M3) c3[r][q][0] = c3[r][q][1] = 0.0;
    }
  const int nk = (ke - kb) / BK;
  // mbarrier pipeline instead of a CTA barrier per stage: every thread's cp.async of a stage
  // complete on the stage's full barrier (cp.async.mbarrier.arrive.noinc, one arrival per
  // thread), warps release a stage on its empty barrier, and a stage is refilled one k-tile
  // after it was consumed (so a warp waits only for the slowest warp of the previous k-tile,
  // not of the current one). All ST stages are filled up front.
  __shared__ __align__(8) uint64_t fullb[ST], emptyb[ST];
  auto bar_addr = [](uint64_t* b) { return (unsigned)__cvta_generic_to_shared(b); };
  auto mb_wait = [&](uint64_t* b, unsigned parity) {
    unsigned done = 0;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(bar_addr(b)), "r"(parity)
          : "memory");
    } while (!done);
  };
  auto arrive_full = [&](int st) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar_addr(&fullb[st])) : "memory");
  };
  if (tid == 0) {
    for (int st = 0; st < ST; ++st) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar_addr(&fullb[st])), "r"(kUpdThreads));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar_addr(&emptyb[st])), "r"(kUpdThreads / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
#pragma unroll
  for (int st = 0; st < ST; ++st)
    if (st < nk) {
      load_stage(st, kb + st * BK);
      arrive_full(st);
    }
  const int cbase = warp * CB * 8 + (lane >> 2);
  const int arow = lane >> 2, kq = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    if (kt >= 1 && kt - 1 + ST < nk) {  // refill the stage k-tile kt - 1 used
      const int st = (kt - 1) % ST;
      mb_wait(&emptyb[st], ((kt - 1) / ST) & 1);
      load_stage(st, kb + (kt - 1 + ST) * BK);
      arrive_full(st);
    }
    mb_wait(&fullb[kt % ST], (kt / ST) & 1);
    const double2* cA = sA + (kt % ST) * BJ * ALD;
    const double2* cB = sB + (kt % ST) * BK * LDB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double br[CB], bi[CB], bs[CB];
#pragma unroll
      for (int q = 0; q < CB; ++q) {
        const int c = cbase + q * 8;
        const double2 b = kfast ? cB[c * BK + ((kk + kq) ^ (BK >= 8 ? (c & 1) << 2 : 0))] : cB[(kk + kq) * LDB + c];
        br[q] = b.x;
        bi[q] = b.y;
        bs[q] = M3 ? b.x + b.y : 0.0;
      }
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const double2 a = cA[(r * 8 + arow) * ALD + kk + kq];
        const double an = M3 ? a.x + a.y : -a.y;
#pragma unroll
        for (int q = 0; q < CB; ++q) {
          if constexpr (M3) {
            dmma_bs(cre[r][q][0], cre[r][q][1], a.x, br[q]);
            dmma_bs(cim[r][q][0], cim[r][q][1], a.y, bi[q]);
            dmma_bs(c3[r][q][0], c3[r][q][1], an, bs[q]);
          } else {
            dmma_bs(cre[r][q][0], cre[r][q][1], a.x, br[q]);
            dmma_bs(cim[r][q][0], cim[r][q][1], a.x, bi[q]);
            dmma_bs(cre[r][q][0], cre[r][q][1], an, bi[q]);
            dmma_bs(cim[r][q][0], cim[r][q][1], a.y, br[q]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar_addr(&emptyb[kt % ST])) : "memory");
  }
  const int bsj = g.bstride[j];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const int row = r * 8 + (lane >> 2);
    const int qb = row / BT;  // row block: the same for the whole fragment (BT % 8 == 0)
    if (qb >= it.nrb) continue;
    double2* out = ring + (int64_t)it.out[qb] * 4096 + (row % BT) * bsj;
#pragma unroll
    for (int q = 0; q < CB; ++q) {
      const int c = warp * CB * 8 + q * 8 + 2 * kq;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double2 v = M3 ? make_double2(cre[r][q][h] - cim[r][q][h], c3[r][q][h] - cre[r][q][h] - cim[r][q][h])
                       : make_double2(cre[r][q][h], cim[r][q][h]);
        double2* o = out + coll[c + h];
        if (it.acc) v = cadd(*o, v);
        *o = v;
      }
    }
  }
}

using FarGroupKernel = void (*)(const TileGeom, const double2*, const int64_t*, const FarGroupItem*, double2*,
                               const double2*);
template <int BT, int G, int CB, bool M3, int KM, int ST, int H>
__global__ void __launch_bounds__(kUpdThreads, 2)
    far_group_kernel(const TileGeom g, const double2* __restrict__ T, const int64_t* __restrict__ tiles,
                     const FarGroupItem* __restrict__ items, double2* __restrict__ ring, const double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 sm[];
  far_group_body<BT, G, CB, M3, KM, ST, H>(g, T, tiles, items[blockIdx.x / H], (int)(blockIdx.x % H), ring, Y, sm);
}

// Padded shared-memory strides of the line-owner kernel: thread t owns the mode-1 line
// (l_2, l_3, ...) = digits of t, so a warp's lanes differ in l_2 (fastest) and a hyperplane puts
// them at l_1 = s - l_2 - ...; a_2 - 1 odd spreads those lanes over all eight 16-byte bank groups.
template <int N, int B>
struct LinePad {
  static constexpr int a1 = B + 2;
  static constexpr int a2 = a1 * B + 1;
  static constexpr int a3 = N >= 4 ? a2 * B + 1 : 0;
  __host__ __device__ static constexpr int at(int m) { return m == 0 ? 1 : m == 1 ? a1 : m == 2 ? a2 : a3; }
  static constexpr int extent = 1 + (B - 1) * (1 + a1 + a2 + a3);
  __device__ static int pad(int l) {
    int a = 0;
#pragma unroll
    for (int m = 0; m < N; ++m) a += ((l >> ((B == 16 ? 4 : 3) * m)) & (B - 1)) * at(m);
    return a;
  }
};

// Line order of the line-owner kernel: lines sorted by d = sum_{m>=2} l_m, so the lanes of a warp
// own lines whose 16-step activity windows ([lv0, lv0 + B - 1], lv0 = (N-1)(B-1) - d) nearly
// coincide; a warp with no active lane skips the step. (Natural order puts l_2 = 0..B-1 in one
// warp, which keeps every warp busy for all (N)(B-1)+1 steps at ~1/3 lane occupancy.)
template <int N, int B>
struct LineOrder {
  uint16_t v[4096 / B];
};
template <int N, int B>
constexpr LineOrder<N, B> make_line_order() {
  LineOrder<N, B> o{};
  constexpr int NL = 4096 / B, LB = B == 16 ? 4 : 3;
  int p = 0;
  for (int d = 0; d <= (N - 1) * (B - 1); ++d)
    for (int l = 0; l < NL; ++l) {
      int s = 0, x = l;
      for (int m = 1; m < N; ++m) {
        s += x & (B - 1);
        x >>= LB;
      }
      if (s == d) o.v[p++] = (uint16_t)l;
    }
  return o;
}
__constant__ LineOrder<3, 16> kLineOrder3 = make_line_order<3, 16>();
__constant__ LineOrder<4, 8> kLineOrder4 = make_line_order<4, 8>();

// Near-coupling push of a solved tile held in shared memory (padded layout LinePad): for every
// mode m with a target (tgt_m[m] >= 0, CTA-uniform), near_out[tgt] (l_m, c) = sum_k Ap_m(l_m, k)
// S(k along m, c) — GEMM (B rows) x (NT columns) x (B k), 3M DMMA; warp w owns columns
// [32 w, 32 w + 32) as RB x 4 fragments of 8 x 8. Column c = the local coordinates of the modes
// != m (earliest fastest). Ap = [N][B][B + 4]: T_m(o_m - B + r, o_m + k).
template <int N, int B, int NT>
__device__ __forceinline__ void push_near(const double2* __restrict__ S, const double2* __restrict__ Ap,
                                          const int* tgt_m, double2* __restrict__ near_out) {
  using PS = LinePad<N, B>;
  constexpr int E = 4096;
  constexpr int LB = B == 16 ? 4 : 3;
  constexpr int ALD = B + 4;
  const int tid = threadIdx.x;
  constexpr int RB = B / 8;
  const int lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, ar = lane >> 2;
  auto col_offsets = [&](int c, int m, int& soff, int& loff) {
    soff = 0;
    loff = 0;
#pragma unroll
    for (int mm = 0; mm < N; ++mm) {
      if (mm == m) continue;
      const int l = c & (B - 1);
      c >>= LB;
      soff += l * PS::at(mm);
      loff += l << (LB * mm);
    }
  };
#pragma unroll 1
  for (int m = 0; m < N; ++m) {
    const int tgt = tgt_m[m];
    if (tgt < 0) continue;  // CTA-uniform
    int sb[4];
#pragma unroll
    for (int qf = 0; qf < 4; ++qf) {
      int lo;
      col_offsets(warp * 32 + qf * 8 + ar, m, sb[qf], lo);
    }
    double2* out = near_out + (int64_t)tgt * E;
    const double2* am = Ap + m * B * ALD;
    double cre[RB][4][2], cim[RB][4][2], c3[RB][4][2];
#pragma unroll
    for (int ri = 0; ri < RB; ++ri)
#pragma unroll
      for (int qf = 0; qf < 4; ++qf)
#pragma unroll
        for (int h = 0; h < 2; ++h) cre[ri][qf][h] = cim[ri][qf][h] = c3[ri][qf][h] = 0.0;
#pragma unroll
    for (int kk = 0; kk < B / 4; ++kk) {
      double a_r[RB], a_i[RB], a_s[RB];
#pragma unroll
      for (int ri = 0; ri < RB; ++ri) {
        const double2 a = am[(ri * 8 + ar) * ALD + kk * 4 + kq];
        a_r[ri] = a.x, a_i[ri] = a.y, a_s[ri] = a.x + a.y;
      }
#pragma unroll
      for (int qf = 0; qf < 4; ++qf) {
        const double2 v = S[(kk * 4 + kq) * PS::at(m) + sb[qf]];
        const double vs = v.x + v.y;
#pragma unroll
        for (int ri = 0; ri < RB; ++ri) {
          dmma_bs(cre[ri][qf][0], cre[ri][qf][1], a_r[ri], v.x);
          dmma_bs(cim[ri][qf][0], cim[ri][qf][1], a_i[ri], v.y);
          dmma_bs(c3[ri][qf][0], c3[ri][qf][1], a_s[ri], vs);
        }
      }
    }
#pragma unroll
    for (int qf = 0; qf < 4; ++qf)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        int so_, lo;
        col_offsets(warp * 32 + qf * 8 + 2 * kq + h, m, so_, lo);
#pragma unroll
        for (int ri = 0; ri < RB; ++ri)
          out[((ri * 8 + ar) << (LB * m)) + lo] =
              make_double2(cre[ri][qf][h] - cim[ri][qf][h], c3[ri][qf][h] - cre[ri][qf][h] - cim[ri][qf][h]);
      }
  }
}

// Diagonal tile, line-owner formulation. Thread t owns the mode-1 line with fixed local
// coordinates (l_2, .., l_N) = base-B digits of t and walks it from row B-1 down to 0, one row
// per local hyperplane: row r is solved at step lv = (N-1)(B-1) - d + (B-1-r), d = sum_{m>=2} l_m.
// Eq. (9)'s sum splits as
//   mode 1:   sum_{k>r} T_1(r, k) y(k, l_2, ..)  — the thread's own history, kept as pending sums
//             q[j] = sum_{k solved} T_1(r-1-j, k) y_k in registers that shift by one row per step
//             (static register indices); T_1's superdiagonals are stored diagonal-major so the
//             lanes' different rows r read consecutive words;
//   mode 2:   T_2(l_2, l_2 + 1 + k) is fixed per thread — held in registers;
//   modes 3+: T_m(l_m, ..) is shared by the lanes of a (half-)warp — a shared-memory broadcast;
// so per term only the neighbour y is read from shared memory, at a compile-time offset from the
// entry. Same partial-subtraction prologue and epilogue as tile_diag_kernel.
// PUSH: once the tile is solved, its couplings to the adjacent tiles behind it (J - e_m, the next
// level's near items) are computed here from the tile still in shared memory —
//   near_out[item] (l_m, c) = sum_k T_m(o_m - B + l_m, o_m + k) Y_J(k along m, c)
// (3M DMMA; near_target[slot N + m] = that item's index at the next level, -1 if none) — which
// replaces the separate near-update launch on the critical path.
// The factor loads go to registers and are stored to shared memory after the tile's own loads are
// in flight (one exposed latency instead of two; 2 % per tile). Measured and removed
// (tools/microbench/lines_bench.cu): a split-phase (mbarrier) step barrier
// with the next row's distance >= 2 terms pre-accumulated in between, a warp-uniform bound on
// the history update, unrolling the PUSH modes, T_2 read from shared memory (128 registers, two
// CTAs per SM, each 2.2x slower), natural line order, and a two-warps-per-32-lines form (512
// threads, 128 registers; wavefront 58 K -> 87 K cycles).
template <int N, int B, int NT>
__device__ __forceinline__ void diag_lines_body(const TileGeom& g, const double2* __restrict__ T, const int64_t tile,
                                                const int4 tr, const double2* __restrict__ far_partial,
                                                const double2* __restrict__ near_partial,
                                                const int* __restrict__ near_target, double2* __restrict__ near_out,
                                                double2* __restrict__ Y, double2* __restrict__ sm) {
  constexpr int E = 4096;
  constexpr int LB = B == 16 ? 4 : 3;
  constexpr int WL = N * (B - 1) + 1;
  static_assert((1 << (LB * N)) == E && E / B == NT, "one thread per mode-1 line of a cubic 4096-entry tile");
  using PS = LinePad<N, B>;
  __shared__ int64_t so[N];
  __shared__ int64_t st[N];
  constexpr bool PUSH = true, T2REG = true, SORT = true;
  const int tid = threadIdx.x;
  NDS_LPROBE(0);
  int tgt_m[N];  // near-coupling targets of the PUSH phase, loaded before the long wavefront
#pragma unroll
  for (int m = 0; m < N; ++m) tgt_m[m] = PUSH ? near_target[m] : -1;
  if (tid == 0) {
    int64_t t = tile;
    for (int m = 0; m < N; ++m) {
      const int64_t I = t % g.nb[m];
      t /= g.nb[m];
      so[m] = I * B;
      st[m] = g.strides[m];
    }
  }
  double2* S = sm;
  double2* Td = S + PS::extent + (PS::extent & 1);  // [N][B][B] row-major: T_m(o_m + row, o_m + col)
  double2* Dq = Td + N * B * B;                     // [B][B]: Dq[j][r] = T_1(r - 1 - j, r)
  constexpr int ALD = B + 4;                        // = 4 mod 8: conflict-free DMMA A fragments
  double2* Ap = Dq + B * B;                         // [N][B][ALD]: T_m(o_m - B + r, o_m + k) (PUSH)
  __syncthreads();
  static_assert(B * B <= NT, "one factor entry per thread");
  double2 tdv[N], apv[N], dqv = make_double2(0.0, 0.0);
  const bool tl = tid < B * B;
  {
    const int r = tid % B, c = tid / B;  // rows fastest: coalesced along T_m's columns
#pragma unroll
    for (int m = 0; m < N; ++m) {
      const double2* Tm = T + g.toff[m];
      const int64_t nm = g.dims[m];
      const bool push_m = PUSH && so[m] >= B;
      tdv[m] = tl ? Tm[(so[m] + r) + (so[m] + c) * nm] : make_double2(0.0, 0.0);
      apv[m] = tl && push_m ? Tm[(so[m] - B + r) + (so[m] + c) * nm] : make_double2(0.0, 0.0);
      if (m == 0) {
        const int j = tid / B, rr = tid % B;
        dqv = tl && rr >= j + 1 ? Tm[(so[0] + rr - 1 - j) + (so[0] + rr) * nm] : make_double2(0.0, 0.0);
      }
    }
  }
  auto store_factors = [&]() {
    if (!tl) return;
    const int r = tid % B, c = tid / B;
#pragma unroll
    for (int m = 0; m < N; ++m) {
      Td[(m * B + r) * B + c] = tdv[m];
      if (PUSH && so[m] >= B) Ap[(m * B + r) * ALD + c] = apv[m];
    }
    Dq[tid] = dqv;
  };
  NDS_LPROBE(1);
  // tr = {far first, far count, near first, near count}; partials two at a time so that 2 x PER
  // loads per thread are in flight (the prologue is latency-bound)
  {
    constexpr int PER = E / NT;
    double2 v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int l = tid + i * NT;
      int64_t gidx = 0;
#pragma unroll
      for (int m = 0; m < N; ++m) gidx += (so[m] + ((l >> (LB * m)) & (B - 1))) * st[m];
      v[i] = Y[gidx];
    }
    store_factors();
    const int np = tr.y + tr.w;
    auto part = [&](int p) {
      return p < tr.y ? far_partial + (int64_t)(tr.x + p) * E + tid : near_partial + (int64_t)(tr.z + p - tr.y) * E + tid;
    };
    int p = 0;
    for (; p + 2 <= np; p += 2) {
      const double2 *p0 = part(p), *p1 = part(p + 1);
      double2 w0[PER], w1[PER];
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        w0[i] = __ldcg(p0 + i * NT);
        w1[i] = __ldcg(p1 + i * NT);
      }
#pragma unroll
      for (int i = 0; i < PER; ++i) v[i] = csub(v[i], cadd(w0[i], w1[i]));
    }
    if (p < np) {
      const double2* p0 = part(p);
#pragma unroll
      for (int i = 0; i < PER; ++i) v[i] = csub(v[i], __ldcg(p0 + i * NT));
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) S[PS::pad(tid + i * NT)] = v[i];
  }
  __syncthreads();
  NDS_LPROBE(2);

  int lm[N];
  int d = 0, pb = 0;
  lm[0] = 0;
  const int line = !SORT ? tid : N == 3 ? kLineOrder3.v[tid] : kLineOrder4.v[tid];
#pragma unroll
  for (int m = 1; m < N; ++m) {
    lm[m] = (line >> (LB * (m - 1))) & (B - 1);
    d += lm[m];
    pb += lm[m] * PS::at(m);
  }
  // T_2(l_2, l_2 + 1 + k): registers (1 CTA / SM), or read per term from Td (128 registers, so a
  // diagonal CTA can share its SM with an update CTA)
  double2 t2r[T2REG ? B - 1 : 1];
  const double2* t2s = Td + (B + lm[1]) * B + lm[1] + 1;
  if constexpr (T2REG) {
#pragma unroll
    for (int k = 0; k < B - 1; ++k) t2r[k] = k < B - 1 - lm[1] ? t2s[k] : make_double2(0.0, 0.0);
  }
  double2 dsum = make_double2(0.0, 0.0);
#pragma unroll
  for (int m = 1; m < N; ++m) dsum = cadd(dsum, Td[(m * B + lm[m]) * B + lm[m]]);
  const int lv0 = (N - 1) * (B - 1) - d;  // step of row B-1
  double2 q[B - 1];
#pragma unroll
  for (int j = 0; j < B - 1; ++j) q[j] = make_double2(0.0, 0.0);

#pragma unroll 1
  for (int lv = 0; lv < WL; ++lv) {
    const int r = B - 1 - (lv - lv0);
    if (lv >= lv0 && r >= 0) {
      const double2* e = S + r + pb;  // this step's entry
      const double2 rden = crecip_fast(cadd(Td[r * (B + 1)], dsum));
      double2 a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = make_double2(0.0, 0.0);
      const int q2 = B - 1 - lm[1];
#pragma unroll
      for (int k = 0; k < B - 1; ++k)
        if (k < q2) a[k & 3] = cfma(a[k & 3], T2REG ? t2r[T2REG ? k : 0] : t2s[k], e[(1 + k) * PS::a1]);
#pragma unroll
      for (int m = 2; m < N; ++m) {
        const double2* tm = Td + (m * B + lm[m]) * B + lm[m] + 1;
        const int qm = B - 1 - lm[m];
#pragma unroll
        for (int k = 0; k < B - 1; ++k)
          if (k < qm) a[(k + 2) & 3] = cfma(a[(k + 2) & 3], tm[k], e[(1 + k) * PS::at(m)]);
      }
      const double2 acc = cadd(cadd(a[0], a[1]), cadd(a[2], cadd(a[3], q[0])));
      const double2 y = cmul(csub(e[0], acc), rden);
      S[r + pb] = y;
      // mode-1 history: q[j] <- q[j+1] + T_1(r-1-j, r) y for the rows r-1-j >= 0 still ahead
#pragma unroll
      for (int j = 0; j < B - 1; ++j)
        if (j < r) q[j] = cfma(j + 1 < B - 1 ? q[j + 1] : make_double2(0.0, 0.0), Dq[j * B + r], y);
    }
    __syncthreads();
  }
  NDS_LPROBE(3);
  {
    constexpr int PER = E / NT;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int l = tid + i * NT;
      int64_t gidx = 0;
#pragma unroll
      for (int m = 0; m < N; ++m) gidx += (so[m] + ((l >> (LB * m)) & (B - 1))) * st[m];
      Y[gidx] = S[PS::pad(l)];
    }
  }
  NDS_LPROBE(4);
  if constexpr (PUSH) push_near<N, B, NT>(S, Ap, tgt_m, near_out);
  NDS_LPROBE(5);
}

template <int N, int B, int NT>
__global__ void __launch_bounds__(NT, 1)
    tile_diag_lines_kernel(const TileGeom g, const double2* __restrict__ T, const int64_t* __restrict__ tiles,
                           const int4* __restrict__ tile_ranges, const double2* __restrict__ far_partial,
                           const double2* __restrict__ near_partial, const int* __restrict__ near_target,
                           double2* __restrict__ near_out, double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 sm[];
  diag_lines_body<N, B, NT>(g, T, tiles[blockIdx.x], tile_ranges[blockIdx.x], far_partial, near_partial,
                                         near_target ? near_target + (int64_t)blockIdx.x * N : nullptr, near_out, Y,
                                         sm);
}

using LinesKernel = void (*)(const TileGeom, const double2*, const int64_t*, const int4*, const double2*,
                             const double2*, const int*, double2*, double2*);
static LinesKernel lines_kernel_for(int n_modes, int b) {
  if (n_modes == 3 && b == 16) return tile_diag_lines_kernel<3, 16, 256>;
  if (n_modes == 4 && b == 8) return tile_diag_lines_kernel<4, 8, 512>;
  return nullptr;
}
static size_t lines_smem_bytes(int n_modes, int b) {
  const int ext = n_modes == 3 ? LinePad<3, 16>::extent : LinePad<4, 8>::extent;
  return (size_t)(ext + (ext & 1)) * 16 + (size_t)(n_modes + 1) * b * b * 16 + (size_t)n_modes * b * (b + 4) * 16;
}
// Threads per diagonal-tile CTA: one per mode-1 line (256 for 16^3, 512 for 8^4).
static int diag_threads_for(int n_modes) { return n_modes == 3 ? 256 : 512; }

// Far-update configurations (measured, c1/c2/c3 solve): one item per
// (target, mode) with an explicit ring slot so each level's items run longest first (LPT: c1
// solve 4.82 -> 4.6 ms); 3M, 4-stage cp.async ring, two CTAs per item (b = 16: 128 columns,
// BK = 8; b = 8: 256 columns, BK = 4). Measured and removed: groups of G = 2 / 4 targets per
// slab read (slower on every config: the kernel is latency/barrier-bound, not traffic-bound, and
// remainder items add partial read-modify-writes), k-split items, BK = 16, one or four column
// CTAs per item, 4M.
struct FarGroupCfg {
  FarGroupKernel kern;
  int g, bk, stages, h;
};
static FarGroupCfg far_group_cfg(int b) {
  if (b == 16) return {far_group_kernel<16, 1, 2, true, 1, 4, 2>, 1, 8, 4, 2};
  if (b == 8) return {far_group_kernel<8, 1, 4, true, 1, 4, 2>, 1, 4, 4, 2};
  return {nullptr, 0, 0, 0, 0};
}
static size_t far_group_smem_bytes(int b) {
  const FarGroupCfg c = far_group_cfg(b);
  if (c.g < 1) return 0;
  const int cols = 4096 / b / c.h, ald = c.bk <= 8 ? 12 : c.bk + 4;
  return (size_t)cols * (8 + 4) + (size_t)c.stages * c.g * b * ald * 16 + (size_t)c.stages * c.bk * (cols + 2) * 16;
}
