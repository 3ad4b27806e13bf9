// v2 of the blocked triangular solve — GEMM regime: cubic tiles of B^N = 4096 entries with B a
// in {8, 16} dividing every n_j (c0, c1: N=3 B=16; c2, c3: N=4 B=8).
// Included by backsub.cu.

#ifdef NDS_LINES_PROBE  // phase probes for tools/microbench/lines_bench.cu only
#define NDS_LPROBE(k) \
  if (threadIdx.x == 0 && blockIdx.x == 0) nds_lines_probe[k] = clock64()
#else
#define NDS_LPROBE(k)
#endif
#ifdef NDS_DIAG_PROBES  // timing probes for tools/microbench/diag_bench.cu only
#define NDS_PROBE(k, v) \
  if (tid == 0 && blockIdx.x == 0) nds_diag_probe[lv * 4 + (k)] = clock64() + (long long)((v) * 0)
#else
#define NDS_PROBE(k, v)
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

// Off-tile coupling of one work item (tile I, mode j, rows [kb, ke) along mode j) as a small
// complex GEMM on the FP64 tensor pipe:
//   partial(l_j, c) = sum_{k in [kb, ke)} T_j(o_j + l_j, k) * Y(k along mode j, c),
// rows l_j (b_j = 8 RB), columns c = the other local coordinates of the tile (cols = 4096 / b_j),
// K streamed from global through an ST-stage cp.async ring of BK = KM 2048 / cols rows (KM 32 KB).
// Every thread owns 8 KM fixed (k, c) slots of each stage; their global / shared offsets are
// computed once. Each warp owns RB x CB fragments (8x8) and reuses its A/B fragments across
// them. The partial is written in tile-local column-major order for the diagonal kernel.
template <int RB, int CB, bool M3, int KM, int ST, int H>
__device__ __forceinline__ void update_body(const TileGeom& g, const double2* __restrict__ T,
                                            const int64_t* __restrict__ tiles, const int4 it, const int half,
                                            double2* __restrict__ out, const double2* __restrict__ Y,
                                            double2* __restrict__ sm) {
  constexpr int BJ = 8 * RB;
  constexpr int TCOLS = 4096 / BJ;       // columns of the tile
  constexpr int COLS = TCOLS / H;        // columns of this CTA (H CTAs per item)
  constexpr int BK = KM * 2048 / TCOLS;
  constexpr int LDB = COLS + 2;          // = 2 mod 8 -> conflict-free B fragments
  constexpr int ALD = BK <= 8 ? 12 : BK + 4;  // = 4 mod 8 -> conflict-free A fragments
  constexpr int SL = 8 * KM / H;         // load slots per thread and stage
  static_assert(CB * 8 * (kUpdThreads / 32) == COLS && BK % 4 == 0 && BJ * BK <= kUpdThreads, "tile shape");
  __shared__ int64_t so[NDS_MAX_MODES];
  __shared__ int64_t s_base;
  const int j = it.y, kb = it.z, ke = it.w;
  const int N = g.n_modes;
  int64_t* colg = (int64_t*)sm;  // global offset of column c
  int* coll = (int*)(colg + COLS);
  double2* sA = (double2*)(coll + COLS);  // [ST][BJ][ALD]
  double2* sB = sA + ST * BJ * ALD;       // [ST][BK][LDB]
  const int tid = threadIdx.x;
  if (tid == 0) {
    int64_t t = tiles[it.x];
    int64_t base = 0;
    for (int m = 0; m < N; ++m) {
      const int64_t I = t % g.nb[m];
      t /= g.nb[m];
      so[m] = I * g.b[m];
      if (m != j) base += so[m] * g.strides[m];
    }
    s_base = base;
  }
  for (int c = tid; c < COLS; c += kUpdThreads) {  // c: local coords of modes != j, earliest fastest
    int rem = c + half * COLS;
    int64_t og = 0;
    int ol = 0;
    for (int m = 0; m < N; ++m) {
      if (m == j) continue;
      const int lm = rem % BJ;
      rem /= BJ;
      og += lm * g.strides[m];
      ol += lm * g.bstride[m];
    }
    colg[c] = og;
    coll[c] = ol;
  }
  __syncthreads();
  const int64_t sj = g.strides[j];
  const double2* Yb = Y + s_base;
  const double2* Tj = T + g.toff[j] + so[j];
  const int64_t nj = g.dims[j];

  // fixed per-thread load slots. Mode 1 (j == 0) is contiguous along k in global memory, so
  // its lanes run along k and the stage is stored k-fastest ([c][8] with the k index XOR-swizzled
  // by bit 0 of c: conflict-free for both the cp.async writes and the fragment reads); other
  // modes run along c into the [k][LDB] layout.
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
  const int a_r = tid % BJ, a_k = tid / BJ;  // rows fastest: coalesced along T_j's columns

  auto load_stage = [&](int stage, int k0) {
    double2* dB = sB + stage * BK * LDB;
    const double2* src = Yb + (int64_t)k0 * sj;
#pragma unroll
    for (int i = 0; i < SL; ++i) cp_async16_bs(dB + sofs[i], src + gofs[i]);
    if (a_loader) cp_async16_bs(sA + stage * BJ * ALD + a_r * ALD + a_k, Tj + a_r + (int64_t)(k0 + a_k) * nj);
  };

  const int lane = tid & 31, warp = tid >> 5;
  // 4M: cre, cim; 3M: cre = Ar Br, cim = Ai Bi, c3 = (Ar + Ai)(Br + Bi) (see zgemm_dmma_kernel)
  double cre[RB][CB][2], cim[RB][CB][2], c3[M3 ? RB : 1][M3 ? CB : 1][2];
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int q = 0; q < CB; ++q) {
      cre[r][q][0] = cre[r][q][1] = cim[r][q][0] = cim[r][q][1] = 0.0;
      if constexpr (M3) c3[r][q][0] = c3[r][q][1] = 0.0;
    }

  const int nk = (ke - kb) / BK;  // host guarantees BK | (ke - kb)
#pragma unroll
  for (int st = 0; st < ST - 1; ++st) {
    if (st < nk) load_stage(st, kb + st * BK);
    cp_commit_bs();
  }
  const int cbase = warp * CB * 8 + (lane >> 2);
  const int arow = lane >> 2, kq = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 2));
    __syncthreads();
    if (kt + ST - 1 < nk) load_stage((kt + ST - 1) % ST, kb + (kt + ST - 1) * BK);
    cp_commit_bs();
    const double2* cA = sA + (kt % ST) * BJ * ALD;
    const double2* cB = sB + (kt % ST) * BK * LDB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double ar[RB], ai[RB], an[RB], br[CB], bi[CB];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const double2 a = cA[(r * 8 + arow) * ALD + kk + kq];
        ar[r] = a.x;
        ai[r] = a.y;
        an[r] = M3 ? a.x + a.y : -a.y;
      }
#pragma unroll
      for (int q = 0; q < CB; ++q) {
        const int c = cbase + q * 8;
        const double2 b = kfast ? cB[c * BK + ((kk + kq) ^ (BK >= 8 ? (c & 1) << 2 : 0))] : cB[(kk + kq) * LDB + c];
        br[q] = b.x;
        bi[q] = b.y;
      }
      if constexpr (M3) {
        double bs[CB];
#pragma unroll
        for (int q = 0; q < CB; ++q) bs[q] = br[q] + bi[q];
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            dmma_bs(cre[r][q][0], cre[r][q][1], ar[r], br[q]);
            dmma_bs(cim[r][q][0], cim[r][q][1], ai[r], bi[q]);
            dmma_bs(c3[r][q][0], c3[r][q][1], an[r], bs[q]);
          }
      } else {
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int q = 0; q < CB; ++q) {
            dmma_bs(cre[r][q][0], cre[r][q][1], ar[r], br[q]);
            dmma_bs(cim[r][q][0], cim[r][q][1], ar[r], bi[q]);
            dmma_bs(cre[r][q][0], cre[r][q][1], an[r], bi[q]);
            dmma_bs(cim[r][q][0], cim[r][q][1], ai[r], br[q]);
          }
      }
    }
  }
  cp_wait0_bs();
  const int bsj = g.bstride[j];
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int q = 0; q < CB; ++q) {
      const int row = r * 8 + (lane >> 2);
      const int c = warp * CB * 8 + q * 8 + 2 * kq;
      if constexpr (M3) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
          out[row * bsj + coll[c + h]] =
              make_double2(cre[r][q][h] - cim[r][q][h], c3[r][q][h] - cre[r][q][h] - cim[r][q][h]);
      } else {
        out[row * bsj + coll[c]] = make_double2(cre[r][q][0], cim[r][q][0]);
        out[row * bsj + coll[c + 1]] = make_double2(cre[r][q][1], cim[r][q][1]);
      }
    }
}

template <int RB, int CB, bool M3, int KM, int ST, int H>
__global__ void __launch_bounds__(kUpdThreads, (M3 && H == 1) ? 1 : 2)
    tile_update_kernel(const TileGeom g, const double2* __restrict__ T, const int64_t* __restrict__ tiles,
                       const int4* __restrict__ items, double2* __restrict__ partial, const double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 sm[];
  update_body<RB, CB, M3, KM, ST, H>(g, T, tiles, items[blockIdx.x / H], (int)(blockIdx.x % H),
                                     partial + (int64_t)(blockIdx.x / H) * 4096, Y, sm);
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
#pragma unroll
  for (int st = 0; st < ST - 1; ++st) {
    if (st < nk) load_stage(st, kb + st * BK);
    cp_commit_bs();
  }
  const int cbase = warp * CB * 8 + (lane >> 2);
  const int arow = lane >> 2, kq = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ST - 2));
    __syncthreads();
    if (kt + ST - 1 < nk) load_stage((kt + ST - 1) % ST, kb + (kt + ST - 1) * BK);
    cp_commit_bs();
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
  }
  cp_wait0_bs();
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

// n terms tp[i grp] * sp[i ss], i < n, into four independent accumulators (loads batched).
__device__ __forceinline__ void dot_run(const double2* tp, const double2* sp, int n, int grp, int ss,
                                        double2 (&acc)[4]) {
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    const double2 t0 = tp[0], t1 = tp[grp], t2 = tp[2 * grp], t3 = tp[3 * grp];
    const double2 s0 = sp[0], s1 = sp[ss], s2 = sp[2 * ss], s3 = sp[3 * ss];
    acc[0] = cfma(acc[0], t0, s0);
    acc[1] = cfma(acc[1], t1, s1);
    acc[2] = cfma(acc[2], t2, s2);
    acc[3] = cfma(acc[3], t3, s3);
    tp += 4 * grp;
    sp += 4 * ss;
  }
  for (; i < n; ++i) {
    acc[0] = cfma(acc[0], tp[0], sp[0]);
    tp += grp;
    sp += ss;
  }
}

// Padded local strides of the diagonal tile in shared memory, chosen so that the entries of a
// local hyperplane (sorted by leading coordinates) fall into distinct 16-byte bank groups:
// N=3, B=16: (1, 17, 274) -> address mod 8 = l1 + l2 + 2 l3; N=4, B=8: (1, 9, 74, 595).
template <int N, int B>
struct PadStrides {
  static constexpr int s1 = B + 1;
  static constexpr int s2 = N >= 3 ? s1 * B + 2 : 0;
  static constexpr int s3 = N >= 4 ? s2 * B + 3 : 0;
  __device__ static constexpr int at(int m) { return m == 0 ? 1 : m == 1 ? s1 : m == 2 ? s2 : s3; }
  static constexpr int extent = 1 + (B - 1) * (1 + s1 + s2 + s3);
  __device__ static int pad(int l) {
    int a = 0;
#pragma unroll
    for (int m = 0; m < N; ++m) a += ((l >> ((B == 16 ? 4 : 3) * m)) & (B - 1)) * at(m);
    return a;
  }
};


// Diagonal tile (cubic, B^N = 4096 entries): S = C_I - sum(partials) (fixed order ->
// deterministic), then the local anti-diagonal wavefront over sum_j l_j = t, highest first.
// Hyperplane step lv (t = N (B - 1) - lv) is described by a host-built table: lvl[lv] =
// lanes-per-entry grp | (busy warps << 8), and thr[lv][tid] = the local entry this thread works
// on (0xffff: none); entries of a hyperplane are sorted by leading coordinates so lanes share
// loop trip counts. An entry's grp lanes split its sum_j sum_{k > l_j} T_j(i_j, k) y(...) terms,
// combine them with warp shuffles, and the leader scales by 1 / sum_j T_j(i_j, i_j). S uses
// padded strides (PadStrides) so a hyperplane's entries sit in distinct shared-memory banks.
template <int N, int B, int NT>
__global__ void __launch_bounds__(NT, 2)
    tile_diag_kernel(const TileGeom g, const double2* __restrict__ T, const int64_t* __restrict__ tiles,
                     const int4* __restrict__ tile_ranges, const double2* __restrict__ far_partial,
                     const double2* __restrict__ near_partial, const uint16_t* __restrict__ thr_g,
                     const int* __restrict__ lvl_g, int wf_levels, double2* __restrict__ Y) {
  constexpr int E = 4096;
  constexpr int LB = B == 16 ? 4 : 3;
  constexpr int WL = N * (B - 1) + 1;  // hyperplanes in a tile
  static_assert((1 << (LB * N)) == E, "cubic 4096-entry tile");
  using PS = PadStrides<N, B>;
  extern __shared__ __align__(16) double2 sm[];
  __shared__ int64_t so[N];
  __shared__ int64_t st[N];
  __shared__ int lvl[WL];
  const int tid = threadIdx.x;
  if (tid == 0) {
    int64_t t = tiles[blockIdx.x];
    for (int m = 0; m < N; ++m) {
      const int64_t I = t % g.nb[m];
      t /= g.nb[m];
      so[m] = I * B;
      st[m] = g.strides[m];
    }
  }
  double2* S = sm;
  double2* Td = S + PS::extent + (PS::extent & 1);  // [N][B][B] row-major: T_m(o_m + row, o_m + col)
  uint16_t* thr = (uint16_t*)(Td + N * B * B);      // [WL][NT]
  {
    const uint4* src = (const uint4*)thr_g;
    uint4* dst = (uint4*)thr;
    for (int i = tid; i < WL * NT / 8; i += NT) dst[i] = src[i];
  }
  for (int i = tid; i < WL; i += NT) lvl[i] = lvl_g[i];
  __syncthreads();
#pragma unroll
  for (int m = 0; m < N; ++m) {
    const double2* Tm = T + g.toff[m];
    const int64_t nm = g.dims[m];
    for (int e = tid; e < B * B; e += NT) {
      const int r = e / B, c = e % B;
      Td[(m * B + r) * B + c] = Tm[(so[m] + r) + (so[m] + c) * nm];
    }
  }
  const int4 tr = tile_ranges[blockIdx.x];  // {far first, far count, near first, near count}
  {
    constexpr int PER = E / NT;  // entries per thread, loads issued together
    double2 v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int l = tid + i * NT;
      int64_t gidx = 0;
#pragma unroll
      for (int m = 0; m < N; ++m) gidx += (so[m] + ((l >> (LB * m)) & (B - 1))) * st[m];
      v[i] = Y[gidx];
    }
    for (int p = 0; p < tr.y; ++p) {
      const double2* pp = far_partial + (int64_t)(tr.x + p) * E + tid;
#pragma unroll
      for (int i = 0; i < PER; ++i) v[i] = csub(v[i], pp[i * NT]);
    }
    for (int p = 0; p < tr.w; ++p) {
      const double2* pp = near_partial + (int64_t)(tr.z + p) * E + tid;
#pragma unroll
      for (int i = 0; i < PER; ++i) v[i] = csub(v[i], pp[i * NT]);
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) S[PS::pad(tid + i * NT)] = v[i];
  }
  __syncthreads();

  const int warp = tid >> 5;
#ifdef NDS_DIAG_CLOCK
  if (tid == 0 && blockIdx.x == 0) nds_diag_clock_start = clock64();
#endif
#pragma unroll 1
  for (int lv = 0; lv < wf_levels; ++lv) {
    const int info = lvl[lv];
    if (warp < (info >> 8)) {  // warp-uniform: this warp holds entries on hyperplane lv
      const int grp = info & 0xff;
      const int lraw = thr[lv * NT + tid];
      NDS_PROBE(0, lraw);
      const bool act = lraw != 0xffff;
      const int l = act ? lraw : 0;
      const int sub = tid & (grp - 1);
      int lm[N];
      int pl = 0;
#pragma unroll
      for (int m = 0; m < N; ++m) {
        lm[m] = (l >> (LB * m)) & (B - 1);
        pl += lm[m] * PS::at(m);
      }
      // denominator first: independent of S, its latency hides under the dot products
      double2 den = make_double2(0.0, 0.0);
#pragma unroll
      for (int m = 0; m < N; ++m) den = cadd(den, Td[m * B * B + lm[m] * (B + 1)]);
      const double2 rden = crecip_fast(den);  // issued before the dot products, off their chain
      NDS_PROBE(1, rden.x);
      double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
      double2 a2 = make_double2(0.0, 0.0), a3 = make_double2(0.0, 0.0);
      // Flattened term loop: every entry of hyperplane lv has exactly lv terms (cubic tile), so
      // the trip count is warp-uniform; term t maps to mode m (t >= qc[m]) and position k = t -
      // qc[m] along it. Offsets are affine in t within a mode: S: sb[m] + t a_m, T: tb[m] + t.
#if !defined(NDS_DIAG_FLAT) && !defined(NDS_DIAG_NODOT)
      if (act) {
#pragma unroll
        for (int m = 0; m < N; ++m) {
          const double2* tp = Td + m * B * B + lm[m] * (B + 1) + 1 + sub;
          const double2* sp = S + pl + (1 + sub) * PS::at(m);
          const int ss = grp * PS::at(m);
          int q = B - 1 - lm[m] - sub;  // this lane's terms: ceil(q / grp)
#pragma unroll 1
          for (; q > 3 * grp; q -= 4 * grp) {  // 4 terms in flight
            const double2 t0 = tp[0], t1 = tp[grp], t2 = tp[2 * grp], t3 = tp[3 * grp];
            const double2 s0 = sp[0], s1 = sp[ss], s2 = sp[2 * ss], s3 = sp[3 * ss];
            a0 = cfma(a0, t0, s0);
            a1 = cfma(a1, t1, s1);
            a2 = cfma(a2, t2, s2);
            a3 = cfma(a3, t3, s3);
            tp += 4 * grp;
            sp += 4 * ss;
          }
          if (q > grp) {
            const double2 t0 = tp[0], t1 = tp[grp], s0 = sp[0], s1 = sp[ss];
            a0 = cfma(a0, t0, s0);
            a1 = cfma(a1, t1, s1);
            tp += 2 * grp;
            sp += 2 * ss;
            q -= 2 * grp;
          }
          if (q > 0) a2 = cfma(a2, tp[0], sp[0]);
        }
      }
#elif !defined(NDS_DIAG_NODOT)
      if (act) {
        int qc[N], sb[N], tb[N];
        int q = 0;
#pragma unroll
        for (int m = 0; m < N; ++m) {
          qc[m] = q;
          sb[m] = pl + (1 - q) * PS::at(m);
          tb[m] = m * B * B + lm[m] * (B + 1) + 1 - q;
          q += B - 1 - lm[m];
        }
        auto term = [&](int t, double2& a) {
          int so = sb[0], sa = PS::at(0), to = tb[0];
#pragma unroll
          for (int m = 1; m < N; ++m)
            if (t >= qc[m]) {
              so = sb[m];
              sa = PS::at(m);
              to = tb[m];
            }
          a = cfma(a, Td[to + t], S[so + t * sa]);
        };
        int t = sub;
#pragma unroll 1
        for (; t + 3 * grp < lv; t += 4 * grp) {
          term(t, a0);
          term(t + grp, a1);
          term(t + 2 * grp, a2);
          term(t + 3 * grp, a3);
        }
        if (t < lv) term(t, a0);
        if (t + grp < lv) term(t + grp, a1);
        if (t + 2 * grp < lv) term(t + 2 * grp, a2);
      }
#endif
      double2 acc = cadd(cadd(a0, a1), cadd(a2, a3));
      NDS_PROBE(2, acc.x);
      for (int o = 1; o < grp; o <<= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (act && sub == 0) S[pl] = cmul(csub(S[pl], acc), rden);
      NDS_PROBE(3, S[pl].x);
    }
    __syncthreads();
#ifdef NDS_DIAG_CLOCK
    if (tid == 0 && blockIdx.x == 0) nds_diag_clock[lv] = clock64();
#endif
  }
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
// VAR bits: 4 = PRO (factor loads issued together with the tile's loads). Measured and removed
// (tools/microbench/lines_bench.cu): a split-phase (mbarrier) step barrier
// with the next row's distance >= 2 terms pre-accumulated in between, a warp-uniform bound on
// the history update, unrolling the PUSH modes, and a two-warps-per-32-lines form (512 threads,
// 128 registers; wavefront 58 K -> 87 K cycles).
template <int N, int B, int NT, bool PUSH, bool T2REG, bool SORT = true, int VAR = 0>
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
  constexpr bool PRO = (VAR & 4) != 0;
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
  // PRO: the factor loads go to registers first and are stored to shared memory only after the
  // tile's own loads are in flight (one exposed latency instead of two)
  static_assert(!PRO || B * B <= NT, "PRO: one factor entry per thread");
  double2 tdv[N], apv[N], dqv = make_double2(0.0, 0.0);
  const bool tl = tid < B * B;
  if constexpr (PRO) {
    const int r = tid % B, c = tid / B;
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
  } else {
#pragma unroll
    for (int m = 0; m < N; ++m) {
      const double2* Tm = T + g.toff[m];
      const int64_t nm = g.dims[m];
      const bool push_m = PUSH && so[m] >= B;
      for (int e = tid; e < B * B; e += NT) {
        const int r = e % B, c = e / B;  // rows fastest: coalesced along T_m's columns
        Td[(m * B + r) * B + c] = Tm[(so[m] + r) + (so[m] + c) * nm];
        if (push_m) Ap[(m * B + r) * ALD + c] = Tm[(so[m] - B + r) + (so[m] + c) * nm];
        if (m == 0) {  // e = j B + r'
          const int j = e / B, rr = e % B;
          Dq[e] = rr >= j + 1 ? Tm[(so[0] + rr - 1 - j) + (so[0] + rr) * nm] : make_double2(0.0, 0.0);
        }
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
    if constexpr (PRO) store_factors();
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
  if constexpr (PUSH) {
    // GEMM (B rows) x (NT columns) x (B k) per mode; warp w owns columns [32 w, 32 w + 32) as
    // RB x 4 fragments of 8 x 8. Column c = the local coordinates of the modes != m (earliest
    // fastest, as in tile_update_kernel's partial layout).
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
  NDS_LPROBE(5);
}

template <int N, int B, int NT, bool PUSH, bool T2REG, bool SORT = true, int VAR = 0>
__global__ void __launch_bounds__(NT, T2REG ? 1 : 2)
    tile_diag_lines_kernel(const TileGeom g, const double2* __restrict__ T, const int64_t* __restrict__ tiles,
                           const int4* __restrict__ tile_ranges, const double2* __restrict__ far_partial,
                           const double2* __restrict__ near_partial, const int* __restrict__ near_target,
                           double2* __restrict__ near_out, double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 sm[];
  diag_lines_body<N, B, NT, PUSH, T2REG, SORT, VAR>(g, T, tiles[blockIdx.x], tile_ranges[blockIdx.x], far_partial, near_partial,
                                         near_target ? near_target + (int64_t)blockIdx.x * N : nullptr, near_out, Y,
                                         sm);
}

using LinesKernel = void (*)(const TileGeom, const double2*, const int64_t*, const int4*, const double2*,
                             const double2*, const int*, double2*, double2*);
static LinesKernel lines_kernel_for(int n_modes, int b, bool push) {
  static const bool t2smem = getenv("NDS_DIAG_T2SMEM") != nullptr;  // A/B experiments
  static const bool natural = getenv("NDS_DIAG_NATURAL") != nullptr;
  // VAR 4 (PRO: factor loads overlapped with the tile's loads) measured 2 % faster per tile
  if (n_modes == 3 && b == 16) {
    if (natural)
      return push ? tile_diag_lines_kernel<3, 16, 256, true, true, false> : tile_diag_lines_kernel<3, 16, 256, false, true, false>;
    if (t2smem) return push ? tile_diag_lines_kernel<3, 16, 256, true, false> : tile_diag_lines_kernel<3, 16, 256, false, false>;
    return push ? tile_diag_lines_kernel<3, 16, 256, true, true, true, 4> : tile_diag_lines_kernel<3, 16, 256, false, true, true, 4>;
  }
  if (n_modes == 4 && b == 8 && natural)
    return push ? tile_diag_lines_kernel<4, 8, 512, true, true, false> : tile_diag_lines_kernel<4, 8, 512, false, true, false>;
  if (n_modes == 4 && b == 8)
    return push ? tile_diag_lines_kernel<4, 8, 512, true, true, true, 4> : tile_diag_lines_kernel<4, 8, 512, false, true, true, 4>;
  return nullptr;
}
static size_t lines_smem_bytes(int n_modes, int b) {
  const int ext = n_modes == 3 ? LinePad<3, 16>::extent : LinePad<4, 8>::extent;
  return (size_t)(ext + (ext & 1)) * 16 + (size_t)(n_modes + 1) * b * b * 16 + (size_t)n_modes * b * (b + 4) * 16;
}

using UpdateKernel = void (*)(const TileGeom, const double2*, const int64_t*, const int4*, double2*, const double2*);
using DiagKernel = void (*)(const TileGeom, const double2*, const int64_t*, const int4*, const double2*,
                            const double2*, const uint16_t*, const int*, int, double2*);

// Update-kernel configurations (measured). b = 16: 3M, BK = 8, 3 stages, two CTAs per item
// (128 columns each, 2 CTAs / SM): c1 solve 4.94 -> 4.36 ms vs one 256-column CTA (1 / SM).
// b = 8: 4M, BK = 4, 3 stages, one CTA per item (2 / SM). NDS_UPD=3m|4m|k16|s4|h1|h2|h4 override
// for A/B experiments.
struct UpdCfg {
  UpdateKernel kern;
  int bk, stages, h;
};
static int update_override() {
  static const int v = [] {
    const char* e = getenv("NDS_UPD");
    if (!e) return -1;
    const std::string s(e);
    return s == "3m" ? 1 : s == "4m" ? 0 : s == "k16" ? 2 : s == "s4" ? 3 : s == "h2" ? 4 : s == "h1" ? 5
         : s == "h4" ? 6 : s == "h2s4" ? 7 : s == "h2s5" ? 8 : s == "h2k16s2" ? 9 : s == "h4k16" ? 10 : -1;
  }();
  return v;
}
static UpdCfg update_cfg_for(int b) {
  const int o = update_override();
  if (b == 8) {
    if (o == 1) return {tile_update_kernel<1, 8, true, 1, 3, 1>, 4, 3, 1};
    if (o == 4) return {tile_update_kernel<1, 4, true, 1, 3, 2>, 4, 3, 2};
    if (o == 6) return {tile_update_kernel<1, 2, true, 1, 3, 4>, 4, 3, 4};
    if (o == 7) return {tile_update_kernel<1, 8, false, 1, 4, 1>, 4, 4, 1};
    if (o == 8) return {tile_update_kernel<1, 8, false, 1, 5, 1>, 4, 5, 1};
    return {tile_update_kernel<1, 8, false, 1, 3, 1>, 4, 3, 1};
  }
  if (b == 16) {
    if (o == 0) return {tile_update_kernel<2, 4, false, 1, 3, 1>, 8, 3, 1};
    if (o == 2) return {tile_update_kernel<2, 4, true, 2, 3, 1>, 16, 3, 1};
    if (o == 3) return {tile_update_kernel<2, 4, true, 1, 4, 1>, 8, 4, 1};
    if (o == 5) return {tile_update_kernel<2, 4, true, 1, 3, 1>, 8, 3, 1};
    if (o == 6) return {tile_update_kernel<2, 1, true, 1, 3, 4>, 8, 3, 4};
    if (o == 7) return {tile_update_kernel<2, 2, true, 1, 4, 2>, 8, 4, 2};
    if (o == 8) return {tile_update_kernel<2, 2, true, 1, 5, 2>, 8, 5, 2};
    if (o == 9) return {tile_update_kernel<2, 2, true, 2, 2, 2>, 16, 2, 2};
    if (o == 10) return {tile_update_kernel<2, 1, true, 2, 3, 4>, 16, 3, 4};
    return {tile_update_kernel<2, 2, true, 1, 3, 2>, 8, 3, 2};
  }
  return {nullptr, 0, 0, 0};
}
static UpdateKernel update_kernel_for(int b) { return update_cfg_for(b).kern; }

// Threads per diagonal-tile CTA: at least the widest local hyperplane (192 for 16^3, 480 for 8^4).
static int diag_threads_for(int n_modes) { return n_modes == 3 ? 256 : 512; }

static DiagKernel diag_kernel_for(int n_modes, int b) {
  if (n_modes == 3 && b == 16) return tile_diag_kernel<3, 16, 256>;
  if (n_modes == 4 && b == 8) return tile_diag_kernel<4, 8, 512>;
  return nullptr;
}
static int update_bk(int b) { return update_cfg_for(b).bk; }
static int update_h(int b) { return update_cfg_for(b).h; }

static size_t update_smem_bytes(int b) {
  const UpdCfg c = update_cfg_for(b);
  const int cols = 4096 / b / c.h, ald = c.bk <= 8 ? 12 : c.bk + 4;
  return (size_t)cols * (8 + 4) + (size_t)c.stages * b * ald * 16 + (size_t)c.stages * c.bk * (cols + 2) * 16;
}

static size_t diag_smem_bytes(int n_modes, int b, int wf_levels) {
  const int ext = n_modes == 3 ? PadStrides<3, 16>::extent : PadStrides<4, 8>::extent;
  return (size_t)(ext + (ext & 1)) * 16 + (size_t)n_modes * b * b * 16 +
         (size_t)wf_levels * diag_threads_for(n_modes) * sizeof(uint16_t);
}

// Far-update configurations (measured, c1/c2/c3 solve): G = 1 — one item per (target, mode), as
// the plain items, but with explicit ring slots so each level's items run longest first (LPT:
// c1 solve 4.82 -> 4.6 ms); 3M, 4-stage cp.async ring, two CTAs per item (b = 16: 128 columns,
// BK = 8; b = 8: 256 columns, BK = 4). Groups of G = 2/4 targets per item (32 rows, half the slab
// traffic per flop) measured slower: the far kernel is not traffic-bound (DMMA pipe ~57 % busy,
// latency/barrier stalls), and the remainder items add partial read-modify-writes.
// NDS_FARGROUP=plain restores the plain per-target items, =2|4 selects G. Also measured for G = 1
// and rejected: BK = 16 (1 CTA/SM by shared memory), one or four column CTAs per item, 4M.
struct FarGroupCfg {
  FarGroupKernel kern;
  int g, bk, stages, h;
};
static FarGroupCfg far_group_cfg(int b) {
  static const std::string env = getenv("NDS_FARGROUP") ? getenv("NDS_FARGROUP") : "";
  if (env == "plain") return {nullptr, 0, 0, 0, 0};
  const int gsel = env.empty() ? 0 : atoi(env.c_str());
  if (b == 16) {
    if (gsel == 2) return {far_group_kernel<16, 2, 2, true, 1, 3, 2>, 2, 8, 3, 2};
    return {far_group_kernel<16, 1, 2, true, 1, 4, 2>, 1, 8, 4, 2};
  }
  if (b == 8) {
    if (gsel == 2) return {far_group_kernel<8, 2, 2, true, 2, 3, 4>, 2, 8, 3, 4};
    if (gsel == 4) return {far_group_kernel<8, 4, 2, true, 2, 3, 4>, 4, 8, 3, 4};
    return {far_group_kernel<8, 1, 4, true, 1, 4, 2>, 1, 4, 4, 2};
  }
  return {nullptr, 0, 0, 0, 0};
}
// 0: plain per-target items (tile_update_kernel, slot = item index); G >= 1: FarGroupItem lists
static int far_group_for(int b) { return far_group_cfg(b).g; }
static int far_group_bk(int b) { return std::max(1, far_group_cfg(b).bk); }
static size_t far_group_smem_bytes(int b) {
  const FarGroupCfg c = far_group_cfg(b);
  if (c.g < 1) return 0;
  const int cols = 4096 / b / c.h, ald = c.bk <= 8 ? 12 : c.bk + 4;
  return (size_t)cols * (8 + 4) + (size_t)c.stages * c.g * b * ald * 16 + (size_t)c.stages * c.bk * (cols + 2) * 16;
}

