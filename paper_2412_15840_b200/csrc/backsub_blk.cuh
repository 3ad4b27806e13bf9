// Triangular solve of the BLOCK-DIAGONALISED cubic route (capi.cu plan_cubic_diag). Included by
// backsub.cu after backsub_v2.cuh (reuses dmma_bs, cp_async16_bs).
//
// The plan replaced every T_j by T'_j = W_j^{-1} T_j W_j, W_j = blockdiag of the eigenvector
// matrices of T_j's D_j x D_j diagonal blocks (D_j a multiple of the tile edge B): T'_j is block
// upper triangular with DIAGONAL D_j x D_j diagonal blocks. In Eq. (9) (sylvester.cpp:88-106) an
// entry then couples only to entries in a HIGHER D_j-block along some mode, so with super-blocks
// of D_j rows the index space is a grid of super-tiles whose levels sum_j floor(i_j / D_j) run
// from high to low, and every entry of a level is independent of the others:
//   y(i) = (c(i) - sum_j sum_{k >= (floor(i_j / D_j) + 1) D_j} T'_j(i_j, k) y(i with i_j -> k))
//          / sum_j T_j(i_j, i_j).
// One launch per level; one CTA per B^N tile of the level's super-tiles PULLS all its couplings:
// per mode j a (B rows) x (B^(N-1) columns) x (K_j = n_j - kb_j rows) complex GEMM on the FP64
// tensor pipe (3M DMMA), the operands streamed through one multi-stage cp.async + mbarrier ring
// that runs across the modes without draining (k-tile t -> (mode, k-tile)); each mode's result is
// subtracted from the tile held in shared memory, then the tile is divided by its denominators
// and stored. No partial buffers, no side streams: the whole solve is `levels` launches
// (c1 with D = 64: 10, against 46 tile hyperplanes of the wavefront route).

struct BlkArgs {
  TileGeom g;            // the COUPLED modes' geometry (modes with D_j < n_j)
  int d[NDS_MAX_MODES];  // diagonalisation block (super-block) extent per coupled mode
  // Uncoupled modes (D_j = n_j: T'_j diagonal) are a batch: tile id = coupled tile + ntc * batch
  // index; the batch index adds boff[b] to the tile origin and bden[b] (their diagonal terms) to
  // every denominator. boff = null: no batch.
  const int64_t* boff;
  const double2* bden;
  int64_t ntc;
};
constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }

template <int N, int B, int BK, int ST, int NT>
struct BlkCfg {
  static constexpr int E = 4096;
  static constexpr int LB = ilog2c(B);
  static constexpr int TC = E / B;        // columns of every mode's GEMM
  static constexpr int NW = NT / 32;
  static constexpr int CB = TC / 8 / NW;  // column fragments per warp
  static constexpr int RB = B / 8;        // row fragments
  static constexpr int LDB = TC + 2;      // row-major B stage stride (modes >= 2)
  static constexpr int ALD = BK <= 8 ? 12 : BK + 4;
  static constexpr int SL = BK * TC / NT;           // B elements per thread per stage
  static constexpr int BSTAGE = BK * LDB;           // >= TC * BK (mode-1 k-fastest layout)
  static constexpr int ASTAGE = B * ALD;
  static constexpr size_t smem() {
    return (size_t)(E + ST * (BSTAGE + ASTAGE)) * sizeof(double2) + (size_t)N * TC * sizeof(int);
  }
};

template <int N, int B, int BK, int ST, int NT, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB)
    blk_level_kernel(const BlkArgs ba, const double2* __restrict__ T, const int64_t* __restrict__ tiles,
                     double2* __restrict__ Y) {
  using C = BlkCfg<N, B, BK, ST, NT>;
  constexpr int kBlkThreads = NT;
  constexpr int E = C::E, LB = C::LB, TC = C::TC, CB = C::CB, RB = C::RB, LDB = C::LDB, ALD = C::ALD;
  constexpr int SL = C::SL;
  static_assert(C::SL * kBlkThreads == BK * TC && BK % 4 == 0 && (1 << (LB * N)) == E, "stage shape");
  extern __shared__ __align__(16) double2 smem[];
  double2* sS = smem;                          // the tile (local index l = sum_m l_m B^m)
  double2* sB = sS + E;                        // [ST][BSTAGE]
  double2* sA = sB + ST * C::BSTAGE;           // [ST][B][ALD]
  int* colg = (int*)(sA + ST * C::ASTAGE);     // [N][TC]: global offset of column c for mode j
  __shared__ __align__(8) uint64_t fullb[ST], emptyb[ST];
  __shared__ int64_t so[N];
  __shared__ int kb_s[N], nk_s[N];
  __shared__ double2 dd[N][B];
  const TileGeom& g = ba.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int64_t tile_id = tiles[blockIdx.x], tb = 0;
  if (ba.boff) {
    tb = tile_id / ba.ntc;
    tile_id -= tb * ba.ntc;
  }
  if (tid < N) {
    int64_t t = tile_id;
    for (int m = 0; m < N; ++m) {
      const int64_t I = t % g.nb[m];
      t /= g.nb[m];
      if (m == tid) {
        so[m] = I * B;
        const int64_t kb = (so[m] / ba.d[m] + 1) * ba.d[m];
        kb_s[m] = (int)kb;
        nk_s[m] = kb < g.dims[m] ? (int)((g.dims[m] - kb) / BK) : 0;
      }
    }
  }
  // column tables: column c of mode j = local coordinates of the modes != j (earliest fastest)
  for (int e = tid; e < N * TC; e += kBlkThreads) {
    const int j = e / TC;
    int x = e % TC, o = 0;
#pragma unroll
    for (int m = 0; m < N; ++m) {
      if (m == j) continue;
      o += (x & (B - 1)) * (int)g.strides[m];
      x >>= LB;
    }
    colg[e] = o;
  }
  auto bar_addr = [](uint64_t* b) { return (unsigned)__cvta_generic_to_shared(b); };
  if (tid == 0) {
    for (int st = 0; st < ST; ++st) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar_addr(&fullb[st])), "r"(kBlkThreads));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar_addr(&emptyb[st])), "r"(kBlkThreads / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid < N * B) dd[tid / B][tid % B] = T[g.toff[tid / B] + (so[tid / B] + tid % B) * (g.dims[tid / B] + 1)];
  int64_t base = ba.boff ? ba.boff[tb] : 0;  // tile origin
  const double2 dext = ba.boff ? ba.bden[tb] : make_double2(0.0, 0.0);
#pragma unroll
  for (int m = 0; m < N; ++m) base += so[m] * g.strides[m];
  int nkt = 0;
#pragma unroll
  for (int m = 0; m < N; ++m) nkt += nk_s[m];

  // ---- producer: k-tile t of the mode sequence (modes with no coupling have nk = 0) ----
  int pj = 0, pkt = 0;  // producer cursor
  auto advance = [&](int& j, int& kt) {
    ++kt;
    while (j < N && kt >= nk_s[j]) {
      kt = 0;
      ++j;
    }
  };
  while (pj < N && nk_s[pj] == 0) ++pj;
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
  // producer per-thread state of its current mode: the SL elements' offsets inside a stage (the
  // same for every k-tile of the mode), rebuilt only when the producer moves to another mode
  int p_mode = -1;
  int64_t p_gofs[SL];
  int p_soff[SL];
  const double2* p_src = nullptr;  // row 0 of mode p_mode through the tile's other coordinates
  int64_t p_sj = 0;
  auto producer_mode = [&](int j) {
    p_mode = j;
    p_sj = g.strides[j];
    p_src = Y + (base - so[j] * p_sj);
    const int* cg = colg + j * TC;
#pragma unroll
    for (int i = 0; i < SL; ++i) {
      const int e = tid + i * kBlkThreads;
      int k, c;
      if (j == 0) {  // mode 1: contiguous along k in HBM — k-fastest smem, XOR swizzle
        k = e % BK;
        c = e / BK;
        p_soff[i] = c * BK + (k ^ (BK >= 8 ? (c & 1) << 2 : 0));
      } else {
        c = e % TC;
        k = e / TC;
        p_soff[i] = k * LDB + c;
      }
      p_gofs[i] = (int64_t)k * p_sj + cg[c];
    }
  };
  auto load_stage = [&](int stage) {  // the producer cursor's k-tile into `stage`
    const int j = pj;
    if (j != p_mode) producer_mode(j);
    const int k0 = kb_s[j] + pkt * BK;
    const double2* src = p_src + (int64_t)k0 * p_sj;
    double2* dB = sB + stage * C::BSTAGE;
#pragma unroll
    for (int i = 0; i < SL; ++i) cp_async16_bs(dB + p_soff[i], src + p_gofs[i]);
    for (int e = tid; e < B * BK; e += kBlkThreads) {  // T'_j(so_j + r, k0 + k), rows fastest (coalesced)
      const int r = e % B, k = e / B;
      cp_async16_bs(sA + stage * C::ASTAGE + r * ALD + k,
                    T + g.toff[j] + (so[j] + r) + (int64_t)(k0 + k) * g.dims[j]);
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar_addr(&fullb[stage])) : "memory");
    advance(pj, pkt);
  };
#pragma unroll
  for (int st = 0; st < ST; ++st)
    if (st < nkt) load_stage(st);
  // the tile itself (C) into shared memory while the first stages are in flight
  {
    constexpr int PER = E / kBlkThreads;
    double2 v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int l = tid + i * kBlkThreads;
      int64_t o = 0;
#pragma unroll
      for (int m = 0; m < N; ++m) o += ((l >> (LB * m)) & (B - 1)) * g.strides[m];
      v[i] = Y[base + o];
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) sS[tid + i * kBlkThreads] = v[i];
  }

  // ---- consumer ----
  double cre[RB][CB][2], cim[RB][CB][2], c3[RB][CB][2];
  auto zero = [&]() {
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int q = 0; q < CB; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) cre[r][q][h] = cim[r][q][h] = c3[r][q][h] = 0.0;
  };
  zero();
  const int cbase = warp * CB * 8 + (lane >> 2);
  const int arow = lane >> 2, kq = lane & 3;
  int cj = 0, ckt = 0;
  while (cj < N && nk_s[cj] == 0) ++cj;
  for (int t = 0; t < nkt; ++t) {
    if (t >= 1 && t - 1 + ST < nkt) {  // refill the stage k-tile t - 1 used
      const int st = (t - 1) % ST;
      mb_wait(&emptyb[st], ((t - 1) / ST) & 1);
      load_stage(st);
    }
    mb_wait(&fullb[t % ST], (t / ST) & 1);
    const double2* cA = sA + (t % ST) * C::ASTAGE;
    const double2* cBs = sB + (t % ST) * C::BSTAGE;
    // all of the k-tile's fragments are loaded before its DMMAs (the layout branch is per k-tile,
    // so the loads of both 4-deep steps issue back to back)
    double2 bv[BK / 4][CB], av[BK / 4][RB];
    if (cj == 0) {  // mode 1: k-fastest swizzled stage
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk)
#pragma unroll
        for (int q = 0; q < CB; ++q) {
          const int c = cbase + q * 8;
          bv[kk][q] = cBs[c * BK + ((kk * 4 + kq) ^ (BK >= 8 ? (c & 1) << 2 : 0))];
        }
    } else {
#pragma unroll
      for (int kk = 0; kk < BK / 4; ++kk)
#pragma unroll
        for (int q = 0; q < CB; ++q) bv[kk][q] = cBs[(kk * 4 + kq) * LDB + cbase + q * 8];
    }
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk)
#pragma unroll
      for (int r = 0; r < RB; ++r) av[kk][r] = cA[(r * 8 + arow) * ALD + kk * 4 + kq];
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double bs[CB];
#pragma unroll
      for (int q = 0; q < CB; ++q) bs[q] = bv[kk][q].x + bv[kk][q].y;
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const double2 a = av[kk][r];
        const double as = a.x + a.y;
#pragma unroll
        for (int q = 0; q < CB; ++q) {
          dmma_bs(cre[r][q][0], cre[r][q][1], a.x, bv[kk][q].x);
          dmma_bs(cim[r][q][0], cim[r][q][1], a.y, bv[kk][q].y);
          dmma_bs(c3[r][q][0], c3[r][q][1], as, bs[q]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar_addr(&emptyb[t % ST])) : "memory");
    if (++ckt == nk_s[cj]) {  // mode cj done: S -= its GEMM (modes in turn: CTA barrier first)
      __syncthreads();
      const int bsj = 1 << (LB * cj);
#pragma unroll
      for (int q = 0; q < CB; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = warp * CB * 8 + q * 8 + 2 * kq + h;
          // local index of column c for mode cj (the modes != cj in order, earliest fastest)
          int x = c, lo = 0;
#pragma unroll
          for (int m = 0; m < N; ++m) {
            if (m == cj) continue;
            lo += (x & (B - 1)) << (LB * m);
            x >>= LB;
          }
#pragma unroll
          for (int r = 0; r < RB; ++r) {
            const int l = lo + (r * 8 + arow) * bsj;
            sS[l] = csub(sS[l], make_double2(cre[r][q][h] - cim[r][q][h], c3[r][q][h] - cre[r][q][h] - cim[r][q][h]));
          }
        }
      zero();
      ckt = 0;
      ++cj;
      while (cj < N && nk_s[cj] == 0) ++cj;
    }
  }
  __syncthreads();
  constexpr int PER = E / kBlkThreads;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int l = tid + i * kBlkThreads;
    double2 den = cadd(dext, dd[0][l & (B - 1)]);
    int64_t o = l & (B - 1);
#pragma unroll
    for (int m = 1; m < N; ++m) {
      const int lm = (l >> (LB * m)) & (B - 1);
      den = cadd(den, dd[m][lm]);
      o += lm * g.strides[m];
    }
    Y[base + o] = cmul(sS[l], crecip_fast(den));
  }
}

using BlkKernel = void (*)(const BlkArgs, const double2*, const int64_t*, double2*);
struct BlkLaunchT {
  BlkKernel kern;
  size_t smem;
  int threads;
};
// Measured (c1 / c3 solve): N = 3 — 256 threads, BK = 8, 3 stages: 1.31 ms (512 threads 1.37,
// 4 stages 1.34, BK = 16 x 2 stages 1.46 / 1.49 with 512 threads); N = 4 — 512 threads, BK = 4,
// 3 stages: 18.1 ms (256 threads 19.9, 4 stages 20.1, BK = 8 x 2 stages 18.9 / 19.3). After the
// producer-offset change (c1 1.195 ms): N = 3 with BK = 4 x 2 stages at 2 CTAs / SM (128
// registers, spills) 1.169, BK = 4 x 3 stages 1.34.
// End of round 2 (c2 is the only BASELINE config left on 8^4 tiles: D = (32, 32, 32, 16), twelve
// short levels): 8^4 with a 4-stage ring 5.11 ms against 5.51 with three (four stages and 256
// threads 5.52, 1024 threads 5.82, BK = 8 x 2 stages 5.26); 16^3 with four stages
// 0.768 (c1) / 10.25 ms (c3) against 0.716 / 9.46 with three.
static BlkLaunchT blk_cfg(int n_modes, int b) {
  if (n_modes == 3 && b == 16) return {blk_level_kernel<3, 16, 8, 3, 256>, BlkCfg<3, 16, 8, 3, 256>::smem(), 256};
  if (n_modes == 4 && b == 8) return {blk_level_kernel<4, 8, 4, 4, 512>, BlkCfg<4, 8, 4, 4, 512>::smem(), 512};
  return {nullptr, 0, 0};
}
