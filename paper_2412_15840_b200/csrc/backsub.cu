// Blocked N-D triangular solve  sum_j T_j x_j Y = C  (T_j upper triangular), in place.
//
// Reference: back_substitute, sylvester.cpp:71-108 — one serial pass over all multi-indices in
// descending flat order (paper Alg. 3), entry update Eq. (9):
//   y(i) = (c(i) - sum_j sum_{k > i_j} T_j(i_j, k) y(i with i_j -> k)) / sum_j T_j(i_j, i_j).
//
// B200 formulation. The index space is cut into tiles of prod_j b_j entries (b_j per mode, tile
// <= kMaxTile entries so a tile fits in shared memory). Every dependency of an entry lies at a
// larger index along exactly one mode, so tile I depends only on tiles I + m e_j (m > 0), and all
// tiles on one tile-hyperplane sum_j I_j = s are independent. Per hyperplane (descending) one
// launch solves all its tiles, one CTA per tile:
//   1. pull: C_I -= sum_j T_j(I_j rows, k > tile) x_j Y   (off-tile updates, coalesced along mode 1)
//   2. diagonal tile: anti-diagonal wavefront over local hyperplanes sum_j l_j = t, each entry
//      divided by sum_j T_j(i_j, i_j) (same summation order as sylvester.cpp:92-96),
//   3. write Y_I back.
#include <algorithm>
#include <numeric>

#include "common.cuh"
#include "kernels.h"

namespace nds {

constexpr int kMaxTile = 4096;   // entries per tile (64 KB of complex128 in shared memory)
constexpr int kSolveThreads = 256;

__global__ void __launch_bounds__(kSolveThreads) tile_level_kernel(const TileGeom g, const double2* __restrict__ T,
                                                                   const int64_t* __restrict__ tiles,
                                                                   const int* __restrict__ wf,
                                                                   const int* __restrict__ wf_off, int wf_levels,
                                                                   double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 S[];
  __shared__ int64_t so[NDS_MAX_MODES];
  __shared__ int se[NDS_MAX_MODES];
  const int N = g.n_modes;
  if (threadIdx.x == 0) {
    int64_t t = tiles[blockIdx.x];
    for (int j = 0; j < N; ++j) {
      const int64_t I = t % g.nb[j];
      t /= g.nb[j];
      so[j] = I * g.b[j];
      const int64_t rest = g.dims[j] - so[j];
      se[j] = (int)(rest < g.b[j] ? rest : g.b[j]);
    }
  }
  __syncthreads();

  // 1. load C_I and subtract the off-tile couplings
  for (int l = threadIdx.x; l < g.tile_entries; l += blockDim.x) {
    int rem = l;
    int64_t gidx = 0;
    bool inside = true;
    for (int j = 0; j < N; ++j) {
      const int lj = rem % g.b[j];
      rem /= g.b[j];
      inside &= lj < se[j];
      gidx += (so[j] + lj) * g.strides[j];
    }
    if (!inside) continue;
    double2 acc = Y[gidx];
    rem = l;
    for (int j = 0; j < N; ++j) {
      const int lj = rem % g.b[j];
      rem /= g.b[j];
      const int64_t nj = g.dims[j];
      const int64_t ij = so[j] + lj;
      const double2* Tj = T + g.toff[j];
      const int64_t st = g.strides[j];
      for (int64_t k = so[j] + se[j]; k < nj; ++k) acc = cfms(acc, __ldg(Tj + ij + k * nj), Y[gidx + (k - ij) * st]);
    }
    S[l] = acc;
  }
  __syncthreads();

  // 2. wavefront over local hyperplanes (descending)
  for (int lv = 0; lv < wf_levels; ++lv) {
    const int p1 = wf_off[lv + 1];
    for (int p = wf_off[lv] + threadIdx.x; p < p1; p += blockDim.x) {
      const int l = wf[p];
      int rem = l;
      bool inside = true;
      for (int j = 0; j < N; ++j) {
        const int lj = rem % g.b[j];
        rem /= g.b[j];
        inside &= lj < se[j];
      }
      if (!inside) continue;
      double2 num = S[l];
      double2 den = make_double2(0.0, 0.0);
      rem = l;
      for (int j = 0; j < N; ++j) {
        const int lj = rem % g.b[j];
        rem /= g.b[j];
        const int64_t nj = g.dims[j];
        const int64_t ij = so[j] + lj;
        const double2* Tj = T + g.toff[j];
        den = cadd(den, __ldg(Tj + ij + ij * nj));
        const int bs = g.bstride[j];
        for (int k = lj + 1; k < se[j]; ++k) num = cfms(num, __ldg(Tj + ij + (so[j] + k) * nj), S[l + (k - lj) * bs]);
      }
      S[l] = cdiv(num, den);
    }
    __syncthreads();
  }

  // 3. store Y_I
  for (int l = threadIdx.x; l < g.tile_entries; l += blockDim.x) {
    int rem = l;
    int64_t gidx = 0;
    bool inside = true;
    for (int j = 0; j < N; ++j) {
      const int lj = rem % g.b[j];
      rem /= g.b[j];
      inside &= lj < se[j];
      gidx += (so[j] + lj) * g.strides[j];
    }
    if (inside) Y[gidx] = S[l];
  }
}


// =============================================================================================
// v2 — GEMM regime (every b_j a power of two >= 8 dividing n_j).
// =============================================================================================

constexpr int kUpdThreads = 256;
constexpr int kALd = 12;  // A stage row stride (complex): = 4 mod 8 -> conflict-free fragments

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

// Off-tile coupling of one work item, as a small complex GEMM on the FP64 tensor pipe:
//   partial(l_j, c) = sum_{k in [kb, ke)} T_j(o_j + l_j, k) * Y(k along mode j, c)
// rows = local index along mode j (b_j), columns c = the other local coordinates of the tile
// (cols = E / b_j), K streamed from global through a 3-stage cp.async ring.
// The partial is written in tile-local column-major order (coalesced for the diagonal kernel).
__global__ void __launch_bounds__(kUpdThreads, 2)
    tile_update_kernel(const TileGeom g, const double2* __restrict__ T, const int64_t* __restrict__ tiles,
                       const int4* __restrict__ items, double2* __restrict__ partial, const double2* __restrict__ Y,
                       int bk) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ int64_t so[NDS_MAX_MODES];
  __shared__ int64_t s_base;
  const int4 it = items[blockIdx.x];
  const int j = it.y, kb = it.z, ke = it.w;
  const int N = g.n_modes;
  const int E = g.tile_entries;
  const int bj = g.b[j];
  const int cols = E / bj;
  const int ldb = cols + 2;  // = 2 mod 8 -> conflict-free B fragments
  int64_t* colg = (int64_t*)sm;           // global offset of column c
  int* coll = (int*)(colg + cols);        // local offset of column c
  double2* sA = (double2*)(coll + cols + (cols & 1));  // [3][bj][kALd]
  double2* sB = sA + 3 * bj * kALd;                     // [3][bk][ldb]
  if (threadIdx.x == 0) {
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
  // column tables: c enumerates the local coordinates of modes != j, earliest mode fastest
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    int rem = c;
    int64_t og = 0;
    int ol = 0;
    for (int m = 0; m < N; ++m) {
      if (m == j) continue;
      const int lm = rem & (g.b[m] - 1);
      rem >>= __ffs(g.b[m]) - 1;
      og += lm * g.strides[m];
      ol += lm * g.bstride[m];
    }
    colg[c] = og;
    coll[c] = ol;
  }
  __syncthreads();
  const int64_t base = s_base;
  const int64_t sj = g.strides[j];
  const int64_t nj = g.dims[j];
  const double2* Tj = T + g.toff[j];
  const int oj = (int)so[j];

  auto load_stage = [&](int stage, int k0) {
    double2* dA = sA + stage * bj * kALd;
    double2* dB = sB + stage * bk * ldb;
    // A: T_j rows oj..oj+bj, cols k0..k0+bk (zero past ke)
    for (int e = threadIdx.x; e < bj * bk; e += blockDim.x) {
      const int r = e / bk, k = e % bk;
      const int gk = k0 + k;
      if (gk < ke)
        cp_async16_bs(dA + r * kALd + k, Tj + (oj + r) + (int64_t)gk * nj);
      else
        dA[r * kALd + k] = make_double2(0.0, 0.0);
    }
    // B: Y rows k0..k0+bk along mode j, all tile columns
    const int total = bk * cols;
    if (j == 0) {  // mode 1 is contiguous along k: k fastest
      for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int k = e % bk, c = e / bk;
        const int gk = k0 + k;
        if (gk < ke)
          cp_async16_bs(dB + k * ldb + c, Y + base + (int64_t)gk * sj + colg[c]);
        else
          dB[k * ldb + c] = make_double2(0.0, 0.0);
      }
    } else {
      for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int c = e % cols, k = e / cols;
        const int gk = k0 + k;
        if (gk < ke)
          cp_async16_bs(dB + k * ldb + c, Y + base + (int64_t)gk * sj + colg[c]);
        else
          dB[k * ldb + c] = make_double2(0.0, 0.0);
      }
    }
  };

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rb_count = bj >> 3;
  // each warp owns 8 fragments (8x8): f = warp * 8 + q
  double cre[8][2], cim[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) cre[q][0] = cre[q][1] = cim[q][0] = cim[q][1] = 0.0;

  const int nk = (ke - kb + bk - 1) / bk;
  load_stage(0, kb);
  cp_commit_bs();
  if (nk > 1) load_stage(1, kb + bk);
  cp_commit_bs();
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait1_bs();
    __syncthreads();
    if (kt + 2 < nk) load_stage((kt + 2) % 3, kb + (kt + 2) * bk);
    cp_commit_bs();
    const double2* cA = sA + (kt % 3) * bj * kALd;
    const double2* cB = sB + (kt % 3) * bk * ldb;
    for (int kk = 0; kk < bk; kk += 4) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int f = warp * 8 + q;
        const int rb = f % rb_count, cb = f / rb_count;
        const double2 a = cA[(rb * 8 + (lane >> 2)) * kALd + kk + (lane & 3)];
        const double2 b = cB[(kk + (lane & 3)) * ldb + cb * 8 + (lane >> 2)];
        dmma_bs(cre[q][0], cre[q][1], a.x, b.x);
        dmma_bs(cim[q][0], cim[q][1], a.x, b.y);
        dmma_bs(cre[q][0], cre[q][1], -a.y, b.y);
        dmma_bs(cim[q][0], cim[q][1], a.y, b.x);
      }
    }
  }
  cp_wait0_bs();
  double2* out = partial + (int64_t)blockIdx.x * E;
  const int bsj = g.bstride[j];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int f = warp * 8 + q;
    const int rb = f % rb_count, cb = f / rb_count;
    const int r = rb * 8 + (lane >> 2);
    const int c = cb * 8 + 2 * (lane & 3);
    out[r * bsj + coll[c]] = make_double2(cre[q][0], cim[q][0]);
    out[r * bsj + coll[c + 1]] = make_double2(cre[q][1], cim[q][1]);
  }
}

// Diagonal tile: S = C_I - sum(partials), then the local anti-diagonal wavefront. On local
// hyperplane t every entry gets `grp` lanes that split its sum_j sum_{k > l_j} terms and combine
// them with warp shuffles; the group leader divides by sum_j T_j(i_j, i_j).
__global__ void __launch_bounds__(kSolveThreads)
    tile_diag_kernel(const TileGeom g, const double2* __restrict__ T, const int64_t* __restrict__ tiles,
                     const int2* __restrict__ tile_items, const double2* __restrict__ partial, int64_t item_base,
                     const int* __restrict__ wf, const int* __restrict__ wf_off, const int* __restrict__ wf_group,
                     int wf_levels, double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 S[];
  __shared__ int64_t so[NDS_MAX_MODES];
  __shared__ int sh_shift[NDS_MAX_MODES];
  const int N = g.n_modes;
  const int E = g.tile_entries;
  double2* Td = S + E;  // diagonal blocks T_j(o_j.., o_j..), b_j x b_j column-major each
  const int64_t slot = blockIdx.x;  // global tile slot offset added by the caller via `tiles`
  if (threadIdx.x == 0) {
    int64_t t = tiles[slot];
    for (int m = 0; m < N; ++m) {
      const int64_t I = t % g.nb[m];
      t /= g.nb[m];
      so[m] = I * g.b[m];
      sh_shift[m] = __ffs(g.bstride[m]) - 1;  // log2 of the local stride (powers of two)
    }
  }
  __syncthreads();
  // diagonal blocks
  {
    int off = 0;
    for (int m = 0; m < N; ++m) {
      const int bm = g.b[m];
      const double2* Tm = T + g.toff[m];
      const int64_t nm = g.dims[m];
      for (int e = threadIdx.x; e < bm * bm; e += blockDim.x) {
        const int r = e % bm, c = e / bm;
        Td[off + e] = Tm[(so[m] + r) + (so[m] + c) * nm];
      }
      off += bm * bm;
    }
  }
  // load C_I minus the partials of this tile (fixed order -> deterministic)
  const int2 ti = tile_items[slot];
  for (int l = threadIdx.x; l < E; l += blockDim.x) {
    int64_t gidx = 0;
    for (int m = 0; m < N; ++m) gidx += (so[m] + ((l >> sh_shift[m]) & (g.b[m] - 1))) * g.strides[m];
    double2 v = Y[gidx];
    for (int p = 0; p < ti.y; ++p) v = csub(v, partial[(int64_t)(ti.x - item_base + p) * E + l]);
    S[l] = v;
  }
  __syncthreads();

  for (int lv = 0; lv < wf_levels; ++lv) {
    const int p0 = wf_off[lv], cnt = wf_off[lv + 1] - p0;
    const int grp = wf_group[lv];
    const int rounds = (cnt * grp + blockDim.x - 1) / blockDim.x;
    for (int rd = 0; rd < rounds; ++rd) {
      const int idx = rd * blockDim.x + threadIdx.x;
      const int e = idx / grp, sub = idx % grp;
      double2 acc = make_double2(0.0, 0.0);
      int l = 0;
      if (e < cnt) {
        l = wf[p0 + e];
        int off = 0;
        for (int m = 0; m < N; ++m) {
          const int bm = g.b[m];
          const int lm = (l >> sh_shift[m]) & (bm - 1);
          const double2* Tm = Td + off;
          const int bs = g.bstride[m];
          for (int k = lm + 1 + sub; k < bm; k += grp) acc = cfma(acc, Tm[lm + k * bm], S[l + (k - lm) * bs]);
          off += bm * bm;
        }
      }
      for (int o = 1; o < grp; o <<= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (e < cnt && sub == 0) {
        double2 den = make_double2(0.0, 0.0);
        int off = 0;
        for (int m = 0; m < N; ++m) {
          const int bm = g.b[m];
          const int lm = (l >> sh_shift[m]) & (bm - 1);
          den = cadd(den, Td[off + lm + lm * bm]);
          off += bm * bm;
        }
        S[l] = cdiv(csub(S[l], acc), den);
      }
    }
    __syncthreads();
  }
  for (int l = threadIdx.x; l < E; l += blockDim.x) {
    int64_t gidx = 0;
    for (int m = 0; m < N; ++m) gidx += (so[m] + ((l >> sh_shift[m]) & (g.b[m] - 1))) * g.strides[m];
    Y[gidx] = S[l];
  }
}

// Tile shape: grow the smallest extents first (earlier modes win ties, keeping tiles contiguous
// along mode 1) while prod b_j <= kMaxTile.
static void choose_tile(int n_modes, const int64_t* dims, int* b) {
  for (int j = 0; j < n_modes; ++j) b[j] = 1;
  int64_t entries = 1;
  for (;;) {
    int best = -1;
    for (int j = 0; j < n_modes; ++j) {
      if (b[j] >= dims[j]) continue;
      const int64_t nb = std::min<int64_t>(dims[j], (int64_t)b[j] * 2);
      if (entries / b[j] * nb > kMaxTile) continue;
      if (best < 0 || b[j] < b[best]) best = j;
    }
    if (best < 0) break;
    const int64_t nb = std::min<int64_t>(dims[best], (int64_t)b[best] * 2);
    entries = entries / b[best] * nb;
    b[best] = (int)nb;
  }
}

static bool gemm_regime(const TileGeom& g) {
  if (g.tile_entries != kMaxTile) return false;
  for (int j = 0; j < g.n_modes; ++j) {
    const int b = g.b[j];
    if (b < 8 || (b & (b - 1)) || g.dims[j] % b) return false;
  }
  return true;
}

static int update_bk(const TileGeom& g, int j) { return (g.tile_entries / g.b[j]) > 256 ? 4 : 8; }

static size_t update_smem(const TileGeom& g, int j) {
  const int cols = g.tile_entries / g.b[j];
  const int bk = update_bk(g, j);
  return (size_t)cols * (8 + 4) + 16 + (size_t)3 * g.b[j] * kALd * 16 + (size_t)3 * bk * (cols + 2) * 16;
}

void solve_plan_build(SolvePlan& sp, int n_modes, const int64_t* dims, const int64_t* toff) {
  TileGeom& g = sp.geom;
  g = TileGeom{};
  g.n_modes = n_modes;
  choose_tile(n_modes, dims, g.b);
  int64_t acc = 1;
  int bacc = 1;
  int64_t ntiles = 1;
  int levels = 1;
  int wf_levels = 1;
  for (int j = 0; j < n_modes; ++j) {
    g.dims[j] = dims[j];
    g.strides[j] = acc;
    acc *= dims[j];
    g.bstride[j] = bacc;
    bacc *= g.b[j];
    g.nb[j] = (dims[j] + g.b[j] - 1) / g.b[j];
    g.toff[j] = toff[j];
    ntiles *= g.nb[j];
    levels += (int)(g.nb[j] - 1);
    wf_levels += g.b[j] - 1;
  }
  g.tile_entries = bacc;
  sp.levels = levels;
  sp.wf_levels = wf_levels;
  sp.v2 = gemm_regime(g);

  // Tiles grouped by hyperplane, highest first (counting sort on the level).
  std::vector<int64_t> lev_count(levels + 1, 0);
  std::vector<int> tile_level(ntiles);
  for (int64_t t = 0; t < ntiles; ++t) {
    int64_t r = t;
    int lv = 0;
    for (int j = 0; j < n_modes; ++j) {
      lv += (int)(r % g.nb[j]);
      r /= g.nb[j];
    }
    tile_level[t] = lv;
    lev_count[levels - 1 - lv]++;
  }
  sp.level_off.assign(levels + 1, 0);
  for (int i = 0; i < levels; ++i) sp.level_off[i + 1] = sp.level_off[i] + lev_count[i];
  std::vector<int64_t> tiles(ntiles);
  {
    std::vector<int64_t> pos(sp.level_off.begin(), sp.level_off.end() - 1);
    for (int64_t t = 0; t < ntiles; ++t) tiles[pos[levels - 1 - tile_level[t]]++] = t;
  }
  // Local wavefront order of a full tile, highest local hyperplane first, and lanes per entry.
  std::vector<int> wf_count(wf_levels + 1, 0), wf(g.tile_entries), wf_lev(g.tile_entries), wf_terms(wf_levels, 0);
  for (int l = 0; l < g.tile_entries; ++l) {
    int r = l, lv = 0, terms = 0;
    for (int j = 0; j < n_modes; ++j) {
      const int lj = r % g.b[j];
      lv += lj;
      terms += g.b[j] - 1 - lj;
      r /= g.b[j];
    }
    wf_lev[l] = lv;
    wf_count[wf_levels - 1 - lv]++;
    wf_terms[wf_levels - 1 - lv] = std::max(wf_terms[wf_levels - 1 - lv], terms);
  }
  std::vector<int> wf_off(wf_levels + 1, 0), wf_group(wf_levels, 1);
  for (int i = 0; i < wf_levels; ++i) {
    wf_off[i + 1] = wf_off[i] + wf_count[i];
    int grp = 1;
    while (grp < 32 && wf_count[i] * grp * 2 <= kSolveThreads && grp * 2 <= std::max(1, wf_terms[i] / 2)) grp *= 2;
    wf_group[i] = grp;
  }
  {
    std::vector<int> pos(wf_off.begin(), wf_off.end() - 1);
    for (int l = 0; l < g.tile_entries; ++l) wf[pos[wf_levels - 1 - wf_lev[l]]++] = l;
  }

  // v2 work items: per level, per tile (level order), per mode with off-tile rows, k-chunks.
  std::vector<int4> items;
  std::vector<int2> tile_items(ntiles, make_int2(0, 0));
  sp.item_off.assign(levels + 1, 0);
  sp.max_level_items = 0;
  if (sp.v2) {
    for (int lv = 0; lv < levels; ++lv) {
      int64_t natural = 0, rows = 0;
      for (int64_t s = sp.level_off[lv]; s < sp.level_off[lv + 1]; ++s) {
        int64_t r = tiles[s];
        for (int j = 0; j < n_modes; ++j) {
          const int64_t I = r % g.nb[j];
          r /= g.nb[j];
          const int64_t K = g.dims[j] - (I + 1) * g.b[j];
          if (K > 0) {
            ++natural;
            rows += K;
          }
        }
      }
      // split k only when the level has too few natural items to fill 2 CTAs per SM
      int64_t kc = INT64_MAX;
      if (natural > 0 && natural < 2 * 148) kc = std::max<int64_t>(32, ((rows + 295) / 296 + 7) / 8 * 8);
      for (int64_t s = sp.level_off[lv]; s < sp.level_off[lv + 1]; ++s) {
        int64_t r = tiles[s];
        const int first = (int)items.size();
        for (int j = 0; j < n_modes; ++j) {
          const int64_t I = r % g.nb[j];
          r /= g.nb[j];
          const int64_t k0 = (I + 1) * g.b[j];
          for (int64_t kb = k0; kb < g.dims[j]; kb += std::min<int64_t>(kc, g.dims[j])) {
            const int64_t ke = std::min<int64_t>(g.dims[j], kc == INT64_MAX ? g.dims[j] : kb + kc);
            items.push_back(make_int4((int)s, j, (int)kb, (int)ke));
          }
        }
        tile_items[s] = make_int2(first, (int)items.size() - first);
      }
      sp.item_off[lv + 1] = (int64_t)items.size();
      sp.max_level_items = std::max(sp.max_level_items, sp.item_off[lv + 1] - sp.item_off[lv]);
    }
  }

  size_t bytes = ntiles * sizeof(int64_t) + (g.tile_entries + 2 * wf_levels + 2) * sizeof(int);
  bytes = (bytes + 15) / 16 * 16;
  const size_t items_off = bytes;
  bytes += items.size() * sizeof(int4) + ntiles * sizeof(int2);
  bytes = (bytes + 255) / 256 * 256;
  const size_t partial_off = bytes;
  bytes += (size_t)sp.max_level_items * g.tile_entries * sizeof(double2) + 256;
  NDS_CUDA(cudaMalloc(&sp.pool, bytes));
  char* base = (char*)sp.pool;
  sp.d_tiles = (int64_t*)base;
  sp.d_wf = (int*)(sp.d_tiles + ntiles);
  sp.d_wf_off = sp.d_wf + g.tile_entries;
  sp.d_wf_group = sp.d_wf_off + wf_levels + 1;
  sp.d_items = (int4*)(base + items_off);
  sp.d_tile_items = (int2*)(sp.d_items + items.size());
  sp.d_partial = (double2*)(base + partial_off);
  NDS_CUDA(cudaMemcpy(sp.d_tiles, tiles.data(), ntiles * sizeof(int64_t), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf, wf.data(), g.tile_entries * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf_off, wf_off.data(), (wf_levels + 1) * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf_group, wf_group.data(), wf_levels * sizeof(int), cudaMemcpyHostToDevice));
  if (!items.empty()) {
    NDS_CUDA(cudaMemcpy(sp.d_items, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice));
    NDS_CUDA(cudaMemcpy(sp.d_tile_items, tile_items.data(), ntiles * sizeof(int2), cudaMemcpyHostToDevice));
  }
}

void solve_plan_free(SolvePlan& sp) {
  if (sp.pool) cudaFree(sp.pool);
  sp.pool = nullptr;
}

int backsub_launch(const SolvePlan& sp, const double2* t_pool, double2* c, cudaStream_t stream, Recorder* rec) {
  static bool attr_set = false;
  if (!attr_set) {
    NDS_CUDA(cudaFuncSetAttribute(tile_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kMaxTile * sizeof(double2))));
    NDS_CUDA(cudaFuncSetAttribute(tile_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
    NDS_CUDA(cudaFuncSetAttribute(tile_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
    attr_set = true;
  }
  const TileGeom& g = sp.geom;
  int launches = 0;
  if (!sp.v2) {
    const size_t smem = (size_t)g.tile_entries * sizeof(double2);
    for (int lv = 0; lv < sp.levels; ++lv) {
      const int64_t count = sp.level_off[lv + 1] - sp.level_off[lv];
      if (count == 0) continue;
      tile_level_kernel<<<(unsigned)count, kSolveThreads, smem, stream>>>(g, t_pool, sp.d_tiles + sp.level_off[lv],
                                                                          sp.d_wf, sp.d_wf_off, sp.wf_levels, c);
      NDS_LAUNCH_CHECK();
      if (rec) rec->mark(stream, kBacksubLevel, lv);
      ++launches;
    }
    return launches;
  }
  size_t upd_smem = 0;
  int bk = 8;
  for (int j = 0; j < g.n_modes; ++j) {
    upd_smem = std::max(upd_smem, update_smem(g, j));
    bk = std::min(bk, update_bk(g, j));
  }
  size_t diag_smem = (size_t)g.tile_entries * sizeof(double2);
  for (int j = 0; j < g.n_modes; ++j) diag_smem += (size_t)g.b[j] * g.b[j] * sizeof(double2);
  for (int lv = 0; lv < sp.levels; ++lv) {
    const int64_t ni = sp.item_off[lv + 1] - sp.item_off[lv];
    if (ni > 0) {
      tile_update_kernel<<<(unsigned)ni, kUpdThreads, upd_smem, stream>>>(g, t_pool, sp.d_tiles, sp.d_items + sp.item_off[lv],
                                                                          sp.d_partial, c, bk);
      NDS_LAUNCH_CHECK();
      if (rec) rec->mark(stream, kBacksubLevel, lv);
      ++launches;
    }
    const int64_t nt = sp.level_off[lv + 1] - sp.level_off[lv];
    tile_diag_kernel<<<(unsigned)nt, kSolveThreads, diag_smem, stream>>>(
        g, t_pool, sp.d_tiles + sp.level_off[lv], sp.d_tile_items + sp.level_off[lv], sp.d_partial, sp.item_off[lv],
        sp.d_wf, sp.d_wf_off, sp.d_wf_group, sp.wf_levels, c);
    NDS_LAUNCH_CHECK();
    if (rec) rec->mark(stream, kBacksubLevel, lv);
    ++launches;
  }
  return launches;
}

}  // namespace nds
