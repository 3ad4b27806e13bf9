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
  // Local wavefront order of a full tile, highest local hyperplane first.
  std::vector<int> wf_count(wf_levels + 1, 0), wf(g.tile_entries), wf_lev(g.tile_entries);
  for (int l = 0; l < g.tile_entries; ++l) {
    int r = l, lv = 0;
    for (int j = 0; j < n_modes; ++j) {
      lv += r % g.b[j];
      r /= g.b[j];
    }
    wf_lev[l] = lv;
    wf_count[wf_levels - 1 - lv]++;
  }
  std::vector<int> wf_off(wf_levels + 1, 0);
  for (int i = 0; i < wf_levels; ++i) wf_off[i + 1] = wf_off[i] + wf_count[i];
  {
    std::vector<int> pos(wf_off.begin(), wf_off.end() - 1);
    for (int l = 0; l < g.tile_entries; ++l) wf[pos[wf_levels - 1 - wf_lev[l]]++] = l;
  }
  const size_t bytes = ntiles * sizeof(int64_t) + (g.tile_entries + wf_levels + 1) * sizeof(int) + 64;
  NDS_CUDA(cudaMalloc(&sp.pool, bytes));
  sp.d_tiles = (int64_t*)sp.pool;
  sp.d_wf = (int*)(sp.d_tiles + ntiles);
  sp.d_wf_off = sp.d_wf + g.tile_entries;
  NDS_CUDA(cudaMemcpy(sp.d_tiles, tiles.data(), ntiles * sizeof(int64_t), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf, wf.data(), g.tile_entries * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf_off, wf_off.data(), (wf_levels + 1) * sizeof(int), cudaMemcpyHostToDevice));
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
    attr_set = true;
  }
  const size_t smem = (size_t)sp.geom.tile_entries * sizeof(double2);
  int launches = 0;
  for (int lv = 0; lv < sp.levels; ++lv) {
    const int64_t count = sp.level_off[lv + 1] - sp.level_off[lv];
    if (count == 0) continue;
    tile_level_kernel<<<(unsigned)count, kSolveThreads, smem, stream>>>(sp.geom, t_pool, sp.d_tiles + sp.level_off[lv],
                                                                        sp.d_wf, sp.d_wf_off, sp.wf_levels, c);
    NDS_LAUNCH_CHECK();
    if (rec) rec->mark(stream, kBacksubLevel, lv);
    ++launches;
  }
  return launches;
}

}  // namespace nds
