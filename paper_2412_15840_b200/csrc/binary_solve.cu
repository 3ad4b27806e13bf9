// Triangular solve for the all-binary regime (every n_j = 2; BASELINE config c4, N = 29).
//
// Reference: back_substitute, sylvester.cpp:71-108. With n_j = 2 every T_j is
// [[t00, t01], [0, t11]] and entry i depends on i + e_j for each mode j with i_j = 0 (coefficient
// t01 of mode j). Tiles are the contiguous 2^m-entry slabs of the first m = min(N, 12) modes
// (one coalesced 64 KB chunk each); the remaining N - m "outer" modes index the tiles. A tile
// depends on the tiles whose outer index differs by one set bit, so all tiles with the same outer
// popcount are independent: one launch per outer level, highest first. Per tile:
//   1. pull: C_I -= sum_{outer j, I_j = 0} t01_j * Y_{I + e_j}  (contiguous neighbour slabs),
//   2. local solve over the 2^m inner entries by popcount level, highest first, entry l:
//        y(l) = (c(l) - sum_{inner j, l_j = 0} t01_j y(l | e_j)) / den(l),
//      den(l) = sum_j T_j(i_j, i_j) over all N modes (inner bits of l, outer bits of I),
//   3. store the slab.
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace nds {

constexpr int kBinSolveThreads = 256;

struct BinSolveGeom {
  int m;              // inner (tile) modes; tile = 2^m entries
  int n_outer;        // N - m
  int wf_levels;      // m + 1
  const double2* t;   // per mode j: T_j (2x2 column-major) at t + 4 j
  int pull;           // 0: decoupled tiles (outer modes diagonalised into the transforms)
};

__global__ void __launch_bounds__(kBinSolveThreads, 3) binary_tile_solve_kernel(const BinSolveGeom g,
                                                                              const int64_t* __restrict__ tiles,
                                                                              const int* __restrict__ wf,
                                                                              const int* __restrict__ wf_off,
                                                                              double2* __restrict__ Y) {
  extern __shared__ __align__(16) double2 S[];  // 2^m entries
  __shared__ double2 t01[64], t00[64], t11[64];
  __shared__ double2 dlo[64], dhi[64];  // den(l) = dlo[l & 63] + dhi[l >> 6] (outer part in dhi)
  __shared__ double2 dout;
  const int tid = threadIdx.x;
  const int N = g.m + g.n_outer;
  const int E = 1 << g.m;
  const int mlo = g.m < 6 ? g.m : 6, mhi = g.m - mlo;
  const int64_t I = tiles[blockIdx.x];  // outer index (bit q = outer mode m + q)
  for (int j = tid; j < N; j += blockDim.x) {
    t00[j] = g.t[4 * j + 0];
    t01[j] = g.t[4 * j + 2];
    t11[j] = g.t[4 * j + 3];
  }
  __syncthreads();
  if (tid == 0) {
    double2 d = make_double2(0.0, 0.0);
    for (int q = 0; q < g.n_outer; ++q) d = cadd(d, ((I >> q) & 1) ? t11[g.m + q] : t00[g.m + q]);
    dout = d;
  }
  __syncthreads();
  if (tid < 64) {  // inner modes 0..mlo-1
    double2 d = make_double2(0.0, 0.0);
    for (int j = 0; j < mlo; ++j) d = cadd(d, ((tid >> j) & 1) ? t11[j] : t00[j]);
    dlo[tid] = d;
  } else if (tid < 128) {  // inner modes mlo..m-1, then the outer modes
    const int x = tid - 64;
    double2 d = make_double2(0.0, 0.0);
    for (int j = 0; j < mhi; ++j) d = cadd(d, ((x >> j) & 1) ? t11[mlo + j] : t00[mlo + j]);
    dhi[x] = cadd(d, dout);
  }
  const int64_t base = I << g.m;
  // 1. load + pull from neighbour slabs (outer modes with bit 0). The running sums live in shared
  //    memory (each thread owns the same entries l = tid + i * 256 throughout, so no barrier), so
  //    registers hold only loads in flight: a whole slab per thread (two slabs, software-
  //    pipelined, spill at 2 CTAs/SM and measured slower). Same per-entry order as the reference:
  //    own value, then q ascending.
  constexpr int PER = 4096 / kBinSolveThreads;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int l = tid + i * kBinSolveThreads;
    if (l < E) S[l] = Y[base + l];
  }
  auto load_slab = [&](int q, double2 (&v)[PER]) {
    const double2* nb = Y + base + ((int64_t)1 << (g.m + q));
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int l = tid + i * kBinSolveThreads;
      v[i] = l < E ? __ldcg(nb + l) : make_double2(0.0, 0.0);
    }
  };
  auto apply = [&](int q, const double2 (&v)[PER]) {
    const double2 c = t01[g.m + q];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int l = tid + i * kBinSolveThreads;
      if (l < E) S[l] = cfms(S[l], c, v[i]);
    }
  };
  for (int q = 0; q < g.n_outer && g.pull; ++q) {
    if ((I >> q) & 1) continue;  // CTA-uniform
    double2 v[PER];
    load_slab(q, v);
    apply(q, v);
  }
  __syncthreads();
  // 2. local popcount wavefront, highest level first; inner-mode terms in mode order (loop fully
  //    unrolled so the neighbour loads issue early; den from the two half tables)
  for (int lv = 0; lv < g.wf_levels; ++lv) {
    const int p1 = wf_off[lv + 1];
    for (int p = wf_off[lv] + tid; p < p1; p += blockDim.x) {
      const int l = wf[p];
      double2 num = S[l];
#pragma unroll
      for (int j = 0; j < 12; ++j)
        if (j < g.m && !((l >> j) & 1)) num = cfms(num, t01[j], S[l | (1 << j)]);
      S[l] = cmul(num, crecip_fast(cadd(dlo[l & 63], dhi[l >> mlo])));
    }
    __syncthreads();
  }
  // 3. store
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int l = tid + i * kBinSolveThreads;
    if (l < E) Y[base + l] = S[l];
  }
}

void binary_solve_plan_build(BinarySolvePlan& bp, int n_modes) {
  const int m = std::min(n_modes, 12);
  bp.m = m;
  bp.n_outer = n_modes - m;
  const int64_t ntiles = (int64_t)1 << bp.n_outer;
  bp.levels = bp.n_outer + 1;
  // tiles by outer popcount, highest first
  std::vector<int64_t> tiles(ntiles);
  bp.level_off.assign(bp.levels + 1, 0);
  std::vector<int64_t> cnt(bp.levels, 0);
  for (int64_t t = 0; t < ntiles; ++t) cnt[bp.n_outer - __builtin_popcountll(t)]++;
  for (int i = 0; i < bp.levels; ++i) bp.level_off[i + 1] = bp.level_off[i] + cnt[i];
  {
    std::vector<int64_t> pos(bp.level_off.begin(), bp.level_off.end() - 1);
    for (int64_t t = ntiles - 1; t >= 0; --t) tiles[pos[bp.n_outer - __builtin_popcountll(t)]++] = t;
  }
  // local entries by popcount, highest first
  const int E = 1 << m;
  std::vector<int> wf(E), wf_off(m + 2, 0), wcnt(m + 1, 0);
  for (int l = 0; l < E; ++l) wcnt[m - __builtin_popcount(l)]++;
  for (int i = 0; i <= m; ++i) wf_off[i + 1] = wf_off[i] + wcnt[i];
  {
    std::vector<int> pos(wf_off.begin(), wf_off.end() - 1);
    for (int l = E - 1; l >= 0; --l) wf[pos[m - __builtin_popcount(l)]++] = l;
  }
  // the fused kernel's order (binary_pass.cu, swizzled tile): within a level, entries
  // round-robin over the 16-byte bank group of their swizzled slot, so the lanes of an 8-lane
  // shared-memory phase hit distinct groups (the term loads XOR the slot with a constant, which
  // keeps them distinct)
  std::vector<uint16_t> wfs(E);
  {
    auto swz = [](int q) { return q ^ (((q >> 3) ^ (q >> 6) ^ (q >> 9)) & 7); };
    for (int lv = 0; lv <= m; ++lv) {
      std::vector<std::vector<int>> bucket(8);
      for (int i = wf_off[lv]; i < wf_off[lv + 1]; ++i) bucket[swz(wf[i]) & 7].push_back(wf[i]);
      int o = wf_off[lv];
      for (size_t r = 0; o < wf_off[lv + 1]; ++r)
        for (int b = 0; b < 8; ++b)
          if (r < bucket[b].size()) wfs[o++] = (uint16_t)bucket[b][r];
    }
  }
  const size_t bytes = ntiles * sizeof(int64_t) + (E + m + 2) * sizeof(int) + E * sizeof(uint16_t) + 16;
  NDS_CUDA(cudaMalloc(&bp.pool, bytes));
  bp.d_tiles = (int64_t*)bp.pool;
  bp.d_wf = (int*)(bp.d_tiles + ntiles);
  bp.d_wf_off = bp.d_wf + E;
  bp.d_wf_swz = (uint16_t*)(bp.d_wf_off + m + 2);
  NDS_CUDA(cudaMemcpy(bp.d_wf_swz, wfs.data(), E * sizeof(uint16_t), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(bp.d_tiles, tiles.data(), ntiles * sizeof(int64_t), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(bp.d_wf, wf.data(), E * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(bp.d_wf_off, wf_off.data(), (m + 2) * sizeof(int), cudaMemcpyHostToDevice));
}

void binary_solve_plan_free(BinarySolvePlan& bp) {
  if (bp.pool) cudaFree(bp.pool);
  bp.pool = nullptr;
}

int binary_solve_launch(const BinarySolvePlan& bp, const double2* t_pool, double2* c, cudaStream_t stream,
                        Recorder* rec, bool decoupled) {
  auto kern = binary_tile_solve_kernel;
  smem_optin(binary_tile_solve_kernel, 4096 * 16);
  BinSolveGeom g{bp.m, bp.n_outer, bp.m + 1, t_pool, decoupled ? 0 : 1};
  const size_t smem = ((size_t)1 << bp.m) * sizeof(double2);
  int launches = 0;
  if (decoupled) {  // every tile independent: one launch, no neighbour pulls
    const int64_t n = bp.level_off.back();
    kern<<<(unsigned)n, kBinSolveThreads, smem, stream>>>(g, bp.d_tiles, bp.d_wf, bp.d_wf_off, c);
    NDS_LAUNCH_CHECK();
    if (rec) rec->mark(stream, kBacksubLevel, 0);
    return 1;
  }
  for (int lv = 0; lv < bp.levels; ++lv) {
    const int64_t n = bp.level_off[lv + 1] - bp.level_off[lv];
    kern<<<(unsigned)n, kBinSolveThreads, smem, stream>>>(g, bp.d_tiles + bp.level_off[lv],
                                                                              bp.d_wf, bp.d_wf_off, c);
    NDS_LAUNCH_CHECK();
    if (rec) rec->mark(stream, kBacksubLevel, lv);
    ++launches;
  }
  return launches;
}

}  // namespace nds

namespace nds {
SolverCache::~SolverCache() {
  for (auto& kv : blk) blk_solve_plan_free(kv.second);
  for (auto& kv : bin_wf) cudaFree(kv.second);
  if (binary)
    binary_solve_plan_free(bsp);
  else
    solve_plan_free(sp);
}
}  // namespace nds
