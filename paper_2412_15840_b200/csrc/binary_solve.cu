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
};

__device__ __forceinline__ unsigned bs_smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bs_mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bs_smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// Per tile (one CTA, 256 threads, 3 CTAs / SM):
//   1. pull — the tile's own slab and its neighbour slabs (outer modes with bit 0, ascending) are
//      streamed through a ring of four 16 KB slots by bulk asynchronous copies (cp.async.bulk,
//      TMA engine) completing on per-slot mbarriers; thread t accumulates its 16 entries
//      l = t + 256 i in registers (own value, then q ascending: the reference's per-entry order);
//      the producer (thread 0) refills a slot as soon as all eight warps released it, so up to
//      four 16 KB pieces per CTA (192 KB per SM) are in flight;
//   2. the ring's 64 KB becomes the tile S; local popcount wavefront, highest level first;
//   3. store the slab.
__global__ void __launch_bounds__(kBinSolveThreads, 3) binary_tile_solve_kernel(const BinSolveGeom g,
                                                                              const int64_t* __restrict__ tiles,
                                                                              const int* __restrict__ wf,
                                                                              const int* __restrict__ wf_off,
                                                                              double2* __restrict__ Y) {
  extern __shared__ __align__(128) double2 S[];  // 2^m entries; first the pull ring (4 x 1024)
  __shared__ double2 t01[64], t00[64], t11[64];
  __shared__ double2 dlo[64], dhi[64];  // den(l) = dlo[l & 63] + dhi[l >> 6] (outer part in dhi)
  __shared__ double2 dout;
  __shared__ __align__(8) uint64_t full[4], empty[4];
  constexpr int kSlot = 1024;  // entries per ring slot (16 KB)
  const int tid = threadIdx.x, lane = tid & 31;
  const int N = g.m + g.n_outer;
  const int E = 1 << g.m;
  const int mlo = g.m < 6 ? g.m : 6, mhi = g.m - mlo;
  const int64_t I = tiles[blockIdx.x];  // outer index (bit q = outer mode m + q)
  for (int j = tid; j < N; j += blockDim.x) {
    t00[j] = g.t[4 * j + 0];
    t01[j] = g.t[4 * j + 2];
    t11[j] = g.t[4 * j + 3];
  }
  const int64_t base = I << g.m;
  // pieces: the own slab, then each neighbour slab (q ascending), E / kSlot pieces per slab
  const int ppb = E >= kSlot ? E / kSlot : 1;        // pieces per slab
  const int pbytes = (E >= kSlot ? kSlot : E) * 16;  // bytes per piece
  int nsrc = 1;
  for (int q = 0; q < g.n_outer; ++q) nsrc += ((I >> q) & 1) ? 0 : 1;
  const int npieces = nsrc * ppb;
  auto piece_src = [&](int i) {  // global address of piece i
    const int src = i / ppb, p = i % ppb;
    int64_t off = base;
    if (src > 0) {  // the src-th zero bit of I
      int seen = 0;
      for (int q = 0; q < g.n_outer; ++q)
        if (!((I >> q) & 1) && ++seen == src) {
          off = base + ((int64_t)1 << (g.m + q));
          break;
        }
    }
    return Y + off + (int64_t)p * kSlot;
  };
  auto issue = [&](int i) {
    const int slot = i & 3;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bs_smem_u32(&full[slot])),
                 "r"(pbytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     bs_smem_u32(S + slot * kSlot)),
                 "l"(piece_src(i)), "r"(pbytes), "r"(bs_smem_u32(&full[slot]))
                 : "memory");
  };
  if (tid == 0) {
    for (int s2 = 0; s2 < 4; ++s2) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bs_smem_u32(&full[s2])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bs_smem_u32(&empty[s2])),
                   "r"(kBinSolveThreads / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int i = 0; i < 4 && i < npieces; ++i) issue(i);
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
  // 1. pull: acc[i] holds entry tid + 256 i; piece p of a slab holds entries [1024 p, 1024 p + 1024)
  constexpr int PER = 4096 / kBinSolveThreads;
  double2 acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = make_double2(0.0, 0.0);
  int piece = 0, q = -1;
  for (int src = 0; src < nsrc; ++src) {
    double2 c = make_double2(0.0, 0.0);
    if (src > 0) {
      do {
        ++q;
      } while ((I >> q) & 1);
      c = t01[g.m + q];
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      if (p < ppb) {
        const int slot = piece & 3;
        if (tid == 0 && piece >= 1 && piece + 3 < npieces) {  // refill the slot piece - 1 used
          bs_mbar_wait(&empty[(piece - 1) & 3], ((piece - 1) >> 2) & 1);
          issue(piece + 3);
        }
        bs_mbar_wait(&full[slot], (piece >> 2) & 1);
        const double2* v = S + slot * kSlot;
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          const int li = tid + i2 * kBinSolveThreads;  // entry within the piece
          if (li < (pbytes >> 4)) {
            const double2 x = v[li];
            acc[p * 4 + i2] = src == 0 ? x : cfms(acc[p * 4 + i2], c, x);
          }
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bs_smem_u32(&empty[slot])) : "memory");
        ++piece;
      }
    }
  }
  __syncthreads();  // every piece consumed: the ring becomes the tile
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int l = tid + i * kBinSolveThreads;
    if (l < E) S[l] = acc[i];
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
  const size_t bytes = ntiles * sizeof(int64_t) + (E + m + 2) * sizeof(int);
  NDS_CUDA(cudaMalloc(&bp.pool, bytes));
  bp.d_tiles = (int64_t*)bp.pool;
  bp.d_wf = (int*)(bp.d_tiles + ntiles);
  bp.d_wf_off = bp.d_wf + E;
  NDS_CUDA(cudaMemcpy(bp.d_tiles, tiles.data(), ntiles * sizeof(int64_t), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(bp.d_wf, wf.data(), E * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(bp.d_wf_off, wf_off.data(), (m + 2) * sizeof(int), cudaMemcpyHostToDevice));
}

void binary_solve_plan_free(BinarySolvePlan& bp) {
  if (bp.pool) cudaFree(bp.pool);
  bp.pool = nullptr;
}

int binary_solve_launch(const BinarySolvePlan& bp, const double2* t_pool, double2* c, cudaStream_t stream,
                        Recorder* rec) {
  static bool attr_set = false;
  auto kern = binary_tile_solve_kernel;
  if (!attr_set) {
    NDS_CUDA(cudaFuncSetAttribute(binary_tile_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 16));
    attr_set = true;
  }
  BinSolveGeom g{bp.m, bp.n_outer, bp.m + 1, t_pool};
  const size_t smem = std::max<size_t>(((size_t)1 << bp.m) * sizeof(double2), 4 * 1024 * sizeof(double2));
  int launches = 0;
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
  if (binary)
    binary_solve_plan_free(bsp);
  else
    solve_plan_free(sp);
}
}  // namespace nds
