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
#include <cstdio>
#include <string>
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


#include "backsub_v2.cuh"
#include "backsub_blk.cuh"

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

// The cubic route needs 4096-entry tiles with the same b in {8, 16} dividing every extent.
static bool gemm_regime(const TileGeom& g) {
  if (g.tile_entries != kMaxTile) return false;
  if (!lines_kernel_for(g.n_modes, g.b[0])) return false;
  for (int j = 0; j < g.n_modes; ++j)
    if (g.b[j] != g.b[0] || g.dims[j] % g.b[j]) return false;
  return true;
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
  std::vector<int64_t> slot_of(ntiles);
  for (int64_t s2 = 0; s2 < ntiles; ++s2) slot_of[tiles[s2]] = s2;
  std::vector<int64_t> tstride(n_modes, 1);
  for (int j = 1; j < n_modes; ++j) tstride[j] = tstride[j - 1] * g.nb[j - 1];

  // Generic tiles: local wavefront order of a full tile, highest local hyperplane first.
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

  // Cubic route work lists. Per level and tile (level order) and mode j with off-tile rows:
  //   near — rows [(I_j + 1) b, (I_j + 2) b): the adjacent block; computed by the diagonal CTA
  //          of tile I + e_j one level earlier (near_target) into the level-parity near buffer;
  //   far  — rows >= (I_j + 2) b: neighbours two or more blocks away, final one level early;
  //          one item per (tile, mode) writing ring slot (lv % fg_ring, slot), longest first.
  std::vector<int4> tile_ranges(ntiles, make_int4(0, 0, 0, 0));
  std::vector<int> near_target;
  std::vector<FarGroupItem> fg_items;
  sp.near_off.assign(levels + 1, 0);
  sp.fg_off.assign(levels + 1, 0);
  sp.max_near = 0;
  sp.fg_ring = 3;  // far(lv) overlaps diag(lv - 1) and far(lv +- 1): three live level regions
  sp.fg_slots = 1;
  if (sp.v2) {
    near_target.assign((size_t)ntiles * n_modes, -1);
    int64_t near_total = 0;
    for (int lv = 0; lv < levels; ++lv) {
      std::vector<FarGroupItem> items;
      int64_t nnear = 0, nslot = 0;
      for (int64_t s2 = sp.level_off[lv]; s2 < sp.level_off[lv + 1]; ++s2) {
        int64_t r = tiles[s2];
        const int64_t far_first = nslot, near_first = nnear;
        for (int j = 0; j < n_modes; ++j) {
          const int64_t I = r % g.nb[j];
          r /= g.nb[j];
          const int64_t b = g.b[j];
          if ((I + 1) * b < g.dims[j]) {
            near_target[(size_t)slot_of[tiles[s2] + tstride[j]] * n_modes + j] = (int)nnear;
            ++nnear;
          }
          if ((I + 2) * b < g.dims[j]) {
            FarGroupItem it{};
            it.tile = (int)s2;
            it.j = j;
            it.kb = (int)((I + 2) * b);
            it.ke = (int)g.dims[j];
            it.rb0 = (int)I;
            it.nrb = 1;
            it.acc = 0;
            for (int q = 0; q < 4; ++q) it.out[q] = -1;
            it.out[0] = (int)nslot++;  // level-relative; the ring region is added below
            items.push_back(it);
          }
        }
        tile_ranges[s2] = make_int4((int)far_first, (int)(nslot - far_first), (int)near_first, (int)(nnear - near_first));
      }
      near_total += nnear;
      sp.near_off[lv + 1] = near_total;
      sp.max_near = std::max(sp.max_near, nnear);
      sp.fg_slots = std::max(sp.fg_slots, nslot);
      // longest first (LPT): the short items fill the launch's tail
      std::stable_sort(items.begin(), items.end(),
                       [](const FarGroupItem& x, const FarGroupItem& y) { return x.ke - x.kb > y.ke - y.kb; });
      for (auto& it : items) fg_items.push_back(it);
      sp.fg_off[lv + 1] = (int64_t)fg_items.size();
    }
    for (int lv = 0; lv < levels; ++lv)
      for (int64_t i = sp.fg_off[lv]; i < sp.fg_off[lv + 1]; ++i)
        fg_items[i].out[0] += (int)((lv % sp.fg_ring) * sp.fg_slots);
  }

  size_t bytes = ntiles * sizeof(int64_t) + (g.tile_entries + wf_levels + 1) * sizeof(int) + 64;
  bytes = (bytes + 15) / 16 * 16;
  const size_t nt_off = bytes;
  bytes += near_target.size() * sizeof(int);
  bytes = (bytes + 15) / 16 * 16;
  const size_t ranges_off = bytes;
  bytes += (size_t)ntiles * sizeof(int4);
  bytes = (bytes + 15) / 16 * 16;
  const size_t fg_items_off = bytes;
  bytes += fg_items.size() * sizeof(FarGroupItem);
  bytes = (bytes + 255) / 256 * 256;
  const size_t partial_off = bytes;
  const size_t tile_bytes = (size_t)g.tile_entries * sizeof(double2);
  if (sp.v2) bytes += ((size_t)sp.fg_ring * sp.fg_slots + 2 * (size_t)sp.max_near) * tile_bytes + 256;
  NDS_CUDA(cudaMalloc(&sp.pool, bytes));
  char* base = (char*)sp.pool;
  sp.d_tiles = (int64_t*)base;
  sp.d_wf = (int*)(sp.d_tiles + ntiles);
  sp.d_wf_off = sp.d_wf + g.tile_entries;
  sp.d_near_target = (int*)(base + nt_off);
  sp.d_tile_ranges = (int4*)(base + ranges_off);
  sp.d_fg_items = (FarGroupItem*)(base + fg_items_off);
  NDS_CUDA(cudaMemcpy(sp.d_tiles, tiles.data(), ntiles * sizeof(int64_t), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf, wf.data(), g.tile_entries * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf_off, wf_off.data(), (wf_levels + 1) * sizeof(int), cudaMemcpyHostToDevice));
  if (sp.v2) {
    sp.d_fg_ring = (double2*)(base + partial_off);
    sp.d_near_partial = sp.d_fg_ring + (size_t)sp.fg_ring * sp.fg_slots * g.tile_entries;
    sp.d_near_partial2 = sp.d_near_partial + (size_t)sp.max_near * g.tile_entries;
    NDS_CUDA(cudaMemcpy(sp.d_near_target, near_target.data(), near_target.size() * sizeof(int), cudaMemcpyHostToDevice));
    NDS_CUDA(cudaMemcpy(sp.d_tile_ranges, tile_ranges.data(), ntiles * sizeof(int4), cudaMemcpyHostToDevice));
    if (!fg_items.empty())
      NDS_CUDA(cudaMemcpy(sp.d_fg_items, fg_items.data(), fg_items.size() * sizeof(FarGroupItem),
                          cudaMemcpyHostToDevice));
    // critical path (diagonal tiles) on a high-priority stream, far updates on low-priority ones
    int lo = 0, hi = 0;
    NDS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    NDS_CUDA(cudaStreamCreateWithPriority(&sp.s_crit, cudaStreamNonBlocking, hi));
    NDS_CUDA(cudaStreamCreateWithPriority(&sp.s_far, cudaStreamNonBlocking, lo));
    NDS_CUDA(cudaStreamCreateWithPriority(&sp.s_far2, cudaStreamNonBlocking, lo));
    sp.ev.resize(2 * levels + 2);
    for (auto& e : sp.ev) NDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
}

void solve_plan_free(SolvePlan& sp) {
  if (sp.pool) cudaFree(sp.pool);
  sp.pool = nullptr;
  for (auto e : sp.ev) cudaEventDestroy(e);
  sp.ev.clear();
  if (sp.s_crit) cudaStreamDestroy(sp.s_crit);
  if (sp.s_far) cudaStreamDestroy(sp.s_far);
  if (sp.s_far2) cudaStreamDestroy(sp.s_far2);
  sp.s_crit = sp.s_far = sp.s_far2 = nullptr;
}

int backsub_launch(const SolvePlan& sp, const double2* t_pool, double2* c, cudaStream_t stream, Recorder* rec,
                   const HeadSync* head, const TailHook* tail) {
  smem_optin(tile_level_kernel, kMaxTile * sizeof(double2));
  for (int b : {8, 16}) smem_optin(far_group_cfg(b).kern, far_group_smem_bytes(b));
  smem_optin(lines_kernel_for(3, 16), 112 * 1024);
  smem_optin(lines_kernel_for(4, 8), 112 * 1024);
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
  const int b = g.b[0];
  const LinesKernel lines = lines_kernel_for(g.n_modes, b);
  const size_t lines_smem = lines_smem_bytes(g.n_modes, b);
  const FarGroupCfg fgc = far_group_cfg(b);
  const size_t fg_smem = far_group_smem_bytes(b);
  const int L = sp.levels;
  cudaEvent_t ev_start = sp.ev[2 * L], ev_end = sp.ev[2 * L + 1];
  // NDS_SOLVE_TRACE=1 (diagnostic, tools/solve_trace.py): per-level start/end events of every
  // launch printed to stderr after the solve.
  static const bool trace = getenv("NDS_SOLVE_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t s, int lv, int k) {
    if (!trace) return;
    NDS_CUDA(cudaEventRecord(tev[(size_t)lv * 6 + k], s));
  };
  if (trace) {
    tev.resize((size_t)L * 6 + 1);
    for (auto& e : tev) NDS_CUDA(cudaEventCreate(&e));
    NDS_CUDA(cudaEventRecord(tev.back(), stream));
  }
  auto ev_diag = [&](int lv) { return sp.ev[lv]; };
  auto ev_far = [&](int lv) { return sp.ev[L + lv]; };
  // fork: the internal streams start after everything already queued on the caller's stream
  NDS_CUDA(cudaEventRecord(ev_start, stream));
  NDS_CUDA(cudaStreamWaitEvent(sp.s_crit, ev_start, 0));
  NDS_CUDA(cudaStreamWaitEvent(sp.s_far, ev_start, 0));
  NDS_CUDA(cudaStreamWaitEvent(sp.s_far2, ev_start, 0));
  if (rec) rec->mark(stream, -1, 0);
  int head_waited = -1;
  for (int lv = 0; lv < L; ++lv) {
    const int64_t nf = sp.fg_off[lv + 1] - sp.fg_off[lv];
    double2* far_buf = sp.d_fg_ring + (size_t)(lv % sp.fg_ring) * sp.fg_slots * g.tile_entries;
    if (nf > 0) {
      // far(lv) needs levels <= lv - 2 only: it overlaps diag(lv - 1) on the critical stream, and
      // even / odd levels use two streams so far(lv) may start while far(lv - 1) drains
      cudaStream_t fs = (lv & 1) ? sp.s_far2 : sp.s_far;
      if (lv >= 2) NDS_CUDA(cudaStreamWaitEvent(fs, ev_diag(lv - 2), 0));
      tmark(fs, lv, 0);
      fgc.kern<<<(unsigned)(nf * fgc.h), kUpdThreads, fg_smem, fs>>>(g, t_pool, sp.d_tiles,
                                                                    sp.d_fg_items + sp.fg_off[lv], sp.d_fg_ring, c);
      NDS_LAUNCH_CHECK();
      tmark(fs, lv, 1);
      NDS_CUDA(cudaEventRecord(ev_far(lv), fs));
      ++launches;
      NDS_CUDA(cudaStreamWaitEvent(sp.s_crit, ev_far(lv), 0));
    }
    double2* near_in = (lv & 1) ? sp.d_near_partial2 : sp.d_near_partial;
    double2* near_out = (lv & 1) ? sp.d_near_partial : sp.d_near_partial2;  // level lv + 1's buffer
    if (head && head->per > 0) {  // C rows of the lowest mode-N block on this level must be ready
      const int N = g.n_modes;
      int64_t rest = 0;
      for (int m = 0; m < N - 1; ++m) rest += g.nb[m] - 1;
      const int64_t sum = (int64_t)(L - 1) - lv;
      const int64_t bmin = std::max<int64_t>(0, sum - rest);
      const int grp = (int)((g.nb[N - 1] - 1 - bmin) / head->per);
      if (grp > head_waited) {
        for (int q = head_waited + 1; q <= grp; ++q) NDS_CUDA(cudaStreamWaitEvent(sp.s_crit, head->ev[q], 0));
        head_waited = grp;
      }
    }
    const int64_t nt = sp.level_off[lv + 1] - sp.level_off[lv];
    tmark(sp.s_crit, lv, 4);
    lines<<<(unsigned)nt, diag_threads_for(g.n_modes), lines_smem, sp.s_crit>>>(
        g, t_pool, sp.d_tiles + sp.level_off[lv], sp.d_tile_ranges + sp.level_off[lv], far_buf, near_in,
        sp.d_near_target + sp.level_off[lv] * g.n_modes, near_out, c);
    NDS_LAUNCH_CHECK();
    tmark(sp.s_crit, lv, 5);
    NDS_CUDA(cudaEventRecord(ev_diag(lv), sp.s_crit));
    ++launches;
    if (tail && tail->fn) tail->fn(tail->ctx, lv, sp.s_crit);
  }
  // join back into the caller's stream
  NDS_CUDA(cudaEventRecord(ev_end, sp.s_crit));
  NDS_CUDA(cudaStreamWaitEvent(stream, ev_end, 0));
  if (rec) rec->mark(stream, kBacksubPersistent, L);
  if (trace) {
    NDS_CUDA(cudaStreamSynchronize(stream));
    for (int lv = 0; lv < L; ++lv) {
      const int64_t nf = sp.fg_off[lv + 1] - sp.fg_off[lv];
      float t[6] = {-1, -1, -1, -1, -1, -1};
      for (int k = 0; k < 6; ++k) {
        if ((k < 2 && nf == 0) || k == 2 || k == 3) continue;
        NDS_CUDA(cudaEventElapsedTime(&t[k], tev.back(), tev[(size_t)lv * 6 + k]));
      }
      fprintf(stderr, "TRACE %d %lld %lld %lld %.1f %.1f %.1f %.1f %.1f %.1f\n", lv,
              (long long)(sp.level_off[lv + 1] - sp.level_off[lv]), (long long)nf, 0LL, t[0] * 1e3, t[1] * 1e3,
              t[2] * 1e3, t[3] * 1e3, t[4] * 1e3, t[5] * 1e3);
    }
    for (auto e : tev) cudaEventDestroy(e);
  }
  return launches;
}

// Geometry of the route: the coupled modes (D_j < n_j) tiled by the instantiated kernel of their
// count (3: 16^3, 4: 8^4 — the tile edge must divide every coupled D_j), the uncoupled modes a
// batch (c3: D = (64, 128, 64, 64) -> 16^3 tiles over modes 1, 3, 4 for each mode-2 index: solve
// 12.6 -> 9.5 ms, 16-row fragments instead of 8); otherwise every mode is tiled (cubic edge b)
// and the uncoupled ones simply have no couplings.
void blk_solve_plan_build(BlkSolvePlan& bp, int n_modes, const int64_t* dims, const int64_t* toff, const int* d,
                          int b) {
  std::vector<int> cm, um;
  for (int j = 0; j < n_modes; ++j) {
    (d[j] < dims[j] ? cm : um).push_back(j);
    bp.dmode[j] = d[j];
  }
  const int nc = (int)cm.size();
  // (two coupled modes are not folded: the 64^2 tile kernel — every warp on all 64 rows — measured
  // 0.78 ms against 0.71 for 16^3 tiles with the uncoupled mode tiled, c1)
  const int bc = nc == 3 ? 16 : nc == 4 ? 8 : 0;
  bool fold = bc > 0 && !um.empty();
  for (int j : cm) fold = fold && d[j] % bc == 0 && dims[j] % bc == 0;
  if (!fold) {  // all modes tiled
    cm.clear();
    um.clear();
    for (int j = 0; j < n_modes; ++j) cm.push_back(j);
  }
  const int bt = fold ? bc : b;
  int64_t gstride[NDS_MAX_MODES];
  {
    int64_t acc = 1;
    for (int j = 0; j < n_modes; ++j) {
      gstride[j] = acc;
      acc *= dims[j];
    }
  }
  TileGeom& g = bp.g;
  g = TileGeom{};
  g.n_modes = (int)cm.size();
  int64_t ntc = 1;
  int bacc = 1, levels = 1;
  for (int i = 0; i < g.n_modes; ++i) {
    const int j = cm[i];
    bp.d[i] = d[j];
    g.dims[i] = dims[j];
    g.strides[i] = gstride[j];
    g.b[i] = bt;
    g.bstride[i] = bacc;
    bacc *= bt;
    g.nb[i] = dims[j] / bt;
    g.toff[i] = toff[j];
    ntc *= g.nb[i];
    levels += (int)(dims[j] / d[j] - 1);
  }
  g.tile_entries = bacc;
  bp.levels = levels;
  bp.ntc = ntc;
  bp.uncoupled = um;
  int64_t nbatch = 1;
  for (int j : um) nbatch *= dims[j];
  bp.nbatch = fold ? nbatch : 1;
  struct Tl {
    int lv;
    int64_t k;  // rows pulled (all modes)
    int64_t id;
  };
  std::vector<Tl> ts((size_t)ntc);
  for (int64_t t = 0; t < ntc; ++t) {
    int64_t r = t, k = 0;
    int lv = 0;
    for (int i = 0; i < g.n_modes; ++i) {
      const int64_t I = r % g.nb[i];
      r /= g.nb[i];
      const int64_t sb = I * g.b[i] / bp.d[i];
      lv += (int)sb;
      k += g.dims[i] - (sb + 1) * bp.d[i];
    }
    ts[t] = {levels - 1 - lv, k, t};
  }
  std::stable_sort(ts.begin(), ts.end(), [](const Tl& x, const Tl& y) { return x.lv != y.lv ? x.lv < y.lv : x.k > y.k; });
  // a level's tiles: its coupled tiles (longest first) for every batch index
  bp.level_off.assign(levels + 1, 0);
  std::vector<int64_t> ids;
  ids.reserve((size_t)(ntc * bp.nbatch));
  for (int lv = 0, i = 0; lv < levels; ++lv) {
    const int i0 = i;
    while (i < (int)ntc && ts[i].lv == lv) ++i;
    for (int64_t tb = 0; tb < bp.nbatch; ++tb)
      for (int q = i0; q < i; ++q) ids.push_back(ts[q].id + ntc * tb);
    bp.level_off[lv + 1] = (int64_t)ids.size();
  }
  const size_t tb_bytes = ids.size() * sizeof(int64_t);
  NDS_CUDA(cudaMalloc(&bp.d_tiles, tb_bytes + (size_t)bp.nbatch * sizeof(int64_t)));
  NDS_CUDA(cudaMemcpy(bp.d_tiles, ids.data(), tb_bytes, cudaMemcpyHostToDevice));
  bp.d_boff = nullptr;
  if (fold) {  // batch origin offsets (mixed radix over the uncoupled modes, earliest fastest)
    std::vector<int64_t> boff((size_t)nbatch);
    for (int64_t tb = 0; tb < nbatch; ++tb) {
      int64_t r = tb, o = 0;
      for (int j : um) {
        o += (r % dims[j]) * gstride[j];
        r /= dims[j];
      }
      boff[tb] = o;
    }
    bp.d_boff = bp.d_tiles + ids.size();
    NDS_CUDA(cudaMemcpy(bp.d_boff, boff.data(), (size_t)nbatch * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
}

void blk_solve_plan_free(BlkSolvePlan& bp) {
  if (bp.d_tiles) cudaFree(bp.d_tiles);
  bp.d_tiles = nullptr;
  bp.d_boff = nullptr;
}

// den_b = sum over the uncoupled modes of T_j(i_j, i_j) for batch index b (diag at g.doff)
__global__ void blk_batch_den_kernel(const Geom g, const double2* __restrict__ diag, BlkBatchModes um,
                                     int64_t nbatch, double2* __restrict__ out) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nbatch; b += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = b;
    double2 s = make_double2(0.0, 0.0);
    for (int i = 0; i < um.count; ++i) {
      const int j = um.mode[i];
      s = cadd(s, diag[g.doff[j] + r % g.dims[j]]);
      r /= g.dims[j];
    }
    out[b] = s;
  }
}

void blk_batch_den_launch(const BlkSolvePlan& bp, const Geom& g, const double2* diag, double2* out,
                          cudaStream_t stream) {
  if (bp.nbatch <= 1 || bp.uncoupled.empty()) return;
  BlkBatchModes um{};
  um.count = (int)bp.uncoupled.size();
  for (int i = 0; i < um.count; ++i) um.mode[i] = bp.uncoupled[i];
  blk_batch_den_kernel<<<(unsigned)std::min<int64_t>((bp.nbatch + 255) / 256, 1024), 256, 0, stream>>>(
      g, diag, um, bp.nbatch, out);
  NDS_LAUNCH_CHECK();
}

int blk_backsub_launch(const BlkSolvePlan& bp, const double2* t_pool, const double2* bden, double2* c,
                       cudaStream_t stream, Recorder* rec) {
  const TileGeom& g = bp.g;
  const BlkLaunchT bl = blk_cfg(g.n_modes, g.b[0]);
  if (!bl.kern) throw Error(NDS_ERR_OTHER, "block-diagonalised solve: no level kernel for this tile geometry");
  smem_optin(bl.kern, bl.smem);
  BlkArgs ba;
  ba.g = g;
  for (int j = 0; j < NDS_MAX_MODES; ++j) ba.d[j] = j < g.n_modes ? bp.d[j] : 1;
  ba.boff = bp.d_boff;
  ba.bden = bden;
  ba.ntc = bp.ntc;
  int launches = 0;
  for (int lv = 0; lv < bp.levels; ++lv) {
    const int64_t nt = bp.level_off[lv + 1] - bp.level_off[lv];
    if (nt == 0) continue;
    bl.kern<<<(unsigned)nt, bl.threads, bl.smem, stream>>>(ba, t_pool, bp.d_tiles + bp.level_off[lv], c);
    NDS_LAUNCH_CHECK();
    if (rec) rec->mark(stream, kBacksubLevel, lv);
    ++launches;
  }
  return launches;
}

}  // namespace nds
