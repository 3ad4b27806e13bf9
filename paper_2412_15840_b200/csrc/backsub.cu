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
#include "backsub_persist.cuh"

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

// v2 needs cubic 4096-entry tiles with b in {8, 16} dividing every extent.
static bool gemm_regime(const TileGeom& g) {
  if (g.tile_entries != kMaxTile) return false;
  if (!diag_kernel_for(g.n_modes, g.b[0])) return false;
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
    // lanes per entry: 1 on wide hyperplanes (ILP inside the lane); on narrow ones split the
    // terms (>= 4 per lane) to shorten the dependency chain.
    while (grp < 32 && wf_count[i] * grp * 2 <= diag_threads_for(n_modes) &&
           grp * 2 <= std::max(1, wf_terms[i] / 4))
      grp *= 2;
    wf_group[i] = grp;
  }
  {
    std::vector<int> pos(wf_off.begin(), wf_off.end() - 1);
    for (int l = 0; l < g.tile_entries; ++l) wf[pos[wf_levels - 1 - wf_lev[l]]++] = l;
    // Within a hyperplane, order entries by their leading coordinates (mode 1 most significant)
    // so that the lanes of a warp share the trip counts of the leading-mode loops (v2 kernel).
    auto key = [&](int l) {
      int k = 0;
      for (int j = 0; j < n_modes; ++j) {
        k = k * g.b[j] + (l % g.b[j]);
        l /= g.b[j];
      }
      return k;
    };
    for (int i = 0; i < wf_levels; ++i)
      std::sort(wf.begin() + wf_off[i], wf.begin() + wf_off[i + 1], [&](int a, int b) { return key(a) < key(b); });
  }

  // v2 work items. Per level and tile (level order) and mode j with off-tile rows:
  //   far  — rows >= (I_j + 2) b_j: neighbours two or more blocks away, ready one level early;
  //          k-split when the level has too few items to fill the GPU;
  //   near — rows [(I_j + 1) b_j, (I_j + 2) b_j): the adjacent block, ready just before diag.
  std::vector<int4> far_items, near_items;
  std::vector<int4> tile_ranges(ntiles, make_int4(0, 0, 0, 0));
  sp.far_off.assign(levels + 1, 0);
  sp.near_off.assign(levels + 1, 0);
  sp.max_far = sp.max_near = 0;
  if (sp.v2) {
    for (int lv = 0; lv < levels; ++lv) {
      int64_t natural = 0, rows = 0;
      for (int64_t s = sp.level_off[lv]; s < sp.level_off[lv + 1]; ++s) {
        int64_t r = tiles[s];
        for (int j = 0; j < n_modes; ++j) {
          const int64_t I = r % g.nb[j];
          r /= g.nb[j];
          const int64_t K = g.dims[j] - (I + 2) * g.b[j];
          if (K > 0) {
            ++natural;
            rows += K;
          }
        }
      }
      int64_t kc = INT64_MAX;
      const int64_t kq = std::max(8, update_bk(g.b[0]));  // item k-ranges are multiples of the stage depth
      if (natural > 0 && natural < 2 * 148) kc = std::max<int64_t>(32, ((rows + 295) / 296 + kq - 1) / kq * kq);
      for (int64_t s = sp.level_off[lv]; s < sp.level_off[lv + 1]; ++s) {
        int64_t r = tiles[s];
        const int f0 = (int)far_items.size(), n0 = (int)near_items.size();
        for (int j = 0; j < n_modes; ++j) {
          const int64_t I = r % g.nb[j];
          r /= g.nb[j];
          const int64_t b = g.b[j];
          if ((I + 1) * b < g.dims[j]) near_items.push_back(make_int4((int)s, j, (int)((I + 1) * b), (int)((I + 2) * b)));
          for (int64_t kb = (I + 2) * b; kb < g.dims[j]; kb += (kc == INT64_MAX ? g.dims[j] : kc)) {
            const int64_t ke = kc == INT64_MAX ? g.dims[j] : std::min<int64_t>(g.dims[j], kb + kc);
            far_items.push_back(make_int4((int)s, j, (int)kb, (int)ke));
          }
        }
        tile_ranges[s] = make_int4(f0 - (int)sp.far_off[lv], (int)far_items.size() - f0, n0 - (int)sp.near_off[lv],
                                   (int)near_items.size() - n0);
      }
      sp.far_off[lv + 1] = (int64_t)far_items.size();
      sp.near_off[lv + 1] = (int64_t)near_items.size();
      sp.max_far = std::max(sp.max_far, sp.far_off[lv + 1] - sp.far_off[lv]);
      sp.max_near = std::max(sp.max_near, sp.near_off[lv + 1] - sp.near_off[lv]);
    }
  }

  // Grouped far updates (fgroup = G > 1): along every mode-j line the far targets (blocks
  // t <= nb_j - 3) form groups of G consecutive blocks from the top, t0, t0 - 1, .., t0 - G' + 1.
  // At the level of t0 one item (k-split like the plain items) covers all of them with the
  // sources every member needs, rows >= (t0 + 2) b; member t0 - q then still needs the q blocks
  // [t0 - q + 2, t0 + 2), added by a remainder item at its own level (sources two or more levels
  // old, so ready). Partials live in a ring of fg_ring level regions (an item writes regions of
  // up to G - 1 later levels), one slot per (target, mode, chunk): the diagonal kernel reads
  // exactly the slots listed in tile_ranges, as with plain items.
  std::vector<FarGroupItem> fg_items;
  sp.fgroup = 0;
  if (sp.v2) {
    const int want = far_group_for(g.b[0]);
    bool ok = want >= 1;
    for (int j = 0; j < n_modes && ok; ++j)
      if (g.b[j] != g.b[0] || (g.nb[j] >= 3 && want * g.b[j] > g.dims[j])) ok = false;
    if (ok) sp.fgroup = want;
  }
  if (sp.fgroup >= 1) {
    const int G = sp.fgroup;
    std::vector<int64_t> slot_of(ntiles);
    for (int64_t s2 = 0; s2 < ntiles; ++s2) slot_of[tiles[s2]] = s2;
    std::vector<int64_t> tstride(n_modes, 1);
    for (int j = 1; j < n_modes; ++j) tstride[j] = tstride[j - 1] * g.nb[j - 1];
    // per (slot, mode): chunk items of the group item covering it, row block within it, remainder
    std::vector<std::vector<int>> chunks((size_t)ntiles * n_modes);
    std::vector<int> rowblk((size_t)ntiles * n_modes, -1), remainder((size_t)ntiles * n_modes, -1);
    std::vector<std::vector<FarGroupItem>> per_level(levels);
    const int64_t kq = std::max(8, far_group_bk(g.b[0]));
    for (int lv = 0; lv < levels; ++lv) {
      int64_t natural = 0, rows = 0;
      auto top_of = [&](int64_t nbj, int64_t t) { return nbj - 3 - ((nbj - 3 - t) / G) * G; };
      for (int64_t s2 = sp.level_off[lv]; s2 < sp.level_off[lv + 1]; ++s2) {
        int64_t r = tiles[s2];
        for (int j = 0; j < n_modes; ++j) {
          const int64_t t = r % g.nb[j];
          r /= g.nb[j];
          if (t > g.nb[j] - 3) continue;
          const int64_t t0 = top_of(g.nb[j], t);
          ++natural;
          rows += t == t0 ? g.dims[j] - (t0 + 2) * g.b[j] : (t0 - t) * g.b[j];
        }
      }
      int64_t kc = INT64_MAX;
      // k-split target: NDS_KSPLIT = CTA-items a small level is spread over (A/B). Default 0 = never
      // split: every chunk is one more partial the diagonal CTA reads on the critical path (c1 tail
      // levels: 3 items -> 21 chunks); unsplit, the small levels' far items still finish under the
      // previous level's diagonal tiles (c1 solve 4.50 -> 4.41 ms)
      static const int64_t ksplit = getenv("NDS_KSPLIT") ? atoll(getenv("NDS_KSPLIT")) : 0;
      if (natural > 0 && natural < ksplit)
        kc = std::max<int64_t>(32, ((rows + ksplit - 1) / ksplit + kq - 1) / kq * kq);
      for (int64_t s2 = sp.level_off[lv]; s2 < sp.level_off[lv + 1]; ++s2) {
        int64_t r = tiles[s2];
        for (int j = 0; j < n_modes; ++j) {
          const int64_t t = r % g.nb[j];
          r /= g.nb[j];
          if (t > g.nb[j] - 3) continue;
          const int64_t t0 = top_of(g.nb[j], t), b = g.b[j];
          if (t == t0) {
            const int gp = (int)std::min<int64_t>(G, t0 + 1);
            const int64_t rb0 = t0 - gp + 1;
            std::vector<int> ids;
            for (int64_t kb = (t0 + 2) * b; kb < g.dims[j]; kb += (kc == INT64_MAX ? g.dims[j] : kc)) {
              const int64_t ke = kc == INT64_MAX ? g.dims[j] : std::min<int64_t>(g.dims[j], kb + kc);
              FarGroupItem it{};
              it.tile = (int)s2;
              it.j = j;
              it.kb = (int)kb;
              it.ke = (int)ke;
              it.rb0 = (int)(gp < G ? 0 : rb0);  // a truncated group starts at block 0
              it.nrb = (int)(gp < G ? t0 + 1 : gp);
              it.acc = 0;
              for (int q = 0; q < 4; ++q) it.out[q] = -1;
              ids.push_back((int)per_level[lv].size() | (lv << 20));
              per_level[lv].push_back(it);
            }
            for (int q = 0; q < gp; ++q) {  // members t0 - q
              const int64_t ms = slot_of[tiles[s2] - q * tstride[j]];
              chunks[(size_t)ms * n_modes + j] = ids;
              rowblk[(size_t)ms * n_modes + j] = (int)(t0 - q - (gp < G ? 0 : rb0));
            }
          } else {
            FarGroupItem it{};
            it.tile = (int)s2;
            it.j = j;
            it.kb = (int)((t + 2) * b);
            it.ke = (int)((t0 + 2) * b);
            it.rb0 = (int)t;
            it.nrb = 1;
            it.acc = 1;
            for (int q = 0; q < 4; ++q) it.out[q] = -1;
            remainder[(size_t)s2 * n_modes + j] = (int)per_level[lv].size() | (lv << 20);
            per_level[lv].push_back(it);
          }
        }
      }
    }
    // slots: per target level, per tile, per mode, per chunk (tile_ranges order)
    int64_t max_slots = 1;
    std::vector<int> slot_idx((size_t)ntiles * n_modes, -1);
    for (int lv = 0; lv < levels; ++lv) {
      int idx = 0;
      for (int64_t s2 = sp.level_off[lv]; s2 < sp.level_off[lv + 1]; ++s2) {
        const int first = idx;
        for (int j = 0; j < n_modes; ++j) {
          const auto& ids = chunks[(size_t)s2 * n_modes + j];
          if (ids.empty()) continue;
          slot_idx[(size_t)s2 * n_modes + j] = idx;
          idx += (int)ids.size();
        }
        tile_ranges[s2].x = first;
        tile_ranges[s2].y = idx - first;
      }
      max_slots = std::max<int64_t>(max_slots, idx);
    }
    sp.fg_ring = G + 2;
    sp.fg_slots = max_slots;
    for (int lv = 0; lv < levels; ++lv)
      for (int64_t s2 = sp.level_off[lv]; s2 < sp.level_off[lv + 1]; ++s2)
        for (int j = 0; j < n_modes; ++j) {
          const auto& ids = chunks[(size_t)s2 * n_modes + j];
          if (ids.empty()) continue;
          const int64_t base = (int64_t)(lv % sp.fg_ring) * max_slots + slot_idx[(size_t)s2 * n_modes + j];
          const int q = rowblk[(size_t)s2 * n_modes + j];
          for (size_t c2 = 0; c2 < ids.size(); ++c2)
            per_level[ids[c2] >> 20][ids[c2] & 0xfffff].out[q] = (int)(base + (int64_t)c2);
          const int rm = remainder[(size_t)s2 * n_modes + j];
          if (rm >= 0) per_level[rm >> 20][rm & 0xfffff].out[0] = (int)base;
        }
    sp.fg_off.assign(levels + 1, 0);
    for (int lv = 0; lv < levels; ++lv) {
      // longest first (LPT): the short remainder items fill the launch's tail
      std::stable_sort(per_level[lv].begin(), per_level[lv].end(), [](const FarGroupItem& a, const FarGroupItem& b2) {
        return (int64_t)(a.ke - a.kb) * (a.acc ? 1 : 2) > (int64_t)(b2.ke - b2.kb) * (b2.acc ? 1 : 2);
      });
      for (const auto& it : per_level[lv]) fg_items.push_back(it);
      sp.fg_off[lv + 1] = (int64_t)fg_items.size();
    }
  }

  // v2 per-thread step tables for the diagonal kernel
  const int dthreads = sp.v2 ? diag_threads_for(n_modes) : 0;
  std::vector<uint16_t> thr((size_t)wf_levels * dthreads, 0xffff);
  std::vector<int> lvl(wf_levels, 0);
  for (int lv = 0; sp.v2 && lv < wf_levels; ++lv) {
    const int grp = wf_group[lv], cnt = wf_off[lv + 1] - wf_off[lv];
    int gsh = 0;
    while ((1 << gsh) < grp) ++gsh;
    for (int t = 0; t < dthreads; ++t) {
      const int e = t >> gsh;
      if (e < cnt) thr[(size_t)lv * dthreads + t] = (uint16_t)wf[wf_off[lv] + e];
    }
    lvl[lv] = grp | (((cnt * grp + 31) / 32) << 8);
  }

  // v2 lines kernel, push mode: for each tile slot J and mode j, the index (relative to its
  // level) of the near item of tile J - e_j that J's diagonal CTA computes, or -1.
  std::vector<int> near_target;
  if (sp.v2) {
    near_target.assign((size_t)ntiles * n_modes, -1);
    std::vector<int64_t> slot_of(ntiles);
    for (int64_t s2 = 0; s2 < ntiles; ++s2) slot_of[tiles[s2]] = s2;
    std::vector<int64_t> tstride(n_modes, 1);
    for (int j = 1; j < n_modes; ++j) tstride[j] = tstride[j - 1] * g.nb[j - 1];
    for (int lv = 0; lv < levels; ++lv)
      for (int64_t n = sp.near_off[lv]; n < sp.near_off[lv + 1]; ++n) {
        const int4 it = near_items[n];
        const int64_t sJ = slot_of[tiles[it.x] + tstride[it.y]];
        near_target[(size_t)sJ * n_modes + it.y] = (int)(n - sp.near_off[lv]);
      }
  }

  // dataflow (persistent) solve tables: N = 3 cubic tiles
  sp.persist = sp.v2 && n_modes == 3 && !far_items.empty() && sp.fgroup == 0;
  std::vector<int> p_level_of, p_level_count, p_far_rel, p_far_dep, p_far_expected, p_push_slot, p_queue;
  if (sp.persist) {
    std::vector<int64_t> slot_of(ntiles);
    for (int64_t s2 = 0; s2 < ntiles; ++s2) slot_of[tiles[s2]] = s2;
    std::vector<int64_t> tstride(n_modes, 1);
    for (int j = 1; j < n_modes; ++j) tstride[j] = tstride[j - 1] * g.nb[j - 1];
    const int H = update_h(g.b[0]);
    p_level_of.resize(ntiles);
    p_level_count.resize(levels);
    p_far_expected.assign(ntiles, 0);
    p_push_slot.assign((size_t)ntiles * n_modes, -1);
    for (int lv = 0; lv < levels; ++lv) {
      p_level_count[lv] = (int)(sp.level_off[lv + 1] - sp.level_off[lv]);
      for (int64_t s2 = sp.level_off[lv]; s2 < sp.level_off[lv + 1]; ++s2) p_level_of[s2] = lv;
      for (int64_t f = sp.far_off[lv]; f < sp.far_off[lv + 1]; ++f) {
        const int4 it = far_items[f];
        p_far_rel.push_back((int)(f - sp.far_off[lv]));
        p_far_dep.push_back((int)slot_of[tiles[it.x] + 2 * tstride[it.y]]);
        p_far_expected[it.x] += H;
      }
    }
    for (int64_t s2 = 0; s2 < ntiles; ++s2) {
      int64_t r = tiles[s2];
      for (int j = 0; j < n_modes; ++j) {
        const int64_t I = r % g.nb[j];
        r /= g.nb[j];
        if (I > 0) p_push_slot[(size_t)s2 * n_modes + j] = (int)slot_of[tiles[s2] - tstride[j]];
      }
    }
    // merged queue: far(lv + 1) CTA-items, then the diagonal tiles of hyperplane lv
    for (int lv = 0; lv < levels; ++lv) {
      if (lv + 1 < levels)
        for (int64_t f = sp.far_off[lv + 1]; f < sp.far_off[lv + 2]; ++f)
          for (int h = 0; h < H; ++h) p_queue.push_back(-(int)(f * H + h) - 1);
      for (int64_t s2 = sp.level_off[lv]; s2 < sp.level_off[lv + 1]; ++s2) p_queue.push_back((int)s2);
    }
  }

  size_t bytes = ntiles * sizeof(int64_t) + (g.tile_entries + 3 * wf_levels + 2) * sizeof(int) +
                 (thr.size() + 8) * sizeof(uint16_t) + 64;
  bytes = (bytes + 15) / 16 * 16;
  const size_t nt_off = bytes;
  bytes += near_target.size() * sizeof(int);
  bytes = (bytes + 15) / 16 * 16;
  const size_t items_off = bytes;
  bytes += (far_items.size() + near_items.size() + ntiles) * sizeof(int4);
  bytes = (bytes + 15) / 16 * 16;
  const size_t fg_items_off = bytes;
  bytes += fg_items.size() * sizeof(FarGroupItem);
  bytes = (bytes + 255) / 256 * 256;
  const size_t partial_off = bytes;
  const size_t tile_bytes = (size_t)g.tile_entries * sizeof(double2);
  const size_t far_bufs = sp.fgroup >= 1 ? (size_t)sp.fg_ring * sp.fg_slots : 2 * (size_t)sp.max_far;
  bytes += (far_bufs + 2 * (size_t)sp.max_near) * tile_bytes + 256;
  bytes = (bytes + 15) / 16 * 16;
  const size_t persist_off = bytes;
  bytes += (p_level_of.size() + p_level_count.size() + p_far_rel.size() + p_far_dep.size() + p_far_expected.size() +
            p_push_slot.size() + p_queue.size()) * sizeof(int) + 64;
  NDS_CUDA(cudaMalloc(&sp.pool, bytes));
  char* base = (char*)sp.pool;
  sp.d_tiles = (int64_t*)base;
  sp.d_wf = (int*)(sp.d_tiles + ntiles);
  sp.d_wf_off = sp.d_wf + g.tile_entries;
  sp.d_wf_group = sp.d_wf_off + wf_levels + 1;
  sp.d_lvl = sp.d_wf_group + wf_levels;
  sp.d_thr = (uint16_t*)(((uintptr_t)(sp.d_lvl + wf_levels) + 15) & ~(uintptr_t)15);
  sp.d_near_target = (int*)(base + nt_off);
  sp.d_far_items = (int4*)(base + items_off);
  sp.d_near_items = sp.d_far_items + far_items.size();
  sp.d_tile_ranges = sp.d_near_items + near_items.size();
  sp.d_fg_items = (FarGroupItem*)(base + fg_items_off);
  if (!fg_items.empty())
    NDS_CUDA(cudaMemcpy(sp.d_fg_items, fg_items.data(), fg_items.size() * sizeof(FarGroupItem), cudaMemcpyHostToDevice));
  sp.d_far_partial[0] = (double2*)(base + partial_off);
  sp.d_far_partial[1] = sp.fgroup >= 1 ? sp.d_far_partial[0] : sp.d_far_partial[0] + (size_t)sp.max_far * g.tile_entries;
  sp.d_fg_ring = sp.d_far_partial[0];
  sp.d_near_partial = sp.d_far_partial[0] + far_bufs * g.tile_entries;
  sp.d_near_partial2 = sp.d_near_partial + (size_t)sp.max_near * g.tile_entries;
  NDS_CUDA(cudaMemcpy(sp.d_tiles, tiles.data(), ntiles * sizeof(int64_t), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf, wf.data(), g.tile_entries * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf_off, wf_off.data(), (wf_levels + 1) * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_wf_group, wf_group.data(), wf_levels * sizeof(int), cudaMemcpyHostToDevice));
  NDS_CUDA(cudaMemcpy(sp.d_lvl, lvl.data(), wf_levels * sizeof(int), cudaMemcpyHostToDevice));
  if (!thr.empty())
    NDS_CUDA(cudaMemcpy(sp.d_thr, thr.data(), thr.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
  if (!near_target.empty())
    NDS_CUDA(cudaMemcpy(sp.d_near_target, near_target.data(), near_target.size() * sizeof(int), cudaMemcpyHostToDevice));
  if (sp.persist) {
    int* q = (int*)(base + persist_off);
    auto put = [&](const std::vector<int>& v, int*& dst) {
      dst = q;
      if (!v.empty()) NDS_CUDA(cudaMemcpy(q, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
      q += v.size();
    };
    put(p_level_of, sp.d_level_of);
    put(p_level_count, sp.d_level_count);
    put(p_far_rel, sp.d_far_rel);
    put(p_far_dep, sp.d_far_dep);
    put(p_far_expected, sp.d_far_expected);
    put(p_push_slot, sp.d_push_slot);
    put(p_queue, sp.d_queue);
    sp.n_queue = (int64_t)p_queue.size();
    sp.n_far_items = (int64_t)far_items.size();
    const PersistCtr pc = PersistCtr::of(ntiles, levels);
    sp.ctr_count = pc.total;
    const size_t ring = (size_t)kRing * (sp.max_far + sp.max_near) * tile_bytes;
    NDS_CUDA(cudaMalloc(&sp.persist_pool, ring + (size_t)pc.total * sizeof(int) + 256));
    sp.d_far_ring = (double2*)sp.persist_pool;
    sp.d_near_ring = sp.d_far_ring + (size_t)kRing * sp.max_far * g.tile_entries;
    sp.d_ctr = (int*)(sp.d_near_ring + (size_t)kRing * sp.max_near * g.tile_entries);
    NDS_CUDA(cudaMallocHost(&sp.h_err, sizeof(int)));
    *sp.h_err = 0;
  }
  if (sp.v2) {
    if (!far_items.empty())
      NDS_CUDA(cudaMemcpy(sp.d_far_items, far_items.data(), far_items.size() * sizeof(int4), cudaMemcpyHostToDevice));
    if (!near_items.empty())
      NDS_CUDA(cudaMemcpy(sp.d_near_items, near_items.data(), near_items.size() * sizeof(int4), cudaMemcpyHostToDevice));
    NDS_CUDA(cudaMemcpy(sp.d_tile_ranges, tile_ranges.data(), ntiles * sizeof(int4), cudaMemcpyHostToDevice));
    // critical path (near + diag) on a high-priority stream, far updates on a low-priority one
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
  if (sp.persist_pool) cudaFree(sp.persist_pool);
  sp.persist_pool = nullptr;
  if (sp.h_err) cudaFreeHost(sp.h_err);
  sp.h_err = nullptr;
  for (auto e : sp.ev) cudaEventDestroy(e);
  sp.ev.clear();
  if (sp.s_crit) cudaStreamDestroy(sp.s_crit);
  if (sp.s_far) cudaStreamDestroy(sp.s_far);
  if (sp.s_far2) cudaStreamDestroy(sp.s_far2);
  sp.s_crit = sp.s_far = sp.s_far2 = nullptr;
}

// NDS_SOLVE=split|unified selects the dataflow (persistent-kernel) solve, an experimental A/B
// path: measured on c1 it is not faster than the level-synchronous launches plus the head
// overlap (split 4.40 ms solve vs 4.30; unified two-queue polling 37 ms), so it is off by default.
bool persist_enabled() {
  static const bool v = getenv("NDS_SOLVE") && (std::string(getenv("NDS_SOLVE")) == "split" ||
                                                std::string(getenv("NDS_SOLVE")) == "unified");
  return v;
}

bool backsub_is_dataflow(const SolvePlan& sp) { return sp.persist && persist_enabled(); }

static int persist_launch(const SolvePlan& sp, const double2* t_pool, double2* c, cudaStream_t stream, Recorder* rec) {
  if (*sp.h_err) throw Error(NDS_ERR_CUDA, "dataflow solve watchdog fired on a previous call (dependency wait timed out)");
  const TileGeom& g = sp.geom;
  const int b = g.b[0];
  const UpdCfg uc = update_cfg_for(b);
  using FarK = void (*)(const PersistArgs);
  const FarK fark = far_persist_kernel<2, 2, true, 1, 3, 2>;
  const FarK diagk = diag_persist_kernel<3, 16, 256>;
  static bool attr = false;
  if (!attr) {
    NDS_CUDA(cudaFuncSetAttribute(fark, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)update_smem_bytes(b)));
    NDS_CUDA(cudaFuncSetAttribute(diagk, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
    attr = true;
  }
  if (uc.h != 2 || uc.bk != 8 || b != 16) throw Error(NDS_ERR_OTHER, "dataflow solve needs the 16-row 3M update");
  PersistArgs a{};
  a.g = g;
  a.T = t_pool;
  a.Y = c;
  a.tiles = sp.d_tiles;
  a.level_of = sp.d_level_of;
  a.level_count = sp.d_level_count;
  a.tile_ranges = sp.d_tile_ranges;
  a.near_target = sp.d_near_target;
  a.push_slot = sp.d_push_slot;
  a.far_items = sp.d_far_items;
  a.far_rel = sp.d_far_rel;
  a.far_dep = sp.d_far_dep;
  a.far_expected = sp.d_far_expected;
  a.n_tiles = sp.level_off.back();
  a.H = uc.h;
  a.n_far_ctas = sp.n_far_items * uc.h;
  a.max_far = sp.max_far;
  a.max_near = sp.max_near;
  a.far_ring = sp.d_far_ring;
  a.near_ring = sp.d_near_ring;
  a.ctr = sp.d_ctr;
  const int L = sp.levels;
  cudaEvent_t ev_start = sp.ev[2 * L], ev_end = sp.ev[2 * L + 1], ev_far_end = sp.ev[0];
  NDS_CUDA(cudaMemsetAsync(sp.d_ctr, 0, (size_t)sp.ctr_count * sizeof(int), stream));
  NDS_CUDA(cudaEventRecord(ev_start, stream));
  NDS_CUDA(cudaStreamWaitEvent(sp.s_crit, ev_start, 0));
  NDS_CUDA(cudaStreamWaitEvent(sp.s_far, ev_start, 0));
  if (rec) rec->mark(stream, -1, 0);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  a.queue = sp.d_queue;
  a.n_queue = sp.n_queue;
  static const bool split = std::string(getenv("NDS_SOLVE")) == "split";
  if (split) {
    // at most one CTA of each kind per SM: both always keep resident CTAs (no deadlock)
    const int gd = (int)std::min<int64_t>(sms, a.n_tiles);
    const int gf = (int)std::min<int64_t>(sms, a.n_far_ctas);
    diagk<<<gd, 256, lines_smem_bytes(3, 16), sp.s_crit>>>(a);
    NDS_LAUNCH_CHECK();
    fark<<<gf, kUpdThreads, update_smem_bytes(b), sp.s_far>>>(a);
    NDS_LAUNCH_CHECK();
    NDS_CUDA(cudaEventRecord(ev_far_end, sp.s_far));
    NDS_CUDA(cudaStreamWaitEvent(sp.s_crit, ev_far_end, 0));
  } else {
    const FarK solvek = solve_persist_kernel<3, 16, 256>;
    static bool attr2 = false;
    if (!attr2) {
      NDS_CUDA(cudaFuncSetAttribute(solvek, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
      attr2 = true;
    }
    const size_t smem = std::max(lines_smem_bytes(3, 16), update_smem_bytes(b));
    const int grid = (int)std::min<int64_t>(2 * sms, a.n_queue);
    solvek<<<grid, 256, smem, sp.s_crit>>>(a);
    NDS_LAUNCH_CHECK();
  }
  NDS_CUDA(cudaMemcpyAsync(sp.h_err, sp.d_ctr + 2, sizeof(int), cudaMemcpyDeviceToHost, sp.s_crit));
  NDS_CUDA(cudaEventRecord(ev_end, sp.s_crit));
  NDS_CUDA(cudaStreamWaitEvent(stream, ev_end, 0));
  if (rec) rec->mark(stream, kBacksubPersistent, L);
  return 2;
}

int backsub_launch(const SolvePlan& sp, const double2* t_pool, double2* c, cudaStream_t stream, Recorder* rec,
                   const HeadSync* head, const TailHook* tail) {
  static bool attr_set = false;
  if (!attr_set) {
    NDS_CUDA(cudaFuncSetAttribute(tile_level_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kMaxTile * sizeof(double2))));
    for (int b : {8, 16}) {
      NDS_CUDA(cudaFuncSetAttribute(update_kernel_for(b), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)update_smem_bytes(b)));
      if (far_group_for(b) >= 1)
        NDS_CUDA(cudaFuncSetAttribute(far_group_cfg(b).kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)far_group_smem_bytes(b)));
    }
    NDS_CUDA(cudaFuncSetAttribute(diag_kernel_for(3, 16), cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
    NDS_CUDA(cudaFuncSetAttribute(diag_kernel_for(4, 8), cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
    for (bool push : {false, true}) {
      NDS_CUDA(cudaFuncSetAttribute(lines_kernel_for(3, 16, push), cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
      NDS_CUDA(cudaFuncSetAttribute(lines_kernel_for(4, 8, push), cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
    }
    attr_set = true;
  }
  const TileGeom& g = sp.geom;
  int launches = 0;
  if (sp.persist && persist_enabled()) return persist_launch(sp, t_pool, c, stream, rec);
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
  const UpdateKernel upd = update_kernel_for(b);
  const DiagKernel diag = diag_kernel_for(g.n_modes, b);
  const size_t upd_smem = update_smem_bytes(b);
  const int uh = update_h(b);  // CTAs per update item (column halves)
  const size_t diag_smem = diag_smem_bytes(g.n_modes, b, sp.wf_levels);
  // NDS_DIAG=wave selects the per-hyperplane entry kernel (A/B experiments); default lines
  static const bool use_lines = !(getenv("NDS_DIAG") && std::string(getenv("NDS_DIAG")) == "wave");
  // NDS_NEAR=kernel: separate near-update launches instead of the diagonal CTAs pushing them
  static const bool push = use_lines && !(getenv("NDS_NEAR") && std::string(getenv("NDS_NEAR")) == "kernel");
  const LinesKernel lines = lines_kernel_for(g.n_modes, b, push);
  const size_t lines_smem = lines_smem_bytes(g.n_modes, b);
  static const int dbg_levels = getenv("NDS_DEBUG_WF_LEVELS") ? atoi(getenv("NDS_DEBUG_WF_LEVELS")) : -1;
  const int wfl = dbg_levels >= 0 ? std::min(dbg_levels, sp.wf_levels) : sp.wf_levels;  // timing experiments only
  const int L = sp.levels;
  cudaEvent_t ev_start = sp.ev[2 * L], ev_end = sp.ev[2 * L + 1];
  // NDS_SOLVE_TRACE=1: per-level start/end events of every launch, printed to stderr (timeline
  // experiments only; adds event records to the streams).
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
  // fork: both internal streams start after everything already queued on the caller's stream
  NDS_CUDA(cudaEventRecord(ev_start, stream));
  NDS_CUDA(cudaStreamWaitEvent(sp.s_crit, ev_start, 0));
  NDS_CUDA(cudaStreamWaitEvent(sp.s_far, ev_start, 0));
  NDS_CUDA(cudaStreamWaitEvent(sp.s_far2, ev_start, 0));
  if (rec) rec->mark(stream, -1, 0);
  int head_waited = -1;
  // far(lv) depends on diag(lv - 2) only: even and odd levels' far launches go to two streams so
  // far(lv) may start while far(lv - 1)'s last CTAs drain (NDS_FAR2=0: one stream)
  static const bool far2 = !(getenv("NDS_FAR2") && std::string(getenv("NDS_FAR2")) == "0");
  const bool grouped = sp.fgroup >= 1;
  const FarGroupCfg fgc = far_group_cfg(b);
  const size_t fg_smem = far_group_smem_bytes(b);
  for (int lv = 0; lv < L; ++lv) {
    const int64_t nf = grouped ? sp.fg_off[lv + 1] - sp.fg_off[lv] : sp.far_off[lv + 1] - sp.far_off[lv];
    const int64_t nn = sp.near_off[lv + 1] - sp.near_off[lv];
    double2* far_buf = grouped ? sp.d_fg_ring + (size_t)(lv % sp.fg_ring) * sp.fg_slots * g.tile_entries
                               : sp.d_far_partial[lv & 1];
    if (nf > 0) {
      // far(lv) needs levels <= lv - 2; it overlaps diag(lv - 1) on the critical stream
      cudaStream_t fs = far2 && (lv & 1) ? sp.s_far2 : sp.s_far;
      if (lv >= 2) NDS_CUDA(cudaStreamWaitEvent(fs, ev_diag(lv - 2), 0));
      tmark(fs, lv, 0);
      if (grouped)
        fgc.kern<<<(unsigned)(nf * fgc.h), kUpdThreads, fg_smem, fs>>>(g, t_pool, sp.d_tiles,
                                                                    sp.d_fg_items + sp.fg_off[lv], sp.d_fg_ring, c);
      else
        upd<<<(unsigned)(nf * uh), kUpdThreads, upd_smem, fs>>>(g, t_pool, sp.d_tiles, sp.d_far_items + sp.far_off[lv],
                                                         far_buf, c);
      NDS_LAUNCH_CHECK();
      tmark(fs, lv, 1);
      NDS_CUDA(cudaEventRecord(ev_far(lv), fs));
      ++launches;
    }
    double2* near_in = push ? (lv & 1 ? sp.d_near_partial2 : sp.d_near_partial) : sp.d_near_partial;
    double2* near_out = (lv & 1) ? sp.d_near_partial : sp.d_near_partial2;  // level lv + 1's buffer
    if (nn > 0 && !push) {
      tmark(sp.s_crit, lv, 2);
      upd<<<(unsigned)(nn * uh), kUpdThreads, upd_smem, sp.s_crit>>>(g, t_pool, sp.d_tiles, sp.d_near_items + sp.near_off[lv],
                                                              sp.d_near_partial, c);
      NDS_LAUNCH_CHECK();
      tmark(sp.s_crit, lv, 3);
      ++launches;
    }
    if (nf > 0) NDS_CUDA(cudaStreamWaitEvent(sp.s_crit, ev_far(lv), 0));
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
    if (use_lines)
      lines<<<(unsigned)nt, diag_threads_for(g.n_modes), lines_smem, sp.s_crit>>>(
          g, t_pool, sp.d_tiles + sp.level_off[lv], sp.d_tile_ranges + sp.level_off[lv], far_buf, near_in,
          sp.d_near_target + sp.level_off[lv] * g.n_modes, near_out, c);
    else
      diag<<<(unsigned)nt, diag_threads_for(g.n_modes), diag_smem, sp.s_crit>>>(
          g, t_pool, sp.d_tiles + sp.level_off[lv], sp.d_tile_ranges + sp.level_off[lv], far_buf, sp.d_near_partial,
          sp.d_thr, sp.d_lvl, wfl, c);
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
      const int64_t nf = sp.fgroup >= 1 ? sp.fg_off[lv + 1] - sp.fg_off[lv] : sp.far_off[lv + 1] - sp.far_off[lv];
      const int64_t nn = push ? 0 : sp.near_off[lv + 1] - sp.near_off[lv];
      float t[6] = {-1, -1, -1, -1, -1, -1};
      for (int k = 0; k < 6; ++k) {
        if ((k < 2 && nf == 0) || ((k == 2 || k == 3) && nn == 0)) continue;
        NDS_CUDA(cudaEventElapsedTime(&t[k], tev.back(), tev[(size_t)lv * 6 + k]));
      }
      fprintf(stderr, "TRACE %d %lld %lld %lld %.1f %.1f %.1f %.1f %.1f %.1f\n", lv,
              (long long)(sp.level_off[lv + 1] - sp.level_off[lv]), (long long)nf, (long long)nn, t[0] * 1e3,
              t[1] * 1e3, t[2] * 1e3, t[3] * 1e3, t[4] * 1e3, t[5] * 1e3);
    }
    for (auto e : tev) cudaEventDestroy(e);
  }
  return launches;
}

}  // namespace nds
