// Dataflow form of the cubic-tile solve (N = 3, 16^3 tiles): two persistent kernels instead of
// three launches per tile hyperplane.
//
//   diagonal kernel: CTAs take tiles in hyperplane order from an atomic queue; tile I starts as
//                    soon as its own far items and the near couplings pushed by its N upper
//                    neighbours I + e_m have landed (per-tile counters), solves, pushes its
//                    couplings to I - e_m, and raises done[I];
//   far kernel:      CTAs take far items (tile I, mode m, k-range, column half) in hyperplane
//                    order; an item starts when done[I + 2 e_m] is set — every tile further along
//                    the line was solved before it (it received their pushes) — and bumps the
//                    target tile's far counter.
// Every wait points to an item strictly earlier in one global order (diag(lv-2) < far(lv) <
// diag(lv)) and each queue is consumed in order by resident CTAs, so the pair cannot deadlock as
// long as both kernels keep at least one resident CTA: each kernel's grid is at most one CTA per
// SM and a diagonal CTA (128 registers x 256 threads, 90 KB) plus an update CTA (122 x 256,
// 60 KB) fit an SM together. Partials live in rings of kRing hyperplanes; a producer writing ring
// slot lv waits until hyperplane lv - kRing has completed. Spins are bounded (watchdog -> error
// flag, the host raises it). Cross-CTA data is read through L2 (__ldcg / cp.async.cg) since L1 is
// not coherent across SMs.
// Included by backsub.cu after backsub_v2.cuh.

constexpr int kRing = 4;

struct PersistArgs {
  TileGeom g;
  const double2* T;
  double2* Y;
  const int64_t* tiles;       // slot -> tile id (hyperplane order)
  const int* level_of;        // slot -> hyperplane
  const int* level_count;     // tiles per hyperplane
  const int4* tile_ranges;    // {far first, far count, near first, near count} (level-relative)
  const int* near_target;     // [slot][N]: item index at the next hyperplane of slot - e_m, or -1
  const int* push_slot;       // [slot][N]: slot of that tile, or -1
  const int4* far_items;      // all far items, hyperplane order
  const int* far_rel;         // item -> index within its hyperplane
  const int* far_dep;         // item -> slot of tile I + 2 e_m
  const int* far_expected;    // slot -> far CTA-items (items x column halves)
  int64_t n_tiles, n_far_ctas, max_far, max_near;
  int H;                      // CTAs per far item
  const int* queue;           // merged work order: slot >= 0 diagonal tile, -(far CTA-item + 1) far
  int64_t n_queue;
  double2* far_ring;          // [kRing][max_far][4096]
  double2* near_ring;         // [kRing][max_near][4096]
  int* ctr;                   // counters, zeroed per solve (layout in PersistCtr)
};

// counter block layout (ints): heads[2], err, pad, done[n], far_done[n], push_done[n], level_done[L]
struct PersistCtr {
  int64_t done, far_done, push_done, level_done, total;
  __host__ __device__ static PersistCtr of(int64_t n_tiles, int levels) {
    PersistCtr c;
    c.done = 4;
    c.far_done = c.done + n_tiles;
    c.push_done = c.far_done + n_tiles;
    c.level_done = c.push_done + n_tiles;
    c.total = c.level_done + levels;
    return c;
  }
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Thread 0 spins until *p >= want (bounded); returns false when the watchdog fired.
__device__ __forceinline__ bool wait_at_least(const int* p, int want, int* err) {
  unsigned spins = 0;
  while (ld_acquire(p) < want) {
    if (ld_acquire(err)) return false;
    __nanosleep(64);
    if (++spins > (1u << 27)) {
      atomicExch(err, 1);
      return false;
    }
  }
  return true;
}

template <int RB, int CB, bool M3, int KM, int ST, int H>
__global__ void __launch_bounds__(kUpdThreads, 2) far_persist_kernel(const PersistArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ int s_idx;
  __shared__ int s_ok;
  const int tid = threadIdx.x;
  const PersistCtr c = PersistCtr::of(a.n_tiles, 0);
  int* err = a.ctr + 2;
  for (;;) {
    if (tid == 0) s_idx = atomicAdd(a.ctr + 1, 1);
    __syncthreads();
    const int64_t idx = s_idx;
    if (idx >= a.n_far_ctas) break;
    const int64_t item = idx / H;
    const int half = (int)(idx % H);
    const int4 it = a.far_items[item];
    const int lv = a.level_of[it.x];
    if (tid == 0) {
      bool ok = wait_at_least(a.ctr + c.done + a.far_dep[item], 1, err);
      if (ok && lv >= kRing) ok = wait_at_least(a.ctr + (c.done + 3 * a.n_tiles) + (lv - kRing), a.level_count[lv - kRing], err);
      s_ok = ok;
      __threadfence();
    }
    __syncthreads();
    if (!s_ok) break;
    double2* out = a.far_ring + ((int64_t)(lv % kRing) * a.max_far + a.far_rel[item]) * 4096;
    update_body<RB, CB, M3, KM, ST, H>(a.g, a.T, a.tiles, it, half, out, a.Y, sm);
    __threadfence();  // every thread: its partial stores are visible device-wide before the signal
    __syncthreads();
    if (tid == 0) {
      atomicAdd(a.ctr + c.far_done + it.x, 1);
    }
  }
}

template <int N, int B, int NT>
__global__ void __launch_bounds__(NT, 2) diag_persist_kernel(const PersistArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ int s_idx;
  __shared__ int s_ok;
  const int tid = threadIdx.x;
  const PersistCtr c = PersistCtr::of(a.n_tiles, 0);
  int* err = a.ctr + 2;
  int* level_done = a.ctr + c.done + 3 * a.n_tiles;
  for (;;) {
    if (tid == 0) s_idx = atomicAdd(a.ctr + 0, 1);
    __syncthreads();
    const int64_t slot = s_idx;
    if (slot >= a.n_tiles) break;
    const int lv = a.level_of[slot];
    const int4 tr = a.tile_ranges[slot];
    if (tid == 0) {
      bool ok = wait_at_least(a.ctr + c.far_done + slot, a.far_expected[slot], err);
      if (ok) ok = wait_at_least(a.ctr + c.push_done + slot, tr.w, err);
      // the pushes below write ring slot lv + 1: hyperplane lv + 1 - kRing must be finished
      if (ok && lv + 1 >= kRing) ok = wait_at_least(level_done + (lv + 1 - kRing), a.level_count[lv + 1 - kRing], err);
      s_ok = ok;
      __threadfence();
    }
    __syncthreads();
    if (!s_ok) break;
    diag_lines_body<N, B, NT, true, false>(
        a.g, a.T, a.tiles[slot], tr, a.far_ring + (int64_t)(lv % kRing) * a.max_far * 4096,
        a.near_ring + (int64_t)(lv % kRing) * a.max_near * 4096, a.near_target + slot * N,
        a.near_ring + (int64_t)((lv + 1) % kRing) * a.max_near * 4096, a.Y, sm);
    __threadfence();  // every thread: Y and pushed partials visible device-wide before the signals
    __syncthreads();
    if (tid == 0) {
      for (int m = 0; m < N; ++m) {
        const int ps = a.push_slot[slot * N + m];
        if (ps >= 0) atomicAdd(a.ctr + c.push_done + ps, 1);
      }
      atomicExch(a.ctr + c.done + slot, 1);
      atomicAdd(level_done + lv, 1);
    }
  }
}

// Both kinds of work in ONE persistent kernel (2 CTAs / SM: 128 registers, 90 KB) with two queues
// (diagonal tiles and far CTA-items, each in hyperplane order). A CTA only ever claims the HEAD of
// a queue, and only once that head's dependencies are met (checked first, then claimed by a
// compare-and-swap), preferring the diagonal queue (the critical path): no CTA ever holds a
// blocked item, so there is nothing to deadlock on, and the far work fills whatever the
// diagonal wavefront leaves idle.
template <int N, int B, int NT>
__global__ void __launch_bounds__(NT, 2) solve_persist_kernel(const PersistArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ int64_t s_w;  // claimed item: slot >= 0 diagonal, -(far CTA-item + 1) far, INT64_MIN done
  const int tid = threadIdx.x;
  const PersistCtr c = PersistCtr::of(a.n_tiles, 0);
  int* err = a.ctr + 2;
  int* level_done = a.ctr + c.done + 3 * a.n_tiles;
  int* dhead = a.ctr + 0;
  int* fhead = a.ctr + 1;
  auto diag_ready = [&](int64_t slot) {
    const int lv = a.level_of[slot];
    const int4 tr = a.tile_ranges[slot];
    if (ld_acquire(a.ctr + c.far_done + slot) < a.far_expected[slot]) return false;
    if (ld_acquire(a.ctr + c.push_done + slot) < tr.w) return false;
    if (lv + 1 >= kRing && ld_acquire(level_done + (lv + 1 - kRing)) < a.level_count[lv + 1 - kRing]) return false;
    return true;
  };
  auto far_ready = [&](int64_t idx) {
    const int64_t item = idx / a.H;
    const int lv = a.level_of[a.far_items[item].x];
    if (ld_acquire(a.ctr + c.done + a.far_dep[item]) == 0) return false;
    if (lv >= kRing && ld_acquire(level_done + (lv - kRing)) < a.level_count[lv - kRing]) return false;
    return true;
  };
  // Roles: the first half of the grid are flex CTAs — they never block: a diagonal tile if the
  // head one is ready, else the far head item if it is ready, else back off; the second half are
  // far workers — they claim far items in order and block on their dependency (as the split
  // form). Blocked CTAs are therefore all far workers, and the flex CTAs always remain free for
  // the diagonal tiles those far items wait on.
  const bool flex = blockIdx.x < gridDim.x / 2;
  for (;;) {
    if (tid == 0) {
      int64_t w = INT64_MIN;
      if (flex) {
        unsigned spins = 0, nap = 32;
        for (;;) {
          const int dh = ld_acquire(dhead);
          if (dh < a.n_tiles && diag_ready(dh)) {
            if (atomicCAS(dhead, dh, dh + 1) == dh) {
              w = dh;
              break;
            }
            continue;
          }
          const int fh = ld_acquire(fhead);
          if (fh < a.n_far_ctas && far_ready(fh)) {
            if (atomicCAS(fhead, fh, fh + 1) == fh) {
              w = -(int64_t)fh - 1;
              break;
            }
            continue;
          }
          if (dh >= a.n_tiles && fh >= a.n_far_ctas) break;  // all claimed: done
          if (ld_acquire(err)) break;
          __nanosleep(nap);  // exponential backoff: idle CTAs must not flood L2 with polls
          nap = nap < 2048 ? 2 * nap : nap;
          if (++spins > (1u << 24)) {
            atomicExch(err, 1);
            break;
          }
        }
      } else {
        const int fh = atomicAdd(fhead, 1);
        if (fh < a.n_far_ctas) {
          const int64_t item = fh / a.H;
          const int lv = a.level_of[a.far_items[item].x];
          bool ok = wait_at_least(a.ctr + c.done + a.far_dep[item], 1, err);
          if (ok && lv >= kRing) ok = wait_at_least(level_done + (lv - kRing), a.level_count[lv - kRing], err);
          if (ok) w = -(int64_t)fh - 1;
        }
      }
      s_w = w;
      __threadfence();
    }
    __syncthreads();
    const int64_t w = s_w;
    if (w == INT64_MIN) break;
    if (w < 0) {  // far CTA-item
      const int64_t idx = -w - 1;
      const int64_t item = idx / a.H;
      const int half = (int)(idx % a.H);
      const int4 it = a.far_items[item];
      const int lv = a.level_of[it.x];
      double2* out = a.far_ring + ((int64_t)(lv % kRing) * a.max_far + a.far_rel[item]) * 4096;
      update_body<2, 2, true, 1, 3, 2>(a.g, a.T, a.tiles, it, half, out, a.Y, sm);
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        atomicAdd(a.ctr + c.far_done + it.x, 1);
      }
    } else {  // diagonal tile
      const int64_t slot = w;
      const int lv = a.level_of[slot];
      diag_lines_body<N, B, NT, true, false>(
          a.g, a.T, a.tiles[slot], a.tile_ranges[slot], a.far_ring + (int64_t)(lv % kRing) * a.max_far * 4096,
          a.near_ring + (int64_t)(lv % kRing) * a.max_near * 4096, a.near_target + slot * N,
          a.near_ring + (int64_t)((lv + 1) % kRing) * a.max_near * 4096, a.Y, sm);
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        for (int m = 0; m < N; ++m) {
          const int ps = a.push_slot[slot * N + m];
          if (ps >= 0) atomicAdd(a.ctr + c.push_done + ps, 1);
        }
        atomicExch(a.ctr + c.done + slot, 1);
        atomicAdd(level_done + lv, 1);
      }
    }
    __syncthreads();
  }
}
