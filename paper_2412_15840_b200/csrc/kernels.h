// Internal launch interface between the C-ABI layer (capi.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <vector>

#include "common.cuh"

namespace nds {

// Device copies of the Schur factors of one problem. Every U_j is kept in the four layouts the
// transform kernels read without a permutation pass: M row-major / column-major for M = U_j
// (inverse transform) and M = U_j^H (forward transform).
struct FactorSet {
  int n_modes = 0;
  int64_t dims[NDS_MAX_MODES] = {};
  double2* u_row[NDS_MAX_MODES] = {};
  double2* u_col[NDS_MAX_MODES] = {};
  double2* uh_row[NDS_MAX_MODES] = {};
  double2* uh_col[NDS_MAX_MODES] = {};
  // Stage-blocked copies for the bulk-copy (TMA) fed transform GEMM, modes with n_j a multiple of
  // 16: per op (0: U, 1: U^H) and CTA shape (0: 64 x 32, 1: 32 x 64), the A operand of the
  // row-major GEMM as [row tile][k tile][BM rows][BK + 4] and the B operand of the mode-1 GEMM
  // as [column tile][k tile][BK][BN + 2] — the padded shared-memory stage images, so one
  // cp.async.bulk moves a whole operand stage (transform.cu).
  double2* ablk[NDS_MAX_MODES][2][2] = {};
  double2* bblk[NDS_MAX_MODES][2][2] = {};
  double2* pool = nullptr;  // one allocation backing all of the above + T + diag
  cudaStream_t stream = nullptr;  // stream the pool was allocated on (stream-ordered free)
  double2* t_pool = nullptr;     // T_j column-major, concatenated (offsets in geom.toff)
  double2* diag_pool = nullptr;  // diag(T_j), concatenated (offsets in geom.doff)
  Geom geom{};
};

// Launch classes (for the per-launch profile read back by bench.py).
enum LaunchKind { kXformGemm = 0, kXformDirect = 1, kBacksubLevel = 2, kElementwise = 3, kBacksubPersistent = 4 };

// Optional CUDA-event recorder: one event after every launch (ev[0] is the start marker).
struct Recorder {
  cudaEvent_t* ev = nullptr;
  int* kind = nullptr;
  int* mode = nullptr;
  int cap = 0;
  int n = 0;
  void mark(cudaStream_t s, int k, int m) {
    if (ev && n < cap) {
      cudaEventRecord(ev[n], s);
      kind[n] = k;
      mode[n] = m;
      ++n;
    }
  }
};

// r = M x_mode x (+ r), M = U_mode or U_mode^H. One launch; returns its LaunchKind.
int mode_product_launch(const FactorSet& f, int mode, bool adjoint, const ModeView& v, const double2* x, double2* r,
                        bool accumulate, cudaStream_t stream);

// A run of `count` binary modes starting at mode `first` (1-based) applied in one fused pass on
// the (inner, 2^count, outer) view, with runs of 2^logR inner entries per tile.
struct BinGroup {
  int first = 0, count = 0, logR = 0;
  int64_t inner = 1, outer = 1;
};
// Fused groups of runs of binary modes among modes [lo, hi) (0-based; hi < 0: all modes).
std::vector<BinGroup> plan_binary_groups(int n_modes, const int64_t* dims, int lo = 0, int hi = -1);
// unit: f's matrices for these modes are unit-diagonal [[1, p], [q, 1]] (the normalised factors
// of the fused all-binary route; their diagonal parts are applied by the fused tile kernel).
int binary_pass_launch(const FactorSet& f, const BinGroup& gr, bool adjoint, const double2* x, double2* r,
                       cudaStream_t stream, bool unit = false);
// Modes 1-12 forward (fwd's U^H), the decoupled 12-mode tile solve (den over all modes; the
// outer modes' coupling diagonalised away), modes 1-12 inverse (inv's U) — one kernel, one read
// and one write of the tensor; gr is the modes-1-12 pass (first 1, count 12, inner 1).
// t_pool: T'_j (2 x 2, all N modes; diagonal for the diagonalised ones), wf / wf_off: the tile
// entries by popcount over the coupled inner modes (levels = their count + 1).
// Host copies of what the device pointers hold (all N modes): the forward / inverse 2 x 2
// matrices (column-major, 4 per mode), T'_j (4 per mode) and, on the normalised route, the scales
// (2 per mode; else nullptr). The round kernel takes its coefficients by value from them.
struct BinHostFactors {
  const double2* fwd = nullptr;
  const double2* inv = nullptr;
  const double2* t = nullptr;
  const double2* e = nullptr;
};
int binary_fused_solve_launch(const FactorSet& fwd, const FactorSet& inv, const BinGroup& gr, const double2* t_pool,
                              int n_outer, const uint16_t* wf, const int* wf_off, int levels, int cmask,
                              const BinHostFactors& host, const double2* x, double2* r, cudaStream_t stream,
                              const double2* unit_scales = nullptr);
// cmask: the inner modes left coupled (bit j = mode j + 1). Up to four: the tile solve is one
// round of the butterfly network (binary_fused_round_kernel; wf unused); more: the popcount
// wavefront kernel.
// unit_scales != nullptr: the normalised route — fwd / inv hold unit-diagonal matrices for all
// modes, unit_scales the deferred diagonal scale e_j[0], e_j[1] of every mode (2 per mode), and
// t_pool's couplings carry the inverse factors' column-scale ratio (binary_pass.cu).

// Plain matrix variant (apply_operator / residual): m_row, m_col are the two layouts of M.
// rows_out > 0: rectangular M (rows_out x n), r has extent rows_out along the mode.
// lda_row > 0: m_row is a column block of a wider row-major matrix (row stride lda_row); only
// valid on the GEMM path with inner >= 8 (the caller checks gemm_rowm_ok).
// blk: the two stage-blocked images of M for the bulk-copy GEMM (FactorSet::ablk / bblk), or null.
int mode_product_matrix_launch(const double2* m_row, const double2* m_col, const ModeView& v, const double2* x,
                               double2* r, bool accumulate, cudaStream_t stream, int64_t rows_out = -1,
                               int64_t lda_row = -1, const double2* const* blk = nullptr);
inline bool gemm_rowm_ok(const ModeView& v) { return v.n >= 16 && v.inner >= 8; }

// ---- triangular solve --------------------------------------------------------------------
struct TileGeom {
  int n_modes;
  int tile_entries;  // prod b_j
  int64_t dims[NDS_MAX_MODES];
  int64_t strides[NDS_MAX_MODES];
  int64_t nb[NDS_MAX_MODES];  // blocks per mode
  int64_t toff[NDS_MAX_MODES];
  int b[NDS_MAX_MODES];       // tile extent per mode
  int bstride[NDS_MAX_MODES]; // strides inside a full tile
};

// Far-update work item (backsub_v2.cuh far_group_body, G = 1): target tile slot, mode, source
// rows [kb, ke) along the mode, and the far-partial ring slot it writes.
struct FarGroupItem {
  int tile;     // tile slot whose other block coordinates define the columns
  int j;        // mode
  int kb, ke;   // source rows along j (absolute; multiple of the stage depth)
  int rb0;      // target block along j
  int nrb;      // valid row blocks (1)
  int acc;      // 1: accumulate into the slot (0 for G = 1)
  int pad;
  int out[4];   // far-partial ring slot per row block
};

struct SolvePlan {
  TileGeom geom{};
  int levels = 0;                 // tile hyperplanes: sum_j (nb_j - 1) + 1
  std::vector<int64_t> level_off; // host copy, size levels + 1
  int64_t* d_tiles = nullptr;     // tile ids sorted by descending level
  int wf_levels = 0;              // hyperplanes inside a full tile
  int* d_wf = nullptr;            // generic tiles: local entries sorted by descending local level
  int* d_wf_off = nullptr;
  int* d_near_target = nullptr;   // cubic: [tile slot][mode] near item of slot - e_mode at the next level
  void* pool = nullptr;
  // Cubic regime (c0-c3: B^N = 4096-entry tiles, B in {8, 16} dividing every n_j): per level,
  // far-update DMMA items (neighbours >= 2 blocks away, ready one level early, low-priority
  // streams) into a ring of level regions, then one diagonal-tile launch that also pushes the
  // near updates (adjacent block) of the next level.
  bool v2 = false;
  std::vector<int64_t> near_off;  // per level: near items (computed by the previous level's diagonal CTAs)
  int4* d_tile_ranges = nullptr;  // per tile slot: {far first, far count, near first, near count} (level-relative)
  double2* d_near_partial = nullptr;   // near partials double-buffered by level parity
  double2* d_near_partial2 = nullptr;
  int64_t max_near = 0;
  std::vector<int64_t> fg_off;         // per level: [fg_off[lv], fg_off[lv + 1]) of d_fg_items
  FarGroupItem* d_fg_items = nullptr;
  double2* d_fg_ring = nullptr;        // far partials: fg_ring level regions of fg_slots tiles
  int fg_ring = 0;
  int64_t fg_slots = 0;
  cudaStream_t s_crit = nullptr, s_far = nullptr, s_far2 = nullptr;  // far: even / odd levels
  std::vector<cudaEvent_t> ev;  // diag(lv), far(lv), start, end
};

// All-binary regime (every n_j = 2, config c4): contiguous 2^min(N,12)-entry tiles, binary outer
// modes, one launch per outer popcount level (binary_solve.cu).
struct BinarySolvePlan {
  int m = 0, n_outer = 0, levels = 0;
  std::vector<int64_t> level_off;
  int64_t* d_tiles = nullptr;
  int* d_wf = nullptr;
  int* d_wf_off = nullptr;
  uint16_t* d_wf_swz = nullptr;  // the same levels, bank-group interleaved for the swizzled tile
  void* pool = nullptr;
};
void binary_solve_plan_build(BinarySolvePlan& bp, int n_modes);
void binary_solve_plan_free(BinarySolvePlan& bp);
// t_pool: T_j (2x2 column-major) at t_pool + 4 j.
// decoupled: the outer modes were diagonalised into the transform passes (capi.cu, all-binary
// route), so every tile is an independent inner-mode solve (den still includes the outer modes).
int binary_solve_launch(const BinarySolvePlan& bp, const double2* t_pool, double2* c, cudaStream_t stream,
                        Recorder* rec = nullptr, bool decoupled = false);

// Block-diagonalised cubic route (backsub_blk.cuh): super-blocks of d[j] rows per mode (multiples
// of the tile edge); the coupled modes (d < n) tiled 64^2 / 16^3 / 8^4 by their count, the
// uncoupled ones a batch (or every mode tiled when no kernel fits); tiles grouped by super-tile
// level sum_j floor(I_j b / d_j) (highest first; within a level longest pull first), one launch
// per level.
struct BlkSolvePlan {
  int d[NDS_MAX_MODES] = {};      // per tiled mode
  int dmode[NDS_MAX_MODES] = {};  // per mode of the problem
  TileGeom g{};               // the tiled modes: the coupled ones (the rest a batch), or all
  int levels = 0;
  int64_t ntc = 1, nbatch = 1;
  std::vector<int> uncoupled;  // batch modes (empty: none folded)
  std::vector<int64_t> level_off;
  int64_t* d_tiles = nullptr;
  int64_t* d_boff = nullptr;  // batch origin offsets (inside d_tiles' allocation), or null
};
struct BlkBatchModes {
  int count;
  int mode[NDS_MAX_MODES];
};
// Dims-only solver structures (tile lists, work items, partial buffers, internal streams), cached
// per context and shared by every plan with the same extents; the block-diagonalised route's
// level lists by super-block extents.
struct SolverCache {
  bool binary = false;
  BinarySolvePlan bsp;
  SolvePlan sp;
  std::map<std::vector<int>, BlkSolvePlan> blk;
  std::map<int, void*> bin_wf;  // all-binary diagonalised route: tile wavefront by coupled-mode mask
  ~SolverCache();
};

void blk_solve_plan_build(BlkSolvePlan& bp, int n_modes, const int64_t* dims, const int64_t* toff, const int* d,
                          int b);
// Per plan: the batch denominators sum_{uncoupled j} T'_j(i_j, i_j) (diag of the route's T').
void blk_batch_den_launch(const BlkSolvePlan& bp, const Geom& g, const double2* diag, double2* out,
                          cudaStream_t stream);
void blk_solve_plan_free(BlkSolvePlan& bp);
int blk_backsub_launch(const BlkSolvePlan& bp, const double2* t_pool, const double2* bden, double2* c,
                       cudaStream_t stream, Recorder* rec = nullptr);
// Schur reordering of the block-diagonalised route (blockdiag.cu): per mode, T_j and U_j (n x n
// column-major at off[m] in the two pools, in place) reordered so the eigenvalue of real-part rank
// R(P) sits at position P, R = digit reversal over the radices rad[m][0..nrad) (least significant
// first: the tile edge, then 2s, then the rest); nrad = 0 skips the mode.
constexpr int kReorderMaxN = 1024;
struct ReorderArgs {
  int n[NDS_MAX_MODES];
  int64_t off[NDS_MAX_MODES];
  int nrad[NDS_MAX_MODES];
  int rad[NDS_MAX_MODES][12];
};
// bar: a device word for the grid barrier (zeroed here).
void schur_reorder_launch(const ReorderArgs& ra, int n_modes, double2* tpool, double2* upool, unsigned int* bar,
                          cudaStream_t stream);
// diag(T_j) of every mode (t_pool at g.toff) into diag (at g.doff).
void diag_extract_launch(const Geom& g, const double2* t_pool, double2* diag, cudaStream_t stream);
// Small plan data written by a kernel from its by-value parameter (no copy-engine traffic, so it
// does not queue behind a tensor streaming in): dst[0, count) = blob.v.
constexpr int kParamBlobMax = 20 * NDS_MAX_MODES;
struct ParamBlob {
  int count;
  double2 v[kParamBlobMax];
};
void param_blob_launch(const ParamBlob& blob, double2* dst, cudaStream_t stream);
// Eigenvector blocks of the route's candidates (blockdiag.cu): job = block at row offset o of
// T_j (n x n at t_pool + toff) with extent d <= 128; V, W = V^{-1} (d x d column-major at
// vpool / wpool + voff) and cond_2(V) into cond[job] (inf on a repeated eigenvalue).
// Candidates are passed by value (no host->device copy in the plan, which runs while the tensor
// streams in): candidate c covers jobs [first[c], first[c + 1]), blocks q = job - first[c].
constexpr int kMaxEigCands = 6 * NDS_MAX_MODES;
// Extents d > 128 (a whole mode, D = n <= 256) use global scratch: 2 d^2 entries per block at
// soff[c] + 2 q d^2.
struct EigCands {
  int count;
  int d[kMaxEigCands];
  int first[kMaxEigCands + 1];
  int64_t n[kMaxEigCands], toff[kMaxEigCands], voff[kMaxEigCands], soff[kMaxEigCands];
};
void block_eig_launch(const double2* t_pool, const EigCands& cands, double2* vpool, double2* wpool, double* cond,
                      double2* scratch, cudaStream_t stream);
// The route's factors of one mode (n x n column-major; V, W = V^{-1}: n / d blocks of d x d):
// minv = U blockdiag(V), mfh = U blockdiag(W)^H, tv = T blockdiag(V) (scratch),
// tprime = blockdiag(W) T blockdiag(V) with diagonal d-blocks = diag(T) exactly, zero below.
void blockdiag_factors_launch(int64_t n, int d, const double2* u, const double2* t, const double2* v, const double2* w,
                              double2* minv, double2* mfh, double2* tv, double2* tprime, cudaStream_t stream);

void solve_plan_build(SolvePlan& sp, int n_modes, const int64_t* dims, const int64_t* toff);
void solve_plan_free(SolvePlan& sp);
// Head overlap: the last forward pass (mode N) produced in row groups of `per` mode-N tile blocks,
// highest first, group g signalled by ev[g]; the diagonal tiles of a level wait only for the
// groups holding their blocks.
struct HeadSync {
  int per = 0;
  const cudaEvent_t* ev = nullptr;
};
// Tail overlap: after the diagonal launch of each level, fn(ctx, lv, critical stream) — used to
// start the first inverse pass on the mode-N slabs of Y that this level completed.
struct TailHook {
  void (*fn)(void* ctx, int lv, cudaStream_t crit) = nullptr;
  void* ctx = nullptr;
};
// In-place Y over C. Returns kernels launched.
int backsub_launch(const SolvePlan& sp, const double2* t_pool, double2* c, cudaStream_t stream,
                   Recorder* rec = nullptr, const HeadSync* head = nullptr, const TailHook* tail = nullptr);

// ---- matrix functions (ODE propagator) -----------------------------------------------------
// exp(t T_m) by the Parlett recurrence, one CTA per listed mode: T_m at t_pool + toff[m]
// (column-major), result at f + foff[m] as [row-major | column-major] n x n.
struct ExpArgs {
  const double2* t_pool;
  const double2* t_row;        // row-major T_m at t_row + foff[m] / 2
  double2* f;
  double t;
  int mode[NDS_MAX_MODES];     // modes handled (0-based), count given at launch
  int64_t n[NDS_MAX_MODES];    // extent of the listed mode (same index as mode[])
  int64_t toff[NDS_MAX_MODES]; // by mode
  int64_t foff[NDS_MAX_MODES]; // by mode
};
int parlett_launch(const ExpArgs& a, int count, cudaStream_t stream);

// ---- elementwise / reductions ------------------------------------------------------------
// Build u_row / u_col / uh_row / uh_col of every mode from the raw column-major U_j (concatenated).
void factor_layouts_launch(const FactorSet& f, const double2* raw, cudaStream_t stream);
// Entries of the stage-blocked operand images of one n x n factor (0 when n is not a multiple
// of 16), and their construction from u_row / u_col / uh_row / uh_col (transform.cu).
int64_t blocked_entries(int64_t n);
// op_mask: bit 0 builds the images of U, bit 1 those of U^H (sets that use one op only).
void blocked_layouts_launch(FactorSet& f, double2* base, cudaStream_t stream, int op_mask = 3);
// min |den| over all entries and the largest flat index with |den| <= tol (-1 if none).
void den_scan(const Geom& g, const double2* diag, double tol, double* min_abs, int64_t* max_bad, cudaStream_t stream,
              void* scratch /* >= 16 bytes device */);
int fast_divide_launch(const Geom& g, const double2* diag, double2* c, cudaStream_t stream);
int real_part_launch(double2* x, int64_t total, cudaStream_t stream);
// z = x + alpha y (z may alias x or y).
int axpy_launch(double2* z, const double2* x, double2 alpha, const double2* y, int64_t total, cudaStream_t stream);
// x += a1 k1 + a2 k2 + a2 k3 + a1 k4 (RK4 update, reference order).
int rk4_combine_launch(double2* x, double2 a1, double2 a2, const double2* k1, const double2* k2, const double2* k3,
                       const double2* k4, int64_t total, cudaStream_t stream);
// Fused RK4 stage (small tensors, N <= 8): K = sum_j A_j x_j in + B, then ST_out = X + c K or,
// in the final stage, X += a1 K1 + a2 K2 + a2 K3 + a1 K.
struct Rk4Stage {
  int n_modes;
  int64_t total;
  int64_t dims[8], strides[8];
  const double2* a_row[8];  // row-major A_j, followed by its column-major copy
  const double2* in;
  const double2* b;
  double2* x;
  double2* k_out;
  double2* st_out;
  double2 c;
  int final_stage;
  const double2 *k1, *k2, *k3;
  double2 a1, a2;
};
int rk4_stage_launch(const Rk4Stage& a, cudaStream_t stream);
// All RK4 steps in one cooperative launch (grid barriers between stages): `steps` steps of h,
// then one of h_last when it is non-zero. Buffers: state, K1..K4, two stage tensors.
struct Rk4Buffers {
  double2* x;
  double2* k[4];
  double2* st[2];
  unsigned int* bar;  // grid-barrier counter, zeroed before the launch
};
int rk4_persistent_launch(const Rk4Stage& base, const Rk4Buffers& buf, int64_t steps, double h, double h_last,
                          cudaStream_t stream);
// *flag |= 1 when x has an Inf or NaN entry.
int nonfinite_launch(const double2* x, int64_t total, int* flag, cudaStream_t stream);
// Max-abs and sum-of-squares of (r - b) and of b, deterministic (per-block partials).
void residual_norms(const double2* r, const double2* b, int64_t total, double* res_max, double* res_2, double* b_max,
                    double* b_2, cudaStream_t stream);

}  // namespace nds
