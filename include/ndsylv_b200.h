/*
 * ndsylv_b200 — B200-native (sm_100a) hot path of the non-recursive N-D Bartels–Stewart
 * solver for  sum_j A_j x_j X = B  (arXiv 2412.15840), behind a plain C ABI.
 *
 * Drop-in boundary. Each entry point below replaces one function of the reference C++ API
 * (/root/reference/proj/include/ndsylv/*.hpp) and keeps its argument meaning, layout and
 * error behaviour; INTEGRATION.md shows the adapter a maintainer adds on the reference side.
 *
 *   Layout: tensors are column-major (first index fastest) arrays of complex128 — the exact
 *   storage of ndsylv::NDTensor::data (tensor.hpp:23-39); matrices are column-major n x n
 *   (ndsylv::Matrix, matrix.hpp:11-30). nds_z is layout-identical to std::complex<double>.
 *   Modes are 1-based where a mode number is passed (kernels.hpp:10-12).
 *
 *   Errors: every call returns an nds_status. The codes mirror the reference's exception
 *   types and the CLI's exit-code mapping (tools/ndsylv_main.cpp:366-381):
 *     SingularOperatorError (types.hpp:31-47) -> NDS_ERR_SINGULAR (=2) + nds_singular filled
 *     std::bad_alloc / device out of memory   -> NDS_ERR_NOMEM (=4)
 *     std::invalid_argument                   -> NDS_ERR_INVALID
 *     ConvergenceError (Schur, schur.cpp:146) -> NDS_ERR_CONVERGENCE
 *     std::overflow_error (tensor.cpp:13)     -> NDS_ERR_OVERFLOW
 *     NonFiniteStateError (types.hpp:62-66)   -> NDS_ERR_NONFINITE
 *   The message of the last failure on a context is returned by nds_last_error().
 *
 *   Threading: one context per host thread; a context owns one CUDA device, one stream and
 *   the workspaces. Host-buffer calls are synchronous (like the reference); the nds_plan_*
 *   device-pointer calls are asynchronous on the context stream. There is no CPU fallback:
 *   without a usable sm_100 device every compute call returns NDS_ERR_CUDA.
 */
#ifndef NDSYLV_B200_H
#define NDSYLV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NDS_MAX_MODES 64 /* NDT1 order limit, README.md "Tensor files" */

typedef struct {
  double re, im;
} nds_z;

typedef enum {
  NDS_OK = 0,
  NDS_ERR_OTHER = 1,
  NDS_ERR_SINGULAR = 2,
  NDS_ERR_FILE = 3,
  NDS_ERR_NOMEM = 4,
  NDS_ERR_INVALID = 5,
  NDS_ERR_CONVERGENCE = 6,
  NDS_ERR_OVERFLOW = 7,
  NDS_ERR_CUDA = 8,
  NDS_ERR_NONFINITE = 9
} nds_status;

/* SolveOptions (sylvester.hpp:19-28): allow_fast_path defaults to true in the reference.
 * NDS_NO_DIAGONALISE (B200 extension): full solves keep the plain Schur factors and the
 * wavefront tile solves even when the block-diagonalised route's guard passes. */
enum { NDS_ALLOW_FAST_PATH = 1u, NDS_REAL_OUTPUT = 2u, NDS_NO_DIAGONALISE = 4u };

/* SolveReport (sylvester.hpp:30-42) plus device-side timings. */
typedef struct {
  double min_abs_denominator;
  int32_t used_normal_fast_path;
  int64_t flop_estimate;
  int64_t schur_flop_estimate;
  int64_t backsub_entries;
  int64_t backsub_multiplies;
  double schur_seconds;     /* host Schur setup (nds_solve only) */
  double transform_seconds; /* forward transform, device time */
  double backsub_seconds;   /* triangular solve (or fast-path divide), device time */
  double inverse_seconds;   /* inverse transform, device time */
  double total_seconds;     /* wall time of the call */
  double h2d_seconds;       /* host->device copy of B (host-buffer calls) */
  double d2h_seconds;       /* device->host copy of X (host-buffer calls) */
  int32_t kernel_launches;  /* device kernels launched by the call */
} nds_report;

/* SingularOperatorError payload: 1-based multi-index of the FIRST offender in the reference's
 * descending visiting order (sylvester.cpp:88-103) and its denominator. */
typedef struct {
  int32_t n_modes;
  int64_t multi_index[NDS_MAX_MODES];
  double den_re, den_im;
} nds_singular;

/* BackSubstituteStats (sylvester.hpp:69-73) */
typedef struct {
  int64_t entries;
  int64_t multiplies;
  double min_abs_denominator;
} nds_backsub_stats;

typedef struct nds_ctx nds_ctx;
typedef struct nds_plan nds_plan;
typedef struct nds_ode nds_ode;

const char* nds_version(void);

/* ---- context ------------------------------------------------------------------------- */
int nds_ctx_create(nds_ctx** out, int device);
void nds_ctx_destroy(nds_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores the own stream.
 * To run on the legacy default stream pass cudaStreamLegacy ((void*)0x1), not NULL. */
int nds_ctx_set_stream(nds_ctx* ctx, void* cuda_stream);
void* nds_ctx_stream(nds_ctx* ctx);
const char* nds_last_error(const nds_ctx* ctx);
/* Release cached device workspaces. */
void nds_ctx_trim(nds_ctx* ctx);

/* ---- reference API, host buffers ----------------------------------------------------- */

/* ndsylv::solve (sylvester.hpp:79, sylvester.cpp:167-227): Schur on the host (timed into
 * rep->schur_seconds), transforms + triangular solve on the GPU. x may alias b. */
int nds_solve(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* a, const nds_z* b, nds_z* x,
              double singular_tol, unsigned flags, nds_report* rep, nds_singular* sing);

/* The same path when the caller already holds the Schur factors A_j = U_j T_j U_j^H
 * (SchurFactors, schur.hpp:9-14) — what ndsylv::solve does after its schur() calls. */
int nds_solve_schur(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* u, const nds_z* const* t,
                    const nds_z* b, nds_z* x, double singular_tol, unsigned flags, nds_report* rep,
                    nds_singular* sing);

/* ndsylv::schur (schur.hpp:19) — host complex Schur (Householder Hessenberg + shifted QR). */
int nds_schur(nds_ctx* ctx, int n, const nds_z* a, nds_z* u, nds_z* t);

/* ndsylv::forward_transform (sylvester.hpp:64): c = U_N^H x_N ( ... U_1^H x_1 b ). c may alias b. */
int nds_forward_transform(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* u, const nds_z* b,
                          nds_z* c);
/* ndsylv::inverse_transform (sylvester.hpp:67): x = U_N x_N ( ... U_1 x_1 y ). x may alias y. */
int nds_inverse_transform(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* u, const nds_z* y,
                          nds_z* x);
/* ndsylv::back_substitute (sylvester.hpp:77): overwrites c with y in place. */
int nds_back_substitute(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* t, nds_z* c,
                        double singular_tol, nds_backsub_stats* stats, nds_singular* sing);
/* ndsylv::mode_product (kernels.hpp:12): r = m x_mode x (mode 1-based). r must not alias x. */
int nds_mode_product(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* m, int mode, const nds_z* x,
                     nds_z* r);
/* ndsylv::apply_operator (sylvester.hpp:61): r = sum_j A_j x_j x. */
int nds_apply_operator(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* a, const nds_z* x,
                       nds_z* r);
/* ndsylv::flop_estimate / schur_flop_estimate (sylvester.hpp:86-90); -1 on invalid/overflow. */
int64_t nds_flop_estimate(int n_modes, const int64_t* dims);
int64_t nds_schur_flop_estimate(int n_modes, const int64_t* dims);

/* ---- plans: device-resident, reusable (B200-native extension) ------------------------- */

/* Uploads the factors, runs the singular check (NDS_ERR_SINGULAR + sing on failure) and
 * decides the route (fast path or triangular solve), like sylvester.cpp:180-213. */
int nds_plan_create(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* u, const nds_z* const* t,
                    double singular_tol, unsigned flags, nds_plan** out, nds_singular* sing);
void nds_plan_destroy(nds_plan* plan);
/* Fills the static report fields (min |den|, route, estimates, counts). */
int nds_plan_report(const nds_plan* plan, nds_report* rep);
int64_t nds_plan_total(const nds_plan* plan);

/* Device pointers, async on the context stream. d_b is not modified; d_x may equal d_b.
 * d_work: NULL (use the context workspace) or a device buffer of plan_total entries. */
int nds_plan_execute(nds_plan* plan, const nds_z* d_b, nds_z* d_x, nds_z* d_work);
/* Stages, device pointers, async. forward/inverse: out may equal in. backsub is in place. */
int nds_plan_forward(nds_plan* plan, const nds_z* d_in, nds_z* d_out, nds_z* d_work);
int nds_plan_backsub(nds_plan* plan, nds_z* d_c);
int nds_plan_inverse(nds_plan* plan, const nds_z* d_in, nds_z* d_out, nds_z* d_work);
/* Host buffers, synchronous: H2D(b), execute, D2H(x); stage device times into rep. */
int nds_plan_execute_host(nds_plan* plan, const nds_z* h_b, nds_z* h_x, nds_report* rep);
/* count right-hand sides through the same plan, synchronous: x[k] = solve(b[k]). With PINNED
 * buffers the solves are pipelined (H2D of b[k+1] and D2H of x[k-1] overlap solve k on separate
 * copy streams; device B / X double-buffered), so the period per right-hand side is
 * max(solve, H2D, D2H); pageable buffers run nds_plan_execute_host per right-hand side. x[k] may
 * alias b[k], no other aliasing. rep: static fields, total_seconds (the whole call) and
 * kernel_launches (all solves). Replaces a loop of ndsylv::solve over the same coefficients
 * (sylvester.cpp:167-227) with the Schur step and the plan done once. */
int nds_plan_execute_host_many(nds_plan* plan, int count, const nds_z* const* h_b, nds_z* const* h_x,
                               nds_report* rep);
/* Kernel launches one nds_plan_execute issues. */
int nds_plan_launches(const nds_plan* plan);
/* Which triangular-solve route the plan takes: the fast-path divide,
 * generic tiles (any shape), cubic 16^3 / 8^4 tiles with DMMA far updates (c0-c3), or the
 * all-binary tiles (c4). -1 for a NULL plan. */
enum { NDS_PATH_FAST = 0, NDS_PATH_GENERIC = 1, NDS_PATH_CUBIC = 2, NDS_PATH_BINARY = 3 };
int nds_plan_solve_path(const nds_plan* plan);
/* Whether FULL solves (nds_plan_execute / _execute_host / nds_solve*) run on diagonalised factors:
 * cubic route — every B x B diagonal block of T_j diagonalised (diagonal tiles become divisions);
 * binary route — the outer modes' 2 x 2 T_j diagonalised (tiles decouple). *cond receives the
 * guard's bound prod_j cond_2 (<= 1e6 when taken; 0 when not evaluated). Returns 1 / 0, -1 for a
 * NULL plan. Stage calls (forward / backsub / inverse) always use the plain factors. */
int nds_plan_diagonalised(const nds_plan* plan, double* cond);
/* Cubic block-diagonalised route: d[j] = the super-block extent D_j of mode j (T_j's D_j x D_j
 * diagonal blocks diagonalised); returns the number of solve levels sum_j (n_j / D_j - 1) + 1,
 * 0 when full solves do not take that route (d untouched), -1 for a NULL plan. */
int nds_plan_superblocks(const nds_plan* plan, int64_t* d);
/* Per-launch device timing: after _begin, every launch of execute/forward/backsub/inverse records
 * a CUDA event on the context stream (up to max_launches). _end synchronises and returns the
 * number of launches written: kind (0 transform GEMM, 1 transform direct, 2 solve level,
 * 3 elementwise, 4 persistent solve), mode (+j inverse / -j forward, or solve level) and ms. */
int nds_plan_profile_begin(nds_plan* plan, int max_launches);
int nds_plan_profile_end(nds_plan* plan, int cap, int* kinds, int* modes, float* ms);

/* ---- device-pointer kernels (test / residual surfaces) -------------------------------- */

/* r = op(m) x_mode x (+ r if accumulate); op = m or m^H (conj_transpose). m is a DEVICE n x n
 * column-major matrix. Async on the context stream. r must not alias x. */
int nds_dev_mode_product(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* d_m, int mode,
                         int conj_transpose, const nds_z* d_x, nds_z* d_r, int accumulate);
/* Rectangular update along one mode, device tensors (multi-GPU slab coupling):
 *   r += M x_mode x,  x of extents dims_x, r of the same extents except rows_out along `mode`,
 *   M a HOST rows_out x dims_x[mode-1] column-major matrix (negate it to subtract). Async. */
int nds_dev_mode_update(nds_ctx* ctx, int n_modes, const int64_t* dims_x, int mode, int64_t rows_out,
                        const nds_z* m, const nds_z* d_x, nds_z* d_r);
/* The same product without accumulation (r = M x_mode x; r need not be initialised): the
 * sharded solver's local mode products. Async on the context stream. */
int nds_dev_mode_apply(nds_ctx* ctx, int n_modes, const int64_t* dims_x, int mode, int64_t rows_out,
                       const nds_z* m, const nds_z* d_x, nds_z* d_r);
/* In-place triangular solve of a device tensor (back_substitute on device memory): T_j HOST
 * upper-triangular matrices. Synchronous; singular check and stats as nds_back_substitute. */
int nds_dev_back_substitute(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* t, nds_z* d_c,
                            double singular_tol, nds_backsub_stats* stats, nds_singular* sing);
/* Device residual: returns max_i |sum_j A_j x_j X - B|_i and the 2-norm, plus |B| norms.
 * a[] are HOST matrices (uploaded), d_x and d_b device tensors. Synchronous. */
int nds_dev_residual(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* a, const nds_z* d_x,
                     const nds_z* d_b, double* res_max, double* res_2, double* b_max, double* b_2);

/* ---- multi-GPU sharded solve ---------------------
 * One rank per GPU. B and X are sharded in layout L_N: rank r owns a contiguous range of the
 * column-major tensor (nds_dist_slab) — a block of the last mode, or for all-binary problems one
 * index of the last log2 P modes. Inside a solve the transforms re-shard once each way by an
 * all-to-all and the triangular solve is pipelined over (rank, block of the last modes) with
 * point-to-point forwarding of solved blocks; all exchanges are NCCL P2P on the rank's own
 * communication stream, ordered against its compute stream by events (no host sync). */
typedef struct nds_comm nds_comm;
typedef struct nds_dist nds_dist;
#define NDS_COMM_ID_BYTES 128
typedef struct {
  int32_t ranks, rank;
  int32_t head_modes, tail_modes, pipe_modes, pipe_blocks;
  int32_t local_solve_path;  /* NDS_PATH_* of the rank's local block solves */
  int32_t launches;          /* kernels of the last solve (this rank) */
  int64_t alltoall_bytes;    /* bytes this rank sends in the two all-to-alls of one solve */
  int64_t pipeline_bytes;    /* bytes this rank forwards to lower ranks in one solve */
  double min_abs_denominator;
} nds_dist_info_t;
/* NCCL unique id (rank 0 creates it, the caller broadcasts the NDS_COMM_ID_BYTES bytes). */
int nds_comm_unique_id(void* id_out);
/* NCCL communicator of rank `rank` of `world` on CUDA device `device` (NCCL is loaded at run
 * time: libnccl.so.2, the copy already in the process if any). */
int nds_comm_create_nccl(nds_comm** out, int device, int rank, int world, const void* id);
/* In-process transport for `world` ranks sharing one device (one host thread per rank; tests):
 * fills out[0..world-1]. */
int nds_comm_create_loopback(int world, nds_comm** out);
void nds_comm_destroy(nds_comm* comm);
/* Rank state for the problem with Schur factors u, t (identical on every rank); comm NULL = one
 * rank. Runs the singular check of the WHOLE operator first, so every rank fails alike
 * (NDS_ERR_SINGULAR + sing with the global first offender) before any exchange. */
int nds_dist_create(nds_ctx* ctx, nds_comm* comm, int n_modes, const int64_t* dims, const nds_z* const* u,
                    const nds_z* const* t, double singular_tol, nds_dist** out, nds_singular* sing);
void nds_dist_destroy(nds_dist* d);
/* Rank r's L_N slab: flat offset and entry count within the full column-major tensor. */
int nds_dist_slab(const nds_dist* d, int rank, int64_t* offset, int64_t* count);
int nds_dist_info(const nds_dist* d, nds_dist_info_t* info);
/* x = solve(b) on this rank's slabs (device pointers), asynchronous on the context stream; every
 * rank of the communicator must call it. */
int nds_dist_solve(nds_dist* d, const nds_z* d_b, nds_z* d_x);
/* One process, n_devices GPUs: ndsylv::solve after its Schur step, sharded over the devices
 * (one host thread, context and NCCL communicator per device), host buffers. */
int nds_solve_multi(int n_devices, const int* devices, int n_modes, const int64_t* dims, const nds_z* const* u,
                    const nds_z* const* t, const nds_z* b, nds_z* x, double singular_tol, nds_singular* sing);

/* ---- ODE  dX/dt = sum_j A_j x_j X + B,  X(0) = X0  (reference ode.hpp) ------ */

/* ndsylv::triangular_exp (schur.hpp:24, schur.cpp:203-228): f = exp(t T), T upper triangular
 * n x n column-major (Parlett recurrence; Taylor scaling and squaring when the diagonal is not
 * well separated).
 * Host, like nds_schur. NDS_ERR_INVALID when T has a nonzero strict lower part. */
int nds_triangular_exp(nds_ctx* ctx, int n, const nds_z* t_mat, double t, nds_z* f);

/* ndsylv::OdePropagator (ode.hpp:18-36, ode.cpp:32-57) from the Schur factors A_j = U_j T_j U_j^H:
 * uploads U_j, T_j, then keeps C = forward(B) and G0 = sum_j T_j x_j forward(X0) + C on the
 * device. Like the reference constructor it does not fail on a singular operator; at() does. */
int nds_ode_create(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* u, const nds_z* const* t,
                   const nds_z* forcing, const nds_z* initial, double singular_tol, unsigned flags, nds_ode** out);
void nds_ode_destroy(nds_ode* ode);
/* OdePropagator::at (ode.cpp:59-87): x = X(time), host buffer, synchronous. On the GPU:
 * G = exp(time T_N) x_N ... exp(time T_1) x_1 G0 - C (the exponentials on the host), one
 * triangular solve, the inverse transform. NDS_ERR_INVALID for a non-finite time;
 * NDS_ERR_SINGULAR + sing as nds_solve. rep: stage device times (transform = exp passes). */
int nds_ode_at(nds_ode* ode, double time, nds_z* x, nds_report* rep, nds_singular* sing);
/* The same into a device tensor, asynchronous on the context stream. */
int nds_ode_at_dev(nds_ode* ode, double time, nds_z* d_x);
/* ndsylv::propagate (ode.hpp:39, ode.cpp:89-91): host Schur of each A_j + create + at. */
int nds_propagate(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* a, const nds_z* forcing,
                  const nds_z* initial, double time, double singular_tol, unsigned flags, nds_z* x, nds_report* rep,
                  nds_singular* sing);
/* ndsylv::rk4_reference (ode.hpp:41-44, ode.cpp:93-129) on the device: classical RK4 with step
 * dt, the last step shortened to land on time; each right-hand side is N mode-product GEMMs
 * plus B; the fixed-size steps are replayed as a CUDA graph. NDS_ERR_INVALID when more than
 * max_steps steps would be needed or dt is not positive and finite; NDS_ERR_NONFINITE when the
 * state leaves finite range. x: host buffer. */
int nds_rk4(nds_ctx* ctx, int n_modes, const int64_t* dims, const nds_z* const* a, const nds_z* forcing,
            const nds_z* initial, double time, double dt, int64_t max_steps, nds_z* x);

/* ---- NDT1 tensor files and the seeded generator -------------------------- */

/* Header of an NDT1 file (tensor_file.hpp:9-15): order and extents (dims has room for 64).
 * NDS_ERR_FILE on I/O failure, bad magic, unsupported version, invalid or overflowing extents. */
int nds_tensor_file_info(const char* path, int* n_modes, int64_t* dims);
/* ndsylv::read_tensor (tensor_file.cpp:67-96) into a host buffer of the file's extents (which
 * must equal n_modes / dims); a short or over-long payload is NDS_ERR_FILE. */
int nds_read_tensor(const char* path, int n_modes, const int64_t* dims, nds_z* out);
/* ndsylv::write_tensor (tensor_file.cpp:48-65). */
int nds_write_tensor(const char* path, int n_modes, const int64_t* dims, const nds_z* data);
/* The same between a file and DEVICE memory, streamed through double-buffered pinned chunks so
 * disk reads overlap the host->device copies (and device->host copies overlap disk writes);
 * for multi-GiB tensors. Synchronous. */
int nds_read_tensor_dev(nds_ctx* ctx, const char* path, int n_modes, const int64_t* dims, nds_z* d_out);
int nds_write_tensor_dev(nds_ctx* ctx, const char* path, int n_modes, const int64_t* dims, const nds_z* d_in);
/* ndsylv::random_problem (rng.hpp:67, rng.cpp:18-25): A_1..A_N then X_true from one xoshiro256++
 * stream (uniform [0,1) + i[0,1)), B = sum_j A_j x_j X_true (computed on the GPU). */
int nds_random_problem(nds_ctx* ctx, int n_modes, const int64_t* dims, uint64_t seed, nds_z* const* a,
                       nds_z* x_true, nds_z* b);
/* ndsylv::random_ode_system (rng.hpp:70, rng.cpp:27-33): A_1..A_N, forcing, initial state. Host. */
int nds_random_ode_system(int n_modes, const int64_t* dims, uint64_t seed, nds_z* const* a, nds_z* forcing,
                          nds_z* initial);

/* ---- harness utility ------------------------------------------------------------------ */
/* Seeded standard normals (Box–Muller over splitmix64 counters, stream-separated), host
 * side, OpenMP-parallel and order-independent: out[i] for i in [0, count). */
void nds_randn(uint64_t seed, uint64_t stream, int64_t count, double* out);

#ifdef __cplusplus
}
#endif

#endif /* NDSYLV_B200_H */
