// Entry-wise kernels of the solve path.
//   den_scan      — singular check + min |den| (sylvester.cpp:101-103, :119-141): den(i) =
//                   sum_j T_j(i_j, i_j) accumulated j = 1..N from 0, |den| = hypot.
//   fast_divide   — normal-coefficient route, c /= den (sylvester.cpp:190-204).
//   real_part     — SolveOptions::real_output (sylvester.cpp:223-224).
//   residual_norms — verification of sum_j A_j x_j X = B on the device (apply_operator,
//                   sylvester.cpp:44-53, is the mode-product kernel with accumulate).

#include "common.cuh"
#include "kernels.h"

namespace nds {


constexpr int kEwThreads = 256;

__device__ __forceinline__ double2 den_at(const Geom& g, const double2* __restrict__ diag, int64_t idx) {
  double2 den = make_double2(0.0, 0.0);
  for (int j = 0; j < g.n_modes; ++j) {
    const int64_t ij = idx % g.dims[j];
    idx /= g.dims[j];
    den = cadd(den, __ldg(diag + g.doff[j] + ij));
  }
  return den;
}

// Eigenvalue sums without per-entry integer division: the leading modes A (product sizeA <= 1024)
// get a shared table dA[a] = sum_{j in A} T_j(i_j, i_j); each row (one index b of the remaining
// modes) adds dB(b) = sum_{j not in A} T_j(i_j, i_j), decoded once per row. den = dA + dB (the
// reference sums j = 1..N left to right; the grouping only changes the last bit).
struct DenSplit {
  int nA;         // leading modes in A
  int sizeA;      // prod of their extents
  int64_t rows;   // total / sizeA
};

static DenSplit den_split(const Geom& g) {
  DenSplit s{0, 1, 0};
  while (s.nA < g.n_modes && s.sizeA * g.dims[s.nA] <= 1024) s.sizeA *= (int)g.dims[s.nA++];
  s.rows = g.total / s.sizeA;
  return s;
}

__device__ __forceinline__ void den_tables(const Geom& g, const DenSplit& s, const double2* __restrict__ diag,
                                           double2* dA) {
  for (int a = threadIdx.x; a < s.sizeA; a += blockDim.x) {
    int rem = a;
    double2 d = make_double2(0.0, 0.0);
    for (int j = 0; j < s.nA; ++j) {
      d = cadd(d, __ldg(diag + g.doff[j] + rem % g.dims[j]));
      rem /= (int)g.dims[j];
    }
    dA[a] = d;
  }
}

__device__ __forceinline__ double2 den_row(const Geom& g, const DenSplit& s, const double2* __restrict__ diag,
                                           int64_t row) {
  double2 d = make_double2(0.0, 0.0);
  for (int j = s.nA; j < g.n_modes; ++j) {
    d = cadd(d, __ldg(diag + g.doff[j] + row % g.dims[j]));
    row /= g.dims[j];
  }
  return d;
}

__global__ void den_scan_kernel(const Geom g, const DenSplit s, const double2* __restrict__ diag, double tol,
                                unsigned long long* __restrict__ min_bits, long long* __restrict__ max_bad) {
  __shared__ double2 dA[1024];
  __shared__ double2 dB;
  den_tables(g, s, diag, dA);
  double local_min = INFINITY;
  long long local_bad = -1;
  for (int64_t row = blockIdx.x; row < s.rows; row += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) dB = den_row(g, s, diag, row);
    __syncthreads();
    const double2 db = dB;
    for (int a = threadIdx.x; a < s.sizeA; a += blockDim.x) {
      const double2 den = cadd(dA[a], db);
      const double v = hypot(den.x, den.y);
      local_min = fmin(local_min, v);
      if (v <= tol) local_bad = max(local_bad, (long long)(row * s.sizeA + a));  // sylvester.cpp:103
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    local_min = fmin(local_min, __shfl_xor_sync(0xffffffffu, local_min, o));
    local_bad = max(local_bad, __shfl_xor_sync(0xffffffffu, local_bad, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(min_bits, (unsigned long long)__double_as_longlong(local_min));  // non-negative: int order
    if (local_bad >= 0) atomicMax(max_bad, local_bad);
  }
}

void den_scan(const Geom& g, const double2* diag, double tol, double* min_abs, int64_t* max_bad, cudaStream_t stream,
              void* scratch) {
  unsigned long long* d_min = (unsigned long long*)scratch;
  long long* d_bad = (long long*)((char*)scratch + 8);
  const unsigned long long init_min = (unsigned long long)0x7ff0000000000000ull;  // +inf
  const long long init_bad = -1;
  NDS_CUDA(cudaMemcpyAsync(d_min, &init_min, 8, cudaMemcpyHostToDevice, stream));
  NDS_CUDA(cudaMemcpyAsync(d_bad, &init_bad, 8, cudaMemcpyHostToDevice, stream));
  const DenSplit s = den_split(g);
  const int64_t blocks = std::min<int64_t>(s.rows, 148 * 16);
  den_scan_kernel<<<(unsigned)blocks, kEwThreads, 0, stream>>>(g, s, diag, tol, d_min, d_bad);
  NDS_LAUNCH_CHECK();
  unsigned long long h_min;
  long long h_bad;
  NDS_CUDA(cudaMemcpyAsync(&h_min, d_min, 8, cudaMemcpyDeviceToHost, stream));
  NDS_CUDA(cudaMemcpyAsync(&h_bad, d_bad, 8, cudaMemcpyDeviceToHost, stream));
  NDS_CUDA(cudaStreamSynchronize(stream));
  long long bits = (long long)h_min;
  double m;
  memcpy(&m, &bits, 8);
  *min_abs = m;
  *max_bad = h_bad;
}

__global__ void fast_divide_kernel(const Geom g, const DenSplit s, const double2* __restrict__ diag,
                                   double2* __restrict__ c) {
  __shared__ double2 dA[1024];
  __shared__ double2 dB;
  den_tables(g, s, diag, dA);
  for (int64_t row = blockIdx.x; row < s.rows; row += gridDim.x) {
    __syncthreads();
    if (threadIdx.x == 0) dB = den_row(g, s, diag, row);
    __syncthreads();
    const double2 db = dB;
    double2* cr = c + row * s.sizeA;
    for (int a = threadIdx.x; a < s.sizeA; a += blockDim.x) cr[a] = cdiv(cr[a], cadd(dA[a], db));
  }
}

int fast_divide_launch(const Geom& g, const double2* diag, double2* c, cudaStream_t stream) {
  const DenSplit s = den_split(g);
  const int64_t blocks = std::min<int64_t>(s.rows, 148 * 16);
  fast_divide_kernel<<<(unsigned)blocks, kEwThreads, 0, stream>>>(g, s, diag, c);
  NDS_LAUNCH_CHECK();
  return 1;
}

struct LayoutArgs {
  int n_modes;
  int n[NDS_MAX_MODES];
  int64_t raw_off[NDS_MAX_MODES];
  double2* ur[NDS_MAX_MODES];
  double2* uc[NDS_MAX_MODES];
  double2* hr[NDS_MAX_MODES];
  double2* hc[NDS_MAX_MODES];
};

__global__ void factor_layouts_kernel(const LayoutArgs a, const double2* __restrict__ raw) {
  const int j = blockIdx.y;
  const int n = a.n[j];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e % n, k = e / n;
    const double2 z = raw[a.raw_off[j] + e];  // U(i, k)
    a.uc[j][i + k * n] = z;
    a.ur[j][i * n + k] = z;
    a.hc[j][k + i * n] = conj2(z);  // U^H(k, i) = conj(U(i, k))
    a.hr[j][k * n + i] = conj2(z);
  }
}

void factor_layouts_launch(const FactorSet& f, const double2* raw, cudaStream_t stream) {
  LayoutArgs a{};
  a.n_modes = f.n_modes;
  int64_t off = 0, maxsq = 1;
  for (int j = 0; j < f.n_modes; ++j) {
    a.n[j] = (int)f.dims[j];
    a.raw_off[j] = off;
    off += f.dims[j] * f.dims[j];
    maxsq = std::max<int64_t>(maxsq, f.dims[j] * f.dims[j]);
    a.ur[j] = f.u_row[j];
    a.uc[j] = f.u_col[j];
    a.hr[j] = f.uh_row[j];
    a.hc[j] = f.uh_col[j];
  }
  const dim3 grid((unsigned)std::min<int64_t>((maxsq + 255) / 256, 1024), (unsigned)f.n_modes);
  factor_layouts_kernel<<<grid, 256, 0, stream>>>(a, raw);
  NDS_LAUNCH_CHECK();
}

__global__ void real_part_kernel(double2* __restrict__ x, int64_t total) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x)
    x[idx].y = 0.0;
}

int real_part_launch(double2* x, int64_t total, cudaStream_t stream) {
  const int64_t blocks = std::min<int64_t>((total + kEwThreads - 1) / kEwThreads, 148 * 32);
  real_part_kernel<<<(unsigned)blocks, kEwThreads, 0, stream>>>(x, total);
  NDS_LAUNCH_CHECK();
  return 1;
}

constexpr int kResBlocks = 148 * 8;

// ---- ODE helpers (reference kernels.cpp:81-88 add_scaled, ode.cpp:98-124 RK4 stages) -------
// Complex scalars multiply as (a.x b.x - a.y b.y, a.x b.y + a.y b.x), the finite-value branch of
// the libgcc product the reference's std::complex uses.
__global__ void axpy_kernel(double2* __restrict__ z, const double2* __restrict__ x, double2 alpha,
                            const double2* __restrict__ y, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = cadd(x[i], cmul(alpha, y[i]));
}

int axpy_launch(double2* z, const double2* x, double2 alpha, const double2* y, int64_t total, cudaStream_t stream) {
  const int64_t blocks = std::min<int64_t>((total + kEwThreads - 1) / kEwThreads, 148 * 32);
  axpy_kernel<<<(unsigned)blocks, kEwThreads, 0, stream>>>(z, x, alpha, y, total);
  NDS_LAUNCH_CHECK();
  return 1;
}

// x += a1 k1; x += a2 k2; x += a2 k3; x += a1 k4 — the reference's four add_scaled calls fused,
// same per-entry operation order (ode.cpp:118-121).
__global__ void rk4_combine_kernel(double2* __restrict__ x, double2 a1, double2 a2, const double2* __restrict__ k1,
                                   const double2* __restrict__ k2, const double2* __restrict__ k3,
                                   const double2* __restrict__ k4, int64_t total) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v = x[i];
    v = cadd(v, cmul(a1, k1[i]));
    v = cadd(v, cmul(a2, k2[i]));
    v = cadd(v, cmul(a2, k3[i]));
    v = cadd(v, cmul(a1, k4[i]));
    x[i] = v;
  }
}

int rk4_combine_launch(double2* x, double2 a1, double2 a2, const double2* k1, const double2* k2, const double2* k3,
                       const double2* k4, int64_t total, cudaStream_t stream) {
  const int64_t blocks = std::min<int64_t>((total + kEwThreads - 1) / kEwThreads, 148 * 32);
  rk4_combine_kernel<<<(unsigned)blocks, kEwThreads, 0, stream>>>(x, a1, a2, k1, k2, k3, k4, total);
  NDS_LAUNCH_CHECK();
  return 1;
}

// *flag |= 1 if any entry is Inf or NaN (NDTensor::all_finite).
__global__ void nonfinite_kernel(const double2* __restrict__ x, int64_t total, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = x[i];
    bad |= !isfinite(v.x) || !isfinite(v.y);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

int nonfinite_launch(const double2* x, int64_t total, int* flag, cudaStream_t stream) {
  const int64_t blocks = std::min<int64_t>((total + kEwThreads - 1) / kEwThreads, 148 * 8);
  nonfinite_kernel<<<(unsigned)blocks, kEwThreads, 0, stream>>>(x, total, flag);
  NDS_LAUNCH_CHECK();
  return 1;
}

// Fused RK4 stage for small tensors (launch-bound regime): one kernel computes the right-hand
// side  K = sum_j A_j x_j IN + B  entry by entry (direct sums along each mode, A_j rows read
// contiguously from the row-major copies) and applies the stage update in its epilogue:
//   stage 0..2: ST_out = X + c K          stage 3: X += a1 K1 + a2 K2 + a2 K3 + a1 K
// (reference ode.cpp:101-123 order per entry). Four launches per step instead of 4 (N + 2).
// Four lanes per entry (each takes every fourth k of every mode; shuffles combine them): for the
// small tensors this path serves, latency chains are what cost, not arithmetic.
constexpr int kRk4Lanes = 4;

__device__ __forceinline__ void rk4_stage_body(const Rk4Stage& a) {
  const int q = threadIdx.x & (kRk4Lanes - 1);
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x / kRk4Lanes;
  const int64_t lane_off = (threadIdx.x & 31) / kRk4Lanes;  // entry offset of this lane within its warp
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kRk4Lanes; base - lane_off < a.total;
       base += gstride) {  // trip count uniform across the warp (shuffles below use the full mask)
    const int64_t e = base;
    const bool active = e < a.total;
    double2 acc = make_double2(0.0, 0.0);
    if (active) {
      int64_t r = e;
      for (int m = 0; m < a.n_modes; ++m) {
        const int64_t n = a.dims[m];
        const int64_t im = r % n;
        r /= n;
        const double2* line = a.in + e - im * a.strides[m];
        // A_1 read column-wise (adjacent entries differ in i_1), the others row-wise (broadcast)
        const double2* ap = m == 0 ? a.a_row[m] + n * n + im : a.a_row[m] + im * n;
        const int64_t astep = m == 0 ? n : 1, xs = a.strides[m];
        double2 t0 = make_double2(0.0, 0.0), t1 = t0;
        int64_t k = q;
        for (; k + kRk4Lanes < n; k += 2 * kRk4Lanes) {
          t0 = cfma(t0, __ldg(ap + k * astep), line[k * xs]);
          t1 = cfma(t1, __ldg(ap + (k + kRk4Lanes) * astep), line[(k + kRk4Lanes) * xs]);
        }
        if (k < n) t0 = cfma(t0, __ldg(ap + k * astep), line[k * xs]);
        acc = cadd(acc, cadd(t0, t1));
      }
    }
#pragma unroll
    for (int o = 1; o < kRk4Lanes; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (!active || q != 0) continue;
    acc = cadd(acc, a.b[e]);
    a.k_out[e] = acc;
    if (a.final_stage) {
      double2 v = a.x[e];
      v = cadd(v, cmul(a.a1, a.k1[e]));
      v = cadd(v, cmul(a.a2, a.k2[e]));
      v = cadd(v, cmul(a.a2, a.k3[e]));
      v = cadd(v, cmul(a.a1, acc));
      a.x[e] = v;
    } else {
      a.st_out[e] = cadd(a.x[e], cmul(a.c, acc));
    }
  }
}

__global__ void rk4_stage_kernel(const Rk4Stage a) { rk4_stage_body(a); }

// All steps in ONE cooperative launch: the four stages of a step are separated by grid-wide
// barriers (each stage reads the whole previous stage buffer), so a step costs four grid syncs
// instead of four kernel launches. Stage buffers rotate exactly as in the four-launch form.
// Sense-free grid barrier: every CTA adds one to the counter and waits for the next multiple of
// gridDim.x. Co-residency of all CTAs is what the cooperative launch guarantees.
__device__ __forceinline__ void rk4_grid_barrier(unsigned int* bar, unsigned int& target) {
  __syncthreads();
  target += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

__global__ void rk4_persistent_kernel(const Rk4Stage base, const Rk4Buffers buf, int64_t steps, double h,
                                      double h_last) {
  unsigned int target = 0;
  for (int64_t st = 0; st < steps + (h_last != 0.0 ? 1 : 0); ++st) {
    const double hh = st < steps ? h : h_last;
    Rk4Stage r = base;
    r.in = buf.x, r.k_out = buf.k[0], r.st_out = buf.st[0], r.c = make_double2(0.5 * hh, 0.0), r.final_stage = 0;
    rk4_stage_body(r);
    rk4_grid_barrier(buf.bar, target);
    r.in = buf.st[0], r.k_out = buf.k[1], r.st_out = buf.st[1];
    rk4_stage_body(r);
    rk4_grid_barrier(buf.bar, target);
    r.in = buf.st[1], r.k_out = buf.k[2], r.st_out = buf.st[0], r.c = make_double2(hh, 0.0);
    rk4_stage_body(r);
    rk4_grid_barrier(buf.bar, target);
    r.in = buf.st[0], r.k_out = buf.k[3], r.final_stage = 1, r.k1 = buf.k[0], r.k2 = buf.k[1], r.k3 = buf.k[2];
    r.a1 = make_double2(hh / 6.0, 0.0), r.a2 = make_double2(hh / 3.0, 0.0);
    rk4_stage_body(r);
    rk4_grid_barrier(buf.bar, target);
  }
}

int rk4_persistent_launch(const Rk4Stage& base, const Rk4Buffers& buf, int64_t steps, double h, double h_last,
                          cudaStream_t stream) {
  int per_sm = 0, sms = 0, dev = 0;
  NDS_CUDA(cudaGetDevice(&dev));
  NDS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  NDS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rk4_persistent_kernel, kEwThreads, 0));
  const int64_t want = (base.total * kRk4Lanes + kEwThreads - 1) / kEwThreads;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per_sm * sms));
  Rk4Stage b0 = base;
  Rk4Buffers b1 = buf;
  void* args[] = {&b0, &b1, &steps, &h, &h_last};
  NDS_CUDA(cudaLaunchCooperativeKernel((const void*)rk4_persistent_kernel, blocks, kEwThreads, args, 0, stream));
  return 1;
}

int rk4_stage_launch(const Rk4Stage& a, cudaStream_t stream) {
  const int64_t blocks = std::min<int64_t>((a.total * kRk4Lanes + kEwThreads - 1) / kEwThreads, 148 * 16);
  rk4_stage_kernel<<<(unsigned)blocks, kEwThreads, 0, stream>>>(a);
  NDS_LAUNCH_CHECK();
  return 1;
}

__global__ void residual_kernel(const double2* __restrict__ r, const double2* __restrict__ b, int64_t total,
                                double* __restrict__ part) {
  double rmax = 0.0, r2 = 0.0, bmax = 0.0, b2 = 0.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const double2 bv = b[idx];
    const double2 d = csub(r[idx], bv);
    const double ad = hypot(d.x, d.y), ab = hypot(bv.x, bv.y);
    rmax = fmax(rmax, ad);
    bmax = fmax(bmax, ab);
    r2 += ad * ad;
    b2 += ab * ab;
  }
  __shared__ double sh[4][kEwThreads];
  sh[0][threadIdx.x] = rmax;
  sh[1][threadIdx.x] = r2;
  sh[2][threadIdx.x] = bmax;
  sh[3][threadIdx.x] = b2;
  __syncthreads();
  for (int s = kEwThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sh[0][threadIdx.x] = fmax(sh[0][threadIdx.x], sh[0][threadIdx.x + s]);
      sh[1][threadIdx.x] += sh[1][threadIdx.x + s];
      sh[2][threadIdx.x] = fmax(sh[2][threadIdx.x], sh[2][threadIdx.x + s]);
      sh[3][threadIdx.x] += sh[3][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = sh[threadIdx.x][0];
}

void residual_norms(const double2* r, const double2* b, int64_t total, double* res_max, double* res_2, double* b_max,
                    double* b_2, cudaStream_t stream) {
  double* d_part;
  NDS_CUDA(cudaMallocAsync(&d_part, kResBlocks * 4 * sizeof(double), stream));
  residual_kernel<<<kResBlocks, kEwThreads, 0, stream>>>(r, b, total, d_part);
  NDS_LAUNCH_CHECK();
  std::vector<double> part(kResBlocks * 4);
  NDS_CUDA(cudaMemcpyAsync(part.data(), d_part, part.size() * sizeof(double), cudaMemcpyDeviceToHost, stream));
  NDS_CUDA(cudaFreeAsync(d_part, stream));
  NDS_CUDA(cudaStreamSynchronize(stream));
  double rm = 0, rs = 0, bm = 0, bs = 0;
  for (int i = 0; i < kResBlocks; ++i) {
    rm = std::max(rm, part[i * 4 + 0]);
    rs += part[i * 4 + 1];
    bm = std::max(bm, part[i * 4 + 2]);
    bs += part[i * 4 + 3];
  }
  *res_max = rm;
  *res_2 = std::sqrt(rs);
  *b_max = bm;
  *b_2 = std::sqrt(bs);
}

}  // namespace nds
