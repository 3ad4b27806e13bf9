// Shared device/host helpers for the ndsylv_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

#include "error.h"
#include "ndsylv_b200.h"

namespace nds {

#define NDS_CUDA(call)                                                                                   \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess)                                                                               \
      throw ::nds::Error(e_ == cudaErrorMemoryAllocation ? NDS_ERR_NOMEM : NDS_ERR_CUDA,                 \
                         std::string(#call) + ": " + cudaGetErrorString(e_));                            \
  } while (0)

#define NDS_LAUNCH_CHECK() NDS_CUDA(cudaGetLastError())

// Dynamic shared-memory opt-in of a kernel before its launch. Function attributes belong to the
// device's context, so the (device, kernel) pairs already raised are remembered — with the
// largest size set — rather than one process-wide flag (several devices in one process:
// nds_solve_multi, one host thread per device in the loopback engine).
inline void smem_optin(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  NDS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = done[{dev, fn}];
  if (cur >= bytes) return;
  NDS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  cur = bytes;
}
template <class K>
inline void smem_optin(K* kern, size_t bytes) {
  smem_optin((const void*)kern, bytes);
}

// Mode-j view of a column-major tensor (reference kernels.cpp:9-21): (inner, n, outer).
struct ModeView {
  int64_t inner, n, outer;
};

inline ModeView mode_view(int n_modes, const int64_t* dims, int mode /*1-based*/) {
  ModeView v{1, dims[mode - 1], 1};
  for (int j = 0; j < mode - 1; ++j) v.inner *= dims[j];
  for (int j = mode; j < n_modes; ++j) v.outer *= dims[j];
  return v;
}

// Geometry of an N-mode tensor passed by value to kernels.
struct Geom {
  int n_modes;
  int64_t total;
  int64_t dims[NDS_MAX_MODES];
  int64_t strides[NDS_MAX_MODES];
  int64_t toff[NDS_MAX_MODES];  // offset of T_j (n_j x n_j, column-major) in the factor pool
  int64_t doff[NDS_MAX_MODES];  // offset of diag(T_j) in the diagonal pool
};

// ---- complex128 arithmetic on double2 --------------------------------------------------
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }
// acc - a*b
__device__ __forceinline__ double2 cfms(double2 acc, double2 a, double2 b) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
// acc + a*b
__device__ __forceinline__ double2 cfma(double2 acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}

// Complex division with the semantics GCC gives std::complex<double>::operator/ in the
// reference (libgcc __divdc3: Smith's method with the Baudin–Smith subnormal-ratio branch and
// range scaling, then C99 Annex G recovery of infinities / zeros).
__device__ __forceinline__ double2 cdiv(double2 num, double2 den) {
  double a = num.x, b = num.y, c = den.x, d = den.y;
  const double RBIG = 8.98846567431157953865e+307;  // DBL_MAX / 2
  const double RMIN = 2.2250738585072014e-308;      // DBL_MIN
  const double RMIN2 = 2.220446049250313e-16;       // DBL_EPSILON
  const double RMINSCAL = 4503599627370496.0;       // 1 / DBL_EPSILON
  const double RMAX2 = RBIG * RMIN2;
  double x, y;
  if (fabs(c) < fabs(d)) {
    if (fabs(d) >= RBIG) { a *= 0.5; b *= 0.5; c *= 0.5; d *= 0.5; }
    if (fabs(d) < RMIN2) {
      a *= RMINSCAL; b *= RMINSCAL; c *= RMINSCAL; d *= RMINSCAL;
    } else if ((fabs(a) < RMIN && fabs(b) < RMAX2 && fabs(d) < RMAX2) ||
               (fabs(b) < RMIN && fabs(a) < RMAX2 && fabs(d) < RMAX2)) {
      a *= RMINSCAL; b *= RMINSCAL; c *= RMINSCAL; d *= RMINSCAL;
    }
    const double ratio = c / d;
    const double denom = __dadd_rn(__dmul_rn(c, ratio), d);
    if (fabs(ratio) > RMIN) {
      x = __dadd_rn(__dmul_rn(a, ratio), b) / denom;
      y = __dsub_rn(__dmul_rn(b, ratio), a) / denom;
    } else {
      x = __dadd_rn(__dmul_rn(c, a / d), b) / denom;
      y = __dsub_rn(__dmul_rn(c, b / d), a) / denom;
    }
  } else {
    if (fabs(c) >= RBIG) { a *= 0.5; b *= 0.5; c *= 0.5; d *= 0.5; }
    if (fabs(c) < RMIN2) {
      a *= RMINSCAL; b *= RMINSCAL; c *= RMINSCAL; d *= RMINSCAL;
    } else if ((fabs(a) < RMIN && fabs(b) < RMAX2 && fabs(c) < RMAX2) ||
               (fabs(b) < RMIN && fabs(a) < RMAX2 && fabs(c) < RMAX2)) {
      a *= RMINSCAL; b *= RMINSCAL; c *= RMINSCAL; d *= RMINSCAL;
    }
    const double ratio = d / c;
    const double denom = __dadd_rn(__dmul_rn(d, ratio), c);
    if (fabs(ratio) > RMIN) {
      x = __dadd_rn(__dmul_rn(b, ratio), a) / denom;
      y = __dsub_rn(b, __dmul_rn(a, ratio)) / denom;
    } else {
      x = __dadd_rn(a, __dmul_rn(d, b / c)) / denom;
      y = __dsub_rn(b, __dmul_rn(d, a / c)) / denom;
    }
  }
  if (isnan(x) && isnan(y)) {  // Annex G recovery
    if (c == 0.0 && d == 0.0 && (!isnan(a) || !isnan(b))) {
      x = copysign(INFINITY, c) * a;
      y = copysign(INFINITY, c) * b;
    } else if ((isinf(a) || isinf(b)) && isfinite(c) && isfinite(d)) {
      a = copysign(isinf(a) ? 1.0 : 0.0, a);
      b = copysign(isinf(b) ? 1.0 : 0.0, b);
      x = INFINITY * (a * c + b * d);
      y = INFINITY * (b * c - a * d);
    } else if ((isinf(c) || isinf(d)) && isfinite(a) && isfinite(b)) {
      c = copysign(isinf(c) ? 1.0 : 0.0, c);
      d = copysign(isinf(d) ? 1.0 : 0.0, d);
      x = 0.0 * (a * c + b * d);
      y = 0.0 * (b * c - a * d);
    }
  }
  return make_double2(x, y);
}

// 1 / d = conj(d) / |d|^2 with an exact power-of-two prescale, so |d|^2 neither overflows
// nor underflows for any finite non-zero d.
__device__ __forceinline__ double2 crecip(double2 d) {
  const double m = fmax(fabs(d.x), fabs(d.y));
  const int e = ((__double2hiint(m) >> 20) & 0x7ff) - 1023;  // exponent field (normal range)
  const double s = __hiloint2double((1023 - e) << 20, 0);   // exactly 2^-e
  const double xr = d.x * s, xi = d.y * s;
  const double inv = 1.0 / (xr * xr + xi * xi);
  return make_double2(xr * inv * s, -xi * inv * s);
}

// 1 / x for a normal positive double: MUFU reciprocal seed + two Newton steps (<= 1 ulp).
__device__ __forceinline__ double drcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// crecip without the IEEE division subroutine (prescaled as crecip, so |d|^2 is normal).
__device__ __forceinline__ double2 crecip_fast(double2 d) {
  const double m = fmax(fabs(d.x), fabs(d.y));
  const int e = ((__double2hiint(m) >> 20) & 0x7ff) - 1023;
  const double s = __hiloint2double((1023 - e) << 20, 0);
  const double xr = d.x * s, xi = d.y * s;
  const double inv = drcp_fast(fma(xr, xr, xi * xi));
  return make_double2(xr * inv * s, -xi * inv * s);
}

inline int ceil_div_i(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace nds
