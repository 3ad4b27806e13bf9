// Do DFMA streams and 128-bit shared-memory traffic overlap on one SM? Three kernels with the same
// launch shape (2 CTAs x 256 threads per SM, 64 KB dynamic shared memory each, like the fused
// all-binary tile kernel): DFMA only, LDS.128 + STS.128 only, and both from DIFFERENT warps of
// the same CTA (even warps compute, odd warps move data) — if the third takes the sum of the
// first two, the two instruction streams share an issue path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_lds_overlap fp64_lds_overlap.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__device__ __forceinline__ void fma_block(double (&a)[16], double m, double c) {
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], m, c);
}

__device__ __forceinline__ void mem_block(double2* S, int tid, double2 (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = S[(tid + 256 * i) & 4095];
#pragma unroll
  for (int i = 0; i < 16; ++i) S[(tid + 256 * ((i + 5) & 15)) & 4095] = v[i];
}

// mode 0: every warp DFMA; 1: every warp LDS/STS; 2: even warps DFMA, odd warps LDS/STS (each
// doing the full per-warp amount of modes 0 / 1); 3: every warp alternates both (sum of work)
__global__ void __launch_bounds__(256, 2) overlap_kernel(int mode, double* out, double m, double c) {
  extern __shared__ __align__(16) double2 S[];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 4096; i += 256) S[i] = make_double2(i, -i);
  __syncthreads();
  double a[16];
  double2 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = tid + i;
    v[i] = make_double2(0, 0);
  }
  const bool do_f = mode == 0 || mode == 3 || (mode == 2 && !(warp & 1));
  const bool do_m = mode == 1 || mode == 3 || (mode == 2 && (warp & 1));
  for (int it = 0; it < kIters; ++it) {
    if (do_f) {
      fma_block(a, m, c);  // 2 x 128 DFMA per thread
      fma_block(a, m, c);
    }
    if (do_m) mem_block(S, tid, v);      // 16 LDS.128 + 16 STS.128 per thread
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i] + v[i].x + v[i].y;
  if (s == 123.456) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(overlap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"DFMA only (all warps)", "LDS/STS.128 only (all warps)", "even warps DFMA, odd warps LDS/STS",
                         "every warp both, alternating"};
  for (int mode = 0; mode < 4; ++mode) {
    overlap_kernel<<<2 * p.multiProcessorCount, 256, 65536>>>(mode, out, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    overlap_kernel<<<2 * p.multiProcessorCount, 256, 65536>>>(mode, out, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // per SM: 16 warps; DFMA warp-instructions and 16-byte shared accesses per SM per iteration
    printf("%-40s %8.3f ms\n", names[mode], ms);
  }
  printf("(mode 2 runs HALF of mode 0's DFMAs and HALF of mode 1's accesses; perfect overlap = max(m0, m1) / 2,\n"
         " none = (m0 + m1) / 2. mode 3 runs all of both; perfect overlap = max(m0, m1), none = m0 + m1.)\n");
  return 0;
}
