// FP64 pipe microbenchmarks for B200 (sm_100a): DFMA vs DMMA (mma.sync f64) throughput.
// Used to pick the inner product engine of the transform kernels and to measure the
// FP64 roofline denominator (MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = c; c1[c] = c + 0.5; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d}\n", p.name, sms, clk);
  double* d; CK(cudaMalloc(&d, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  // DFMA: blocks x threads x iters x chains FMAs, 2 flops each.
  for (int bpsm : {2, 4, 8}) {
    int threads = 256, iters = 20000;
    int blocks = sms * bpsm;
    dfma_kernel<8><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * blocks * threads * (double)iters * 8;
    printf("{\"kernel\": \"dfma\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", bpsm, best, flops / best / 1e9);
  }
  // Sustained DFMA for ~3 s (clock under power cap)
  {
    int threads = 256, iters = 200000, blocks = sms * 4;
    cudaEventRecord(e0);
    int reps = 0;
    for (; reps < 12; ++reps) dfma_kernel<8><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * (double)iters * 8 * reps;
    printf("{\"kernel\": \"dfma_sustained\", \"ms\": %.1f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
  }
  // DMMA m8n8k4: 8*8*4 FMAs per warp-instruction.
  for (int bpsm : {2, 4, 8}) {
    int threads = 256, iters = 4000;
    int blocks = sms * bpsm;
    dmma_kernel<8><<<blocks, threads>>>(d, 10);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      dmma_kernel<8><<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256.0 * (blocks * threads / 32) * (double)iters * 8;
    printf("{\"kernel\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", bpsm, best, flops / best / 1e9);
  }
  {
    int threads = 256, iters = 40000, blocks = sms * 4;
    cudaEventRecord(e0);
    int reps = 0;
    for (; reps < 12; ++reps) dmma_kernel<8><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256.0 * (blocks * threads / 32) * (double)iters * 8 * reps;
    printf("{\"kernel\": \"dmma_sustained\", \"ms\": %.1f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
  }
  // HBM copy
  {
    size_t n = (size_t)1 << 28;  // 4 GiB per buffer of double2
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    cudaMemset(a, 0, n * 16);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      copy_kernel<<<sms * 8, 512>>>(a, b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"kernel\": \"copy_double2\", \"ms\": %.3f, \"gbs\": %.1f}\n", best, 2.0 * n * 16 / best / 1e6);
  }
  return 0;
}
