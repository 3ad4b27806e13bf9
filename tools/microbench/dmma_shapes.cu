// FP64 tensor-core (mma.sync .f64) throughput per instruction shape on B200 (sm_100a):
// m8n8k4 (the shape the transform / update kernels use) vs the sm_90+ shapes m16n8k4,
// m16n8k8, m16n8k16. Reports TFLOP/s (2 flops per MAC) for several independent accumulator
// chains per warp and warps per SM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/dmma_shapes.cu -o tools/microbench/dmma_shapes
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void m16n8k8(double* out, int iters) {
  double a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  b[0] = 1.0 + threadIdx.x * 1e-4;
  b[1] = b[0] + 1;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

template <int CH>
__global__ void m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + threadIdx.x * 1e-4 + i;
  double c[CH][4];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5) out[0] = s;
}

template <class K>
static void run(const char* name, K k, double macs_per_inst, int ch, int sms) {
  double* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wps : {4, 8, 16}) {
    const int threads = 32 * wps / 2, blocks = sms * 2, iters = 4000;
    k<<<blocks, threads>>>(d, 10);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * macs_per_inst * ch * iters * (double)blocks * (threads / 32);
    printf("%-9s chains %d warps/SM %2d : %7.2f TFLOP/s  (%s)\n", name, ch, wps, flops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(d);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  run("m8n8k4", m8n8k4<8>, 8 * 8 * 4, 8, sms);
  run("m16n8k4", m16n8k4<8>, 16 * 8 * 4, 8, sms);
  run("m16n8k8", m16n8k8<8>, 16 * 8 * 8, 8, sms);
  run("m16n8k16", m16n8k16<4>, 16 * 8 * 16, 4, sms);
  run("m16n8k16", m16n8k16<8>, 16 * 8 * 16, 8, sms);
  return 0;
}
