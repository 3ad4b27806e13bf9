// Latency microbenchmark: dependent chains of DFMA, DADD, LDS.128 (single warp).
#include <cstdio>
__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double2* out, int n, long long* cyc) {
  __shared__ double2 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_double2(i & 1023, 0);
  __syncthreads();
  int idx = threadIdx.x;
  double2 v;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { v = s[idx]; idx = ((int)v.x + 1) & 1023; }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_div(double* out, double a, int n, long long* cyc) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = a / x + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* d; double2* d2; long long* c; long long h;
  cudaMalloc(&d, 4096); cudaMalloc(&d2, 8192); cudaMalloc(&c, 8);
  const int n = 1000;
  k_dfma<<<1, 32>>>(d, 1.0000001, 1e-9, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DFMA latency  %.1f cycles\n", (double)h / n);
  k_lds<<<1, 32>>>(d2, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("LDS.128 chain %.1f cycles (incl. F2I+IADD)\n", (double)h / n);
  k_div<<<1, 32>>>(d, 3.0, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DDIV+DADD     %.1f cycles\n", (double)h / n);
  for (int t : {32, 256, 512}) { k_bar<<<1, t>>>(n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("bar.sync %3d thr %.1f cycles\n", t, (double)h / n); }
  return 0;
}
