// Microbenchmark of the v2 diagonal-tile kernel: 148 CTAs each solving one 16^3 tile (N=3)
// with the library's own wavefront tables; reports time per launch for several wavefront depths.
#include <cstdio>
#include <vector>
#define NDS_DIAG_CLOCK
__device__ long long nds_diag_clock[128];
__device__ long long nds_diag_clock_start;
__device__ long long nds_diag_probe[512];
#include "../../paper_2412_15840_b200/csrc/backsub.cu"

using namespace nds;

int main() {
  const int64_t dims[3] = {16, 16, 16};
  const int64_t toff[3] = {0, 256, 512};
  SolvePlan sp;
  solve_plan_build(sp, 3, dims, toff);
  printf("levels %d wf_levels %d v2 %d\n", sp.levels, sp.wf_levels, (int)sp.v2);
  std::vector<double2> T(768), Y(4096);
  for (int j = 0; j < 3; ++j)
    for (int c = 0; c < 16; ++c)
      for (int r = 0; r < 16; ++r)
        T[j * 256 + r + c * 16] = r > c ? make_double2(0, 0) : r == c ? make_double2(2.0 + 0.1 * r, 0.3) : make_double2(0.01 * (r + c), -0.02);
  for (int i = 0; i < 4096; ++i) Y[i] = make_double2(1.0 + 0.001 * i, 0.5);
  double2 *dT, *dY;
  int64_t* dtiles;
  int2* ditems;
  const int G = 148 * 2;
  cudaMalloc(&dT, 768 * 16);
  cudaMalloc(&dY, 4096 * 16);
  cudaMalloc(&dtiles, G * 8);
  cudaMalloc(&ditems, G * 16);
  cudaMemset(dtiles, 0, G * 8);
  cudaMemset(ditems, 0, G * 16);
  cudaMemcpy(dT, T.data(), 768 * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), 4096 * 16, cudaMemcpyHostToDevice);
  auto k = diag_kernel_for(3, 16);
  const int kDiagThreads = diag_threads_for(3);
  const size_t smem = diag_smem_bytes(3, 16, sp.wf_levels);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int grid : {1, 148}) {
    for (int L : {0, 1, 5, 10, 20, 30, 46}) {
      for (int w = 0; w < 3; ++w)
        k<<<grid, kDiagThreads, smem>>>(sp.geom, dT, dtiles, (const int4*)ditems, nullptr, nullptr, sp.d_thr, sp.d_lvl, L, dY);
      cudaEventRecord(e0);
      const int reps = 20;
      for (int r = 0; r < reps; ++r)
        k<<<grid, kDiagThreads, smem>>>(sp.geom, dT, dtiles, (const int4*)ditems, nullptr, nullptr, sp.d_thr, sp.d_lvl, L, dY);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("grid %3d levels %2d : %8.2f us/launch  err=%s\n", grid, L, ms * 1000 / reps, cudaGetErrorString(cudaGetLastError()));
    }
  }
  {
    auto kl = lines_kernel_for(3, 16, false);
    const size_t lsmem = lines_smem_bytes(3, 16);
    cudaFuncSetAttribute(kl, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
    for (int grid : {1, 148, 296}) {
      for (int w = 0; w < 3; ++w)
        kl<<<grid, kDiagThreads, lsmem>>>(sp.geom, dT, dtiles, (const int4*)ditems, nullptr, nullptr, nullptr, nullptr, dY);
      cudaEventRecord(e0);
      const int reps = 20;
      for (int r = 0; r < reps; ++r)
        kl<<<grid, kDiagThreads, lsmem>>>(sp.geom, dT, dtiles, (const int4*)ditems, nullptr, nullptr, nullptr, nullptr, dY);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("lines grid %3d : %8.2f us/launch  err=%s\n", grid, ms * 1000 / reps, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // per-level cycles of CTA 0 for a full single-tile run
  k<<<1, kDiagThreads, smem>>>(sp.geom, dT, dtiles, (const int4*)ditems, nullptr, nullptr, sp.d_thr, sp.d_lvl, sp.wf_levels, dY);
  cudaDeviceSynchronize();
  long long clk[128], c0;
  cudaMemcpyFromSymbol(clk, nds_diag_clock, sizeof(clk));
  cudaMemcpyFromSymbol(&c0, nds_diag_clock_start, sizeof(c0));
  std::vector<int> off(sp.wf_levels + 1), grp(sp.wf_levels);
  cudaMemcpy(off.data(), sp.d_wf_off, off.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(grp.data(), sp.d_wf_group, grp.size() * 4, cudaMemcpyDeviceToHost);
  long long probe[512];
  cudaMemcpyFromSymbol(probe, nds_diag_probe, sizeof(probe));
  long long prev = c0;
  for (int lv = 0; lv < sp.wf_levels; ++lv) {
    printf("lv %2d cnt %3d grp %2d cycles %6lld  [thr %lld rden %lld dot %lld upd %lld bar %lld]\n", lv, off[lv + 1] - off[lv], grp[lv], clk[lv] - prev,
           probe[lv*4] - prev, probe[lv*4+1] - probe[lv*4], probe[lv*4+2] - probe[lv*4+1], probe[lv*4+3] - probe[lv*4+2], clk[lv] - probe[lv*4+3]);
    prev = clk[lv];
  }
  return 0;
}
