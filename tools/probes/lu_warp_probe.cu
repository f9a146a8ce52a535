// Probe: standalone timing of the warp-register LU (k_lu_warp) against the row-block
// k_lu_solve for several n (CUDA events, 200 back-to-back launches), bitwise comparison of
// the solutions, plus a residual check. Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 --expt-relaxed-constexpr tools/probes/lu_warp_probe.cu -o tools/probes/lu_warp_probe
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>
#include <random>
#include "retired/lu_warp.cuh"
using namespace nlrom;

template <class K>
float time_it(K kern, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) kern();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) kern();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : 0;
  cudaFuncSetAttribute(k_lu_solve<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_lu_warp<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_lu_warp<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_lu_warp<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int n : {5, 15, 30, 31, 32, 45, 60, 63}) {
    if (only && n != only) continue;
    std::vector<double> S(n * n), phi(n);
    std::mt19937 g(n);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto& x : S) x = U(g);
    for (auto& x : phi) x = U(g);
    double *dS, *dphi, *ddr, *dr;
    int* st;
    cudaMalloc(&dS, n * n * 8); cudaMalloc(&dphi, n * 8); cudaMalloc(&ddr, n * 8); cudaMalloc(&dr, n * 8);
    cudaMalloc(&st, 4);
    cudaMemcpy(dS, S.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dphi, phi.data(), n * 8, cudaMemcpyHostToDevice);
    std::vector<double> x_ref(n), x(n);
    const float t_ref = time_it([&] {
      k_lu_solve<4><<<1, 256, lu_smem_bytes(n)>>>(dS, dphi, ddr, dr, n, 0, st, nullptr, 0, nullptr, nullptr, 0, 0);
    }, 200);
    cudaMemcpy(x_ref.data(), ddr, n * 8, cudaMemcpyDeviceToHost);
#ifdef LU_CYCLES
    long long cyc[2];
    cudaMemcpyFromSymbol(cyc, g_lu_cycles, sizeof cyc);
    printf("n=%2d  k_lu_solve pivot loop %lld cycles (%.0f per step)\n", n, cyc[1] - cyc[0], (double)(cyc[1] - cyc[0]) / n);
#endif
    cudaMemset(ddr, 0, n * 8);
    const int nw = luw_warps(n, 0);
    const size_t sm = luw_smem_bytes(nw, 0);
    const float t_w = time_it([&] {
      if (nw == 1) k_lu_warp<1><<<1, 256, sm>>>(dS, dphi, ddr, dr, n, 0, st, nullptr, 0, nullptr, nullptr, 0, 0);
      else if (nw == 2) k_lu_warp<2><<<1, 256, sm>>>(dS, dphi, ddr, dr, n, 0, st, nullptr, 0, nullptr, nullptr, 0, 0);
      else k_lu_warp<3><<<1, 256, sm>>>(dS, dphi, ddr, dr, n, 0, st, nullptr, 0, nullptr, nullptr, 0, 0);
    }, 200);
    cudaMemcpy(x.data(), ddr, n * 8, cudaMemcpyDeviceToHost);
    int stat = -1;
    cudaMemcpy(&stat, st, 4, cudaMemcpyDeviceToHost);
    double res = 0;
    for (int i = 0; i < n; ++i) {
      double s = phi[i];
      for (int j = 0; j < n; ++j) s += S[i * n + j] * x[j];
      res = fmax(res, fabs(s));
    }
    printf("n=%2d  k_lu_solve %6.2f us  k_lu_warp<%d> %6.2f us  bitwise %s  residual %.1e  status %d  err=%s\n", n,
           t_ref, nw, t_w, memcmp(x.data(), x_ref.data(), n * 8) == 0 ? "equal" : "DIFFER", res, stat,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
