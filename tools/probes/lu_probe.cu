// Probe: standalone timing of the in-CTA LU solves (row-block k_lu_solve<4> vs column-cyclic
// k_lu_cols) for several n (CUDA events, 200 back-to-back launches) and the residual.
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_2102_11026_b200/csrc/solve_kernels.cuh"
using namespace nlrom;
int main() {
  for (int n : {8, 16, 32, 48, 60, 63}) {
    std::vector<double> S(n * n), phi(n);
    std::mt19937 g(1);
    std::uniform_real_distribution<double> U(-1, 1);
    for (auto& x : S) x = U(g);
    for (int i = 0; i < n; ++i) S[i * n + i] += 0.5;
    for (auto& x : phi) x = U(g);
    double *dS, *dphi, *ddr, *dr;
    int* st;
    cudaMalloc(&dS, n * n * 8); cudaMalloc(&dphi, n * 8); cudaMalloc(&ddr, n * 8); cudaMalloc(&dr, n * 8);
    cudaMalloc(&st, 4);
    cudaMemcpy(dS, S.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dphi, phi.data(), n * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_lu_solve<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    auto check = [&](const char* name, float ms) {
      std::vector<double> x(n);
      cudaMemcpy(x.data(), ddr, n * 8, cudaMemcpyDeviceToHost);
      double res = 0;
      for (int i = 0; i < n; ++i) {
        double s = phi[i];
        for (int j = 0; j < n; ++j) s += S[i * n + j] * x[j];
        res = fmax(res, fabs(s));
      }
      printf("n=%2d %-12s %7.2f us/solve  residual %.2e  err=%s\n", n, name, ms * 1000 / 200, res,
             cudaGetErrorString(cudaGetLastError()));
    };
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    for (int w = 0; w < 3; ++w) k_lu_solve<4><<<1, 256, lu_smem_bytes(n)>>>(dS, dphi, ddr, dr, n, 0, st, nullptr, 0, nullptr, nullptr, 0, 0);
    cudaEventRecord(a);
    for (int r = 0; r < 200; ++r) k_lu_solve<4><<<1, 256, lu_smem_bytes(n)>>>(dS, dphi, ddr, dr, n, 0, st, nullptr, 0, nullptr, nullptr, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    check("k_lu_solve", ms);
    for (int w = 0; w < 3; ++w) k_lu_cols<<<1, 256, luc_smem_bytes()>>>(dS, dphi, ddr, dr, n, 0, st, nullptr, 0, nullptr, nullptr, 0, 0);
    cudaEventRecord(a);
    for (int r = 0; r < 200; ++r) k_lu_cols<<<1, 256, luc_smem_bytes()>>>(dS, dphi, ddr, dr, n, 0, st, nullptr, 0, nullptr, nullptr, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    check("k_lu_cols", ms);
  }
#ifdef LU_TRACE
  long long tr[80];
  cudaMemcpyFromSymbol(tr, g_lu_trace, sizeof tr);
  printf("pdl %lld load %lld steps(total) %lld sync %lld backsub %lld\n", tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2],
         tr[4] - tr[3], tr[5] - tr[4]);
  for (int k = 0; k < 62; ++k) printf("%lld ", tr[9 + k] - tr[8 + k]);
  printf("\n");
  long long t2[16];
  cudaMemcpyFromSymbol(t2, g_lu_trace2, sizeof t2);
  printf("k_lu_solve step 10 (thread 0): search+redux %lld | rcp %lld | loads+update %lld | barrier %lld | total %lld\n",
         t2[1] - t2[0], t2[2] - t2[1], t2[3] - t2[2], t2[4] - t2[3], t2[4] - t2[0]);
#endif
}
