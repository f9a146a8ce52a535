// Probe: the split LU (k_lu_front on S_base, k_lu_back with the vhp block) against the one-shot
// k_lu_solve on S_base + diag(0, V) at n = 60, n_p = 30: solution difference and in-kernel
// cycle counts of the phases (LU_CYCLES).
#include <cstdio>
#include <vector>
#include <random>
#include "retired/lu_split.cuh"
using namespace nlrom;
int main() {
  const int n = 60, n_p = 30, nq = 30, FC = n + 1 + nq;
  std::mt19937 g(3);
  std::uniform_real_distribution<double> U(-1, 1);
  std::vector<double> S(n * n), phi(n), Gt(2 * nq * nq);
  for (auto& x : S) x = U(g);
  for (auto& x : phi) x = U(g);
  for (auto& x : Gt) x = 0.3 * U(g);
  double *dS, *dphi, *dGt, *dF, *drd, *ddr, *dr, *ddr2;
  int *dpiv, *dflag, *dst;
  cudaMalloc(&dS, n * n * 8); cudaMalloc(&dphi, n * 8); cudaMalloc(&dGt, Gt.size() * 8); cudaMalloc(&dF, n * FC * 8);
  cudaMalloc(&drd, n * 8); cudaMalloc(&ddr, n * 8); cudaMalloc(&dr, n * 8); cudaMalloc(&ddr2, n * 8);
  cudaMalloc(&dpiv, n * 4); cudaMalloc(&dflag, 4); cudaMalloc(&dst, 4);
  cudaMemcpy(dS, S.data(), n * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dphi, phi.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dGt, Gt.data(), Gt.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_lu_solve<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_lu_front<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_lu_back<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  LuSplitArgs a{n, n_p, 0, FC, dS, dphi, nullptr, dF, dpiv, drd, dflag, dGt, nq, ddr, dr, 0, dst, nullptr};
  for (int rep = 0; rep < 3; ++rep) {
    k_lu_solve<4><<<1, 256, lu_smem_bytes(n, nq)>>>(dS, dphi, ddr2, dr, n, 0, dst, nullptr, 0, nullptr, dGt, nq, n_p);
    k_lu_front<6><<<1, 256, LuSplitPlan<6>::bytes(0)>>>(a);
    k_lu_back<2><<<1, 256, LuSplitPlan<2>::bytes(nq)>>>(a);
  }
  cudaDeviceSynchronize();
  std::vector<double> x(n), x2(n);
  cudaMemcpy(x.data(), ddr, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(x2.data(), ddr2, n * 8, cudaMemcpyDeviceToHost);
  double e = 0, m = 0;
  for (int i = 0; i < n; ++i) { e = fmax(e, fabs(x[i] - x2[i])); m = fmax(m, fabs(x2[i])); }
  long long c[8];
  cudaMemcpyFromSymbol(c, g_lus_cycles, sizeof c);
  printf("split vs one-shot: max |dx| / max |x| = %.2e   err=%s\n", e / m, cudaGetErrorString(cudaGetLastError()));
  printf("front steps %lld cycles (%.0f/step); back staging+ZV %lld, steps %lld (%.0f/step), solve %lld\n", c[1] - c[0],
         (double)(c[1] - c[0]) / n_p, c[3] - c[2], c[4] - c[3], (double)(c[4] - c[3]) / nq, c[5] - c[4]);
  return 0;
}
