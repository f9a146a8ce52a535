// Probe: standalone timing of the in-CTA LU solve for several n (CUDA events, 200 reps).
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
    for (int i = 0; i < n; ++i) S[i * n + i] += n;
    for (auto& x : phi) x = U(g);
    double *dS, *dphi, *ddr, *dr;
    int* st;
    cudaMalloc(&dS, n * n * 8); cudaMalloc(&dphi, n * 8); cudaMalloc(&ddr, n * 8); cudaMalloc(&dr, n * 8);
    cudaMalloc(&st, 4);
    cudaMemcpy(dS, S.data(), n * n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dphi, phi.data(), n * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_lu_solve<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k_lu_solve<4><<<1, 256, lu_smem_bytes(n)>>>(dS, dphi, ddr, dr, n, 0, st);
    cudaEventRecord(a);
    for (int r = 0; r < 200; ++r) k_lu_solve<4><<<1, 256, lu_smem_bytes(n)>>>(dS, dphi, ddr, dr, n, 0, st);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<double> x(n); cudaMemcpy(x.data(), ddr, n * 8, cudaMemcpyDeviceToHost);
    double res = 0;
    for (int i = 0; i < n; ++i) { double s = phi[i]; for (int j = 0; j < n; ++j) s += S[i * n + j] * x[j]; res = fmax(res, fabs(s)); }
    printf("n=%d  %.2f us/solve  residual %.2e  err=%s\n", n, ms * 1000 / 200, res, cudaGetErrorString(cudaGetLastError()));
  }
}
