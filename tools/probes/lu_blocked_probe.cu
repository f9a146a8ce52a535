// Probe: k_lu_blocked (8-column panels in one warp) vs k_lu_solve (one barrier per pivot):
// bitwise equality of dr (same pivots, same fma sequence per element) on random systems with
// and without the staged vhp block / extra right-hand sides, and the device time per solve
// (CUDA events, 200 back-to-back launches, one CTA).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          tools/probes/lu_blocked_probe.cu -o tools/probes/lu_blocked_probe
#include <cstdio>
#include <cstring>
#include <vector>
#include <random>
#include "../../paper_2102_11026_b200/csrc/solve_kernels.cuh"
#ifndef LU_PW
#define LU_PW 4
#endif
using namespace nlrom;

template <int NB>
int run(int n, int n_p, int nx, bool vhp) {
  if (lu_nb(n + nx) != NB) {  // the kernels' shared memory is sized by lu_nb(n + nx)
    printf("n=%d nx=%d needs NB=%d, not %d\n", n, nx, lu_nb(n + nx), NB);
    return 1;
  }
  const int nq = n - n_p;
  std::mt19937 g(n * 7 + nx);
  std::uniform_real_distribution<double> U(-1, 1);
  std::vector<double> S(n * n), phi(n), X((size_t)nx * n), Gt((size_t)2 * nq * nq);
  for (auto& x : S) x = U(g);
  for (int i = 0; i < n; ++i) S[i * n + i] += 0.3;
  for (auto& x : phi) x = U(g);
  for (auto& x : X) x = U(g);
  for (auto& x : Gt) x = U(g) * 0.1;
  double *dS, *dphi, *ddr1, *ddr2, *dr, *dX, *dxo1, *dxo2, *dG;
  int* st;
  cudaMalloc(&dS, n * n * 8); cudaMalloc(&dphi, n * 8); cudaMalloc(&ddr1, n * 8); cudaMalloc(&ddr2, n * 8);
  cudaMalloc(&dr, n * 8); cudaMalloc(&dX, (nx + 1) * n * 8); cudaMalloc(&dxo1, (nx + 1) * n * 8);
  cudaMalloc(&dxo2, (nx + 1) * n * 8); cudaMalloc(&dG, (2 * nq * nq + 1) * 8); cudaMalloc(&st, 4);
  cudaMemcpy(dS, S.data(), n * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dphi, phi.data(), n * 8, cudaMemcpyHostToDevice);
  if (nx) cudaMemcpy(dX, X.data(), nx * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dG, Gt.data(), 2 * nq * nq * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_lu_solve<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  
  cudaFuncSetAttribute(k_lu_lookahead<NB, LU_PW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const double* G = vhp ? dG : nullptr;
  const size_t s1 = lu_smem_bytes(n + nx, nq), s2 = lu_lookahead_smem_bytes(n + nx, nq);
  auto one = [&](bool blocked, double* ddr, double* dxo) {
    if (blocked) k_lu_lookahead<NB, LU_PW><<<1, 256, s2>>>(dS, dphi, ddr, dr, n, 0, st, nx ? dX : nullptr, nx, dxo, G, nq, n_p);
    else k_lu_solve<NB><<<1, 256, s1>>>(dS, dphi, ddr, dr, n, 0, st, nx ? dX : nullptr, nx, dxo, G, nq, n_p);
  };
  one(false, ddr1, dxo1);
  one(true, ddr2, dxo2);
  cudaDeviceSynchronize();
  std::vector<double> a(n), b(n), xa((size_t)nx * n + 1), xb((size_t)nx * n + 1);
  cudaMemcpy(a.data(), ddr1, n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), ddr2, n * 8, cudaMemcpyDeviceToHost);
  if (nx) {
    cudaMemcpy(xa.data(), dxo1, nx * n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(xb.data(), dxo2, nx * n * 8, cudaMemcpyDeviceToHost);
  }
  const bool same = !memcmp(a.data(), b.data(), n * 8) && (!nx || !memcmp(xa.data(), xb.data(), nx * n * 8));
  double md = 0;
  for (int i = 0; i < n; ++i) md = fmax(md, fabs(a[i] - b[i]));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float t[2];
  for (int v = 0; v < 2; ++v) {
    for (int w = 0; w < 5; ++w) one(v, ddr2, dxo2);
    cudaEventRecord(e0);
    for (int r = 0; r < 200; ++r) one(v, ddr2, dxo2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t[v], e0, e1);
  }
#ifdef LU_TRACE
  if (n == 60) {
    one(true, ddr2, dxo2);
    cudaDeviceSynchronize();
    long long tr[70];
    cudaMemcpyFromSymbol(tr, g_lu_trace, sizeof tr);
    long long tu[64];
    cudaMemcpyFromSymbol(tu, g_lu_trace_u, sizeof tu);
    printf("  phases (cycles): staging %lld  factor %lld  solve+store %lld  | total %lld\n", tr[65] - tr[64],
           tr[66] - tr[65], tr[67] - tr[66], tr[67] - tr[64]);
    for (int p = 0; p < 15; ++p)
      printf("  panel %d: factor %lld  wait %lld  lookahead %lld | upd: spin %lld chains %lld rows %lld (fact pub at +%lld)\n", p,
             tr[4 * p + 1] - tr[4 * p], tr[4 * p + 2] - tr[4 * p + 1], p < 14 ? tr[4 * (p + 1)] - tr[4 * p + 2] : -1LL,
             tu[4 * p + 1] - tu[4 * p], tu[4 * p + 2] - tu[4 * p + 1], tu[4 * p + 3] - tu[4 * p + 2],
             tu[4 * p + 1] - tr[4 * p + 1]);
  }
#endif
  printf("n=%3d n_p=%2d nx=%d vhp=%d NB=%d  k_lu_solve %6.2f us  k_lu_lookahead %6.2f us  %s (max |d| %.1e)  %s\n", n,
         n_p, nx, (int)vhp, NB, t[0] * 5, t[1] * 5, same ? "BITWISE" : "DIFFER", md,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(dS); cudaFree(dphi); cudaFree(ddr1); cudaFree(ddr2); cudaFree(dr); cudaFree(dX); cudaFree(dxo1);
  cudaFree(dxo2); cudaFree(dG); cudaFree(st);
  return same ? 0 : 1;
}

int main(int argc, char** argv) {
  int bad = 0;
  if (argc > 1) {  // profiling: n = 60 only
    bad += run<4>(60, 30, 0, true);
    return bad;
  }
  bad += run<4>(15, 10, 0, true);
  bad += run<4>(60, 30, 0, true);
  bad += run<4>(60, 30, 0, false);
  bad += run<4>(15, 10, 3, true);
  bad += run<6>(70, 30, 0, true);
  bad += run<6>(90, 30, 3, true);
  bad += run<8>(124, 60, 0, true);
  bad += run<8>(100, 30, 0, true);
  printf("%s\n", bad ? "LU_PROBE_FAIL" : "LU_PROBE_OK");
  return bad;
}
