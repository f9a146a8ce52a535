// Probe: persistent warp-specialised TMA GEMM (gemm_ws.cuh) vs the cp.async GEMM (gemm_f64.cuh)
// on the two decoder shapes: batched hidden layer (M = K = 256, C = 4096 x 96) and the cfg2
// output layer (M = 6720, K = 256, C = 124). Checks the two agree bitwise.
#include <cstdio>
#include <vector>
#include <random>
#include "gemm_ws.cuh"
using namespace nlrom;

template <class F>
float timeit(F f, int reps) {
  f();
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <class CfgOld, class CfgWs>
void run(const char* name, int M, int K, int C) {
  std::mt19937_64 rng(3);
  std::uniform_real_distribution<double> U(-1, 1);
  std::vector<double> hA((size_t)M * K), hB((size_t)C * K);
  for (auto& x : hA) x = U(rng);
  for (auto& x : hB) x = U(rng);
  double *A, *B, *Y1, *Y2;
  cudaMalloc(&A, hA.size() * 8);
  cudaMalloc(&B, hB.size() * 8);
  cudaMalloc(&Y1, (size_t)C * M * 8);
  cudaMalloc(&Y2, (size_t)C * M * 8);
  cudaMemcpy(A, hA.data(), hA.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), hB.size() * 8, cudaMemcpyHostToDevice);
  GemmArgs g{A, B, K, K, M, C, K, 0, 0};
  EpiStore e1{Y1, M, 0, nullptr, 1 << 30, nullptr}, e2{Y2, M, 0, nullptr, 1 << 30, nullptr};
  const double fl = 2.0 * M * K * (double)C;
  float t1 = timeit([&] { launch_gemm<CfgOld>(g, e1, 0); }, 10);
  float t2 = 0;
  try {
    t2 = timeit([&] { launch_gemm_ws<CfgWs>(g, e2, 0); }, 10);
  } catch (const Error& e) {
    printf("error: %s\n", e.what());
  }
  std::vector<double> y1((size_t)C * M), y2((size_t)C * M);
  cudaMemcpy(y1.data(), Y1, y1.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(y2.data(), Y2, y2.size() * 8, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (size_t i = 0; i < y1.size(); ++i) {
    md = fmax(md, fabs(y1[i] - y2[i]));
    mx = fmax(mx, fabs(y1[i]));
  }
  printf("%-24s cp.async %.3f ms %.1f TF/s | ws-TMA %.3f ms %.1f TF/s | max|diff| %.3e (max %.2e) err=%s\n", name, t1,
         fl / t1 / 1e9, t2, fl / t2 / 1e9, md, mx, cudaGetErrorString(cudaGetLastError()));
  cudaFree(A); cudaFree(B); cudaFree(Y1); cudaFree(Y2);
}

int main() {
  run<GemmCfg<48, 128, 2, 4, 1, 32, 3>, WsCfg<48, 128, 2, 4, 6>>("output ws 2x4 (8 warps)", 6720, 256, 124);
  run<GemmCfg<48, 128, 2, 4, 1, 32, 3>, WsCfg<48, 128, 2, 8, 6>>("output ws 2x8 (16 warps)", 6720, 256, 124);
  run<GemmCfg<48, 128, 2, 4, 1, 32, 3>, WsCfg<48, 128, 1, 8, 6>>("output ws 1x8 (8 warps)", 6720, 256, 124);
  run<GemmCfg<48, 128, 2, 4, 1, 32, 3>, WsCfg<48, 128, 3, 4, 6>>("output ws 3x4 (12 warps)", 6720, 256, 124);
  run<GemmCfg<48, 128, 2, 4, 1, 32, 3>, WsCfg<48, 128, 6, 4, 6>>("output ws 6x4 (24 warps)", 6720, 256, 124);
  return 0;
}
