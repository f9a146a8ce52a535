// Probe: fp64 DMMA GEMM tile configurations for the batched (many-sims) decoder layers.
// Y_t[c][m] = sum_k W[m][k] X_t[c][k], M = K = 256 (hidden width), C = sims * jet columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2102_11026_b200/csrc \
//        gemm_probe.cu -o gemm_probe
#include <cstdio>
#include <vector>
#include "gemm_f64.cuh"
#include "epilogues.cuh"

using namespace nlrom;

template <class Cfg, class Epi>
float run(const GemmArgs& g, const Epi& e, int reps) {
  cudaStream_t st = 0;
  launch_gemm<Cfg>(g, e, st);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) launch_gemm<Cfg>(g, e, st);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms / reps;
}

template <class Cfg>
void probe(const char* name, const GemmArgs& g, double* Y, double* bias, double* cache) {
  EpiStore es{Y, g.M, 0, bias, 1 << 30, nullptr};
  EpiAct<2, ACT_SIN_MD> ea{Y, g.M, 0, bias, nullptr};
  const double fl = 2.0 * g.M * g.K * (double)g.C;
  float t1 = run<Cfg>(g, es, 5);
  float t2 = run<Cfg>(g, ea, 5);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_tn_kernel<Cfg, EpiStore>, Cfg::NT, Cfg::SMEM_BYTES);
  printf("%-34s smem %6d B  occ %d  store %.3f ms %.1f TF/s   sin-epi %.3f ms %.1f TF/s\n", name, Cfg::SMEM_BYTES,
         occ, t1, fl / t1 / 1e9, t2, fl / t2 / 1e9);
}

int main() {
  const int M = 256, K = 256, C = 4096 * 96;
  double *A, *B, *Y, *bias;
  cudaMalloc(&A, (size_t)M * K * 8);
  cudaMalloc(&B, (size_t)C * K * 8);
  cudaMalloc(&Y, (size_t)C * M * 8);
  cudaMalloc(&bias, M * 8);
  cudaMemset(A, 0, (size_t)M * K * 8);
  cudaMemset(B, 0, (size_t)C * K * 8);
  cudaMemset(bias, 0, M * 8);
  GemmArgs g{A, B, K, K, M, C, K, 0, 0};
  probe<GemmCfg<64, 128, 2, 4, 1, 32, 3>>("64x128 w2x4 bk32 s3 (current)", g, Y, bias, nullptr);
  probe<GemmCfg<64, 128, 2, 4, 1, 16, 3>>("64x128 w2x4 bk16 s3", g, Y, bias, nullptr);
  probe<GemmCfg<64, 128, 2, 4, 1, 16, 4>>("64x128 w2x4 bk16 s4", g, Y, bias, nullptr);
  probe<GemmCfg<128, 128, 2, 4, 1, 16, 3>>("128x128 w2x4 bk16 s3", g, Y, bias, nullptr);
  probe<GemmCfg<128, 128, 4, 4, 1, 16, 3>>("128x128 w4x4 bk16 s3", g, Y, bias, nullptr);
  probe<GemmCfg<128, 64, 4, 2, 1, 16, 4>>("128x64 w4x2 bk16 s4", g, Y, bias, nullptr);
  probe<GemmCfg<64, 64, 2, 2, 1, 16, 4>>("64x64 w2x2 bk16 s4", g, Y, bias, nullptr);
  probe<GemmCfg<128, 128, 2, 2, 1, 16, 3>>("128x128 w2x2 bk16 s3", g, Y, bias, nullptr);
  probe<GemmCfg<256, 64, 4, 2, 1, 16, 3>>("256x64 w4x2 bk16 s3", g, Y, bias, nullptr);
  probe<GemmCfg<64, 256, 2, 4, 1, 16, 3>>("64x256 w2x4 bk16 s3", g, Y, bias, nullptr);
  return 0;
}
