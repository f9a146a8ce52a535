// Probe: the tcgen05 kind::i8 Ozaki fp64 GEMM (csrc/ozaki_tc.cuh) against a CPU long-double
// GEMM on random data with widely varying column scales, and its device time vs the fp64
// DMMA big-tile kernels at the cfg5 hidden-layer shape (M = K = 256).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          -lineinfo tools/probes/ozaki_probe.cu -o tools/probes/ozaki_probe
#include <cstdio>
#include <cstdlib>
#ifndef OZ_BN
#define OZ_BN 32
#endif
#include <vector>
#include <random>
#include "../../paper_2102_11026_b200/csrc/ozaki_chain.cuh"
#include "../../paper_2102_11026_b200/csrc/gemm_ws.cuh"
using namespace nlrom;

namespace nlrom {
void upload_matrix(DBuf& dst, const double* h, int rows, int cols, int ld, int rows_alloc) {
  const int ra = rows_alloc < 0 ? rows : rows_alloc;
  std::vector<double> tmp((size_t)ra * ld, 0.0);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) tmp[(size_t)r * ld + c] = h[(size_t)r * cols + c];
  dst.alloc(tmp.size());
  NL_CUDA(cudaMemcpy(dst.p, tmp.data(), tmp.size() * 8, cudaMemcpyHostToDevice));
}
}  // namespace nlrom

// B operand as digit tiles (the digit chain's layout, ozaki_chain.cuh): [C/64][K/32][S][64 x 32 B]
static void prepare_b_digits(const std::vector<double>& B, int C, int K, std::vector<unsigned char>& tiles,
                             std::vector<int>& exps) {
  using namespace oz;
  const int tc_n = (C + 63) / 64, nk = K / BK;
  const int BST = Cfg<64>::B_STAGE, BSL = Cfg<64>::B_SLICE;
  tiles.assign((size_t)tc_n * nk * BST, 0);
  exps.assign((size_t)tc_n * 64, 0);
  for (int c = 0; c < C; ++c) {
    double amax = 0.0;
    for (int k = 0; k < K; ++k) amax = std::max(amax, std::fabs(B[(size_t)c * K + k]));
    // the producer's rule: exp_of of the high-word bound of the column maximum
    const unsigned hw = (unsigned)(__builtin_bit_cast(unsigned long long, amax) >> 32);
    const int E = hw ? exp_of(__builtin_bit_cast(double, ((unsigned long long)hw << 32) | 0xFFFFFFFFull)) : 0;
    exps[c] = E;
    for (int k = 0; k < K; ++k) {
      const long long qb = balanced((long long)std::trunc(std::ldexp(B[(size_t)c * K + k], QBITS - E)));
      unsigned char* st = tiles.data() + ((size_t)(c / 64) * nk + k / BK) * BST;
      for (int t = 0; t < S; ++t) st[t * BSL + core_off(c % 64, k % BK)] = (unsigned char)digit(qb, t);
    }
  }
}

int main(int argc, char** argv) {
  const int M = 256, K = 256;
  const int C = argc > 1 ? atoi(argv[1]) : 1000;
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(-1, 1);
  std::vector<double> A((size_t)M * K), B((size_t)C * K);
  for (int m = 0; m < M; ++m) {
    const double rs = std::ldexp(1.0, (int)(U(g) * 6));
    for (int k = 0; k < K; ++k) A[(size_t)m * K + k] = U(g) * rs;
  }
  for (int c = 0; c < C; ++c) {
    const double cs = std::ldexp(1.0, (int)(U(g) * 30));  // columns from 2^-30 to 2^30
    for (int k = 0; k < K; ++k) B[(size_t)c * K + k] = U(g) * cs * (k % 7 == 0 ? 1e-3 : 1.0);
  }
  std::vector<unsigned char> tiles;
  std::vector<int> exps;
  ozaki_prepare_a(A.data(), K, M, K, tiles, exps);
  unsigned char* dT;
  int* dE;
  NL_CUDA(cudaMalloc(&dT, tiles.size()));
  NL_CUDA(cudaMalloc(&dE, exps.size() * 4));
  NL_CUDA(cudaMemcpy(dT, tiles.data(), tiles.size(), cudaMemcpyHostToDevice));
  NL_CUDA(cudaMemcpy(dE, exps.data(), exps.size() * 4, cudaMemcpyHostToDevice));
  DBuf dA, dB, dY((size_t)C * M), dY2((size_t)C * M);
  upload_matrix(dA, A.data(), M, K, K, -1);
  upload_matrix(dB, B.data(), C, K, K, -1);
  GemmArgs ga{dA.p, dB.p, K, K, M, C, K, 0, 0};
  OzakiA oa{dT, dE};
  launch_ozaki<OZ_BN>(oa, OzakiBExp{nullptr, 0}, ga, EpiStore{dY.p, M, 0, nullptr, 1, nullptr}, 0);
  NL_CUDA(cudaDeviceSynchronize());
  std::vector<double> Y((size_t)C * M);
  NL_CUDA(cudaMemcpy(Y.data(), dY.p, Y.size() * 8, cudaMemcpyDeviceToHost));
  double worst = 0, worst_rel = 0;
  for (int c = 0; c < C; ++c)
    for (int m = 0; m < M; ++m) {
      long double s = 0, sa = 0;
      for (int k = 0; k < K; ++k) {
        s += (long double)A[(size_t)m * K + k] * B[(size_t)c * K + k];
        sa += fabsl((long double)A[(size_t)m * K + k] * B[(size_t)c * K + k]);
      }
      const double e = (double)(fabsl((long double)Y[(size_t)c * M + m] - s) / (sa > 0 ? sa : 1));
      worst = std::max(worst, e);
      if (fabsl(s) > 1e-3 * sa) worst_rel = std::max(worst_rel, (double)(fabsl((long double)Y[(size_t)c * M + m] - s) / fabsl(s)));
    }
  printf("C=%d  max |y - ref| / sum|a||b| = %.3e   max rel (well-conditioned) = %.3e  %s\n", C, worst, worst_rel,
         worst < 2e-15 ? "OZAKI_OK" : "OZAKI_BAD");
#if OZ_BN == 64
  {  // B from digit tiles: bitwise equal to the converter path when the column scales agree
    std::vector<unsigned char> bt;
    std::vector<int> be;
    prepare_b_digits(B, C, K, bt, be);
    unsigned char* dBt;
    int* dBe;
    NL_CUDA(cudaMalloc(&dBt, bt.size()));
    NL_CUDA(cudaMalloc(&dBe, be.size() * 4));
    NL_CUDA(cudaMemcpy(dBt, bt.data(), bt.size(), cudaMemcpyHostToDevice));
    NL_CUDA(cudaMemcpy(dBe, be.data(), be.size() * 4, cudaMemcpyHostToDevice));
    OzakiBExp bd{nullptr, 0};
    bd.dig = dBt;
    bd.dexp = dBe;
    DBuf dY3((size_t)C * M);
    launch_ozaki<64, EpiStore, true>(oa, bd, ga, EpiStore{dY3.p, M, 0, nullptr, 1, nullptr}, 0);
    NL_CUDA(cudaDeviceSynchronize());
    std::vector<double> Y3((size_t)C * M);
    NL_CUDA(cudaMemcpy(Y3.data(), dY3.p, Y3.size() * 8, cudaMemcpyDeviceToHost));
    double w3 = 0;
    for (size_t i = 0; i < Y3.size(); ++i) w3 = std::max(w3, std::fabs(Y3[i] - Y[i]));
    printf("BDIG vs converter: max |diff| = %.3e (%s)\n", w3, w3 == 0 ? "bitwise" : "DIFFERENT");
  }
#endif
  // timing at the cfg5 hidden-layer shape
  const int CT = 393216;
  DBuf bigB((size_t)CT * K), bigY((size_t)CT * M);
  {
    std::vector<double> hb((size_t)CT * K);
    for (auto& x : hb) x = U(g);
    NL_CUDA(cudaMemcpy(bigB.p, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice));
  }
  GemmArgs gb{dA.p, bigB.p, K, K, M, CT, K, 0, 0};
  unsigned* dEx;  // precomputed column scales (1 part per column): high word of 1.0 (|x| < 1)
  NL_CUDA(cudaMalloc(&dEx, CT * 4));
  {
    std::vector<unsigned> ex(CT, 0x3FF00000u);
    NL_CUDA(cudaMemcpy(dEx, ex.data(), CT * 4, cudaMemcpyHostToDevice));
  }
  const OzakiBExp pre{dEx, 1}, self{nullptr, 0};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float t_oz = 0, t_ozp = 0, t_ws = 0;
  for (int rep = 0; rep < 2; ++rep) {
    launch_ozaki<OZ_BN>(oa, self, gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
    launch_gemm_ws<WsCfg<64, 128, 4, 4, 4>>(gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
  }
  cudaEventRecord(e0);
  for (int rep = 0; rep < 5; ++rep) launch_ozaki<OZ_BN>(oa, self, gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&t_oz, e0, e1);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 5; ++rep) launch_ozaki<OZ_BN>(oa, pre, gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&t_ozp, e0, e1);
  cudaEventRecord(e0);
  for (int rep = 0; rep < 5; ++rep) launch_gemm_ws<WsCfg<64, 128, 4, 4, 4>>(gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&t_ws, e0, e1);
  const double fl = 2.0 * M * K * (double)CT;
  float t_dig = 0;
#if OZ_BN == 64
  {
    std::vector<double> hb((size_t)CT * K);
    NL_CUDA(cudaMemcpy(hb.data(), bigB.p, hb.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<unsigned char> bt;
    std::vector<int> be;
    prepare_b_digits(hb, CT, K, bt, be);
    unsigned char* dBt;
    int* dBe;
    NL_CUDA(cudaMalloc(&dBt, bt.size()));
    NL_CUDA(cudaMalloc(&dBe, be.size() * 4));
    NL_CUDA(cudaMemcpy(dBt, bt.data(), bt.size(), cudaMemcpyHostToDevice));
    NL_CUDA(cudaMemcpy(dBe, be.data(), be.size() * 4, cudaMemcpyHostToDevice));
    OzakiBExp bd{nullptr, 0};
    bd.dig = dBt;
    bd.dexp = dBe;
    launch_ozaki<64, EpiStore, true>(oa, bd, gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) launch_ozaki<64, EpiStore, true>(oa, bd, gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t_dig, e0, e1);
#ifdef OZ_TRACE
    unsigned long long z[12] = {};
    cudaMemcpyToSymbol(g_oz_trace, z, sizeof z);
    launch_ozaki<64, EpiStore, true>(oa, bd, gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(z, g_oz_trace, sizeof z);
    printf("BDIG per CTA (cycles): MMA wait tempty %.0f  wait A+B %.0f | drain wait tfull %.0f\n", z[0] / 148.0,
           z[1] / 148.0, z[4] / 148.0);
#endif
    printf("BDIG (B digit tiles by TMA, EpiStore): %.3f ms (%.1f fp64-equiv TFLOP/s)\n", t_dig / 5,
           fl / (t_dig / 5 * 1e-3) / 1e12);
    // the digit chain's middle layer: B digits in, EpiJetDig (jet sin + digit tiles) out
    {
      unsigned char* dOut;
      int* dOutE;
      NL_CUDA(cudaMalloc(&dOut, bt.size()));
      NL_CUDA(cudaMalloc(&dOutE, be.size() * 4));
      DBuf bias(M);
      NL_CUDA(cudaMemset(bias.p, 0, M * 8));
      DBuf cache((size_t)(CT / 96) * 40 * M);
      EpiJetDig ed{bias.p, getenv("OZ_NOCACHE") ? nullptr : cache.p, M, 32, 3, 20, dOut, dOutE};
      float t_jd = 0;
      launch_ozaki<64, EpiJetDig, true>(oa, bd, gb, ed, 0);
      cudaEventRecord(e0);
      for (int rep = 0; rep < 5; ++rep) launch_ozaki<64, EpiJetDig, true>(oa, bd, gb, ed, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&t_jd, e0, e1);
#ifdef OZ_TRACE
      cudaMemcpyToSymbol(g_oz_trace, z, sizeof z);
      launch_ozaki<64, EpiJetDig, true>(oa, bd, gb, ed, 0);
      cudaDeviceSynchronize();
      cudaMemcpyFromSymbol(z, g_oz_trace, sizeof z);
      printf("BDIG+EpiJetDig per CTA (cycles): MMA wait tempty %.0f  wait A+B %.0f | epi wait tfull %.0f  drain %.0f  "
             "functor %.0f (jet %.0f, colmax %.0f, exchange %.0f, convert %.0f, fence+bar %.0f, bulk read %.0f)\n",
             z[0] / 148.0, z[1] / 148.0, z[4] / 148.0, z[5] / 148.0, z[6] / 148.0, z[2] / 148.0, z[3] / 148.0,
             z[7] / 148.0, z[8] / 148.0, z[10] / 148.0, z[9] / 148.0);
#endif
      printf("BDIG + EpiJetDig: %.3f ms  (%s)\n", t_jd / 5, cudaGetErrorString(cudaGetLastError()));
    }
  }
#endif
#ifdef OZ_TRACE
  {
    unsigned long long z[12] = {};
    cudaMemcpyToSymbol(g_oz_trace, z, sizeof z);
    launch_ozaki<OZ_BN>(oa, pre, gb, EpiStore{bigY.p, M, 0, nullptr, 1, nullptr}, 0);
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(z, g_oz_trace, sizeof z);
    const double ctas = 148;
    printf("per CTA (cycles): MMA wait tempty %.0f  wait A %.0f  wait B %.0f | epi wait tfull %.0f  drain %.0f\n",
           z[0] / ctas, z[1] / ctas, z[2] / ctas, z[4] / ctas, z[5] / ctas);
  }
#endif
  printf("BN=%d M=K=256, C=%d: ozaki tcgen05 %.3f ms (%.1f fp64-equiv TFLOP/s), with given exponents %.3f ms (%.1f)   "
         "DMMA ws %.3f ms (%.1f TFLOP/s)  %s\n", OZ_BN, CT, t_oz / 5, fl / (t_oz / 5 * 1e-3) / 1e12, t_ozp / 5,
         fl / (t_ozp / 5 * 1e-3) / 1e12, t_ws / 5, fl / (t_ws / 5 * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  return worst < 2e-15 ? 0 : 1;
}
