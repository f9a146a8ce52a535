// Small "Gram" products out = X^T Y on shared-memory row panels, on the fp64 tensor pipe.
//   X: [K][ldx], Y: [K][ldy] (row k = one DOF row of J~ / of the weighted partner), out: n x m
// Used for the per-CTA partial sums J~_C^T (w K J~_C) (cubature) and J~^T [M R | a] (assembly).
// Each warp owns groups of 4 horizontally adjacent 8x8 output tiles (4 independent DMMA
// accumulator chains); smem leading dimensions should be = 4 or 12 (mod 16) doubles
// for conflict-free fragment loads (use gram_ld()).
#pragma once
#include "gemm_f64.cuh"

namespace nlrom {

__host__ __device__ inline int gram_ld(int n) { return ((n + 7) / 8) * 8 + 4; }

__device__ inline void gram_dmma(const double* __restrict__ X, int ldx, const double* __restrict__ Y, int ldy, int K,
                                 int n, int m, double* __restrict__ out, int ldo, bool accumulate = false) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int ti = (n + 7) / 8, tj = (m + 7) / 8, tjg = (tj + 3) / 4;
  for (int t = warp; t < ti * tjg; t += nw) {
    const int bi = t / tjg, bj0 = (t % tjg) * 4;
    double c[4][2] = {};
    const int i = bi * 8 + (lane >> 2);
    for (int k = 0; k < K; k += 4) {
      const int kk = k + (lane & 3);
      const bool kin = kk < K;
      const double a = (kin && i < n) ? X[kk * ldx + i] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = (bj0 + u) * 8 + (lane >> 2);
        const double b = (kin && j < m) ? Y[kk * ldy + j] : 0.0;
        dmma(c[u][0], c[u][1], a, b);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = (bj0 + u) * 8 + 2 * (lane & 3);
      if (i < n) {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (j + e < m) {
            double* o = out + (size_t)i * ldo + j + e;
            *o = accumulate ? (*o + c[u][e]) : c[u][e];
          }
      }
    }
  }
}

}  // namespace nlrom
