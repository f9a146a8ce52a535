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


// Gram with one extra right-hand column: out = X^T Y[:, 0:n] (n x n, ldo) and fout = X^T Y[:, n].
// The cubature stores G_e = w_e K_e J~_e in the G panel's columns 0..n-1 and w_e f_e in its
// padding column n, so the force projection rides along in the same DMMA loop. Predicate-free
// loads: K must be a multiple of 4, and rows / columns past n (garbage in the panels' padding,
// or the next shared-memory region) only reach output tiles that are not stored; needs
// ldx >= 8 ceil(n / 8) and ldy > n (gram_ld).
template <int GW>
__device__ inline void gram_dmma_kf_t(const double* __restrict__ X, int ldx, const double* __restrict__ Y, int ldy,
                                      int K, int n, double* __restrict__ out, int ldo, double* __restrict__ fout,
                                      bool accumulate) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int m = n + 1;
  const int ti = (n + 7) / 8, tj = (m + 7) / 8, tjg = (tj + GW - 1) / GW;
  for (int t = warp; t < ti * tjg; t += nw) {
    const int bi = t / tjg, bj0 = (t % tjg) * GW;
    double c[GW][2] = {};
    const int i = bi * 8 + (lane >> 2);
    const double* xp = X + (lane & 3) * ldx + i;
    const double* yp = Y + (lane & 3) * ldy + bj0 * 8 + (lane >> 2);
#pragma unroll 4
    for (int k = 0; k < K; k += 4) {
      const double a = xp[k * ldx];
#pragma unroll
      for (int u = 0; u < GW; ++u) dmma(c[u][0], c[u][1], a, yp[k * ldy + u * 8]);
    }
#pragma unroll
    for (int u = 0; u < GW; ++u) {
      const int j = (bj0 + u) * 8 + 2 * (lane & 3);
      if (i < n) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double* o = j + e < n ? out + (size_t)i * ldo + j + e : (j + e == n ? fout + i : nullptr);
          if (o) *o = accumulate ? (*o + c[u][e]) : c[u][e];
        }
      }
    }
  }
}

__device__ inline void gram_dmma_kf(const double* __restrict__ X, int ldx, const double* __restrict__ Y, int ldy,
                                    int K, int n, double* __restrict__ out, int ldo, double* __restrict__ fout,
                                    bool accumulate) {
  const int ti = (n + 7) / 8, tj = (n + 8) / 8;
  if (ti * ((tj + 3) / 4) < (int)(blockDim.x >> 5))
    gram_dmma_kf_t<2>(X, ldx, Y, ldy, K, n, out, ldo, fout, accumulate);
  else
    gram_dmma_kf_t<4>(X, ldx, Y, ldy, K, n, out, ldo, fout, accumulate);
}

// Per-element G_e = w_e K_e J~_e on the DMMA pipe: K_e (12 x 12, row-major, [el][144]) times
// the element's 12 J~ rows (Js panel rows el*12 .. el*12+11, pitch ldp), scaled by w[el] and
// written to the G panel (same pitch, columns 0..n-1). Rows padded 12 -> 16 (two 8-row tiles;
// rows 12..15 read the next element's K or the force panel and are never stored), k = 12 in
// 3 steps. One warp per (element, row tile): its 3 A fragments are loaded once and reused over
// all 8-column tiles.
__device__ inline void ke_j_dmma(const double* __restrict__ Ks, const double* __restrict__ Js, double* __restrict__ Gs,
                                 int ldp, int epc, int n, const double* __restrict__ w) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nt = (n + 7) / 8;
  const int r0 = lane >> 2, kq = lane & 3;
  for (int t = warp; t < epc * 2; t += nw) {
    const int el = t >> 1, row = (t & 1) * 8 + r0;
    const double* K = Ks + el * 144 + row * 12 + kq;
    const double* J = Js + ((size_t)el * 12 + kq) * ldp + r0;
    double* g = Gs + ((size_t)el * 12 + row) * ldp + 2 * kq;
    const double we = w[el];
    const double a0 = K[0], a1 = K[4], a2 = K[8];
#pragma unroll 2
    for (int nj = 0; nj < nt; ++nj) {
      double c0 = 0.0, c1 = 0.0;
      dmma(c0, c1, a0, J[nj * 8]);
      dmma(c0, c1, a1, J[4 * ldp + nj * 8]);
      dmma(c0, c1, a2, J[8 * ldp + nj * 8]);
      const int ocol = nj * 8 + 2 * kq;
      if (row < 12) {
        if (ocol < n) g[nj * 8] = we * c0;
        if (ocol + 1 < n) g[nj * 8 + 1] = we * c1;
      }
    }
  }
}

}  // namespace nlrom
