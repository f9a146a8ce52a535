// Substructured scene (SURVEY.md §8e, cfg4 puffer ball): the context's sims are strings
// sharing one DAE / cubature model, each with a fixed rotation R_s (string frame -> world),
// attached to a translating core (3 DOFs, replicated on every rank). Model and notation:
// oracle/coupled.py (module docstring). Per Newton iteration and rank:
//
//   k_cp_fext     f_eff,s = R_s^T f_ext,s - M T R_s^T Dc / h^2   (the coupling enters the string
//                 residual / system Jacobian as an effective load, so phase E / J run unchanged)
//   k_cp_blocks   per string: K_s = T^T M J~ (3 x n), T^T M dJ (3 x n_q), t_s = T^T f_fict,
//                 C_s = (1 + ah) K_s^T R_s^T (n x 3: extra right-hand sides of the LU)
//   k_lu_solve    [S_s | -phi_s | C_s] -> dr0_s = -S^-1 phi_s, X_s = S^-1 C_s
//   k_cp_partial  16 doubles: sum_s E_s [X_s | dr0_s] (3 x 4), the strings' part of phi_c (3),
//                 sum_s ||phi_s||^2, E_s = R_s((1 + ah) K_s + [0, T^T M dJ_s])
//   -- allreduce of the 16 doubles over ranks (NCCL, host side) --
//   k_cp_update   phi_c, ||phi||, Schur solve (Z - sum E X) dc = -phi_c - sum E dr0 (3 x 3, LU-pp)
//   k_cp_apply    r_s = r_base,s + t (dr0_s - X_s dc), c = c_base + t dc
#pragma once
#include "common.cuh"

namespace nlrom {

// core state layout (doubles): c, c_bar, cdot_bar, c_base, dc, phi_c (6 x 3) + norm
enum { CORE_C = 0, CORE_CBAR = 3, CORE_CDBAR = 6, CORE_CBASE = 9, CORE_DC = 12, CORE_PHIC = 15, CORE_NORM = 18,
       CORE_SIZE = 19 };
constexpr int CP_PARTIAL = 16;

__device__ __forceinline__ void cp_delta(const double* core, double ah, double h, double* Dc) {
#pragma unroll
  for (int a = 0; a < 3; ++a) Dc[a] = (1.0 + ah) * (core[CORE_C + a] - core[CORE_CBAR + a]) - h * core[CORE_CDBAR + a];
}

// grid-stride over n_sims * N: f_eff = floc - m (R^T Dc)[dof % 3] / h^2
__global__ void k_cp_fext(const double* __restrict__ floc, const double* __restrict__ R,
                          const double* __restrict__ core, const double* __restrict__ mass, int N, int S, double h,
                          double ah, double* __restrict__ fext) {
  pdl_wait();
  pdl_launch();
  double Dc[3];
  cp_delta(core, ah, h, Dc);
  const double ih2 = 1.0 / (h * h);
  const long long tot = (long long)S * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
       idx += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(idx / N), i = (int)(idx % N), d = i % 3;
    const double* Rs = R + (size_t)s * 9;
    const double dl = Rs[0 * 3 + d] * Dc[0] + Rs[1 * 3 + d] * Dc[1] + Rs[2 * 3 + d] * Dc[2];  // (R^T Dc)_d
    fext[idx] = floc[idx] - mass[i] * dl * ih2;
  }
}

// one CTA (256 threads) per string: axis sums over the free-DOF rows (vertex-major, xyz interleaved)
// of m J~ (n columns), m dJ (n_q) and m hvv (1); then C_s = (1 + ah) K^T R^T.
// blocks[s] = [K (3 x n) | TMdJ (3 x n_q) | t (3)], Cb[s] = 3 columns of n.
__global__ void __launch_bounds__(256) k_cp_blocks(const double* __restrict__ Jt, int ldjt, const double* __restrict__ dJ,
                                                   int lddj, const double* __restrict__ hvv,
                                                   const double* __restrict__ mass, const double* __restrict__ R,
                                                   int N, int n, int n_q, int drop_fict, double ah,
                                                   double* __restrict__ blocks, double* __restrict__ Cb) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[8][3][32];
  __shared__ double Ks[3][128];
  const int s = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncol = n + n_q + 1, nv = N / 3;
  const int bsz = 3 * (n + n_q) + 3;
  const double* Js = Jt + (size_t)s * N * ldjt;
  const double* Ds = dJ + (size_t)s * N * lddj;
  const double* hs = hvv + (size_t)s * N;
  double* out = blocks + (size_t)s * bsz;
  for (int c0 = 0; c0 < ncol; c0 += 32) {
    const int j = c0 + lane;
    double acc[3] = {0.0, 0.0, 0.0};
    if (j < ncol)
      for (int v = warp; v < nv; v += 8) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const int row = 3 * v + d;
          double val;
          if (j < n) val = Js[(size_t)row * ldjt + j];
          else if (j < n + n_q) val = Ds[(size_t)row * lddj + (j - n)];
          else val = drop_fict ? 0.0 : hs[row];
          acc[d] = fma(mass[row], val, acc[d]);
        }
      }
#pragma unroll
    for (int d = 0; d < 3; ++d) red[warp][d][lane] = acc[d];
    __syncthreads();
    if (warp < 3 && j < ncol) {
      const int d = warp;
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sum += red[w][d][lane];
      if (j < n) {
        out[d * n + j] = sum;
        Ks[d][j] = sum;
      } else if (j < n + n_q) {
        out[3 * n + d * n_q + (j - n)] = sum;
      } else {
        out[3 * (n + n_q) + d] = sum;  // t_s = T^T (M hvv) = T^T f_fict
      }
    }
    __syncthreads();
  }
  const double* Rs = R + (size_t)s * 9;
  for (int idx = threadIdx.x; idx < 3 * n; idx += blockDim.x) {
    const int a = idx / n, i = idx % n;  // C[i][a] = (1+ah) sum_d K[d][i] R[a][d]
    Cb[((size_t)s * 3 + a) * n + i] =
        (1.0 + ah) * (Ks[0][i] * Rs[a * 3 + 0] + Ks[1][i] * Rs[a * 3 + 1] + Ks[2][i] * Rs[a * 3 + 2]);
  }
}

struct CpPartialArgs {
  const double* R; const double* blocks; const double* fsum; const double* core;
  const double* r; const double* rbar; const double* rdbar; const double* phi;
  const double* X; const double* dr0;
  int S, n, n_p, n_q;
  double h, ah, m_string;
  int jac;
  double* out;  // CP_PARTIAL doubles
};

// one CTA: per-string terms summed in a fixed order (thread-strided, then a fixed tree)
__global__ void __launch_bounds__(256) k_cp_partial(CpPartialArgs A) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[CP_PARTIAL][256];
  double acc[CP_PARTIAL];
#pragma unroll
  for (int k = 0; k < CP_PARTIAL; ++k) acc[k] = 0.0;
  double Dc[3];
  cp_delta(A.core, A.ah, A.h, Dc);
  const int n = A.n, bsz = 3 * (n + A.n_q) + 3;
  for (int s = threadIdx.x; s < A.S; s += blockDim.x) {
    const double* Rs = A.R + (size_t)s * 9;
    const double* K = A.blocks + (size_t)s * bsz;
    const double* TMdJ = K + 3 * n;
    const double* t = K + 3 * (n + A.n_q);
    const size_t o = (size_t)s * n;
    double Kc[3] = {t[0], t[1], t[2]};
    double pp = 0.0;
    for (int i = 0; i < n; ++i) {
      const double cs = (1.0 + A.ah) * (A.r[o + i] - A.rbar[o + i]) - A.h * A.rdbar[o + i];
      Kc[0] = fma(K[i], cs, Kc[0]);
      Kc[1] = fma(K[n + i], cs, Kc[1]);
      Kc[2] = fma(K[2 * n + i], cs, Kc[2]);
      pp = fma(A.phi[o + i], A.phi[o + i], pp);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
      acc[12 + a] += A.m_string * Dc[a] + Rs[a * 3 + 0] * Kc[0] + Rs[a * 3 + 1] * Kc[1] + Rs[a * 3 + 2] * Kc[2] -
                     A.h * A.h * A.fsum[(size_t)s * 3 + a];
    acc[15] += pp;
    if (A.jac) {
      // B[d][col] = sum_i ((1+ah) K[d][i] + [i >= n_p] TMdJ[d][i - n_p]) Xcol[i]; E X = R B
      double B[3][4] = {};
      for (int i = 0; i < n; ++i) {
        double Xi[4];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) Xi[cc] = A.X[((size_t)s * 3 + cc) * n + i];
        Xi[3] = A.dr0[o + i];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double e = (1.0 + A.ah) * K[d * n + i];
          if (i >= A.n_p) e += TMdJ[d * A.n_q + (i - A.n_p)];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) B[d][cc] = fma(e, Xi[cc], B[d][cc]);
        }
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
          acc[a * 4 + cc] += Rs[a * 3 + 0] * B[0][cc] + Rs[a * 3 + 1] * B[1][cc] + Rs[a * 3 + 2] * B[2][cc];
    }
  }
#pragma unroll
  for (int k = 0; k < CP_PARTIAL; ++k) red[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
#pragma unroll
      for (int k = 0; k < CP_PARTIAL; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x < CP_PARTIAL) A.out[threadIdx.x] = red[threadIdx.x][0];
}

// one thread: phi_c, ||phi||, and (mode >= 1) the Schur solve for dc; c_base = c.
__global__ void k_cp_update(const double* __restrict__ tot, double* __restrict__ core, double h, double ah,
                            double m_core, double m_total, double k_core, const double* __restrict__ f_core,
                            int mode) {
  pdl_wait();
  pdl_launch();
  if (threadIdx.x != 0) return;
  double Dc[3], phic[3];
  cp_delta(core, ah, h, Dc);
  double sq = tot[15];
  for (int a = 0; a < 3; ++a) {
    phic[a] = m_core * Dc[a] + h * h * (k_core * core[CORE_C + a] - f_core[a]) + tot[12 + a];
    core[CORE_PHIC + a] = phic[a];
    sq += phic[a] * phic[a];
  }
  core[CORE_NORM] = sqrt(sq);
  if (mode == 0) return;
  const double z = (1.0 + ah) * m_total + h * h * k_core;
  double M[3][4];
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) M[a][b] = (a == b ? z : 0.0) - tot[a * 4 + b];
    M[a][3] = -phic[a] - tot[a * 4 + 3];
  }
  for (int k = 0; k < 3; ++k) {  // Gaussian elimination with partial pivoting
    int p = k;
    for (int i = k + 1; i < 3; ++i)
      if (fabs(M[i][k]) > fabs(M[p][k])) p = i;
    if (p != k)
      for (int j = 0; j < 4; ++j) { const double tmp = M[k][j]; M[k][j] = M[p][j]; M[p][j] = tmp; }
    for (int i = k + 1; i < 3; ++i) {
      const double l = M[i][k] / M[k][k];
      for (int j = k; j < 4; ++j) M[i][j] -= l * M[k][j];
    }
  }
  double dc[3];
  for (int k = 2; k >= 0; --k) {
    double v = M[k][3];
    for (int j = k + 1; j < 3; ++j) v -= M[k][j] * dc[j];
    dc[k] = v / M[k][k];
  }
  for (int a = 0; a < 3; ++a) {
    core[CORE_DC + a] = dc[a];
    core[CORE_CBASE + a] = core[CORE_C + a];
  }
}

// r = r_base + t (dr0 - X dc), c = c_base + t dc
__global__ void k_cp_apply(double* __restrict__ r, const double* __restrict__ rbase, const double* __restrict__ dr0,
                           const double* __restrict__ X, double* __restrict__ core, int S, int n, double t) {
  pdl_wait();
  pdl_launch();
  const double dc0 = core[CORE_DC], dc1 = core[CORE_DC + 1], dc2 = core[CORE_DC + 2];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < S * n; idx += gridDim.x * blockDim.x) {
    const int s = idx / n, i = idx % n;
    const double* Xs = X + (size_t)s * 3 * n;
    const double d = dr0[idx] - Xs[i] * dc0 - Xs[n + i] * dc1 - Xs[2 * n + i] * dc2;
    r[idx] = rbase[idx] + t * d;
  }
  if (blockIdx.x == 0 && threadIdx.x < 3) core[CORE_C + threadIdx.x] = core[CORE_CBASE + threadIdx.x] + t * core[CORE_DC + threadIdx.x];
}

}  // namespace nlrom
