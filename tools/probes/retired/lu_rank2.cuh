// Two pivot steps per CTA barrier: k_lu_solve's row-block LU (registers + shared mirror,
// implicit pivoting, Gauss-Jordan form) with the steps k and k + 1 fused into one rank-2 update.
//
// Per double step every warp redundantly (no communication):
//   1. p1 = argmax_unused |a_ik|, r1 = 1 / a_p1,k, l1_i = a_ik r1;
//   2. column k + 1 after step k for its rows: u_i = fma(-l1_i, a_p1,k+1, a_i,k+1);
//      p2 = argmax_unused' |u_i|, r2 = 1 / u_p2;
// then every thread updates its register block for columns j >= k + 2 (ONE barrier per double
// step, after the stores):
//   a'_ij = fma(-l1_i, a_p1,j, a_ij)   (i != p1)      step k
//   a''_ij = fma(-l2_i, a'_p2,j, a'_ij) (i != p2)    step k + 1, l2_i = a'_i,k+1 r2
// with the same fma sequence as two single steps, so the result is bitwise identical to
// k_lu_solve (same pivots, same roundings). Columns k, k + 1 are not written in the double
// step. The two pivot rows are read by every thread with their OLD values, so their owners
// put the new values into a side buffer PR (rows p1, p2) instead of the shared mirror; the
// next double step reads the multipliers of those two rows from PR (later steps write the
// rows back to the mirror as ordinary rows; after the loop every owner stores its block).
#pragma once
#include "../../../paper_2102_11026_b200/csrc/solve_kernels.cuh"

namespace nlrom {

template <int NB>
__global__ void __launch_bounds__(256) k_lu_solve2(const double* __restrict__ S, const double* __restrict__ phi,
                                                    double* __restrict__ dr, double* __restrict__ r, int n, int apply,
                                                    int* __restrict__ status, const double* __restrict__ xrhs, int nx,
                                                    double* __restrict__ xout, const double* __restrict__ Gt, int ldg,
                                                    int n_p) {
  pdl_wait();
  pdl_launch();
  constexpr int D = 16 * NB;
  constexpr int LDF = D + 1;
  extern __shared__ double M[];        // [D][LDF] | vhp block [n_q][n_q]
  __shared__ int pivrow[D];
  __shared__ double rdiag[D];
  __shared__ double PR[2][D];          // new values of the last double step's pivot rows
  const int sim = blockIdx.x;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31;
  const double* Ss = S + (size_t)sim * n * n;
  const int nq = n - n_p;
  double* Vs = M + D * LDF;
  for (int idx = tid; idx < D * D; idx += 256) {
    const int i = idx / D, j = idx % D;
    double* dst = M + i * LDF + j;
    if (i < n && j < n) cp_async8(dst, Ss + (size_t)i * n + j);
    else if (i < n && j == n) cp_async8(dst, phi + (size_t)sim * n + i);
    else if (i < n && j > n && j <= n + nx) cp_async8(dst, xrhs + ((size_t)sim * nx + (j - n - 1)) * n + i);
    else *dst = 0.0;
  }
  if (Gt)
    for (int idx = tid; idx < nq * nq; idx += 256) {
      const int k = idx / nq, i = idx % nq;
      cp_async8(Vs + idx, Gt + ((size_t)sim * 2 * nq + 2 * k + 1) * ldg + i);
    }
  cp_async_all_wait();
  __syncthreads();
  double A[NB][NB];
#pragma unroll
  for (int a = 0; a < NB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int i = ty + 16 * a, j = tx + 16 * b;
      double v = M[i * LDF + j];
      if (j == n) v = -v;
      if (Gt && i >= n_p && j >= n_p && i < n && j < n) v += Vs[(j - n_p) * nq + (i - n_p)];
      A[a][b] = v;
    }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < NB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) M[(ty + 16 * a) * LDF + tx + 16 * b] = A[a][b];
  unsigned long long used_lo = 0ull, used_hi = 0ull;
  for (int i = n; i < D; ++i) {
    if (i < 64) used_lo |= 1ull << i;
    else used_hi |= 1ull << (i - 64);
  }
  auto is_used = [&](int i) -> bool {
    return i < 64 ? ((used_lo >> i) & 1ull) : ((used_hi >> (i - 64)) & 1ull);
  };
  auto mark = [&](int i) {
    if (i < 64) used_lo |= 1ull << i;
    else used_hi |= 1ull << (i - 64);
  };
  // exact argmax over unused rows of v(i) (IEEE bits of |v| >= 0), lowest row on ties
  auto argmax = [&](const double (&val)[D / 32], int& piv) -> bool {
    double best = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < D / 32; ++u) {
      const int i = lane + 32 * u;
      if (!is_used(i)) {
        const double v = fabs(val[u]);
        if (v > best) { best = v; bi = i; }
      }
    }
    const unsigned long long key = (best >= 0.0) ? (unsigned long long)__double_as_longlong(best) : 0ull;
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    piv = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)bi : 0x7fffffffu);
    return (mhi | mlo) && piv < n;
  };
  int q1 = -1, q2 = -1;  // pivot rows of the previous double step (their new values live in PR)
  // value of column j of row i at the start of a double step (PR for last step's pivot rows)
  auto colval = [&](int i, int j) -> double {
    return i == q1 ? PR[0][j] : (i == q2 ? PR[1][j] : M[i * LDF + j]);
  };
  bool bad = false;
  __syncthreads();
  int k = 0;
  for (; k + 1 < n; k += 2) {
    // ---- step k: pivot search on column k (unused rows are never q1 / q2)
    double ck[D / 32], ck1[D / 32];
#pragma unroll
    for (int u = 0; u < D / 32; ++u) {
      ck[u] = M[(lane + 32 * u) * LDF + k];
      ck1[u] = M[(lane + 32 * u) * LDF + k + 1];
    }
    int p1;
    if (!argmax(ck, p1)) { bad = true; break; }
    mark(p1);
    const double a1k = M[p1 * LDF + k], a1k1 = M[p1 * LDF + k + 1];
    const double r1 = recip_fast(a1k);
    // ---- step k + 1: column k + 1 after step k, pivot search
    double uk1[D / 32];
#pragma unroll
    for (int u = 0; u < D / 32; ++u) uk1[u] = fma(-(ck[u] * r1), a1k1, ck1[u]);
    int p2;
    if (!argmax(uk1, p2)) { bad = true; break; }
    mark(p2);
    const double l1p2 = M[p2 * LDF + k] * r1;
    const double u2 = fma(-l1p2, a1k1, M[p2 * LDF + k + 1]);
    const double r2 = recip_fast(u2);
    if (tid == 0) {
      pivrow[k] = p1;
      rdiag[k] = r1;
      pivrow[k + 1] = p2;
      rdiag[k + 1] = r2;
    }
    // operands: pivot rows (old values) for this thread's columns, multipliers of its rows
    double pr1[NB], pr2[NB], l1[NB], ak1[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      pr1[b] = M[p1 * LDF + tx + 16 * b];
      pr2[b] = M[p2 * LDF + tx + 16 * b];
    }
#pragma unroll
    for (int a = 0; a < NB; ++a) {
      const int i = ty + 16 * a;
      l1[a] = colval(i, k) * r1;
      ak1[a] = colval(i, k + 1);
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) pr2[b] = fma(-l1p2, pr1[b], pr2[b]);  // a'_p2,j
    // no barrier here: this step writes only columns >= k + 2 of non-pivot rows of the mirror
    // and PR[.][>= k + 2], while it reads columns k, k + 1, the pivot rows and PR[.][k, k + 1]
#pragma unroll
    for (int a = 0; a < NB; ++a) {
      const int i = ty + 16 * a;
      const bool r_p1 = i == p1, r_p2 = i == p2;
      // step k: every row but p1; step k + 1: every row but p2
      const double m1 = r_p1 ? 0.0 : l1[a];
      const double a1 = r_p1 ? ak1[a] : fma(-l1[a], a1k1, ak1[a]);  // a'_i,k+1
      const double m2 = r_p2 ? 0.0 : a1 * r2;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (NB > 4 && 16 * b + 15 <= k + 1) continue;  // column block already eliminated (uniform)
        const int j = tx + 16 * b;
        if (i < n && j > k + 1) {
          double v = A[a][b];
          if (!r_p1) v = fma(-m1, pr1[b], v);
          if (!r_p2) v = fma(-m2, pr2[b], v);
          A[a][b] = v;
          if (r_p1) PR[0][j] = v;
          else if (r_p2) PR[1][j] = v;
          else M[i * LDF + j] = v;
        }
      }
    }
    q1 = p1;
    q2 = p2;
    __syncthreads();
  }
  if (!bad && k < n) {  // odd n: one single step (k = n - 1), as in k_lu_solve
    double ck[D / 32];
#pragma unroll
    for (int u = 0; u < D / 32; ++u) ck[u] = M[(lane + 32 * u) * LDF + k];
    int p1;
    if (!argmax(ck, p1)) {
      bad = true;
    } else {
      mark(p1);
      const double r1 = recip_fast(M[p1 * LDF + k]);
      if (tid == 0) {
        pivrow[k] = p1;
        rdiag[k] = r1;
      }
      double pr1[NB], l1[NB];
#pragma unroll
      for (int b = 0; b < NB; ++b) pr1[b] = M[p1 * LDF + tx + 16 * b];
#pragma unroll
      for (int a = 0; a < NB; ++a) l1[a] = colval(ty + 16 * a, k);
      __syncthreads();
#pragma unroll
      for (int a = 0; a < NB; ++a) {
        const int i = ty + 16 * a;
        const double la = l1[a] * r1;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int j = tx + 16 * b;
          if (i < n && i != p1 && j > k) A[a][b] = fma(-la, pr1[b], A[a][b]);
        }
      }
    }
  }
  if (bad) {
    if (tid == 0) status[sim] = 1;
    return;
  }
  // the right-hand-side columns of every row from the registers (PR rows included)
#pragma unroll
  for (int a = 0; a < NB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int i = ty + 16 * a, j = tx + 16 * b;
      if (i < n && j >= n) M[i * LDF + j] = A[a][b];
    }
  __syncthreads();
  for (int t = tid; t < n * (1 + nx); t += blockDim.x) {
    const int kk = t % n, col = t / n;
    const double x = M[pivrow[kk] * LDF + n + col] * rdiag[kk];
    if (col == 0) {
      dr[(size_t)sim * n + kk] = x;
      if (apply) r[(size_t)sim * n + kk] += x;
    } else {
      xout[((size_t)sim * nx + col - 1) * n + kk] = x;
    }
  }
  if (tid == 0) status[sim] = 0;
}

}  // namespace nlrom
