// Retired: 8-column panels in one warp with CTA-wide trailing updates (bitwise equal to
// k_lu_solve, as fast at n = 60; superseded by k_lu_lookahead). Not compiled into the library.
#pragma once
#include "../../../paper_2102_11026_b200/csrc/solve_kernels.cuh"
namespace nlrom {
inline size_t lu_blocked_smem_bytes(int n, int nq = 0) {
  const int D = 16 * lu_nb(n);
  return lu_smem_bytes(n, nq) + (size_t)D * 8 * 8 + (size_t)8 * (D + 1) * 8;
}
// Blocked form of k_lu_solve (same pivots, same multipliers, same fma sequence per element:
// bitwise-equal results, tools/probes/lu_blocked_probe.cu). The per-pivot-step work that must be
// serial runs in ONE warp on 8-column panels held in registers (lane owns rows lane + 32u):
// exact argmax by integer REDUX, the pivot row's panel entries by shuffles, multipliers and the
// rank-1 update of the remaining panel columns -- no CTA barrier inside a panel. Per panel the
// CTA then (1) forms the pivot rows' trailing entries u_kj = A[p_k][j] after the panel's earlier
// steps (a thread per column), (2) applies the panel's 8 rank-1 updates to its register block
// in step order and writes it back to the shared mirror: 3 barriers per 8 pivots instead of one
// per pivot with a full matrix write-back each. Gauss-Jordan (every non-pivot row eliminated)
// and implicit pivoting as k_lu_solve.
template <int NB>
__global__ void __launch_bounds__(256) k_lu_blocked(const double* __restrict__ S, const double* __restrict__ phi,
                                                     double* __restrict__ dr, double* __restrict__ r, int n, int apply,
                                                     int* __restrict__ status, const double* __restrict__ xrhs, int nx,
                                                     double* __restrict__ xout, const double* __restrict__ Gt, int ldg,
                                                     int n_p) {
  pdl_wait();
  pdl_launch();
  constexpr int D = 16 * NB;
  constexpr int LDF = D + 1;
  constexpr int PW = 8;                // panel width
  constexpr int R = D / 32;            // panel rows per lane
  extern __shared__ double M[];        // [D][LDF] | vhp block [n_q][n_q] | Mul [D][PW] | U [PW][LDF]
  __shared__ int pivrow[D];
  __shared__ double rdiag[D];
  __shared__ int bad_s;
  const int sim = blockIdx.x;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31, warp = tid >> 5;
  const double* Ss = S + (size_t)sim * n * n;
  const int nq = n - n_p;
  double* Vs = M + D * LDF;
  double* Mul = Vs + nq * nq;
  double* Ub = Mul + D * PW;
  const int ncol = n + 1 + nx;         // live columns (matrix, -phi, extra right-hand sides)
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
  if (tid == 0) bad_s = 0;
  cp_async_all_wait();
  __syncthreads();
  // rhs = -phi, S_base + diag(0, vhp); every element is read and rewritten by its own thread
#pragma unroll
  for (int a = 0; a < NB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int i = ty + 16 * a, j = tx + 16 * b;
      double v = M[i * LDF + j];
      if (j == n) v = -v;
      if (Gt && i >= n_p && j >= n_p && i < n && j < n) v += Vs[(j - n_p) * nq + (i - n_p)];
      M[i * LDF + j] = v;
    }
  // the panel warp's rows lane + 32 u: pivot already (rows >= n never are)
  bool used[R];
#pragma unroll
  for (int u = 0; u < R; ++u) used[u] = lane + 32 * u >= n;
  __syncthreads();
#ifdef LU_TRACE
  if (tid == 0) g_lu_trace[0] = clock64();
#endif
  for (int c0 = 0; c0 < n; c0 += PW) {
    const int kw = min(PW, n - c0);
#ifdef LU_TRACE
    if (tid == 0) g_lu_trace[1 + 4 * (c0 / PW)] = clock64();
#endif
    if (warp == 0) {
      // ---- panel: pivots c0 .. c0 + kw - 1 in registers, no CTA barrier
      double pv[R][PW];
#pragma unroll
      for (int u = 0; u < R; ++u)
#pragma unroll
        for (int c = 0; c < PW; ++c) pv[u][c] = M[(lane + 32 * u) * LDF + c0 + c];
      bool bad = false;
#pragma unroll
      for (int kk = 0; kk < PW; ++kk) {
        if (kk >= kw || bad) break;
        double best = -1.0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const double v = fabs(pv[u][kk]);
          if (!used[u] && v > best) { best = v; bi = lane + 32 * u; }
        }
        // exact argmax of |a_ik| over unused rows, lowest row on ties (LAPACK idamax order)
        const unsigned long long key = (best >= 0.0) ? (unsigned long long)__double_as_longlong(best) : 0ull;
        const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        // 1 / |p| from the reduced key, overlapping the row-index reduction and the shuffles
        const double rabs = recip_fast(__hiloint2double((int)mhi, (int)mlo));
        const int piv = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)bi : 0x7fffffffu);
        if (!(mhi | mlo) || piv >= n) { bad = true; break; }
        const int up = piv >> 5, lp = piv & 31;
#pragma unroll
        for (int u = 0; u < R; ++u) used[u] = used[u] || (u == up && lane == lp);
        // the pivot row's panel entries kk .. kw-1 from their owner lane
        double prow[PW];
#pragma unroll
        for (int c = kk; c < PW; ++c) {
          double mine = pv[0][c];
#pragma unroll
          for (int u = 1; u < R; ++u) mine = (up == u) ? pv[u][c] : mine;
          prow[c] = __shfl_sync(0xffffffffu, mine, lp);
        }
        const double rp = copysign(rabs, prow[kk]);  // == recip_fast(p): the Newton steps are odd in p
        if (lane == 0) {
          pivrow[c0 + kk] = piv;
          rdiag[c0 + kk] = rp;
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
          const int i = lane + 32 * u;
          const double m = (i < n && i != piv) ? pv[u][kk] * rp : 0.0;
          Mul[i * PW + kk] = m;
#pragma unroll
          for (int c = kk + 1; c < PW; ++c) pv[u][c] = fma(-m, prow[c], pv[u][c]);
        }
      }
      if (bad && lane == 0) bad_s = 1;
    }
    __syncthreads();
#ifdef LU_TRACE
    if (tid == 0) g_lu_trace[2 + 4 * (c0 / PW)] = clock64();
#endif
    if (bad_s) break;
    // ---- pivot rows' trailing entries: u_kj = A[p_k][j] after the panel's steps < k
    // (all loads issued before the chain and the stores)
    const int jlo = c0 + kw;
    if (jlo + tid < ncol) {
      const int j = jlo + tid;
      int pk[PW];
      double raw[PW], mk[PW][PW];
#pragma unroll
      for (int kk = 0; kk < PW; ++kk) pk[kk] = kk < kw ? pivrow[c0 + kk] : 0;
#pragma unroll
      for (int kk = 0; kk < PW; ++kk) {
        raw[kk] = M[pk[kk] * LDF + j];
#pragma unroll
        for (int k2 = 0; k2 < kk; ++k2) mk[kk][k2] = Mul[pk[kk] * PW + k2];
      }
      double u[PW];
#pragma unroll
      for (int kk = 0; kk < PW; ++kk) {
        double v = raw[kk];
#pragma unroll
        for (int k2 = 0; k2 < kk; ++k2) v = fma(-mk[kk][k2], u[k2], v);
        u[kk] = v;
      }
#pragma unroll
      for (int kk = 0; kk < PW; ++kk)
        if (kk < kw) Ub[kk * LDF + j] = u[kk];
    }
    __syncthreads();
#ifdef LU_TRACE
    if (tid == 0) g_lu_trace[3 + 4 * (c0 / PW)] = clock64();
#endif
    // ---- the panel's rank-1 updates on every row's trailing block (shared matrix), in step order;
    // the thread's u values and multipliers are loaded once, before any store
    {
      // NB <= 4: every operand of the thread's 4 x 4 block in registers; wider blocks (n > 63)
      // row by row to stay within the register file
      constexpr int AR = NB <= 4 ? NB : 1;
      double ub[NB][PW];
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int j = tx + 16 * b;
#pragma unroll
        for (int kk = 0; kk < PW; ++kk) ub[b][kk] = (kk < kw && 16 * b + 15 >= jlo) ? Ub[kk * LDF + j] : 0.0;
      }
#pragma unroll
      for (int a0 = 0; a0 < NB; a0 += AR) {
        double m[AR][PW], v[AR][NB];
#pragma unroll
        for (int a = 0; a < AR; ++a) {
          const int i = ty + 16 * (a0 + a);
#pragma unroll
          for (int kk = 0; kk < PW; ++kk) m[a][kk] = kk < kw ? Mul[i * PW + kk] : 0.0;
#pragma unroll
          for (int b = 0; b < NB; ++b) v[a][b] = (16 * b + 15 >= jlo) ? M[i * LDF + tx + 16 * b] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < AR; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if (16 * b + 15 < jlo) continue;  // column block eliminated (uniform)
#pragma unroll
            for (int kk = 0; kk < PW; ++kk) v[a][b] = fma(-m[a][kk], ub[b][kk], v[a][b]);
          }
#pragma unroll
        for (int a = 0; a < AR; ++a)
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            const int j = tx + 16 * b;
            if (j >= jlo && j < ncol) M[(ty + 16 * (a0 + a)) * LDF + j] = v[a][b];
          }
      }
    }
    __syncthreads();
  }
  if (bad_s) {
    if (tid == 0) status[sim] = 1;
    return;
  }
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
