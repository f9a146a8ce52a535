// Retired LU variants (bitwise equal to k_lu_solve, measured slower on B200).
// Not compiled into libnlrom_b200.so.
#pragma once
#include "../../../paper_2102_11026_b200/csrc/solve_kernels.cuh"
namespace nlrom {
// Look-ahead form of k_lu_solve (same arithmetic, same pivots, bitwise equal results): the
// pivot search and reciprocal of step k + 1 run before step k's barrier on a register copy of
// column k + 1 that every warp updates itself, so the barrier -> argmax -> 1/p -> update chain
// of the row-block kernel loses its argmax and 1/p legs. Column k + 1 as of step k - 1 is read
// from a double-buffered side copy (nxt) written by its owners, never from M, which the owners
// overwrite during step k.
template <int NB>
__global__ void __launch_bounds__(256) k_lu_la(const double* __restrict__ S, const double* __restrict__ phi,
                                                   double* __restrict__ dr, double* __restrict__ r, int n, int apply,
                                                   int* __restrict__ status, const double* __restrict__ xrhs, int nx,
                                                   double* __restrict__ xout, const double* __restrict__ Gt, int ldg,
                                                   int n_p) {
  // every input waits: in a captured graph the event edge from the side branch (S_base, phi)
  // into this PDL launch is programmatic too, so nothing is complete before the wait
  pdl_wait();
  pdl_launch();
  constexpr int D = 16 * NB;           // covered rows / columns (n + 1 <= D)
  constexpr int LDF = D + 1;
  extern __shared__ double M[];        // [D][LDF] | vhp block [n_q][n_q]
  __shared__ int pivrow[D];
  __shared__ double rdiag[D];
  __shared__ double nxt[2][D];          // column k + 1 as of the end of step k - 1 (slot (k + 1) & 1)
  const int sim = blockIdx.x;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31;
  const double* Ss = S + (size_t)sim * n * n;
  const int nq = n - n_p;
  double* Vs = M + D * LDF;            // vhp[k][i] = G_t[2k+1][i] (k_reduce_S without G_t built S_base)
  // stage [S | phi | extra rhs] and the vhp block with async copies (one round trip for all)
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
      if (j == n) v = -v;  // rhs = -phi
      if (Gt && i >= n_p && j >= n_p && i < n && j < n) v += Vs[(j - n_p) * nq + (i - n_p)];  // S_base + diag(0, vhp)
      A[a][b] = v;
    }
  __syncthreads();
  // the shared copy holds the full matrix from here on (the first pivot row is read from it)
#pragma unroll
  for (int a = 0; a < NB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      M[(ty + 16 * a) * LDF + tx + 16 * b] = A[a][b];
      if (tx + 16 * b == 1) nxt[1][ty + 16 * a] = A[a][b];
    }
  // rows >= n are never pivots
  unsigned long long used_lo = 0ull, used_hi = 0ull;  // rows 0..63, 64..127
  for (int i = n; i < D; ++i) {
    if (i < 64) used_lo |= 1ull << i;
    else used_hi |= 1ull << (i - 64);
  }
  auto is_used = [&](int i) -> bool {
    return i < 64 ? ((used_lo >> i) & 1ull) : ((used_hi >> (i - 64)) & 1ull);
  };
  bool bad = false;
  __syncthreads();
#ifdef LU_CYCLES
  if (tid == 0) g_lu_cycles[0] = clock64();
#endif
  // argmax of |c| over the unused rows lane + 32u (LAPACK idamax ties: lowest row); the pivot
  // value comes back from its owner lane, bitwise the element the row-block update stores
  constexpr int U = D / 32;
  auto find_pivot = [&](const double (&c)[U], int& piv, double& pv) -> bool {
    double best = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = lane + 32 * u;
      if (!is_used(i)) {
        const double v = fabs(c[u]);
        if (v > best) { best = v; bi = i; }
      }
    }
    const unsigned long long key = (best >= 0.0) ? (unsigned long long)__double_as_longlong(best) : 0ull;
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    piv = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)bi : 0x7fffffffu);
    if (!(mhi | mlo) || piv >= n) return false;
    double sel = c[0];
#pragma unroll
    for (int u = 1; u < U; ++u)
      if ((piv >> 5) == u) sel = c[u];
    pv = __shfl_sync(0xffffffffu, sel, piv & 31);
    if (piv < 64) used_lo |= 1ull << piv;
    else used_hi |= 1ull << (piv - 64);
    return true;
  };
  double c0[U];
#pragma unroll
  for (int u = 0; u < U; ++u) c0[u] = M[(lane + 32 * u) * LDF];
  int piv;
  double rp;
  {
    double pv;
    if (n > 0 && !find_pivot(c0, piv, pv)) bad = true;
    else rp = recip_fast(pv);
  }
  for (int k = 0; k < n && !bad; ++k) {
    // step k's pivot (piv, rp) and column k (c0) were found during step k - 1: every warp
    // updates column k + 1 for its rows itself (the same fma the row-block owners do) and
    // searches step k + 1's pivot before the barrier instead of after it
    if (tid == 0) {
      pivrow[k] = piv;
      rdiag[k] = rp;
    }
    const bool ahead = k + 1 < n;
    const double* prow = M + piv * LDF;
    double pr[NB], l[NB], c1[U];
    bool act[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) pr[b] = prow[tx + 16 * b];
#pragma unroll
    for (int a = 0; a < NB; ++a) {
      const int i = ty + 16 * a;
      act[a] = (i < n) && (i != piv);  // Gauss-Jordan: every row but the pivot row is eliminated
      l[a] = M[i * LDF + k];
    }
    const double p1 = ahead ? prow[k + 1] : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) c1[u] = nxt[(k + 1) & 1][lane + 32 * u];
    // step k + 1's pivot chain first: the trailing update below is independent of it and
    // fills the REDUX / shuffle / reciprocal latencies
    int piv_n = piv;
    double rp_n = rp;
    if (ahead) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = lane + 32 * u;
        if (i < n && i != piv) c1[u] = fma(-(c0[u] * rp), p1, c1[u]);
        c0[u] = c1[u];
      }
      double pv;
      if (!find_pivot(c0, piv_n, pv)) { bad = true; break; }
      rp_n = recip_fast(pv);
    }
#pragma unroll
    for (int a = 0; a < NB; ++a) {
      const int i = ty + 16 * a;
      const double la = l[a] * rp;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        if (NB > 4 && 16 * b + 15 <= k) continue;  // column block already eliminated (uniform)
        const int j = tx + 16 * b;
        if (act[a] && j > k) {
          A[a][b] = fma(-la, pr[b], A[a][b]);
          M[i * LDF + j] = A[a][b];
        }
        if (j == k + 2) nxt[k & 1][i] = A[a][b];
      }
    }
    piv = piv_n;
    rp = rp_n;
    __syncthreads();
  }
#ifdef LU_CYCLES
  if (tid == 0) g_lu_cycles[1] = clock64();
#endif
  if (bad) {
    if (tid == 0) status[sim] = 1;
    return;
  }
  // Gauss-Jordan: the pivot rows form a diagonal system, x_k = rhs[piv_k] / a[piv_k][k]
  // (no sequential back substitution). Column n is -phi, columns n+1.. the extra right-hand sides.
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

// Column-cyclic variant for n <= 64 and n + 1 + nx <= 72 columns: warp w owns columns
// w, w + 8, ...; lane holds rows lane and lane + 32 of them in registers. Pivot step k is
// produced by ONE warp (the owner of column k: pivot search with REDUX, reciprocal,
// multipliers into shared memory) and consumed by the other seven through a named barrier
// (bar.arrive / bar.sync, two alternating ids), so a step costs one producer->consumer
// hand-off instead of a full CTA barrier plus redundant pivot searches in every warp.
// Same arithmetic as k_lu_solve (m = a_ik / a_pk, a_ij -= m a_pj on unused rows).

constexpr int LUC_CPW = 9, LUC_D = 64, LUC_LDF = 8 * LUC_CPW + 1;
#ifdef LU_TRACE
__device__ long long g_lu_trace[80];
__device__ long long g_lu_trace2[16];
#define LU_MARK(i) \
  if (threadIdx.x == 0) g_lu_trace[i] = clock64();
#define LU_MARK2(w, i) \
  if (threadIdx.x == 32 * (w)) g_lu_trace2[i] = clock64();
#else
#define LU_MARK(i)
#define LU_MARK2(w, i)
#endif
inline size_t luc_smem_bytes() { return (size_t)LUC_D * LUC_LDF * 8; }

__global__ void __launch_bounds__(256) k_lu_cols(const double* __restrict__ S, const double* __restrict__ phi,
                                                 double* __restrict__ dr, double* __restrict__ r, int n, int apply,
                                                 int* __restrict__ status, const double* __restrict__ xrhs, int nx,
                                                 double* __restrict__ xout, const double* __restrict__ Gt, int ldg,
                                                 int n_p) {
  LU_MARK(0);
  pdl_wait();
  pdl_launch();
  LU_MARK(1);
  constexpr int CPW = LUC_CPW, D = LUC_D, LDF = LUC_LDF;
  extern __shared__ double M[];  // [D][LDF]: eliminated matrix for the back substitution
  __shared__ double mul[2][D];
  __shared__ int pivrow[D];
  __shared__ double rdiag[D];
  const unsigned FULL = 0xffffffffu;
  const int sim = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(FULL, tid >> 5, 0);  // provably warp-uniform
  const int ncol = n + 1 + nx;
  const double* Ss = S + (size_t)sim * n * n;
  double A[CPW][2];
#pragma unroll
  for (int j = 0; j < CPW; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = warp + 8 * j, row = lane + 32 * h;
      double v = 0.0;
      if (row < n) {
        if (c < n) {
          v = Ss[(size_t)row * n + c];
          if (Gt && row >= n_p && c >= n_p) v += Gt[((size_t)sim * 2 * (n - n_p) + 2 * (c - n_p) + 1) * ldg + (row - n_p)];
        }
        else if (c == n) v = -phi[(size_t)sim * n + row];
        else if (c < ncol) v = xrhs[((size_t)sim * nx + (c - n - 1)) * n + row];
      }
      A[j][h] = v;
    }
  bool used0 = lane >= n, used1 = lane + 32 >= n;
  bool bad = false;
  LU_MARK(2);
  // pivot step k by its owner warp: search column k (slot k >> 3), publish multipliers and the
  // pivot row through shared memory, release the consumers of barrier 1 + (k & 1)
  auto produce = [&](int k, int& piv, double& m0, double& m1) -> bool {
    const int jk = k >> 3;
    if (k == 11) LU_MARK2(3, 3);
    double ak0 = 0.0, ak1 = 0.0;
#pragma unroll
    for (int j = 0; j < CPW; ++j)
      if (j == jk) { ak0 = A[j][0]; ak1 = A[j][1]; }
    const double v0 = used0 ? -1.0 : fabs(ak0), v1 = used1 ? -1.0 : fabs(ak1);
    double best = v0;
    int bi = lane;
    if (v1 > best) { best = v1; bi = lane + 32; }
    const unsigned long long key = (best >= 0.0) ? (unsigned long long)__double_as_longlong(best) : 0ull;
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_max_sync(FULL, hi);
    const unsigned mlo = __reduce_max_sync(FULL, hi == mhi ? lo : 0u);
    piv = (int)__reduce_min_sync(FULL, (hi == mhi && lo == mlo) ? (unsigned)bi : 0x7fffffffu);
    if (k == 11) LU_MARK2(3, 4);
    const bool ok = (mhi | mlo) && piv < n;
    const double pv = __shfl_sync(FULL, piv < 32 ? ak0 : ak1, piv & 31);  // convergent: every lane
    if (ok) {
      const double rp = 1.0 / pv;
      if (k == 11 && rp != 12345.0) LU_MARK2(3, 5);
      // the pivot row is marked used by the caller once its step k-1 updates are done
      m0 = (used0 || piv == lane) ? 0.0 : ak0 * rp;
      m1 = (used1 || piv == lane + 32) ? 0.0 : ak1 * rp;
      mul[k & 1][lane] = m0;
      mul[k & 1][lane + 32] = m1;
      if (lane == 0) {
        pivrow[k] = piv;
        rdiag[k] = rp;
      }
    } else if (lane == 0) {
      pivrow[k] = -1;
    }
    if (k == 11) LU_MARK2(3, 6);
    named_bar_arrive(1 + (k & 1), 256);
    return ok;
  };
  // column update of one owned slot j for pivot step k (shuffle executed by the whole warp)
  auto update = [&](int j, int piv, double m0, double m1, bool on) {
    double src = 0.0;
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj)
      if (jj == j) src = (piv < 32) ? A[jj][0] : A[jj][1];
    const double pr = __shfl_sync(FULL, src, piv & 31);
#pragma unroll
    for (int jj = 0; jj < CPW; ++jj)
      if (on && jj == j) {
        if (!used0) A[jj][0] = fma(-m0, pr, A[jj][0]);
        if (!used1) A[jj][1] = fma(-m1, pr, A[jj][1]);
      }
  };
  int piv = 0;
  double m0 = 0.0, m1 = 0.0;
  if (warp == 0 && n > 0) {
    if (!produce(0, piv, m0, m1)) bad = true;
    if (piv == lane) used0 = true;
    if (piv == lane + 32) used1 = true;
  }
  for (int k = 0; k < n && !bad; ++k) {
    LU_MARK(8 + k);
    if (warp != (k & 7)) {  // consumer of step k (the owner already holds piv, m0, m1)
      if (k == 10) LU_MARK2(3, 0);
      named_bar_sync(1 + (k & 1), 256);
      if (k == 10) LU_MARK2(3, 1);
      piv = pivrow[k];
      if (piv < 0) { bad = true; break; }
      if (piv == lane) used0 = true;
      if (piv == lane + 32) used1 = true;
      m0 = mul[k & 1][lane];
      m1 = mul[k & 1][lane + 32];
    }
    const int next = k + 1;
    // this warp's first owned column after k: for the owner of k + 1 it IS column k + 1
    const int j1 = (k >= warp) ? ((k - warp) >> 3) + 1 : 0;
    const int c1 = warp + 8 * j1;
    update(j1, piv, m0, m1, c1 < ncol);
    if (k == 10) LU_MARK2(3, 2);
    int piv_n = 0;
    double m0_n = 0.0, m1_n = 0.0;
    const bool owner_next = next < n && warp == (next & 7);
    if (owner_next && !produce(next, piv_n, m0_n, m1_n)) bad = true;  // look-ahead: publish step k + 1
#pragma unroll
    for (int j = 0; j < CPW; ++j) {
      const int c = warp + 8 * j;
      const double pr = __shfl_sync(FULL, piv < 32 ? A[j][0] : A[j][1], piv & 31);
      if (j > j1 && c < ncol) {
        if (!used0) A[j][0] = fma(-m0, pr, A[j][0]);
        if (!used1) A[j][1] = fma(-m1, pr, A[j][1]);
      }
    }
    const int jskip = owner_next ? 1 : -1;
    if (jskip >= 0) {
      piv = piv_n;
      m0 = m0_n;
      m1 = m1_n;
      if (piv == lane) used0 = true;
      if (piv == lane + 32) used1 = true;
    }
  }
  LU_MARK(3);
  __syncthreads();
  LU_MARK(4);
  if (bad) {
    if (tid == 0) status[sim] = 1;
    return;
  }
#pragma unroll
  for (int j = 0; j < CPW; ++j) {
    const int c = warp + 8 * j;
    if (c < ncol) {
      M[lane * LDF + c] = A[j][0];
      M[(lane + 32) * LDF + c] = A[j][1];
    }
  }
  __syncthreads();
  if (warp <= nx) {  // back substitution: warp 0 for -phi, warp w for extra right-hand side w
    const int col = n + warp;
    constexpr int NU = 2;
    double bv[NU];
    const double* rowp[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int t = lane + 32 * u;
      rowp[u] = M + (t < n ? pivrow[t] : 0) * LDF;
      bv[u] = (t < n) ? rowp[u][col] : 0.0;
    }
#pragma unroll 4
    for (int t = n - 1; t >= 0; --t) {
      const int owner = t & 31, slot = t >> 5;
      const double rd = rdiag[t];
      double uc[NU];
#pragma unroll
      for (int u = 0; u < NU; ++u) uc[u] = rowp[u][t];
      double bt = (slot == 0) ? bv[0] : bv[1];
      bt = __shfl_sync(FULL, bt, owner);
      const double xt = bt * rd;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const int tt = lane + 32 * u;
        if (tt < t) bv[u] = fma(-uc[u], xt, bv[u]);
        else if (tt == t) bv[u] = xt;
      }
    }
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int t = lane + 32 * u;
      if (t < n) {
        if (warp == 0) {
          dr[(size_t)sim * n + t] = bv[u];
          if (apply) r[(size_t)sim * n + t] += bv[u];
        } else {
          xout[((size_t)sim * nx + warp - 1) * n + t] = bv[u];
        }
      }
    }
    if (tid == 0) status[sim] = 0;
  }
  LU_MARK(5);
}

}  // namespace nlrom
