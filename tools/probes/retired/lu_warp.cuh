// Warp-register LU-pp solve of the Eq. 11 Newton system for n <= 64
// unknowns and n + 1 + nx <= 32 NW augmented columns: cfg1 / cfg4 / cfg5 need one warp,
// cfg2 (n = 60) two. Larger systems (cfg3 corners) use the row-block k_lu_solve.
//
// Warp w owns columns [32w, 32w + 32) of [S | -phi | extra rhs]; each lane holds rows lane
// and lane + 32 of them in registers (64 doubles). Pivot step k is produced by the owner
// warp of column k entirely inside that warp -- exact argmax by integer REDUX on the IEEE
// bits (lowest row on ties, as LAPACK idamax), pivot-row values by shuffles, fast reciprocal
// -- with no CTA-wide barrier. The producer publishes the pivot row and the 64 multipliers of
// step k to shared memory and arrives on mbarrier k; the warps to its right consume the steps
// in order as they come (every step has its own slot, so a consumer never blocks the
// producer). When a warp has produced its 32 columns, the next warp -- which has consumed
// every earlier step meanwhile -- produces the following ones.
//
// Same algorithm and arithmetic as k_lu_solve (Gauss-Jordan form: every row but the pivot
// row is eliminated, x_k = rhs[piv_k] / a[piv_k][k]; m = a_ik * (1 / a_pk),
// a_ij = fma(-m, a_pj, a_ij)), so the two kernels agree bit for bit.
#pragma once
#include "../../../paper_2102_11026_b200/csrc/solve_kernels.cuh"  // recip_fast, cp_async8, mbarrier helpers

namespace nlrom {

constexpr int LUW_MAXN = 64;
inline int luw_warps(int n, int nx) { return (n + 1 + nx + 31) / 32; }
inline size_t luw_smem_bytes(int nw, int nq) {
  return (size_t)(64 * (32 * nw + 1) + 64 * 64 + 64) * 8 + (size_t)nq * nq * 8 + 64 * 8 + 64 * 4 + 16;
}

template <int NW>
__global__ void __launch_bounds__(256) k_lu_warp(const double* __restrict__ S, const double* __restrict__ phi,
                                                  double* __restrict__ dr, double* __restrict__ r, int n, int apply,
                                                  int* __restrict__ status, const double* __restrict__ xrhs, int nx,
                                                  double* __restrict__ xout, const double* __restrict__ Gt, int ldg,
                                                  int n_p) {
  pdl_wait();  // every input comes from earlier grids (see k_lu_solve)
  pdl_launch();
  constexpr int LDF = 32 * NW + 1;  // odd: the lanes reading one column hit distinct banks
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) double sm[];
  double* M = sm;                   // [64][LDF] staging, later the rhs rows for the solve
  double* Lb = M + 64 * LDF;        // [step][64 rows] multipliers
  double* rdiag = Lb + 64 * 64;     // [step] 1 / pivot
  const int nq = n - n_p;
  double* Vs = rdiag + 64;          // vhp[k][i] = G_t[2k+1][i]
  uint64_t* bars = reinterpret_cast<uint64_t*>(Vs + (Gt ? nq * nq : 0));
  int* pivrow = reinterpret_cast<int*>(bars + 64);
  __shared__ int bad_flag;
  const int sim = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ncol = n + 1 + nx;
  const double* Ss = S + (size_t)sim * n * n;
  for (int idx = tid; idx < 64 * 32 * NW; idx += blockDim.x) {
    const int i = idx / (32 * NW), j = idx % (32 * NW);
    double* dst = M + i * LDF + j;
    if (i < n && j < n) cp_async8(dst, Ss + (size_t)i * n + j);
    else if (i < n && j == n) cp_async8(dst, phi + (size_t)sim * n + i);
    else if (i < n && j > n && j < ncol) cp_async8(dst, xrhs + ((size_t)sim * nx + (j - n - 1)) * n + i);
    else *dst = 0.0;
  }
  if (Gt)
    for (int idx = tid; idx < nq * nq; idx += blockDim.x) {
      const int k = idx / nq, i = idx % nq;
      cp_async8(Vs + idx, Gt + ((size_t)sim * 2 * nq + 2 * k + 1) * ldg + i);
    }
  if (tid < 64) mbar_init(bars + tid, 32);
  if (tid == 0) bad_flag = 0;
  cp_async_all_wait();
  __syncthreads();
  double A0[32], A1[32];
  const int c0 = 32 * warp;
  if (warp < NW) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const int j = c0 + c;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        double v = M[i * LDF + j];
        if (j == n) v = -v;  // rhs = -phi
        if (Gt && i >= n_p && j >= n_p && i < n && j < n) v += Vs[(j - n_p) * nq + (i - n_p)];  // + diag(0, vhp)
        if (h == 0) A0[c] = v;
        else A1[c] = v;
      }
    }
  }
  __syncthreads();  // the last CTA-wide barrier: M is free from here on
  if (warp >= NW) return;
  bool used0 = lane >= n, used1 = lane + 32 >= n;  // rows >= n are never pivots
  const bool consumers = warp + 1 < NW;
  // ---- consume the steps produced by the warps to the left (all of this warp's columns are > k)
  const int kc = min(c0, n);
  for (int k = 0; k < kc; ++k) {
    mbar_wait_cta(bars + k, 0);
    if (*reinterpret_cast<volatile int*>(&bad_flag)) return;
    const int piv = pivrow[k];
    const double la0 = Lb[k * 64 + lane], la1 = Lb[k * 64 + 32 + lane];
    const int pl = piv & 31;
    const bool ps = piv >= 32;
    if (lane == pl) {
      if (ps) used1 = true;
      else used0 = true;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double pj = __shfl_sync(FULL, ps ? A1[j] : A0[j], pl);
      A0[j] = fma(-la0, pj, A0[j]);
      A1[j] = fma(-la1, pj, A1[j]);
    }
  }
  // ---- produce the steps of this warp's columns. A rolled loop (the code runs once per
  // launch from a cold instruction cache, so it has to be small): the pivot column is always
  // register 0 and the update writes column j + 1 into register j, so the remaining columns
  // shift left by one per step at no extra instruction cost.
  int sh = 0;  // columns consumed by this warp's own pivot steps
  if (c0 < n) {
    const int kend = min(n, c0 + 32);
#pragma unroll 1
    for (int k = c0; k < kend; ++k, ++sh) {
      double best = -1.0;
      int bi = 0x7fffffff;
      if (!used0) {
        const double v = fabs(A0[0]);
        if (v > best) { best = v; bi = lane; }
      }
      if (!used1) {
        const double v = fabs(A1[0]);
        if (v > best) { best = v; bi = lane + 32; }
      }
      const unsigned long long key = (best >= 0.0) ? (unsigned long long)__double_as_longlong(best) : 0ull;
      const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
      const unsigned mhi = __reduce_max_sync(FULL, hi);
      const unsigned mlo = __reduce_max_sync(FULL, hi == mhi ? lo : 0u);
      const int piv = (int)__reduce_min_sync(FULL, (hi == mhi && lo == mlo) ? (unsigned)bi : 0x7fffffffu);
      if (!(mhi | mlo) || piv >= n) {  // zero (or NaN) pivot column: singular
        if (lane == 0) {
          bad_flag = 1;
          status[sim] = 1;
        }
        __syncwarp();
        if (consumers)
          for (int k2 = k; k2 < n; ++k2) mbar_arrive(bars + k2);  // wake the consumers: they see bad_flag
        return;
      }
      const int pl = piv & 31;
      const bool ps = piv >= 32;
      const double pk = __shfl_sync(FULL, ps ? A1[0] : A0[0], pl);
      const double rp = recip_fast(pk);
      const bool own0 = lane == pl && !ps, own1 = lane == pl && ps;
      used0 |= own0;
      used1 |= own1;
      const double la0 = own0 ? 0.0 : A0[0] * rp;  // Gauss-Jordan: every row but the pivot row
      const double la1 = own1 ? 0.0 : A1[0] * rp;
      if (lane == 0) {
        pivrow[k] = piv;
        rdiag[k] = rp;
      }
      if (consumers) {
        Lb[k * 64 + lane] = la0;
        Lb[k * 64 + 32 + lane] = la1;
        mbar_arrive(bars + k);  // release: pivrow / Lb of step k
      }
#pragma unroll
      for (int j = 0; j < 31; ++j) {
        const double pj = __shfl_sync(FULL, ps ? A1[j + 1] : A0[j + 1], pl);
        A0[j] = fma(-la0, pj, A0[j + 1]);
        A1[j] = fma(-la1, pj, A1[j + 1]);
      }
      A0[31] = 0.0;
      A1[31] = 0.0;
    }
  }
  // ---- solve: the warps holding right-hand-side columns (they have applied all n steps);
  // column j now sits in register j - c0 - sh
  if (c0 + 32 <= n || c0 >= ncol) return;
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const int j = c0 + sh + c;
    if (j >= n && j < ncol) {
      M[lane * LDF + j] = A0[c];
      M[(lane + 32) * LDF + j] = A1[c];
    }
  }
  __syncwarp();
  const int jlo = max(n, c0), jhi = min(ncol, c0 + 32);
  for (int t = lane; t < n * (jhi - jlo); t += 32) {
    const int kk = t % n, j = jlo + t / n;
    const double x = M[pivrow[kk] * LDF + j] * rdiag[kk];
    if (j == n) {
      dr[(size_t)sim * n + kk] = x;
      if (apply) r[(size_t)sim * n + kk] += x;
    } else {
      xout[((size_t)sim * nx + (j - n - 1)) * n + kk] = x;
    }
  }
  if (lane == 0 && jlo == n) status[sim] = 0;
}

}  // namespace nlrom
