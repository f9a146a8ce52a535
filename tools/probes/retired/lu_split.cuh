// Split Gauss-Jordan LU-pp of the Eq. 11 Newton system (n <= 64) around the vhp block.
//
// S = S_base + diag(0, V): V (the vhp, n_q x n_q) only touches the columns n_p .. n-1, so the
// first n_p pivot steps of LU with partial pivoting (pivot search in columns 0 .. n_p-1 over all
// rows) are the same for S_base and S, and by linearity the transformed trailing columns are
//   T(S)[:, n_p:] = T(S_base)[:, n_p:] + Z[:, n_p:] V,   Z = the accumulated row operations.
// k_lu_front runs those n_p steps on [S_base | -phi | extra rhs | e_{n_p} .. e_{n-1}] (the unit
// columns accumulate Z[:, n_p:]) on a side branch while the vhp chain still runs; k_lu_back adds
// Z[:, n_p:] V once V exists and finishes the n_q remaining steps, then x_k = rhs[piv_k] / a_pk.
// Same pivot search (exact argmax on the IEEE bits, lowest row on ties), same multipliers and
// updates as k_lu_solve; only the V contribution is summed in a different order (roundoff).
// Thread (ty, tx) of 256 owns rows ty + 16a (a < 4) and columns tx + 16b (b < NBC).
#pragma once
#include "../../../paper_2102_11026_b200/csrc/solve_kernels.cuh"

namespace nlrom {

struct LuSplitArgs {
  int n, n_p, nx, FC;       // FC = n + 1 + nx + n_q columns of the front matrix
  const double* S;          // front: S_base (n_sims, n, n)
  const double* phi;        // front: (n_sims, n)
  const double* xrhs;       // front: (n_sims, nx, n) extra right-hand sides
  double* F;                // front out / back in: (n_sims, n, FC)
  int* piv;                 // (n_sims, n) pivot rows per step
  double* rdiag;            // (n_sims, n) 1 / pivot per step
  int* flag;                // (n_sims) front found a zero pivot
  const double* Gt;         // back: vhp[k][i] = Gt[2k+1][i]
  int ldg;
  double* dr;
  double* r;
  int apply;
  int* status;
  double* xout;             // back: (n_sims, nx, n)
};

#ifdef LU_CYCLES
__device__ long long g_lus_cycles[8];  // tools/probes/lu_split_probe.cu
#define LUS_MARK(i) \
  if (threadIdx.x == 0 && blockIdx.x == 0) g_lus_cycles[i] = clock64();
#else
#define LUS_MARK(i)
#endif

template <int NBC>
struct LuSplitPlan {
  static constexpr int C = 16 * NBC, LDF = C + 1;
  static size_t bytes(int nq) { return (size_t)64 * LDF * 8 + (size_t)nq * nq * 8 + 64 * 12 + 16; }
};

// The pivot steps k in [k0, k1) with the pivot column at local column k - coff.
// Returns false on a zero / NaN pivot column (singular).
template <int NBC>
__device__ __forceinline__ bool lu_gj_steps(double (&A)[4][NBC], double* M, int k0, int k1, int coff, int n,
                                            unsigned long long& used, int* pivrow, double* rdg) {
  constexpr int LDF = LuSplitPlan<NBC>::LDF;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31;
  for (int k = k0; k < k1; ++k) {
    const int kc = k - coff;
    double best = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int i = lane + 32 * u;
      if (!((used >> i) & 1ull)) {
        const double v = fabs(M[i * LDF + kc]);
        if (v > best) { best = v; bi = i; }
      }
    }
    const unsigned long long key = (best >= 0.0) ? (unsigned long long)__double_as_longlong(best) : 0ull;
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    const int piv = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)bi : 0x7fffffffu);
    if (!(mhi | mlo) || piv >= n) return false;
    used |= 1ull << piv;
    const double rp = recip_fast(M[piv * LDF + kc]);
    if (tid == 0) {
      pivrow[k] = piv;
      rdg[k] = rp;
    }
    const double* prow = M + piv * LDF;
    double pr[NBC], l[4];
    bool act[4];
#pragma unroll
    for (int b = 0; b < NBC; ++b) pr[b] = prow[tx + 16 * b];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = ty + 16 * a;
      act[a] = (i < n) && (i != piv);
      l[a] = M[i * LDF + kc];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = ty + 16 * a;
      const double la = l[a] * rp;
#pragma unroll
      for (int b = 0; b < NBC; ++b) {
        const int j = tx + 16 * b;
        if (act[a] && j > kc) {
          A[a][b] = fma(-la, pr[b], A[a][b]);
          M[i * LDF + j] = A[a][b];
        }
      }
    }
    __syncthreads();
  }
  return true;
}

template <int NBC>
__global__ void __launch_bounds__(256) k_lu_front(LuSplitArgs a) {
  pdl_wait();  // S_base, phi from earlier grids
  pdl_launch();
  constexpr int LDF = LuSplitPlan<NBC>::LDF, C = LuSplitPlan<NBC>::C;
  extern __shared__ __align__(16) double M[];  // [64][LDF]
  __shared__ int pivrow[64];
  __shared__ double rdg[64];
  const int sim = blockIdx.x, tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int n = a.n, nx = a.nx, ncut = n + 1 + nx;
  const double* Ss = a.S + (size_t)sim * n * n;
  for (int idx = tid; idx < 64 * C; idx += 256) {
    const int i = idx / C, j = idx % C;
    double* dst = M + i * LDF + j;
    if (i < n && j < n) cp_async8(dst, Ss + (size_t)i * n + j);
    else if (i < n && j == n) cp_async8(dst, a.phi + (size_t)sim * n + i);
    else if (i < n && j > n && j < ncut) cp_async8(dst, a.xrhs + ((size_t)sim * nx + (j - n - 1)) * n + i);
    else *dst = (i < n && j >= ncut && j < a.FC && i == a.n_p + (j - ncut)) ? 1.0 : 0.0;
  }
  cp_async_all_wait();
  __syncthreads();
  double A[4][NBC];
#pragma unroll
  for (int aa = 0; aa < 4; ++aa)
#pragma unroll
    for (int b = 0; b < NBC; ++b) {
      const int i = ty + 16 * aa, j = tx + 16 * b;
      double v = M[i * LDF + j];
      if (j == n) v = -v;  // rhs = -phi
      A[aa][b] = v;
    }
  __syncthreads();
#pragma unroll
  for (int aa = 0; aa < 4; ++aa)
#pragma unroll
    for (int b = 0; b < NBC; ++b) M[(ty + 16 * aa) * LDF + tx + 16 * b] = A[aa][b];
  unsigned long long used = n >= 64 ? 0ull : (~0ull << n);  // rows >= n are never pivots
  __syncthreads();
  LUS_MARK(0);
  const bool ok = lu_gj_steps<NBC>(A, M, 0, a.n_p, 0, n, used, pivrow, rdg);
  LUS_MARK(1);
  if (tid == 0) a.flag[sim] = ok ? 0 : 1;
  if (!ok) return;
  // the transformed matrix (rows < n) and the first n_p pivots
  double* Fs = a.F + (size_t)sim * n * a.FC;
#pragma unroll
  for (int aa = 0; aa < 4; ++aa)
#pragma unroll
    for (int b = 0; b < NBC; ++b) {
      const int i = ty + 16 * aa, j = tx + 16 * b;
      if (i < n && j < a.FC) Fs[(size_t)i * a.FC + j] = A[aa][b];
    }
  for (int k = tid; k < a.n_p; k += 256) {
    a.piv[(size_t)sim * n + k] = pivrow[k];
    a.rdiag[(size_t)sim * n + k] = rdg[k];
  }
}

template <int NBC>
__global__ void __launch_bounds__(256) k_lu_back(LuSplitArgs a) {
  pdl_wait();  // the front's output, the vhp
  pdl_launch();
  constexpr int LDF = LuSplitPlan<NBC>::LDF, C = LuSplitPlan<NBC>::C;
  extern __shared__ __align__(16) double M[];  // [64][LDF] | V [n_q][n_q] | Z [64][n_q] reuse
  __shared__ int pivrow[64];
  __shared__ double rdg[64];
  const int sim = blockIdx.x, tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const int n = a.n, n_p = a.n_p, nq = n - n_p, nx = a.nx, ncut = n + 1 + nx;
  if (a.flag[sim]) {
    if (tid == 0) a.status[sim] = 1;
    return;
  }
  LUS_MARK(2);
  double* Vs = M + 64 * LDF;  // V[q][c] = vhp(row n_p + q, col n_p + c) = Gt[2c+1][q]
  const double* Fs = a.F + (size_t)sim * n * a.FC;
  // local columns: c < n_q -> column n_p + c; n_q -> rhs; n_q + 1 + x -> extra rhs x
  for (int idx = tid; idx < 64 * C; idx += 256) {
    const int i = idx / C, c = idx % C;
    double* dst = M + i * LDF + c;
    const int j = c < nq ? n_p + c : (c < nq + 1 + nx ? n + (c - nq) : -1);
    if (i < n && j >= 0) cp_async8(dst, Fs + (size_t)i * a.FC + j);
    else *dst = 0.0;
  }
  for (int idx = tid; idx < nq * nq; idx += 256) {
    const int c = idx / nq, q = idx % nq;
    cp_async8(Vs + q * nq + c, a.Gt + ((size_t)sim * 2 * nq + 2 * c + 1) * a.ldg + q);
  }
  for (int k = tid; k < n_p; k += 256) {
    pivrow[k] = a.piv[(size_t)sim * n + k];
    rdg[k] = a.rdiag[(size_t)sim * n + k];
  }
  cp_async_all_wait();
  __syncthreads();
  // T'[:, n_p + c] = T[:, n_p + c] + sum_q Z[:, q] V[q][c]   (Z[:, q] = front column ncut + q)
  double A[4][NBC];
#pragma unroll
  for (int aa = 0; aa < 4; ++aa)
#pragma unroll
    for (int b = 0; b < NBC; ++b) {
      const int i = ty + 16 * aa, c = tx + 16 * b;
      double v = M[i * LDF + c];
      if (i < n && c < nq) {
        const double* Zi = Fs + (size_t)i * a.FC + ncut;
        double s0 = 0.0, s1 = 0.0;
        int q = 0;
        for (; q + 1 < nq; q += 2) {
          s0 = fma(Zi[q], Vs[q * nq + c], s0);
          s1 = fma(Zi[q + 1], Vs[(q + 1) * nq + c], s1);
        }
        if (q < nq) s0 = fma(Zi[q], Vs[q * nq + c], s0);
        v += s0 + s1;
      }
      A[aa][b] = v;
    }
  __syncthreads();
#pragma unroll
  for (int aa = 0; aa < 4; ++aa)
#pragma unroll
    for (int b = 0; b < NBC; ++b) M[(ty + 16 * aa) * LDF + tx + 16 * b] = A[aa][b];
  unsigned long long used = n >= 64 ? 0ull : (~0ull << n);
  for (int k = 0; k < n_p; ++k) used |= 1ull << pivrow[k];
  __syncthreads();
  LUS_MARK(3);
  const bool ok = lu_gj_steps<NBC>(A, M, n_p, n, n_p, n, used, pivrow, rdg);
  LUS_MARK(4);
  if (!ok) {
    if (tid == 0) a.status[sim] = 1;
    return;
  }
  // Gauss-Jordan: x_k = rhs[piv_k] / a[piv_k][k] (rhs columns hold every step's elimination)
  for (int t = tid; t < n * (1 + nx); t += 256) {
    const int kk = t % n, col = t / n;
    const double x = M[pivrow[kk] * LDF + nq + col] * rdg[kk];
    if (col == 0) {
      a.dr[(size_t)sim * n + kk] = x;
      if (a.apply) a.r[(size_t)sim * n + kk] += x;
    } else {
      a.xout[((size_t)sim * nx + col - 1) * n + kk] = x;
    }
  }
  if (tid == 0) a.status[sim] = 0;
  LUS_MARK(5);
}

}  // namespace nlrom
