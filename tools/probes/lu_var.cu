
#include <cstdio>
#include <vector>
#include <random>
#include "../../paper_2102_11026_b200/csrc/solve_kernels.cuh"
using namespace nlrom;
__global__ void k_empty(int* st) { if (threadIdx.x == 0) st[0] = 0; }
template <int NB, int MODE>
__global__ void __launch_bounds__(256) k_lu_var(const double* __restrict__ S, const double* __restrict__ phi,
                                                   double* __restrict__ dr, double* __restrict__ r, int n, int apply,
                                                   int* __restrict__ status) {
  constexpr int D = 16 * NB;           // covered rows / columns (n + 1 <= D)
  constexpr int LDF = D + 1;
  extern __shared__ double M[];        // [D][LDF]
  __shared__ int pivrow[D];
  __shared__ double rdiag[D];
  const int sim = blockIdx.x;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31;
  const double* Ss = S + (size_t)sim * n * n;
  // stage [S | phi] into shared memory with async copies (one round trip for all elements)
  for (int idx = tid; idx < D * D; idx += 256) {
    const int i = idx / D, j = idx % D;
    double* dst = M + i * LDF + j;
    if (i < n && j < n) cp_async8(dst, Ss + (size_t)i * n + j);
    else if (i < n && j == n) cp_async8(dst, phi + (size_t)sim * n + i);
    else *dst = 0.0;
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
      A[a][b] = v;
    }
  __syncthreads();
#pragma unroll
  for (int a = 0; a < NB; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if (tx + 16 * b == n) M[(ty + 16 * a) * LDF + n] = A[a][b];
  if (MODE == 1) { if (tid == 0) status[sim] = (int)A[0][0]; return; }
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
  for (int k = 0; k < n; ++k) {
    // every warp: argmax over the column (rows lane + 32u)
    double best = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int u = 0; u < D / 32; ++u) {
      const int i = lane + 32 * u;
      if (!is_used(i)) {
        const double v = fabs(M[i * LDF + k]);
        if (v > best) { best = v; bi = i; }
      }
    }
    const unsigned long long key = (best >= 0.0) ? (unsigned long long)__double_as_longlong(best) : 0ull;
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    const int piv = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)bi : 0x7fffffffu);
    if (!(mhi | mlo) || piv >= n) { bad = true; break; }
    if (piv < 64) used_lo |= 1ull << piv;
    else used_hi |= 1ull << (piv - 64);
    // one fp64 division per warp (MUFU-based division is slow when every thread issues it)
    double rp = 0.0;
    if (lane == 0) rp = 1.0 / M[piv * LDF + k];
    rp = __shfl_sync(0xffffffffu, rp, 0);
    if (tid == 0) {
      pivrow[k] = piv;
      rdiag[k] = rp;
    }
    // all operands are loaded before any store: the pivot row and column k are never
    // written in this step, but the compiler cannot prove it (would serialise LDS/STS)
    const double* prow = M + piv * LDF;
    double pr[NB], l[NB];
    bool act[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) pr[b] = prow[tx + 16 * b];
#pragma unroll
    for (int a = 0; a < NB; ++a) {
      const int i = ty + 16 * a;
      act[a] = !is_used(i);
      l[a] = M[i * LDF + k];
    }
#pragma unroll
    for (int a = 0; a < NB; ++a) {
      const int i = ty + 16 * a;
      const double la = l[a] * rp;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int j = tx + 16 * b;
        if (act[a] && j > k) {
          A[a][b] = fma(-la, pr[b], A[a][b]);
          M[i * LDF + j] = A[a][b];
        }
      }
    }
    __syncthreads();
  }
  if (bad) {
    if (tid == 0) status[sim] = 1;
    return;
  }
  if (MODE == 2) { if (tid == 0) status[sim] = (int)A[0][0]; return; }
  if (tid < 32) {
    constexpr int NU = (D + 31) / 32;
    double bv[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int t = lane + 32 * u;
      bv[u] = (t < n) ? M[pivrow[t] * LDF + n] : 0.0;
    }
    for (int t = n - 1; t >= 0; --t) {
      const int owner = t & 31, slot = t >> 5;
      double bt = 0.0;
#pragma unroll
      for (int u = 0; u < NU; ++u)
        if (u == slot) bt = bv[u];
      bt = __shfl_sync(0xffffffffu, bt, owner);
      const double xt = bt * rdiag[t];
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const int tt = lane + 32 * u;
        if (tt < t) bv[u] = fma(-M[pivrow[tt] * LDF + t], xt, bv[u]);
        else if (tt == t) bv[u] = xt;
      }
    }
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      const int t = lane + 32 * u;
      if (t < n) {
        dr[(size_t)sim * n + t] = bv[u];
        if (apply) r[(size_t)sim * n + t] += bv[u];
      }
    }
    if (lane == 0) status[sim] = 0;
  }
}


template <int MODE> float run(int n, double* dS, double* dphi, double* ddr, double* dr, int* st) {
  cudaFuncSetAttribute(k_lu_var<4, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k_lu_var<4, MODE><<<1, 256, lu_smem_bytes(n)>>>(dS, dphi, ddr, dr, n, 0, st);
  cudaEventRecord(a);
  for (int r = 0; r < 200; ++r) k_lu_var<4, MODE><<<1, 256, lu_smem_bytes(n)>>>(dS, dphi, ddr, dr, n, 0, st);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000 / 200;
}
int main() {
  for (int n : {8, 60}) {
  std::vector<double> S(n * n), phi(n);
  std::mt19937 g(1); std::uniform_real_distribution<double> U(-1, 1);
  for (auto& x : S) x = U(g);
  for (int i = 0; i < n; ++i) S[i * n + i] += n;
  for (auto& x : phi) x = U(g);
  double *dS, *dphi, *ddr, *dr; int* st;
  cudaMalloc(&dS, n * n * 8); cudaMalloc(&dphi, n * 8); cudaMalloc(&ddr, n * 8); cudaMalloc(&dr, n * 8); cudaMalloc(&st, 4);
  cudaMemcpy(dS, S.data(), n * n * 8, cudaMemcpyHostToDevice); cudaMemcpy(dphi, phi.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 200; ++r) k_empty<<<1, 256>>>(st);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("n=%d empty %.2f us | load-only %.2f | load+elim %.2f | full %.2f\n", n, ms * 1000 / 200, run<1>(n, dS, dphi, ddr, dr, st),
         run<2>(n, dS, dphi, ddr, dr, st), run<0>(n, dS, dphi, ddr, dr, st));
  }
  return 0;
}
