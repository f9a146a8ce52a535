// Non-GEMM kernels of the reduced Newton step: seeds, wnet, StVK cubature,
// assembly, reductions, in-CTA LU with partial pivoting.
#pragma once
#include "cluster_async.cuh"
#include "common.cuh"
#include "mc_device.cuh"
#include "gram_dmma.cuh"

namespace nlrom {

// ----------------------------------------------------------------- bundle seed
// X0_t rows (per sim, groups of G = 4 + 4 nk columns):
//   base   : q | v | 0 | w           (1, s, s^2, r)
//   tangent: e_k | 0 | 0 | 0         (t, ts, ts^2, tr)
// v = q - q_bar (0 when drop_fict), w = (3 + alpha dt) v - dt qdot_bar
// (drop_fict: (1 + alpha dt) v - dt qdot_bar), see rdsim oracle / DESIGN.md.
__global__ void k_seed_jet(const double* __restrict__ r, const double* __restrict__ rbar,
                           const double* __restrict__ rdbar, double* __restrict__ X0, int ldx, int n_p, int n_q,
                           int n, int G, int gps, int n_sims, double dt, double alpha, int drop_fict) {
  pdl_wait();
  pdl_launch();
  const int cols = gps * G;
  const long long total = (long long)n_sims * cols * n_q;
  const int nk = (G - 4) / 4;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int i = t % n_q;
    long long cc = t / n_q;
    int c = cc % cols;
    int sim = cc / cols;
    int g = c / G, cl = c % G;
    const double* rs = r + (size_t)sim * n;
    double q = rs[n_p + i];
    double qb = rbar[(size_t)sim * n + n_p + i];
    double qdb = rdbar[(size_t)sim * n + n_p + i];
    double v = q - qb;
    double val = 0.0;
    if (cl < 4) {
      if (cl == 0) val = q;
      else if (cl == 1) val = drop_fict ? 0.0 : v;
      else if (cl == 3) val = (drop_fict ? (1.0 + alpha * dt) : (3.0 + alpha * dt)) * v - dt * qdb;
    } else {
      int k = (cl - 4) / 4, s = (cl - 4) % 4;
      int kg = g * nk + k;
      if (s == 0 && kg == i) val = 1.0;
    }
    X0[((size_t)sim * cols + c) * ldx + i] = val;
  }
}

// Reference-structure seeds for the individual diffops.
// Column c = pass * S + slot; value for input coordinate i.
//   op JVP: 1 pass order 1 (i1 = v); JAC: n_q passes (i1 = e_j); HVV: 1 pass order 2 (v, v);
//   HV: n_q passes order 2 (e_j, v); SVV: n_q passes order 3 (e_j, v, v); VALUE/VJP: order 0.
//   scale = eps (literal multicomplex, mode 1) or 1 (scaled multi-dual, mode 0).
__global__ void k_seed_ref(const double* __restrict__ q, const double* __restrict__ vec, double* __restrict__ X0,
                           int ldx, int n_q, int op, int S, int npass, double scale) {
  pdl_wait();
  pdl_launch();
  const long long total = (long long)npass * S * n_q;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int i = t % n_q;
    int c = t / n_q;
    int pass = c / S, s = c % S;
    double val = 0.0;
    double ej = (pass == i) ? 1.0 : 0.0;
    double v = vec ? vec[i] : 0.0;
    if (s == 0) val = q[i];
    else if (op == NLROM_OP_JVP) val = (s == 1) ? v * scale : 0.0;
    else if (op == NLROM_OP_JACOBIAN || op == NLROM_OP_VHP) val = (s == 1) ? ej * scale : 0.0;
    else if (op == NLROM_OP_HVV) val = (s == 1 || s == 2) ? v * scale : 0.0;
    else if (op == NLROM_OP_HV) val = (s == 1) ? ej * scale : (s == 2 ? v * scale : 0.0);
    else if (op == NLROM_OP_SVV) val = (s == 1) ? ej * scale : ((s == 2 || s == 4) ? v * scale : 0.0);
    X0[(size_t)c * ldx + i] = val;
  }
}

// Extract slot `slot` of every pass from Y_t (ncols x ldy) into out (N, npass) row-major, / div.
__global__ void k_extract_slot(const double* __restrict__ Y, int ldy, int N, int S, int npass, int slot, double div,
                               double* __restrict__ out) {
  pdl_wait();
  pdl_launch();
  const long long total = (long long)N * npass;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int j = t % npass;
    int m = t / npass;
    out[t] = Y[((size_t)j * S + slot) * ldy + m] / div;
  }
}

// ------------------------------------------------------------------------ wnet
// Split-K GEMV: part[s][sim][m] = sum_{k in chunk s} A[m][k] x[sim][k]   (A: M x K row-major, lda)
// Each warp works on 4 rows at once so 4 independent loads per lane are in flight.
__global__ void k_gemv_splitk(const double* __restrict__ A, int lda, const double* __restrict__ x, long long strideX,
                              int M, int K, int chunk, double* __restrict__ part, int n_sims) {
  pdl_wait();
  pdl_launch();
  const int s = blockIdx.x;
  const int sim = blockIdx.y;
  const int k0 = s * chunk, k1 = min(K, k0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double* xs = x + (size_t)sim * strideX;
  for (int m0 = warp * 4; m0 < M; m0 += nw * 4) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = k0 + lane; k < k1; k += 32) {
      const double xv = xs[k];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (m0 + u < M) acc[u] = fma(A[(size_t)(m0 + u) * lda + k], xv, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double v = acc[u];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && m0 + u < M) part[((size_t)s * n_sims + sim) * M + m0 + u] = v;
    }
  }
}

// Same split-K GEMV with every load of a lane issued up front: CH k-values per lane (chunk =
// 32 CH columns), 8 rows per warp, 8 interleaved shuffle trees.
template <int CH>
__global__ void __launch_bounds__(256) k_gemv_splitk_t(const double* __restrict__ A, int lda,
                                                       const double* __restrict__ x, long long strideX, int M, int K,
                                                       double* __restrict__ part, int n_sims) {
  pdl_wait();
  pdl_launch();
  const int s = blockIdx.x, sim = blockIdx.y;
  const int k0 = s * 32 * CH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double* xs = x + (size_t)sim * strideX;
  double xv[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    const int k = k0 + lane + 32 * c;
    xv[c] = (k < K) ? xs[k] : 0.0;
  }
  for (int m0 = warp * 8; m0 < M; m0 += nw * 8) {
    double a[8][CH];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int k = k0 + lane + 32 * c;
        a[u][c] = (m0 + u < M && k < K) ? A[(size_t)(m0 + u) * lda + k] : 0.0;
      }
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc[u] = 0.0;
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[u] = fma(a[u][c], xv[c], acc[u]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
    if (lane < 8 && m0 + lane < M) {
      double v = acc[0];
#pragma unroll
      for (int u = 1; u < 8; ++u)
        if (lane == u) v = acc[u];
      part[((size_t)s * n_sims + sim) * M + m0 + lane] = v;
    }
  }
}

// Weight-net tail, grid (ceil(|C|/64), n_sims): every CTA rebuilds h1..h3 (tiny) and
// evaluates 64 rows of the C-restricted last layer:
//   h1 = sin(sum parts + b1), h2 = sin(W2 h1 + b2), h3 = sin(W3 h2 + b3),
//   w_C = (W4[C] h3 + b4[C])^2   (square keeps w >= 0)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// hout = sin(W hin + b): warp-per-row dot products into hout, then one thread per row
// evaluates the (long, fp64) sin so the sins run in parallel, not one per warp in sequence.
__device__ void wnet_dense_sin(const double* __restrict__ W, const double* __restrict__ b, const double* hin,
                               double* hout, int wn) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int m = warp; m < wn; m += nw) {
    double acc = 0.0;
    for (int k = lane; k < wn; k += 32) acc = fma(W[(size_t)m * wn + k], hin[k], acc);
    acc = warp_sum(acc);
    if (lane == 0) hout[m] = acc + b[m];
  }
  __syncthreads();
  for (int m = threadIdx.x; m < wn; m += blockDim.x) hout[m] = sin(hout[m]);
}

__global__ void k_wnet_tail(const double* __restrict__ part, int n_split, int wn, const double* __restrict__ b1,
                            const double* __restrict__ W2, const double* __restrict__ b2, const double* __restrict__ W3,
                            const double* __restrict__ b3, const double* __restrict__ W4C, const double* __restrict__ b4C,
                            int n_cub, double* __restrict__ wC, int n_sims) {
  // Every global input is staged with async copies in two batches (constants before the
  // programmatic-dependency wait, the producer's partial sums after it): each dependent
  // global round trip costs ~0.5-1 us here, so none may sit inside a loop.
  extern __shared__ double sh[];
  const int sim = blockIdx.y;
  const int j0 = blockIdx.x * 64;
  const int nrows4 = max(0, min(64, n_cub - j0));
  double* h1 = sh;                    // [wn]
  double* h2 = h1 + wn;               // [wn]
  double* bs = h2 + wn;               // b1 | b2 | b3 | b4[rows]   [3 wn + 64]
  double* W2s = bs + 3 * wn + 64;     // [wn][wn]
  double* W3s = W2s + wn * wn;        // [wn][wn]
  double* W4s = W3s + wn * wn;        // [64][wn]
  double* ps = W4s + 64 * wn;         // [n_split][wn] partial sums of layer 1
  for (int t = threadIdx.x; t < wn * wn; t += blockDim.x) {
    cp_async8(W2s + t, W2 + t);
    cp_async8(W3s + t, W3 + t);
  }
  for (int t = threadIdx.x; t < nrows4 * wn; t += blockDim.x) cp_async8(W4s + t, W4C + (size_t)j0 * wn + t);
  for (int t = threadIdx.x; t < wn; t += blockDim.x) {
    cp_async8(bs + t, b1 + t);
    cp_async8(bs + wn + t, b2 + t);
    cp_async8(bs + 2 * wn + t, b3 + t);
  }
  for (int t = threadIdx.x; t < nrows4; t += blockDim.x) cp_async8(bs + 3 * wn + t, b4C + j0 + t);
  pdl_wait();
  pdl_launch();
  for (int t = threadIdx.x; t < n_split * wn; t += blockDim.x)
    cp_async8(ps + t, part + ((size_t)(t / wn) * n_sims + sim) * wn + t % wn);
  cp_async_all_wait();
  __syncthreads();
  for (int m = threadIdx.x; m < wn; m += blockDim.x) {
    double acc[4] = {bs[m], 0.0, 0.0, 0.0};
    int s2 = 0;
    for (; s2 + 3 < n_split; s2 += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += ps[(s2 + u) * wn + m];
    for (; s2 < n_split; ++s2) acc[0] += ps[s2 * wn + m];
    h1[m] = sin((acc[0] + acc[1]) + (acc[2] + acc[3]));
  }
  __syncthreads();
  wnet_dense_sin(W2s, bs + wn, h1, h2, wn);
  __syncthreads();
  wnet_dense_sin(W3s, bs + 2 * wn, h2, h1, wn);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int jj = warp; jj < nrows4; jj += nw) {
    double acc = 0.0;
    for (int k = lane; k < wn; k += 32) acc = fma(W4s[(size_t)jj * wn + k], h1[k], acc);
    acc = warp_sum(acc) + bs[3 * wn + jj];
    if (lane == 0) wC[(size_t)sim * n_cub + j0 + jj] = acc * acc;
  }
}

// Same tail with TMA bulk staging (one copy per weight matrix / bias / partial block, on two
// mbarriers: constants before the dependency wait, the producer's partials after it) and
// tpr = blockDim / wn threads per output row (short FMA chains + a 2-level shuffle) instead of
// a warp per row. Needs wn even, blockDim % wn == 0, partials contiguous per sim.
__device__ __forceinline__ double wnet_row_tpr(const double* __restrict__ W, int wn, const double* hin, int m, int q,
                                               int tpr) {
  const int per = wn / tpr;
  double acc = 0.0;
  if ((per & (per - 1)) == 0) {
    const int rot = m & (per - 1);
    for (int i = 0; i < per; ++i) {
      const int k = q + tpr * ((i + rot) & (per - 1));  // rotated walk: rows of a warp hit different banks
      acc = fma(W[(size_t)m * wn + k], hin[k], acc);
    }
  } else {
    for (int i = 0; i < per; ++i) {
      const int k = q + tpr * ((i + m) % per);
      acc = fma(W[(size_t)m * wn + k], hin[k], acc);
    }
  }
  for (int o = tpr >> 1; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return acc;
}

// Weight-net layer 1 from the decoder's last hidden activation (folded weights, see the upload
// in ctx.cu): part[sim][m] = sum_k F[m][k] x[k], x = [h (w) | p (n_p) | 1]; h is the base jet
// column of the hidden chain's output (compact column sim * cs). Runs on a side branch while the
// output layer executes; k_wnet_tail2 (n_split = 1) adds b1 and finishes the net. The folded
// matrix (wn x ldF, constant) lands in shared memory by one TMA bulk copy issued BEFORE the
// dependency wait, i.e. while the hidden chain still runs.
inline size_t wnet_head_smem(int rows, int ldF) { return (size_t)rows * ldF * 8 + 1024 * 8 + 16; }

// grid (wn / rows per CTA, n_sims): each CTA lands only its rows of F by TMA (8 rows = 18 KB at
// cfg2 instead of all 64 = 147 KB in one CTA: the single bulk copy was the kernel's latency)
__global__ void __launch_bounds__(256) k_wnet_head(const double* __restrict__ H, int ldH, int cs,
                                                   const double* __restrict__ r, int n, int n_p, int w,
                                                   const double* __restrict__ F, int ldF, int wn,
                                                   double* __restrict__ part) {
  extern __shared__ __align__(16) double hs[];
  const int rpc = wn / gridDim.x;     // rows of this CTA (divides wn; 256 / rpc a power of two <= 32)
  const int r0 = blockIdx.x * rpc;
  double* Fs = hs;                    // [rpc][ldF]
  double* x = Fs + (size_t)rpc * ldF;  // [<= 1024]
  uint64_t* bar = reinterpret_cast<uint64_t*>(x + 1024);
  const int sim = blockIdx.y, tid = threadIdx.x;
  const int K = w + n_p + 1;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const uint32_t bytes = (uint32_t)(rpc * ldF * 8);
    mbar_expect_tx(bar, bytes);
    tma_g2s(Fs, F + (size_t)r0 * ldF, bytes, bar);
  }
  pdl_wait();
  pdl_launch();
  for (int k = tid; k < K; k += blockDim.x)
    x[k] = k < w ? H[(size_t)sim * cs * ldH + k] : (k < w + n_p ? r[(size_t)sim * n + (k - w)] : 1.0);
  __syncthreads();
  mbar_wait(bar, 0);
  const int tpr = blockDim.x / rpc;  // threads per output row
  const int m = tid / tpr, q = tid % tpr;
  double a0 = 0.0, a1 = 0.0;
  if (m < rpc) {
    const double* Fm = Fs + (size_t)m * ldF;
    int k = q;
    for (; k + tpr < K; k += 2 * tpr) {
      a0 = fma(Fm[k], x[k], a0);
      a1 = fma(Fm[k + tpr], x[k + tpr], a1);
    }
    if (k < K) a0 = fma(Fm[k], x[k], a0);
  }
  double acc = a0 + a1;
  for (int o = tpr >> 1; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (m < rpc && q == 0) part[(size_t)sim * wn + r0 + m] = acc;
}

__global__ void __launch_bounds__(256) k_wnet_tail2(const double* __restrict__ part, int n_split, int wn,
                                                    const double* __restrict__ b1, const double* __restrict__ W2,
                                                    const double* __restrict__ b2, const double* __restrict__ W3,
                                                    const double* __restrict__ b3, const double* __restrict__ W4C,
                                                    const double* __restrict__ b4C, int n_cub, double* __restrict__ wC,
                                                    int n_sims) {
  extern __shared__ __align__(16) double sh[];
  const int sim = blockIdx.y, tid = threadIdx.x;
  const int j0 = blockIdx.x * 64;
  const int nrows4 = max(0, min(64, n_cub - j0));
  double* h1 = sh;
  double* h2 = h1 + wn;
  double* bs = h2 + wn;            // b1 | b2 | b3   [3 wn]
  double* W2s = bs + 3 * wn + 64;
  double* W3s = W2s + wn * wn;
  double* W4s = W3s + wn * wn;     // [64][wn]
  double* ps = W4s + 64 * wn;      // [n_split][wn]
  uint64_t* bar = reinterpret_cast<uint64_t*>(ps + n_split * wn);
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
    const uint32_t mat = (uint32_t)(wn * wn * 8), vec = (uint32_t)(wn * 8);
    mbar_expect_tx(bar, 2 * mat + (uint32_t)(nrows4 * wn * 8) + 3 * vec);
    tma_g2s(W2s, W2, mat, bar);
    tma_g2s(W3s, W3, mat, bar);
    if (nrows4) tma_g2s(W4s, W4C + (size_t)j0 * wn, (uint32_t)(nrows4 * wn * 8), bar);
    tma_g2s(bs, b1, vec, bar);
    tma_g2s(bs + wn, b2, vec, bar);
    tma_g2s(bs + 2 * wn, b3, vec, bar);
  }
  pdl_wait();
  pdl_launch();
  if (tid == 0) {
    const uint32_t pb = (uint32_t)(n_split * wn * 8);
    mbar_expect_tx(bar + 1, pb);
    tma_g2s(ps, part + (size_t)sim * (n_split == 1 ? wn : 0), pb, bar + 1);
  }
  __syncthreads();
  mbar_wait(bar + 1, 0);
  mbar_wait(bar, 0);
  for (int m = tid; m < wn; m += blockDim.x) {
    double acc[4] = {bs[m], 0.0, 0.0, 0.0};
    int s2 = 0;
    for (; s2 + 3 < n_split; s2 += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += ps[(s2 + u) * wn + m];
    for (; s2 < n_split; ++s2) acc[0] += ps[s2 * wn + m];
    h1[m] = sin((acc[0] + acc[1]) + (acc[2] + acc[3]));
  }
  __syncthreads();
  const int tpr = blockDim.x / wn, m = tid / tpr, q = tid % tpr;
  {
    const double v = wnet_row_tpr(W2s, wn, h1, m, q, tpr);
    if (q == 0) h2[m] = sin(v + bs[wn + m]);
  }
  __syncthreads();
  {
    const double v = wnet_row_tpr(W3s, wn, h2, m, q, tpr);
    if (q == 0) h1[m] = sin(v + bs[2 * wn + m]);
  }
  __syncthreads();
  for (int r0 = 0; r0 < nrows4; r0 += wn) {
    const int jj = r0 + m;
    const bool ok = jj < nrows4;
    const double v = wnet_row_tpr(W4s, wn, h1, ok ? jj : 0, q, tpr);
    if (q == 0 && ok) {
      const double z = v + b4C[j0 + jj];
      wC[(size_t)sim * n_cub + j0 + jj] = z * z;
    }
  }
}

// -------------------------------------------------------------------- cubature
// One warp per element: StVK (P1 tet, one-point quadrature) force f_e and stiffness
// K_e, weighted by w_e; then the CTA projects with the element's
// 12 rows of J~ = [U, J]:  f~ += w_e J~_e^T f_e,  K~ += J~_e^T (w_e K_e) J~_e.
struct CubArgs {
  const int* elems;        // (E,) element ids (nullptr: identity 0..E-1)
  int n_elems;
  const int* elem_rows;    // (T, 12) free-DOF rows or -1
  const double* Dm_inv;    // (T, 9)
  const double* vol;       // (T)
  const double* w;         // (n_sims, E) weights (nullptr: 1)
  const double* u;         // (n_sims, N)
  const double* Jt;        // (n_sims, N, ldjt)
  int N, n, ldjt;
  double mu, lam;
  int epc;                 // elements per CTA
  double* fe_w;            // (n_sims, E, 12) weighted element forces
  double* part_f;          // (n_sims, nchunk, n)
  double* part_K;          // (n_sims, nchunk, n*n)
  int nchunk;
  double* Ke_out;          // optional (E, 144): w-scaled element stiffness
  double* fred_out;        // optional (E, n): per-element J~_e^T (w f_e)
  int early = 0;           // 1: the producer grid is the weight net (J~, u complete at launch)
  int skip_fe = 0;         // 1: do not write fe_w (a concurrent force-only launch owns it)
  const int* rows_g = nullptr;     // optional (n_elems, 12) set-gathered DOF rows
  const double* Dm_g = nullptr;    // optional (n_elems, 9) set-gathered Dm^-1
  const double* vol_g = nullptr;   // optional (n_elems) set-gathered volumes
  int cpc = 1;             // element chunks per CTA: the Gram accumulates in shared memory over
                           // cpc chunks and each CTA writes ONE partial (nchunk = partials per
                           // sim); > 1 only with J~ and without fred_out
};

__device__ __forceinline__ void mat3_mul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) C[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
}

// Programmatic-launch overlap: everything that does not depend on the weight net (the DOF rows,
// the J~ / u gathers, the element physics and G_e = K_e J~_e, all unweighted) runs BEFORE the
// dependency wait, i.e. while the weight-net kernels still execute; the element weights scale
// f_e and the G_e rows afterwards (the Gram is linear in w_e). Safe because the producer
// (k_wnet_tail*) issues launch_dependents only after its own wait, so the output layer that
// wrote J~ and u has completed when this grid starts.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) k_cubature(CubArgs a) {
  if (!a.early) pdl_wait();  // producer wrote J~ / u itself: wait before the gathers
  extern __shared__ double sh[];
  const int n = a.n;
  const int epc = a.epc;
  const int ldp = gram_ld(n);              // row pitch of the J~ / G panels
  double* Js = sh;                         // [epc*12][ldp]
  double* Gs = Js + (size_t)epc * 12 * ldp;  // [epc*12][ldp]  (w K J)
  double* Ks = Gs + (size_t)epc * 12 * ldp;  // [epc][12][12]
  double* Fs = Ks + (size_t)epc * 144;     // [epc][12]
  const int sim = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double* u = a.u + (size_t)sim * a.N;
  const double* Jt = a.Jt ? a.Jt + (size_t)sim * a.N * a.ldjt : nullptr;
  int* Rw = reinterpret_cast<int*>(Fs + (size_t)epc * 12);  // [epc][12]
  double* Kacc = reinterpret_cast<double*>(Rw + epc * 12);  // [n][n] + [n] (K~, f~ partials) when cpc > 1
  __shared__ double wsh[64];
  __shared__ uint64_t gbar;  // J~ row gather by TMA bulk copies (one mbarrier phase per chunk)
  const bool pref = a.rows_g != nullptr && epc * 12 <= (int)blockDim.x;
  const bool bulk = pref && Jt && (a.ldjt & 1) == 0 && (ldp & 1) == 0;
  if (bulk && threadIdx.x == 0) {
    mbar_init(&gbar, 1);
    fence_mbar_init();
  }
  int nxt = -1;
  for (int ck = 0; ck < a.cpc; ++ck) {
  const int chunk = blockIdx.x * a.cpc + ck;  // element chunk
  if (ck > 0) {
    if (chunk * epc >= a.n_elems) break;      // uniform over the CTA
    __syncthreads();                          // the previous chunk's Gram read Js / Gs / Fs
  }

  // stage the chunk's 12 DOF rows per element, then gather the J~ rows (independent loads).
  // Set-gathered rows: held in a register one chunk ahead (loaded while the previous chunk
  // computes), so a chunk starts without a global round trip.
  if (pref) {
    if (ck == 0 && threadIdx.x < epc * 12) {
      const int ei = chunk * epc + threadIdx.x / 12;
      nxt = ei < a.n_elems ? a.rows_g[(size_t)chunk * epc * 12 + threadIdx.x] : -1;
    }
    if (threadIdx.x < epc * 12) Rw[threadIdx.x] = nxt;
  } else
  for (int idx = threadIdx.x; idx < epc * 12; idx += blockDim.x) {
    const int ei = chunk * epc + idx / 12;
    int row = -1;
    if (ei < a.n_elems) {
      const int e = a.elems ? a.elems[ei] : ei;
      row = a.elem_rows[(size_t)e * 12 + idx % 12];
    }
    Rw[idx] = row;
  }
  const int nrows = __syncthreads_count(bulk && threadIdx.x < epc * 12 && nxt >= 0);
  if (bulk) {
    // one TMA bulk copy per valid J~ row (issued by the row's owner thread; even n so the size
    // is a multiple of 16 bytes), fixed-DOF rows zero-filled; lands while the physics runs
    const uint32_t B = (uint32_t)((n + 1) & ~1) * 8u;
    if (threadIdx.x == 0) mbar_expect_tx(&gbar, (uint32_t)nrows * B);
    if (threadIdx.x < epc * 12) {
      double* dst = Js + threadIdx.x * ldp;
      if (nxt >= 0) {
        fence_proxy_async();
        tma_g2s(dst, Jt + (size_t)nxt * a.ldjt, B, &gbar);
      } else {
        for (int j = 0; j < n; ++j) dst[j] = 0.0;
      }
    }
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (Jt && (a.ldjt & 1) == 0 && (ldp & 1) == 0) {  // 16-byte chunks (both pitches even)
      // n <= 32: a half-warp per J~ row (two rows per warp instruction), else a warp per row
      const int half = n <= 32 ? 1 : 0;
      const int sub = half ? lane >> 4 : 0, sl = half ? lane & 15 : lane, step = half ? 32 : 64;
      for (int rr = (warp << half) + sub; rr < epc * 12; rr += nw << half) {
        const int row = Rw[rr];
        double* dst = Js + rr * ldp;
        for (int j = 2 * sl; j < n; j += step) {
          if (row >= 0) cp_async16(dst + j, Jt + (size_t)row * a.ldjt + j, true);
          else dst[j] = dst[j + 1] = 0.0;
        }
      }
    } else
    for (int rr = warp; Jt && rr < epc * 12; rr += nw) {  // warp per J~ row: no div / mod
      const int row = Rw[rr];
      double* dst = Js + rr * ldp;
      {
        for (int j = lane; j < n; j += 32) {
          if (row >= 0) cp_async8(dst + j, Jt + (size_t)row * a.ldjt + j);
          else dst[j] = 0.0;
        }
      }
    }
  }
  if (pref && ck + 1 < a.cpc && threadIdx.x < epc * 12) {  // next chunk's rows, in flight during this one
    const int ei = (chunk + 1) * epc + threadIdx.x / 12;
    nxt = ei < a.n_elems ? a.rows_g[(size_t)(chunk + 1) * epc * 12 + threadIdx.x] : -1;
  }
  // element physics: two elements per warp (one per half-warp; lanes 0..11 of a half own the
  // element's 12 DOFs). A padding element (past the set) gets V = 0 and Dm^-1 = 0, so its force
  // and stiffness come out exactly zero without divergent control flow around the shuffles.
  const int hw = lane >> 4, hl = lane & 15;
  for (int el0 = 2 * warp; el0 < epc; el0 += 2 * nw) {
    const int el = el0 + hw;
    const int ei = chunk * epc + el;
    const bool valid = el < epc && ei < a.n_elems;
    const int e = !valid ? 0 : a.Dm_g ? ei : (a.elems ? a.elems[ei] : ei);  // index into Dm / vol
    const double* Dm = a.Dm_g ? a.Dm_g : a.Dm_inv;
    const double* vl = a.vol_g ? a.vol_g : a.vol;
    double ue = 0.0;
    if (valid && hl < 12) {
      const int row = Rw[el * 12 + hl];
      ue = row >= 0 ? u[row] : 0.0;
    }
    double uv[12];
#pragma unroll
    for (int l = 0; l < 12; ++l) uv[l] = __shfl_sync(0xffffffffu, ue, l, 16);
    double Di[9];
#pragma unroll
    for (int l = 0; l < 9; ++l) Di[l] = valid ? Dm[(size_t)e * 9 + l] : 0.0;
    const double V = valid ? vl[e] : 0.0;
    const double we = 1.0;  // weights applied after the dependency wait (row weights of the Gram)
    // G rows: g_i (i=1..3) = rows of Dm^-1, g_0 = -sum
    double G[12];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      G[3 + b] = Di[b];
      G[6 + b] = Di[3 + b];
      G[9 + b] = Di[6 + b];
      G[b] = -(Di[b] + Di[3 + b] + Di[6 + b]);
    }
    // Ds (columns u_i - u_0), F = I + Ds Dm^-1
    double Ds[9], F[9];
#pragma unroll
    for (int aa = 0; aa < 3; ++aa)
#pragma unroll
      for (int i = 0; i < 3; ++i) Ds[aa * 3 + i] = uv[(i + 1) * 3 + aa] - uv[aa];
    mat3_mul(Ds, Di, F);
    F[0] += 1.0;
    F[4] += 1.0;
    F[8] += 1.0;
    double E[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        E[i * 3 + j] = 0.5 * (F[i] * F[j] + F[3 + i] * F[3 + j] + F[6 + i] * F[6 + j] - (i == j ? 1.0 : 0.0));
    const double trE = E[0] + E[4] + E[8];
    double S[9];
#pragma unroll
    for (int l = 0; l < 9; ++l) S[l] = 2.0 * a.mu * E[l];
    S[0] += a.lam * trE;
    S[4] += a.lam * trE;
    S[8] += a.lam * trE;
    double P[9];
    mat3_mul(F, S, P);
    if (hl < 12 && el < epc) {
      const int i = hl / 3, aa = hl % 3;
      // row i of G and row aa of P by selects (no dynamically indexed local arrays)
      double gi[3], pa[3];
#pragma unroll
      for (int y = 0; y < 3; ++y) {
        gi[y] = i == 0 ? G[y] : i == 1 ? G[3 + y] : i == 2 ? G[6 + y] : G[9 + y];
        pa[y] = aa == 0 ? P[y] : aa == 1 ? P[3 + y] : P[6 + y];
      }
      double f = V * (pa[0] * gi[0] + pa[1] * gi[1] + pa[2] * gi[2]);
      Fs[el * 12 + hl] = we * f;
      if (!Jt && !a.Ke_out) continue;  // force-only launch: no element stiffness
      // stiffness column for DOF (jv, d) = (i, aa) = hl: dF_ab = delta_ad g_jv[b]
      const int d = aa;
      double dF[9];
#pragma unroll
      for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int y = 0; y < 3; ++y) dF[x * 3 + y] = (x == d) ? gi[y] : 0.0;
      double dE[9];
#pragma unroll
      for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int y = 0; y < 3; ++y)
          dE[x * 3 + y] = 0.5 * (dF[x] * F[y] + dF[3 + x] * F[3 + y] + dF[6 + x] * F[6 + y] + F[x] * dF[y] +
                                 F[3 + x] * dF[3 + y] + F[6 + x] * dF[6 + y]);
      const double trdE = dE[0] + dE[4] + dE[8];
      double dS[9];
#pragma unroll
      for (int l = 0; l < 9; ++l) dS[l] = 2.0 * a.mu * dE[l];
      dS[0] += a.lam * trdE;
      dS[4] += a.lam * trdE;
      dS[8] += a.lam * trdE;
      double t1[9], t2[9];
      mat3_mul(dF, S, t1);
      mat3_mul(F, dS, t2);
#pragma unroll
      for (int l = 0; l < 9; ++l) t1[l] += t2[l];
#pragma unroll
      for (int r = 0; r < 12; ++r) {
        int ri = r / 3, ra = r % 3;
        double kv = V * (t1[ra * 3] * G[ri * 3] + t1[ra * 3 + 1] * G[ri * 3 + 1] + t1[ra * 3 + 2] * G[ri * 3 + 2]);
        Ks[el * 144 + r * 12 + hl] = we * kv;
      }
    }
  }
  // ---- the weight net's output is needed from here on
  pdl_wait();
  pdl_launch();
  for (int el = threadIdx.x; el < epc; el += blockDim.x) {
    const int ei = chunk * epc + el;
    wsh[el] = (a.w && ei < a.n_elems) ? a.w[(size_t)sim * a.n_elems + ei] : 1.0;
  }
  if (bulk) mbar_wait_cta(&gbar, (uint32_t)(ck & 1));  // the J~ rows of this chunk
  else cp_async_all_wait();
  __syncthreads();  // physics done (Ks, Fs), weights staged, J~ rows landed
  const bool gram = Jt && !a.fred_out;
  // G_e = w_e K_e J~_e (12 x n) on the DMMA pipe
  if (gram) ke_j_dmma(Ks, Js, Gs, ldp, epc, n, wsh);
  for (int t = threadIdx.x; t < epc * 12; t += blockDim.x) {
    const int el = t / 12, ei = chunk * epc + el;
    const double v = Fs[t] * wsh[el];
    Fs[t] = v;
    if (gram) Gs[t * ldp + n] = v;  // padding column n carries w f into the Gram
    if (ei < a.n_elems && !a.skip_fe) a.fe_w[((size_t)sim * a.n_elems + ei) * 12 + t % 12] = v;
  }
  if (a.Ke_out)
    for (int t = threadIdx.x; t < epc * 144; t += blockDim.x) {
      const int el = t / 144, ei = chunk * epc + el;
      if (ei < a.n_elems) a.Ke_out[(size_t)ei * 144 + t % 144] = wsh[el] * Ks[t];
    }
  if (!Jt) return;
  if (a.fred_out) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < epc * n; idx += blockDim.x) {
      int el = idx / n, i = idx % n;
      int ei = chunk * epc + el;
      if (ei >= a.n_elems) continue;
      double acc = 0.0;
      for (int l = 0; l < 12; ++l) acc = fma(Js[(el * 12 + l) * ldp + i], Fs[el * 12 + l], acc);
      a.fred_out[(size_t)ei * n + i] = acc;
    }
    return;
  }
  __syncthreads();
  // partial K~ = J~_C^T (w K J~_C) and f~ = J~_C^T (w f) over the chunk's rows, one DMMA Gram
  const int R = epc * 12;
  if (a.cpc == 1)
    gram_dmma_kf(Js, ldp, Gs, ldp, R, n, a.part_K + ((size_t)sim * a.nchunk + blockIdx.x) * n * n, n,
                 a.part_f + ((size_t)sim * a.nchunk + blockIdx.x) * n, false);
  else
    gram_dmma_kf(Js, ldp, Gs, ldp, R, n, Kacc, n, Kacc + n * n, ck > 0);  // warp-owned tiles: no race
  }  // chunks of this CTA
  if (a.cpc > 1) {
    __syncthreads();
    double* pK = a.part_K + ((size_t)sim * a.nchunk + blockIdx.x) * n * n;
    double* pf = a.part_f + ((size_t)sim * a.nchunk + blockIdx.x) * n;
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) pK[t] = Kacc[t];
    for (int t = threadIdx.x; t < n; t += blockDim.x) pf[t] = Kacc[n * n + t];
  }
}

// -------------------------------------------------------------------- cubature, many sims
// One CTA per sim (cfg5: 4096 sims x |C| = 100, n = 30). The reduced stiffness is projected
// through the deformation-gradient map instead of the 12 DOF rows of J~:
//   B_e = dF/dr (9 x n):  B[(a,y)] = sum_v G[v][y] J~[row(v,a)]    (G: rows of Dm^-1, g_0 = -sum)
//   K~ += w_e V_e B_e^T dP(B_e),  f~ += w_e V_e B_e^T vec(P_e)      (dP = dF S + F dS: dP/dF of StVK)
// which is J~_e^T (w K_e J~_e) and J~_e^T (w f_e) exactly (K_e = V G^T (dP/dF) G), with a 9-row
// Gram per element instead of 12 and no 12 x 12 K_e. The constant U columns of J~ give constant
// B columns, precomputed per set element at upload (BU, L2-resident); only the n_q J columns of
// the element rows are gathered per sim. dP/dF is symmetric (a Hessian of the StVK energy), so
// only the Gram's upper 8 x 8 tiles are computed (10 of 16 at n = 30) and mirrored on store.
// Per CTA: physics of up to CS_SUPER elements (thread per element: F, S, w V, Dm^-1 to shared
// memory, weighted element forces to fe_w), then chunks of CS_EPC elements: the chunk's J rows
// land by cp.async (prefetched during the previous chunk's Gram), thread per (element, column)
// builds the B and w V dP(B) panels, and the warps run the DMMA Gram over the panels, k-steps
// dealt round-robin over the sim so every warp carries every tile: accumulators stay in
// registers for the whole sim and are summed over warps once, in a fixed order (deterministic).
struct CubSimsArgs {
  const int* rows_g;    // (n_elems, 12) free-DOF rows (-1 fixed)
  const double* Dm_g;   // (n_elems, 9)
  const double* vol_g;  // (n_elems)
  const double* BU;     // (n_elems, 9, n_p): B columns of the constant U block
  int n_elems;
  const double* w;      // (n_sims, n_elems) weights (nullptr: 1)
  const double* u;      // (n_sims, N)
  const double* Jt;     // (n_sims, N, ldjt): [U | J]
  int N, n, n_p, ldjt;
  double mu, lam;
  double* fe_w;         // (n_sims, n_elems, 12) weighted element forces
  double* part_f;       // (n_sims, n)   one partial per sim
  double* part_K;       // (n_sims, n*n)
  int skip_fe;
};
constexpr int CS_EPC = 8, CS_SUPER = 128, CS_FS = 25;  // FS: F 9 | S 6 | w V | Dm^-1 9
__host__ __device__ inline int cub_sims_ldq(int n_q) { return (n_q + 1) & ~1; }
inline size_t cub_sims_smem(int n, int n_p, int ti) {
  const int ldp = gram_ld(n), nt = ti * (ti + 1) / 2;
  const size_t panels = (size_t)2 * CS_EPC * 9 * ldp;
  return ((size_t)CS_SUPER * CS_FS + (size_t)CS_EPC * 12 * cub_sims_ldq(n - n_p) +
          std::max(panels, (size_t)8 * nt * 64)) * 8;
}

__device__ __forceinline__ void stvk_dP(const double* F, const double* S6, double lam2, double mu, const double* dF,
                                        double* dP) {
  // X = F^T dF, dS = mu (X + X^T) + lam tr(X) I, dP = dF S + F dS   (S6: S00 S11 S22 S01 S02 S12)
  double X[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) X[i * 3 + j] = F[i] * dF[j] + F[3 + i] * dF[3 + j] + F[6 + i] * dF[6 + j];
  const double tr = lam2 * (X[0] + X[4] + X[8]);
  const double dS00 = 2.0 * mu * X[0] + tr, dS11 = 2.0 * mu * X[4] + tr, dS22 = 2.0 * mu * X[8] + tr;
  const double dS01 = mu * (X[1] + X[3]), dS02 = mu * (X[2] + X[6]), dS12 = mu * (X[5] + X[7]);
  const double dS[9] = {dS00, dS01, dS02, dS01, dS11, dS12, dS02, dS12, dS22};
  const double S[9] = {S6[0], S6[3], S6[4], S6[3], S6[1], S6[5], S6[4], S6[5], S6[2]};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      dP[a * 3 + j] = dF[a * 3] * S[j] + dF[a * 3 + 1] * S[3 + j] + dF[a * 3 + 2] * S[6 + j] + F[a * 3] * dS[j] +
                      F[a * 3 + 1] * dS[3 + j] + F[a * 3 + 2] * dS[6 + j];
}

template <int TI, int MINB>
__global__ void __launch_bounds__(256, MINB) k_cub_sims(CubSimsArgs a) {
  constexpr int NT = TI * (TI + 1) / 2;  // upper 8 x 8 tiles of the (n x n+1) Gram
  extern __shared__ __align__(16) double sh[];
  const int n = a.n, n_p = a.n_p, nq = n - n_p, ldq = cub_sims_ldq(nq), ldp = gram_ld(n);
  double* FS = sh;                               // [CS_SUPER][CS_FS]
  double* Jg = FS + CS_SUPER * CS_FS;            // [CS_EPC * 12][ldq]  J columns of the chunk's rows
  double* Bp = Jg + CS_EPC * 12 * ldq;           // [CS_EPC * 9][ldp]   B rows (+ reduction space)
  double* Wp = Bp + CS_EPC * 9 * ldp;            // [CS_EPC * 9][ldp]   w V dP(B) rows | w V vec(P)
  const int sim = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* u = a.u + (size_t)sim * a.N;
  const double* Jq = a.Jt + (size_t)sim * a.N * a.ldjt + n_p;
  const bool v16 = ((n_p | a.ldjt) & 1) == 0;    // 16-byte aligned J columns
  pdl_wait();
  pdl_launch();
  // J rows of elements c0 .. c0 + CS_EPC - 1 into Jg by cp.async, two threads per row (measured
  // faster than one TMA bulk copy per 160-byte row: 0.70 vs 0.98 ms at cfg5), fixed rows zeroed
  auto gather = [&](int c0) {
    constexpr int TPR = 2;
    if (tid < CS_EPC * 12 * TPR) {
      const int rr = tid / TPR, h = tid % TPR;
      const int ei = c0 + rr / 12;
      const int row = ei < a.n_elems ? a.rows_g[(size_t)c0 * 12 + rr] : -1;
      double* dst = Jg + rr * ldq;
      const double* src = Jq + (size_t)max(row, 0) * a.ldjt;
      if (v16) {
        for (int k = 2 * h; k < nq; k += 2 * TPR) {
          if (row >= 0) cp_async16(dst + k, src + k, true);
          else dst[k] = dst[k + 1] = 0.0;
        }
      } else {
        for (int k = h; k < nq; k += TPR) {
          if (row >= 0) cp_async8(dst + k, src + k);
          else dst[k] = 0.0;
        }
      }
    }
    cp_async_commit();
  };
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  int ks_glob = 0;
  const double lam = a.lam, mu = a.mu;
  // this thread's panel tasks (chunk-invariant): (element, column) over the n columns, then the
  // CS_EPC force columns (j = n; they fall in one warp); <= 2 per thread since n < 32
  int tk_el[2], tk_j[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int t = tid + q * 256;
    const bool fcol = t >= CS_EPC * n;
    tk_el[q] = t < CS_EPC * (n + 1) ? (fcol ? t - CS_EPC * n : t / n) : -1;
    tk_j[q] = fcol ? n : t - (t / n) * n;
  }
  gather(0);
  for (int s0 = 0; s0 < a.n_elems; s0 += CS_SUPER) {
    const int ns = min(CS_SUPER, a.n_elems - s0);
    if (tid < ns) {
      // ------------------------------------------------ element physics (thread per element)
      const int ei = s0 + tid;
      double uv[12], Di[9];
#pragma unroll
      for (int l = 0; l < 12; ++l) {
        const int row = a.rows_g[(size_t)ei * 12 + l];
        uv[l] = row >= 0 ? u[row] : 0.0;
      }
#pragma unroll
      for (int l = 0; l < 9; ++l) Di[l] = a.Dm_g[(size_t)ei * 9 + l];
      const double V = a.vol_g[ei];
      const double we = a.w ? a.w[(size_t)sim * a.n_elems + ei] : 1.0;
      double F[9];
#pragma unroll
      for (int aa = 0; aa < 3; ++aa)
#pragma unroll
        for (int y = 0; y < 3; ++y) {
          double f = 0.0;
#pragma unroll
          for (int i = 0; i < 3; ++i) f = fma(uv[(i + 1) * 3 + aa] - uv[aa], Di[i * 3 + y], f);
          F[aa * 3 + y] = f + (aa == y ? 1.0 : 0.0);
        }
      double C[6];  // F^T F: 00 11 22 01 02 12
      C[0] = F[0] * F[0] + F[3] * F[3] + F[6] * F[6];
      C[1] = F[1] * F[1] + F[4] * F[4] + F[7] * F[7];
      C[2] = F[2] * F[2] + F[5] * F[5] + F[8] * F[8];
      C[3] = F[0] * F[1] + F[3] * F[4] + F[6] * F[7];
      C[4] = F[0] * F[2] + F[3] * F[5] + F[6] * F[8];
      C[5] = F[1] * F[2] + F[4] * F[5] + F[7] * F[8];
      const double trE = 0.5 * (C[0] + C[1] + C[2] - 3.0);
      double S6[6];
#pragma unroll
      for (int l = 0; l < 3; ++l) S6[l] = mu * (C[l] - 1.0) + lam * trE;
#pragma unroll
      for (int l = 3; l < 6; ++l) S6[l] = mu * C[l];
      double* fs = FS + tid * CS_FS;
#pragma unroll
      for (int l = 0; l < 9; ++l) fs[l] = F[l];
#pragma unroll
      for (int l = 0; l < 6; ++l) fs[9 + l] = S6[l];
      fs[15] = we * V;
#pragma unroll
      for (int l = 0; l < 9; ++l) fs[16 + l] = Di[l];
      if (!a.skip_fe) {
        // f_e[(v, aa)] = V sum_y P[aa][y] G[v][y],  P = F S
        const double S[9] = {S6[0], S6[3], S6[4], S6[3], S6[1], S6[5], S6[4], S6[5], S6[2]};
        double P[9];
        mat3_mul(F, S, P);
        double* fo = a.fe_w + ((size_t)sim * a.n_elems + ei) * 12;
#pragma unroll
        for (int aa = 0; aa < 3; ++aa) {
          double pg[3];
#pragma unroll
          for (int i = 0; i < 3; ++i)
            pg[i] = P[aa * 3] * Di[i * 3] + P[aa * 3 + 1] * Di[i * 3 + 1] + P[aa * 3 + 2] * Di[i * 3 + 2];
          fo[aa] = -we * V * (pg[0] + pg[1] + pg[2]);
#pragma unroll
          for (int i = 0; i < 3; ++i) fo[(i + 1) * 3 + aa] = we * V * pg[i];
        }
      }
    }
    for (int c0 = s0; c0 < s0 + ns; c0 += CS_EPC) {
      cp_async_all_wait();
      __syncthreads();  // the chunk's J rows landed, FS written, the previous Gram done with B / W
      // ---------------------------------------------------- B and w V dP(B) panels
      const int ne = min(CS_EPC, a.n_elems - c0);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int el = tk_el[q], j = tk_j[q];
        if (el < 0) continue;
        double* bcol = Bp + el * 9 * ldp + j;
        double* wcol = Wp + el * 9 * ldp + j;
        if (el >= ne) {
#pragma unroll
          for (int k = 0; k < 9; ++k) bcol[k * ldp] = wcol[k * ldp] = 0.0;
          continue;
        }
        const double* fs = FS + (c0 - s0 + el) * CS_FS;
        double F[9], S6[6];
#pragma unroll
        for (int l = 0; l < 9; ++l) F[l] = fs[l];
#pragma unroll
        for (int l = 0; l < 6; ++l) S6[l] = fs[9 + l];
        const double wv = fs[15];
        if (j == n) {  // force column: w V vec(P)
          const double S[9] = {S6[0], S6[3], S6[4], S6[3], S6[1], S6[5], S6[4], S6[5], S6[2]};
          double P[9];
          mat3_mul(F, S, P);
#pragma unroll
          for (int k = 0; k < 9; ++k) wcol[k * ldp] = wv * P[k];  // (B column n only reaches unstored outputs)
          continue;
        }
        double dF[9];
        if (j < n_p) {
          const double* bu = a.BU + (size_t)(c0 + el) * 9 * n_p + j;
#pragma unroll
          for (int k = 0; k < 9; ++k) dF[k] = bu[k * n_p];
        } else {
          const double* jr = Jg + el * 12 * ldq + (j - n_p);
          double x[12];
#pragma unroll
          for (int l = 0; l < 12; ++l) x[l] = jr[l * ldq];
#pragma unroll
          for (int aa = 0; aa < 3; ++aa)
#pragma unroll
            for (int y = 0; y < 3; ++y) {
              double f = 0.0;
#pragma unroll
              for (int i = 0; i < 3; ++i) f = fma(x[(i + 1) * 3 + aa] - x[aa], fs[16 + i * 3 + y], f);
              dF[aa * 3 + y] = f;
            }
        }
        double dP[9];
        stvk_dP(F, S6, lam, mu, dF, dP);
#pragma unroll
        for (int k = 0; k < 9; ++k) {
          bcol[k * ldp] = dF[k];
          wcol[k * ldp] = wv * dP[k];
        }
      }
      __syncthreads();  // panels complete; Jg free
      if (c0 + CS_EPC < a.n_elems) gather(c0 + CS_EPC);  // lands during the Gram
      // ---------------------------------------------------- Gram: upper tiles of B^T W
      constexpr int KS = CS_EPC * 9 / 4;
      const int kq = lane & 3, r8 = lane >> 2;
      for (int ks = (warp - ks_glob) & 7; ks < KS; ks += 8) {
        const double* bx = Bp + (4 * ks + kq) * ldp + r8;
        const double* wy = Wp + (4 * ks + kq) * ldp + r8;
        double av[TI], bv[TI];
#pragma unroll
        for (int t = 0; t < TI; ++t) {
          av[t] = bx[8 * t];
          bv[t] = wy[8 * t];
        }
        int t = 0;
#pragma unroll
        for (int bi = 0; bi < TI; ++bi)
#pragma unroll
          for (int bj = bi; bj < TI; ++bj, ++t) dmma(acc[t][0], acc[t][1], av[bi], bv[bj]);
      }
      ks_glob = (ks_glob + KS) & 7;
    }
  }
  // ------------------------------------------------------------ fixed-order sum over warps
  __syncthreads();
  double* red = Bp;  // [8][NT][64]
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    red[(warp * NT + t) * 64 + 2 * lane] = acc[t][0];
    red[(warp * NT + t) * 64 + 2 * lane + 1] = acc[t][1];
  }
  __syncthreads();
  double* K = a.part_K + (size_t)sim * n * n;
  double* f = a.part_f + (size_t)sim * n;
  for (int idx = tid; idx < NT * 64; idx += blockDim.x) {
    const int t = idx >> 6, q = idx & 63, ln = q >> 1, e = q & 1;
    double v = 0.0;
#pragma unroll
    for (int w8 = 0; w8 < 8; ++w8) v += red[(w8 * NT + t) * 64 + q];
    int bi = 0, rem = t;
    while (rem >= TI - bi) { rem -= TI - bi; ++bi; }
    const int bj = bi + rem;
    const int i = bi * 8 + (ln >> 2), j = bj * 8 + 2 * (ln & 3) + e;
    if (i >= n) continue;
    if (j < n) {
      K[(size_t)i * n + j] = v;
      if (bi != bj) K[(size_t)j * n + i] = v;
    } else if (j == n) {
      f[i] = v;
    }
  }
}

// Deterministic scatter of weighted element forces into the free-DOF vector (CSR over rows).
__global__ void k_scatter_rows(const int* __restrict__ row_ids, const int* __restrict__ row_ptr,
                               const int* __restrict__ entries, int n_rows, const double* __restrict__ fe_w,
                               int n_elems, double* __restrict__ f, int N, int n_sims) {
  pdl_wait();
  pdl_launch();
  const long long total = (long long)n_rows * n_sims;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int i = t % n_rows;
    int sim = t / n_rows;
    double acc = 0.0;
    for (int j = row_ptr[i]; j < row_ptr[i + 1]; ++j) acc += fe_w[(size_t)sim * n_elems * 12 + entries[j]];
    f[(size_t)sim * N + row_ids[i]] = acc;
  }
}

}  // namespace nlrom
