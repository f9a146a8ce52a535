// Assembly of the reduced Newton system, its reductions, the in-CTA LU solve and the
// top of the vhp backward (rdsim.residual / system_jacobian / step).
#pragma once
#include "cluster_async.cuh"
#include "common.cuh"
#include "mc_device.cuh"
#include "gram_dmma.cuh"

namespace nlrom {

// -------------------------------------------------------------------- assembly
// Per chunk of rows n (one CTA):
//   a_n = M_n (J~_n . c) + [M_n hvv_n] + dt^2 (f_n - fext_n),  c = (1+alpha dt)(r - r_bar) - dt rdot_bar
//   part[i][j] = sum_n J~_n[i] M_n R_n[j],  R_n = (1+alpha dt) J~_n + [0, dJ_n]      (n x n)
//   partphi[i] = sum_n J~_n[i] a_n                                                   (n)
// The n x n accumulation is register-blocked 4 x 4 per thread.
struct AsmArgs {
  const double* Jt; int ldjt;
  const double* dJ; int lddj;
  const double* mass;
  const double* hvv;
  const double* f;       // scattered cubature / exact force (n_sims, N)
  const double* fext;    // (n_sims, N)
  const double* r; const double* rbar; const double* rdbar;
  double* a;             // (n_sims, N)
  double* part;          // (n_sims, nchunk, n*n)
  double* partphi;       // (n_sims, nchunk, n)
  int N, n, n_p, n_q, rows_per_cta, nchunk;
  double dt, alpha;
  int drop_fict;
  int mode;              // 0: both, 1: mass block only (part), 2: a and J~^T a only (a, partphi)
};

__global__ void k_assemble(AsmArgs A) {
  pdl_wait();
  pdl_launch();
  extern __shared__ double sh[];
  const int n = A.n;
  const int RC = A.rows_per_cta;            // multiple of 4
  const int ldp = gram_ld(n);
  double* Js = sh;                          // [RC][ldp]  J~ rows
  double* Rs = Js + (size_t)RC * ldp;       // [RC][ldp]  M R rows, column n = a
  double* cs = Rs + (size_t)RC * ldp;       // [n]
  double* ms = cs + n;                      // [RC] mass
  double* fs = ms + RC;                     // [RC] row constant of a: dt^2 (f - fext) + M hvv
  const int chunk = blockIdx.x, sim = blockIdx.y;
  const double ah = A.alpha * A.dt;
  const int row0 = chunk * RC;
  const double* Jt = A.Jt + (size_t)sim * A.N * A.ldjt;
  const double* dJ = A.dJ + (size_t)sim * A.N * A.lddj;
  // stage J~ rows into Js and dJ rows into Rs[:, n_p:] (async copies: all loads in flight)
  for (int idx = threadIdx.x; idx < RC * n; idx += blockDim.x) {
    const int rl = idx / n, j = idx % n;
    const int row = row0 + rl;
    double* js = Js + rl * ldp + j;
    double* rs = Rs + rl * ldp + j;
    if (row < A.N) {
      cp_async8(js, Jt + (size_t)row * A.ldjt + j);
      if (A.mode != 2 && j >= A.n_p) cp_async8(rs, dJ + (size_t)row * A.lddj + (j - A.n_p));
    } else {
      *js = 0.0;
      *rs = 0.0;
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const size_t o = (size_t)sim * n + i;
    cs[i] = (1.0 + ah) * (A.r[o] - A.rbar[o]) - A.dt * A.rdbar[o];
  }
  for (int rl = threadIdx.x; rl < RC; rl += blockDim.x) {
    const int row = row0 + rl;
    double m = 0.0, fc = 0.0;
    if (row < A.N) {
      const size_t o = (size_t)sim * A.N + row;
      m = A.mass[row];
      if (A.mode != 1) {
        fc = A.dt * A.dt * (A.f[o] - A.fext[o]);
        if (!A.drop_fict) fc += m * A.hvv[o];
      }
    }
    ms[rl] = m;
    fs[rl] = fc;
  }
  cp_async_all_wait();
  __syncthreads();
  if (A.mode != 2)
    for (int idx = threadIdx.x; idx < RC * n; idx += blockDim.x) {
      const int rl = idx / n, j = idx % n;
      const double dj = (j >= A.n_p) ? Rs[rl * ldp + j] : 0.0;
      Rs[rl * ldp + j] = ((1.0 + ah) * Js[rl * ldp + j] + dj) * ms[rl];
    }
  // a_n (one warp per row) into column n of Rs
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int rl = warp; A.mode != 1 && rl < RC; rl += nw) {
    const int row = row0 + rl;
    double acc = 0.0;
    for (int j = lane; j < n; j += 32) acc = fma(Js[rl * ldp + j], cs[j], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      double av = 0.0;
      if (row < A.N) {
        av = ms[rl] * acc + fs[rl];
        A.a[(size_t)sim * A.N + row] = av;
      }
      Rs[rl * ldp + n] = av;
    }
  }
  __syncthreads();
  // [J~^T M R | J~^T a] for the chunk on the DMMA pipe: n x (n + 1), split into part / partphi
  double* P = A.part + ((size_t)sim * A.nchunk + chunk) * n * n;
  double* Pp = A.partphi + ((size_t)sim * A.nchunk + chunk) * n;
  if (A.mode != 2) gram_dmma(Js, ldp, Rs, ldp, RC, n, n, P, n);
  if (A.mode != 1) gram_dmma(Js, ldp, Rs + n, ldp, RC, n, 1, Pp, 1);
}

// Mass block of the system matrix for chunks of RC rows (the side-branch half of the assembly,
// mode 1 of k_assemble): partA[p] = sum over the CTA's cpm row chunks of
// J~_rows^T M [(1+ah) U, (1+ah) J + dJ]_rows. J~ rows (global pitch ldjt == the Gram panel pitch),
// dJ rows and the masses land by three TMA bulk copies per chunk (one mbarrier phase each); the
// Gram product runs on the DMMA pipe. cpm > 1 (many sims): the Gram accumulates in shared
// memory and each CTA writes one partial (nchunk = partials per sim), so the partial traffic and
// its reduction shrink by cpm.
__global__ void __launch_bounds__(256) k_assemble_mass(const double* __restrict__ Jt, int ldjt,
                                                       const double* __restrict__ dJ, int lddj,
                                                       const double* __restrict__ mass, int N, int n, int n_p,
                                                       int RC, int nchunk, double ah, double* __restrict__ part,
                                                       int cpm) {
  pdl_wait();
  pdl_launch();
  extern __shared__ __align__(16) double sh[];
  const int ldp = ldjt;
  double* Js = sh;                     // [RC][ldp]
  double* Rs = Js + (size_t)RC * ldp;  // [RC][ldp]
  double* Ds = Rs + (size_t)RC * ldp;  // [RC][lddj]
  double* ms = Ds + (size_t)RC * lddj; // [RC]
  uint64_t* bar = reinterpret_cast<uint64_t*>(ms + RC);
  double* Kacc = reinterpret_cast<double*>(bar + 2);  // [n][n] when cpm > 1
  const int sim = blockIdx.y, tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  for (int ck = 0; ck < cpm; ++ck) {
    const int chunk = blockIdx.x * cpm + ck;
    const int row0 = chunk * RC;
    if (row0 >= N) break;  // uniform over the CTA
    const int nrow = min(RC, N - row0);
    __syncthreads();  // barrier init visible; the previous chunk's Gram is done with Js / Rs
    if (tid == 0) {
      fence_proxy_async();
      const uint32_t bj = (uint32_t)(nrow * ldjt * 8), bd = (uint32_t)(nrow * lddj * 8), bm = (uint32_t)(nrow * 8);
      mbar_expect_tx(bar, bj + bd + (nrow % 2 == 0 ? bm : 0));
      tma_g2s(Js, Jt + ((size_t)sim * N + row0) * ldjt, bj, bar);
      tma_g2s(Ds, dJ + ((size_t)sim * N + row0) * lddj, bd, bar);
      if (nrow % 2 == 0) tma_g2s(ms, mass + row0, bm, bar);
    }
    if (nrow % 2 != 0)
      for (int i = tid; i < nrow; i += blockDim.x) ms[i] = mass[row0 + i];
    for (int t = tid; t < (RC - nrow) * ldp; t += blockDim.x) {  // zero tail rows of the last chunk
      Js[(size_t)nrow * ldp + t] = 0.0;
      Rs[(size_t)nrow * ldp + t] = 0.0;
    }
    __syncthreads();
    mbar_wait(bar, (uint32_t)(ck & 1));
    for (int t = tid; t < nrow * n; t += blockDim.x) {
      const int rl = t / n, j = t % n;
      const double dj = (j >= n_p) ? Ds[rl * lddj + (j - n_p)] : 0.0;
      Rs[rl * ldp + j] = ((1.0 + ah) * Js[rl * ldp + j] + dj) * ms[rl];
    }
    __syncthreads();
    if (cpm == 1) gram_dmma(Js, ldp, Rs, ldp, RC, n, n, part + ((size_t)sim * nchunk + blockIdx.x) * n * n, n);
    else gram_dmma(Js, ldp, Rs, ldp, RC, n, n, Kacc, n, ck > 0);  // warp-owned tiles: no race
  }
  if (cpm > 1) {
    __syncthreads();
    double* P = part + ((size_t)sim * nchunk + blockIdx.x) * n * n;
    for (int t = tid; t < n * n; t += blockDim.x) P[t] = Kacc[t];
  }
}

// The critical-path half of the assembly for one chunk of RC <= 128 rows, with the weighted
// element forces gathered per row through a full-row CSR (no separate scatter launch):
//   a_row = m (J~_row . c) + dt^2 (f_row - fext_row) + m hvv_row,   f_row = sum_{(e,l) -> row} w_e f_e[l]
//   partphi[chunk] = J~_chunk^T a_chunk
// 256 threads: 2 per row for the dot products and the gather, then 4 row quarters x 64 columns.
struct AsmAArgs {
  const double* Jt; int ldjt;
  const double* mass; const double* hvv; const double* fext;
  const double* r; const double* rbar; const double* rdbar;
  const int* rowptr;       // (N + 1): CSR over all free-DOF rows
  const int* entries;      // element slot * 12 + l
  const double* fe_w;      // (n_sims, n_elems, 12)
  int n_elems;
  double* a; double* partphi;
  int N, n, RC, nchunk;
  double dt, alpha;
  int drop_fict;
  // optional, fused (P W_L)^T a for the vhp chain: gpart[sim][chunk][M] = sum_rows PW[row][:] a_row
  const double* PW; int ldPW, M;
  double* gpart;
};

// Programmatic-launch overlap: the J~ . c dot products (J~, hvv: output layer; r, r_bar,
// rdot_bar: state) run before the dependency wait -- the producer (k_cubature) launches
// dependents only after its own wait, so the output layer has completed -- and only the
// gathered element forces (cubature output) are read after it.
// With A.gpart (RC <= 32, M <= 256): the seed of the vhp chain, (P W_L)^T a, is accumulated here
// per chunk (the chain's prologue sums the chunk partials): each thread owns one column of P W_L
// and loads its RC entries (constants) before the dependency wait.
constexpr int ASMA_GROWS = 32;
// GP = false (no vhp seed partials: the batched path): 8 threads per row for the dot products and
// the gather (coalesced 64-byte row segments, 4 rows per warp) and no (P W_L) registers, so 4x the
// resident warps (cfg5: 0.67 ms, 24% warps active with the 2-threads-per-row GP layout).
template <bool GP>
__global__ void __launch_bounds__(256) k_assemble_a(AsmAArgs A) {
  __shared__ double cs[128];
  __shared__ double as[128];
  __shared__ double red[4][64];
  const int chunk = blockIdx.x, sim = blockIdx.y, tid = threadIdx.x;
  const int n = A.n;
  const double ah = A.alpha * A.dt;
  double pw[GP ? ASMA_GROWS : 1];
  const bool gcol = GP && A.gpart && tid < A.M;
  if (GP && A.gpart) {
#pragma unroll
    for (int rl = 0; rl < ASMA_GROWS; ++rl) {
      const int row = chunk * A.RC + rl;
      pw[rl] = (gcol && rl < A.RC && row < A.N) ? A.PW[(size_t)row * A.ldPW + tid] : 0.0;
    }
  }
  for (int i = tid; i < n; i += blockDim.x) {
    const size_t o = (size_t)sim * n + i;
    cs[i] = (1.0 + ah) * (A.r[o] - A.rbar[o]) - A.dt * A.rdbar[o];
  }
  __syncthreads();
  const int row0 = chunk * A.RC;
  const double* Jsim = A.Jt + (size_t)sim * A.N * A.ldjt;
  if constexpr (!GP) {
    pdl_wait();
    pdl_launch();
    for (int rl0 = 0; rl0 < A.RC; rl0 += 32) {
      const int rl = rl0 + (tid >> 3), h = tid & 7;
      const int row = row0 + rl;
      double acc = 0.0, fs = 0.0;
      if (rl < A.RC && row < A.N) {
        const double* Jr = Jsim + (size_t)row * A.ldjt;
        for (int j = h; j < n; j += 8) acc = fma(Jr[j], cs[j], acc);
        const double* fw = A.fe_w + (size_t)sim * A.n_elems * 12;
        for (int k = A.rowptr[row] + h; k < A.rowptr[row + 1]; k += 8) fs += fw[A.entries[k]];
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        fs += __shfl_xor_sync(0xffffffffu, fs, o);
      }
      if (h == 0 && rl < A.RC) {
        double av = 0.0;
        if (row < A.N) {
          const size_t o = (size_t)sim * A.N + row;
          const double m = A.mass[row];
          av = m * acc + A.dt * A.dt * (fs - A.fext[o]);
          if (!A.drop_fict) av += m * A.hvv[o];
          A.a[o] = av;
        }
        as[rl] = av;
      }
    }
  } else {
    const int rl = tid >> 1, h = tid & 1;
    const int row = row0 + rl;
    double acc = 0.0, fs = 0.0;
    if (rl < A.RC && row < A.N) {
      const double* Jr = Jsim + (size_t)row * A.ldjt;
      for (int j = h; j < n; j += 2) acc = fma(Jr[j], cs[j], acc);
    }
    pdl_wait();
    pdl_launch();
    if (rl < A.RC && row < A.N) {
      const double* fw = A.fe_w + (size_t)sim * A.n_elems * 12;
      for (int k = A.rowptr[row] + h; k < A.rowptr[row + 1]; k += 2) fs += fw[A.entries[k]];
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    fs += __shfl_xor_sync(0xffffffffu, fs, 1);
    if (h == 0 && rl < A.RC) {
      double av = 0.0;
      if (row < A.N) {
        const size_t o = (size_t)sim * A.N + row;
        const double m = A.mass[row];
        av = m * acc + A.dt * A.dt * (fs - A.fext[o]);
        if (!A.drop_fict) av += m * A.hvv[o];
        A.a[o] = av;
      }
      as[rl] = av;
    }
  }
  __syncthreads();
  if (GP && A.gpart) {
    double g0 = 0.0, g1 = 0.0;
#pragma unroll
    for (int rl = 0; rl < ASMA_GROWS; rl += 2) {
      g0 = fma(pw[rl], as[rl], g0);
      g1 = fma(pw[rl + 1], as[rl + 1], g1);
    }
    if (gcol) A.gpart[((size_t)sim * A.nchunk + chunk) * A.M + tid] = g0 + g1;
  }
  const int q = tid >> 6, jl = tid & 63;
  for (int j0 = 0; j0 < n; j0 += 64) {
    const int j = j0 + jl;
    double acc = 0.0;
    if (j < n)
      for (int rl = q; rl < A.RC; rl += 4) {
        const int row = row0 + rl;
        if (row < A.N) acc = fma(Jsim[(size_t)row * A.ldjt + j], as[rl], acc);
      }
    red[q][jl] = acc;
    __syncthreads();
    if (q == 0 && j < n)
      A.partphi[((size_t)sim * A.nchunk + chunk) * n + j] = (red[0][jl] + red[1][jl]) + (red[2][jl] + red[3][jl]);
    __syncthreads();
  }
}

// Many small systems (n <= 32: cfg5 solves 4096 of n = 30 per Newton iteration): one warp per
// system instead of one CTA. Lane i owns row i of [S + diag(0, vhp) | -phi] in registers; partial
// pivoting (max |a_ik| over rows i >= k, the lowest row on ties, as the CTA kernels) and Gauss-Jordan
// elimination by shuffles -- no shared memory, no barriers; with k and j unrolled at compile time
// only the live columns j >= k are exchanged. Same outputs as k_lu_lookahead (dr, r += dr when
// apply, status 1 on a zero / non-finite pivot without writing dr).
__global__ void __launch_bounds__(256, 2) k_lu_warp(const double* __restrict__ S, const double* __restrict__ phi,
                                                 double* __restrict__ dr, double* __restrict__ r, int n, int apply,
                                                 int* __restrict__ status, const double* __restrict__ Gt, int ldg,
                                                 int n_p, int n_sims) {
  pdl_wait();
  pdl_launch();
  constexpr int NP = 33;   // n + 1 <= 33 columns [A | b]
  const int lane = threadIdx.x & 31;
  const int sim = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (sim >= n_sims) return;   // warp-uniform
  const int nq = n - n_p;
  double a[NP];
  const double* Sr = S + (size_t)sim * n * n + (size_t)lane * n;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    double v = 0.0;
    if (lane < n) {
      if (j < n) v = Sr[j];
      else if (j == n) v = -phi[(size_t)sim * n + lane];
      if (Gt && lane >= n_p && j >= n_p && j < n) v += Gt[((size_t)sim * 2 * nq + 2 * (j - n_p) + 1) * ldg + (lane - n_p)];
    }
    a[j] = v;
  }
  bool bad = false;
#pragma unroll
  for (int k = 0; k < NP - 1; ++k) {
    if (k >= n) break;   // uniform
    // pivot row p: max |a_ik| over i >= k, the lowest i on ties
    double v = (lane >= k && lane < n) ? fabs(a[k]) : -1.0;
    int p = lane;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int op = __shfl_xor_sync(0xffffffffu, p, o);
      if (ov > v || (ov == v && op < p)) {
        v = ov;
        p = op;
      }
    }
    if (!(v > 0.0) || !isfinite(v)) bad = true;
    // rows k and p exchange their live columns
    const int src = lane == k ? p : (lane == p ? k : lane);
#pragma unroll
    for (int j = k; j < NP; ++j) a[j] = __shfl_sync(0xffffffffu, a[j], src);
    const double rp = 1.0 / __shfl_sync(0xffffffffu, a[k], k);
    const double l = a[k] * rp;
#pragma unroll
    for (int j = k + 1; j < NP; ++j) {
      const double pkj = __shfl_sync(0xffffffffu, a[j], k);
      if (lane != k) a[j] = fma(-l, pkj, a[j]);
    }
  }
  if (bad) {
    if (lane == 0) status[sim] = 1;
    return;
  }
  // x_i = b_i / a_ii (row i is on lane i after the exchanges)
  double d = 1.0, b = 0.0;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    if (j == lane) d = a[j];
    if (j == n) b = a[j];
  }
  if (lane < n) {
    const double x = b * (1.0 / d);
    dr[(size_t)sim * n + lane] = x;
    if (apply) r[(size_t)sim * n + lane] += x;
  }
  if (lane == 0) status[sim] = 0;
}

// phi = sum_chunks partphi (one CTA per sim; 8 chunk groups per output, smem combine), ||phi||_2
__global__ void k_reduce_phi(const double* __restrict__ partphi, int nchunk, int n, double* __restrict__ phi,
                             double* __restrict__ norm) {
  pdl_wait();
  pdl_launch();
  extern __shared__ double sh[];  // [8][n]
  const int sim = blockIdx.x;
  const int groups = blockDim.x / 32 > 0 ? 8 : 1;
  for (int t = threadIdx.x; t < 8 * n; t += blockDim.x) {
    int i = t % n, gidx = t / n;
    double acc = 0.0;
    for (int c = gidx; c < nchunk; c += 8) acc += partphi[((size_t)sim * nchunk + c) * n + i];
    sh[gidx * n + i] = acc;
  }
  __syncthreads();
  __shared__ double red[32];
  double sq = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double acc = 0.0;
#pragma unroll
    for (int gidx = 0; gidx < 8; ++gidx) acc += sh[gidx * n + i];
    phi[(size_t)sim * n + i] = acc;
    sq += acc * acc;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    norm[sim] = sqrt(s);
  }
  (void)groups;
}

// S = sum part_A + dt^2 sum part_K + diag(0, vhp);  vhp[i][k] = G_t[2k+1][i].
// grid (ceil(n*n/32), n_sims), block 256: 32 outputs x 8 partial groups.
__global__ void k_reduce_S(const double* __restrict__ partA, int nchA, const double* __restrict__ partK, int nchK,
                           const double* __restrict__ Gt, int ldg, int n, int n_p, int n_q, double dt,
                           double* __restrict__ S) {
  pdl_wait();
  pdl_launch();
  // block-stride over 32-output blocks: the side-branch launch uses few CTAs so that it does not
  // hold SMs the concurrently scheduled 16-CTA clusters of the vhp chain need
  __shared__ double red[8][32];
  const int sim = blockIdx.y;
  const int lane = threadIdx.x & 31, gidx = threadIdx.x >> 5;
  const int nn = n * n;
  for (int ob = blockIdx.x; ob * 32 < nn; ob += gridDim.x) {
    const int idx = ob * 32 + lane;
    double a = 0.0, k = 0.0;
    if (idx < nn) {
      for (int c = gidx; c < nchA; c += 8) a += partA[((size_t)sim * nchA + c) * nn + idx];
      for (int c = gidx; c < nchK; c += 8) k += partK[((size_t)sim * nchK + c) * nn + idx];
    }
    red[gidx][lane] = a + dt * dt * k;
    __syncthreads();
    if (gidx == 0 && idx < nn) {
      double acc = 0.0;
#pragma unroll
      for (int g2 = 0; g2 < 8; ++g2) acc += red[g2][lane];
      const int i = idx / n, j = idx % n;
      if (Gt && i >= n_p && j >= n_p) acc += Gt[((size_t)sim * 2 * n_q + 2 * (j - n_p) + 1) * ldg + (i - n_p)];
      S[(size_t)sim * nn + idx] = acc;
    }
    __syncthreads();
  }
}

// k_reduce_S for many sims (each with few partials): one thread per output element (k_reduce_S's
// 8-way CTA split left 7 of 8 threads idle and launched 29 x n_sims CTAs: cfg5 0.35 ms)
__global__ void k_reduce_S_flat(const double* __restrict__ partA, int nchA, const double* __restrict__ partK,
                                int nchK, const double* __restrict__ Gt, int ldg, int n, int n_p, int n_q, double dt,
                                double* __restrict__ S, int n_sims) {
  pdl_wait();
  pdl_launch();
  const int nn = n * n;
  const long long total = (long long)n_sims * nn;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const int sim = (int)(t / nn), idx = (int)(t % nn);
    double a = 0.0, k = 0.0;
    for (int c = 0; c < nchA; ++c) a += partA[((size_t)sim * nchA + c) * nn + idx];
    for (int c = 0; c < nchK; ++c) k += partK[((size_t)sim * nchK + c) * nn + idx];
    double acc = a + dt * dt * k;
    const int i = idx / n, j = idx % n;
    if (Gt && i >= n_p && j >= n_p) acc += Gt[((size_t)sim * 2 * n_q + 2 * (j - n_p) + 1) * ldg + (i - n_p)];
    S[t] = acc;
  }
}

// sum of cubature partials (cubature_integrate): f~ (n), K~ (n,n)
__global__ void k_reduce_cub(const double* __restrict__ part_f, const double* __restrict__ part_K, int nch, int n,
                             double* __restrict__ f_red, double* __restrict__ K_red) {
  pdl_wait();
  pdl_launch();
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n * n + n; t += gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (t < n * n) {
      for (int c = 0; c < nch; ++c) acc += part_K[(size_t)c * n * n + t];
      K_red[t] = acc;
    } else {
      int i = t - n * n;
      for (int c = 0; c < nch; ++c) acc += part_f[(size_t)c * n + i];
      f_red[i] = acc;
    }
  }
}

// --------------------------------------------------------------------------- LU
// One CTA (256 threads = 16 x 16) per sim: elimination with partial pivoting on
// [S | -phi | extra rhs]. The matrix lives in shared memory; thread (ty, tx)
// owns the NB x NB elements (ty + 16a, tx + 16b), keeps them in registers and writes
// them back after every update. Every warp finds the pivot itself (exact argmax of
// |A[i][k]| over unused rows via integer warp reductions on the IEEE bits, lowest row on
// ties, as LAPACK idamax), so a pivot step needs ONE barrier: within a step only
// columns > k of non-pivot rows are written while the pivot row and column k are read.
// Pivoting is implicit (rows are marked used instead of swapped). Gauss-Jordan form: the
// used rows are eliminated too, which costs no latency here (every thread updates its block
// in parallel anyway) and turns the sequential back substitution into one division per
// unknown. Same pivot sequence as LU-pp; results agree to roundoff. If `apply`, r += dr.
// status[sim] = 1 on a zero pivot.
// 1/p on the pivot critical path: MUFU reciprocal seed + two Newton steps (error <= 1 ulp;
// the IEEE-rounded division costs ~3x the latency here). |p| is a partial pivot, never
// denormal for a non-singular Newton matrix.
__device__ __forceinline__ double recip_fast(double p) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
  double e = fma(-p, r, 1.0);
  r = fma(r, e, r);
  e = fma(-p, r, 1.0);
  return fma(r, e, r);
}

#ifdef LU_CYCLES
__device__ long long g_lu_cycles[2];  // tools/probes/lu_warp_probe.cu: cycles of the pivot loop
#endif

template <int NB>
__global__ void __launch_bounds__(256) k_lu_solve(const double* __restrict__ S, const double* __restrict__ phi,
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
    for (int b = 0; b < NB; ++b) M[(ty + 16 * a) * LDF + tx + 16 * b] = A[a][b];
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
    const double rp = recip_fast(M[piv * LDF + k]);
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
      act[a] = (i < n) && (i != piv);  // Gauss-Jordan: every row but the pivot row is eliminated
      l[a] = M[i * LDF + k];
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
      }
    }
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

#ifndef LU_RB
#define LU_RB 16   // trailing-update row block (tools/probes/lu_blocked_probe.cu -DLU_RB=8)
#endif
#ifdef LU_TRACE
__device__ long long g_lu_trace[4 * 16 + 6];   // tools/probes/lu_blocked_probe.cu -DLU_TRACE: panels | start, staged, factored, end
__device__ long long g_lu_trace_u[4 * 16];
#endif
// Look-ahead panel LU (same pivots, same multipliers, same fma sequence per element as
// k_lu_solve: bitwise-equal results, tools/probes/lu_blocked_probe.cu). One warp owns the pivot
// chain: it factors an 8-column panel in registers (exact REDUX argmax, reciprocal of |p| from the
// reduced key while the row index reduction and the pivot-row shuffles run, multipliers, rank-1
// updates of the remaining panel columns), publishes the panel's multipliers, and then brings the
// NEXT panel's 8 columns up to date itself (pivot-row entries from its own registers, the
// u-chain of the panel's pivot rows, 8 fmas per element) -- so it never waits for the trailing
// update. Warps 1-7 apply each published panel to the columns beyond the next panel; a column is
// owned by one warp for the whole factorisation (column j -> warp 1 + j mod 7), so updates of one
// column need no cross-warp ordering. Hand-offs are counters in shared memory (the panel warp
// waits for the trailing update of panel P-1 before reading panel P+1's columns), no CTA barrier
// inside the factorisation. Gauss-Jordan form and implicit pivoting as k_lu_solve.
template <int NB, int PW = 4>
__global__ void __launch_bounds__(256) k_lu_lookahead(const double* __restrict__ S, const double* __restrict__ phi,
                                                       double* __restrict__ dr, double* __restrict__ r, int n, int apply,
                                                       int* __restrict__ status, const double* __restrict__ xrhs, int nx,
                                                       double* __restrict__ xout, const double* __restrict__ Gt, int ldg,
                                                       int n_p) {
  pdl_wait();
  pdl_launch();
#ifdef LU_TRACE
  if (threadIdx.x == 0) g_lu_trace[64] = clock64();
#endif
  constexpr int D = 16 * NB;
  constexpr int LDF = D + 1;
  constexpr int R = D / 32;            // rows per lane (PW: panel width)
#ifndef LU_SOLO
#define LU_SOLO 0   // 1: warp 4 idles so the pivot-chain warp has its scheduler (SMSP 0) to itself
#endif
  constexpr int NU = LU_SOLO ? 6 : 7;  // trailing-update warps
  extern __shared__ double M[];        // [D][LDF] | vhp block [n_q][n_q] | Mul [2][D][PW]
  __shared__ int pivrow[D];
  __shared__ double rdiag[D];
  __shared__ volatile int fact_cnt;    // panels factored (multipliers published)
  __shared__ volatile int upd_cnt[NU]; // panels applied by each update warp
  __shared__ volatile int bad_s;
  const int sim = blockIdx.x;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31, warp = tid >> 5;
  const double* Ss = S + (size_t)sim * n * n;
  const int nq = n - n_p;
  double* Vs = M + D * LDF;
  double* Mul = Vs + ((nq * nq + 1) & ~1);   // 16-byte aligned multiplier panels
  const int ncol = n + 1 + nx;
  const int npan = (n + PW - 1) / PW;
  if constexpr (NB > 6) {
    // wide matrices: asynchronous copies, then one pass (negate phi, add the vhp block); the
    // one-pass register staging below measured slower here (n = 100, 124)
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
#pragma unroll
    for (int a = 0; a < NB; ++a)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int i = ty + 16 * a, j = tx + 16 * b;
        double v = M[i * LDF + j];
        if (j == n) v = -v;  // rhs = -phi
        if (Gt && i >= n_p && j >= n_p && i < n && j < n) v += Vs[(j - n_p) * nq + (i - n_p)];
        M[i * LDF + j] = v;
      }
  } else {
    // staging in one pass: every thread loads its (row, column) entries of [S + diag(0, V) | -phi |
    // extra rhs] straight from global memory (all loads in flight at once; the vhp block V[i][j] =
    // Gt[2 j + 1][i] of the sim) and stores them once. Thread (ty, tx) owns rows ty + 16 a, columns
    // tx + 16 b.
    double stg[NB][NB];
#pragma unroll
    for (int a = 0; a < NB; ++a)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int i = ty + 16 * a, j = tx + 16 * b;
        double v = 0.0;
        if (i < n) {
          if (j < n) v = Ss[(size_t)i * n + j];
          else if (j == n) v = -phi[(size_t)sim * n + i];
          else if (j <= n + nx) v = xrhs[((size_t)sim * nx + (j - n - 1)) * n + i];
        }
        stg[a][b] = v;
      }
    if (Gt) {
#pragma unroll
      for (int a = 0; a < NB; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int i = ty + 16 * a, j = tx + 16 * b;
          if (i >= n_p && j >= n_p && i < n && j < n)
            stg[a][b] += Gt[((size_t)sim * 2 * nq + 2 * (j - n_p) + 1) * ldg + (i - n_p)];
        }
    }
#pragma unroll
    for (int a = 0; a < NB; ++a)
#pragma unroll
      for (int b = 0; b < NB; ++b) M[(ty + 16 * a) * LDF + tx + 16 * b] = stg[a][b];
  }
  // the iterate's entries this thread will update at the end (apply), fetched while the LU runs
  double r_old[(D + 255) / 256];
#pragma unroll
  for (int q = 0; q < (D + 255) / 256; ++q) {
    const int t = tid + 256 * q;
    r_old[q] = (NB <= 6 && apply && t < n) ? r[(size_t)sim * n + t] : 0.0;
  }
  if (tid == 0) {
    fact_cnt = 0;
    bad_s = 0;
  }
  if (tid < NU) upd_cnt[tid] = 0;
  __syncthreads();
#ifdef LU_TRACE
  if (threadIdx.x == 0) g_lu_trace[65] = clock64();
#endif
  if (warp == 0) {
    // ------------------------------------------------------------------ pivot-chain warp
    bool used[R];
#pragma unroll
    for (int u = 0; u < R; ++u) used[u] = lane + 32 * u >= n;
    double pv[R][PW];
#pragma unroll
    for (int u = 0; u < R; ++u)
#pragma unroll
      for (int c = 0; c < PW; ++c) pv[u][c] = c < n ? M[(lane + 32 * u) * LDF + c] : 0.0;
    for (int P = 0; P < npan; ++P) {
      const int c0 = P * PW, kw = min(PW, n - c0);
      double* MulP = Mul + (P & 1) * D * PW;
      bool bad = false;
#ifdef LU_TRACE
      if (lane == 0 && P < 16) g_lu_trace[4 * P] = clock64();
#endif
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
        const unsigned long long key = (best >= 0.0) ? (unsigned long long)__double_as_longlong(best) : 0ull;
        const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        const double rabs = recip_fast(__hiloint2double((int)mhi, (int)mlo));
        const int piv = (int)__reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? (unsigned)bi : 0x7fffffffu);
        if (!(mhi | mlo) || piv >= n) { bad = true; break; }
        const int up = piv >> 5, lp = piv & 31;
#pragma unroll
        for (int u = 0; u < R; ++u) used[u] = used[u] || (u == up && lane == lp);
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
          MulP[i * PW + kk] = m;
#pragma unroll
          for (int c = kk + 1; c < PW; ++c) pv[u][c] = fma(-m, prow[c], pv[u][c]);
        }
      }
      __syncwarp();
      if (bad) {
        if (lane == 0) {
          bad_s = 1;
          __threadfence_block();
          fact_cnt = 1 << 30;
        }
        break;
      }
      if (lane == 0) {
        __threadfence_block();
        fact_cnt = P + 1;   // the update warps may apply panel P
      }
#ifdef LU_TRACE
      if (lane == 0 && P < 16) g_lu_trace[4 * P + 1] = clock64();
#endif
      if (P + 1 < npan) {
        // next panel's columns: up to date through panel P - 1 once the update warps are done with it
        if (P >= 1) {
          if (lane == 0)
            while (upd_cnt[0] < P) {}
          __syncwarp();
        }
#ifdef LU_TRACE
        if (lane == 0 && P < 16) g_lu_trace[4 * P + 2] = clock64();
#endif
        const int c1 = c0 + PW, kw1 = min(PW, n - c1);
        int pk[PW];
        double mrow[R][PW], mk[PW][PW];
#pragma unroll
        for (int kk = 0; kk < PW; ++kk) {
          pk[kk] = kk < kw ? pivrow[c0 + kk] : 0;  // pivrow / MulP of this panel: this warp's own stores
#pragma unroll
          for (int k2 = 0; k2 < PW; ++k2) mk[kk][k2] = (kk < kw && k2 < kk) ? MulP[pk[kk] * PW + k2] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < R; ++u)
#pragma unroll
          for (int kk = 0; kk < PW; ++kk) mrow[u][kk] = kk < kw ? MulP[(lane + 32 * u) * PW + kk] : 0.0;
        // 4 columns at a time: the panel's pivot rows at these columns straight from the shared
        // matrix (up to date through panel P - 1, broadcast loads), their u-chains (independent
        // across the 4 columns), then every lane's rows
        static_assert(PW % 4 == 0, "panel width");
#pragma unroll
        for (int c4 = 0; c4 < PW; c4 += 4) {
          double raw[4][PW], x[4][R];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const bool live = c4 + c < kw1;
#pragma unroll
            for (int kk = 0; kk < PW; ++kk) raw[c][kk] = (live && kk < kw) ? M[pk[kk] * LDF + c1 + c4 + c] : 0.0;
#pragma unroll
            for (int u = 0; u < R; ++u) x[c][u] = live ? M[(lane + 32 * u) * LDF + c1 + c4 + c] : 0.0;
          }
          double uk[4][PW];
#pragma unroll
          for (int kk = 0; kk < PW; ++kk)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double v = raw[c][kk];
#pragma unroll
              for (int k2 = 0; k2 < kk; ++k2) v = fma(-mk[kk][k2], uk[c][k2], v);
              uk[c][kk] = v;
            }
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int u = 0; u < R; ++u) {
              double v = x[c][u];
#pragma unroll
              for (int kk = 0; kk < PW; ++kk) v = fma(-mrow[u][kk], uk[c][kk], v);
              pv[u][c4 + c] = v;
            }
        }
      }
    }
  } else if (!(LU_SOLO && warp == 4)) {
    // ------------------------------------------------------------------ trailing-update warps
    // work unit = (32-column group, 16-row block), lanes = columns; unit u belongs to warp 1 + u % 7
    // for the whole factorisation. Per panel: every unit's u-chain from the pivot rows (read by all
    // units before any unit writes: named barrier), then its rows.
    constexpr int RB = LU_RB, NRB = D / RB;
    const int uw = (LU_SOLO && warp > 4) ? warp - 2 : warp - 1, ut = tid - 32;
    const int ngrp = (ncol + 31) / 32;
    for (int P = 0; P < npan; ++P) {
#ifdef LU_TRACE
      if (ut == 0 && P < 16) g_lu_trace_u[4 * P] = clock64();
#endif
      if (lane == 0)
        while (fact_cnt < P + 1) {}
      __syncwarp();   // the publisher fenced before its flag store; our loads follow the flag read
      if (bad_s) break;
#ifdef LU_TRACE
      if (ut == 0 && P < 16) g_lu_trace_u[4 * P + 1] = clock64();
#endif
      const int c0 = P * PW, kw = min(PW, n - c0);
      const double* MulP = Mul + (P & 1) * D * PW;
      const int c1 = c0 + PW;
      const int jlo = (P + 1 < npan) ? c1 + min(PW, n - c1) : c0 + kw;   // beyond the next panel
      int pk[PW];
      double mk[PW][PW];
#pragma unroll
      for (int kk = 0; kk < PW; ++kk) {
        pk[kk] = kk < kw ? pivrow[c0 + kk] : 0;
#pragma unroll
        for (int k2 = 0; k2 < PW; ++k2) mk[kk][k2] = (kk < kw && k2 < kk) ? MulP[pk[kk] * PW + k2] : 0.0;
      }
      // u-chains of this warp's units (one per column group it owns: the same for all its row blocks)
      constexpr int MAXU = (4 * NRB + NU - 1) / NU;   // units per warp (<= 4 column groups)
      double uk[MAXU][PW];
      int nu = 0;
#pragma unroll
      for (int q = 0; q < MAXU; ++q) {
        const int unit = uw + q * NU, g = unit / NRB;
        const int j = g * 32 + lane;
        const bool live = g < ngrp && j >= jlo && j < ncol;
#pragma unroll
        for (int kk = 0; kk < PW; ++kk) {
          double v = (live && kk < kw) ? M[pk[kk] * LDF + j] : 0.0;
#pragma unroll
          for (int k2 = 0; k2 < kk; ++k2) v = fma(-mk[kk][k2], uk[q][k2], v);
          uk[q][kk] = v;
        }
        nu += g < ngrp;
      }
      named_bar_sync(1, 32 * NU);   // all pivot-row entries read before any unit writes
#ifdef LU_TRACE
      if (ut == 0 && P < 16) g_lu_trace_u[4 * P + 2] = clock64();
#endif
#pragma unroll
      for (int q = 0; q < MAXU; ++q) {
        const int unit = uw + q * NU, g = unit / NRB, blk = unit % NRB;
        const int j = g * 32 + lane;
        if (g >= ngrp || g * 32 + 31 < jlo) continue;   // warp-uniform
        const bool live = j >= jlo && j < ncol;
        // all loads of the block before its stores (the compiler cannot tell rows apart)
        double v[RB];
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
          const int i = blk * RB + rr;
          v[rr] = (live && i < n) ? M[i * LDF + j] : 0.0;
        }
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
          // the row's PW multipliers as 16-byte broadcast loads (half the shared-memory wavefronts)
          const double2* mi = reinterpret_cast<const double2*>(MulP + (blk * RB + rr) * PW);
#pragma unroll
          for (int k2 = 0; k2 < PW / 2; ++k2) {
            const double2 m2 = mi[k2];   // (entries kk >= kw of a short last panel are never written)
            if (2 * k2 < kw) v[rr] = fma(-m2.x, uk[q][2 * k2], v[rr]);
            if (2 * k2 + 1 < kw) v[rr] = fma(-m2.y, uk[q][2 * k2 + 1], v[rr]);
          }
        }
#pragma unroll
        for (int rr = 0; rr < RB; ++rr) {
          const int i = blk * RB + rr;
          if (live && i < n) M[i * LDF + j] = v[rr];
        }
      }
#ifdef LU_TRACE
      if (ut == 0 && P < 16) g_lu_trace_u[4 * P + 3] = clock64();
#endif
      named_bar_sync(1, 32 * NU);   // this panel's writes done before the next panel's reads
      if (ut == 0) {
        __threadfence_block();
        upd_cnt[0] = P + 1;
      }
      (void)nu;
    }
  }
  __syncthreads();
#ifdef LU_TRACE
  if (threadIdx.x == 0) g_lu_trace[66] = clock64();
#endif
  if (bad_s) {
    if (tid == 0) status[sim] = 1;
    return;
  }
  for (int t = tid; t < n * (1 + nx); t += blockDim.x) {
    const int kk = t % n, col = t / n;
    const double x = M[pivrow[kk] * LDF + n + col] * rdiag[kk];
    if (col == 0) {
      dr[(size_t)sim * n + kk] = x;
      if (apply) {
        if constexpr (NB <= 6) r[(size_t)sim * n + kk] = r_old[t / 256] + x;   // t < n <= D: this thread's prefetch
        else r[(size_t)sim * n + kk] += x;
      }
    } else {
      xout[((size_t)sim * nx + col - 1) * n + kk] = x;
    }
  }
  if (tid == 0) status[sim] = 0;
#ifdef LU_TRACE
  __syncthreads();
  if (threadIdx.x == 0) g_lu_trace[67] = clock64();
#endif
}

// n: unknowns + extra right-hand sides (D >= n + 1 columns incl. -phi)
inline int lu_nb(int n) { return (n + 1 <= 64) ? 4 : (n + 1 <= 96) ? 6 : 8; }
// n: unknowns + extra rhs; nq: size of the vhp block staged beside the matrix
inline size_t lu_smem_bytes(int n, int nq = 0) {
  const int D = 16 * lu_nb(n);
  return (size_t)D * (D + 1) * 8 + (size_t)nq * nq * 8;
}
// k_lu_lookahead: + double-buffered panel multipliers [2][D][PW <= 8]
inline size_t lu_lookahead_smem_bytes(int n, int nq = 0) {
  const int D = 16 * lu_nb(n);
  return lu_smem_bytes(n, nq) + (size_t)2 * D * 8 * 8 + 16;
}


// r = base + t * dr ; rdot = (r - r_bar)/dt ; elementwise product
__global__ void k_axpy(double* __restrict__ out, const double* __restrict__ base, const double* __restrict__ d,
                       double t, int n) {
  pdl_wait();
  pdl_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = base[i] + t * d[i];
}
__global__ void k_rdot(const double* __restrict__ r, const double* __restrict__ rbar, double* __restrict__ rdot,
                       double inv_dt, int n) {
  pdl_wait();
  pdl_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) rdot[i] = (r[i] - rbar[i]) * inv_dt;
}
// nlrom_step's host hand-off without copy-engine nodes: the step graph's first kernel reads the
// pinned staging (r_bar | rdot_bar | f_ext) over the bus and forms the predictor (k_axpy), its last
// writes r, rdot, ||phi|| and the pivot status into pinned memory (k_rdot) -- the same arithmetic
// as k_axpy / k_rdot, two kernel nodes instead of seven memcpy nodes.
__global__ void k_step_in(const double* __restrict__ hin, double* __restrict__ rbar, double* __restrict__ rdbar,
                          double* __restrict__ fext, double* __restrict__ r, double t, int nn, long long nf) {
  pdl_wait();
  pdl_launch();
  const long long tot = nf > nn ? nf : nn;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
    if (i < nn) {
      const double base = hin[i], d = hin[nn + i];
      rbar[i] = base;
      rdbar[i] = d;
      r[i] = base + t * d;
    }
    if (i < nf) fext[i] = hin[2 * (long long)nn + i];
  }
}
__global__ void k_step_out(const double* __restrict__ r, const double* __restrict__ rbar, double* __restrict__ rdot,
                           double inv_dt, int nn, const double* __restrict__ extra, int nextra,
                           const int* __restrict__ status, int n_sims, double* __restrict__ ho, int* __restrict__ hs) {
  pdl_wait();
  pdl_launch();
  const int tot = max(nn, max(nextra, status ? n_sims : 0));
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    if (i < nn) {
      const double ri = r[i];
      const double rd = (ri - rbar[i]) * inv_dt;
      rdot[i] = rd;
      ho[i] = ri;
      ho[nn + i] = rd;
    }
    if (i < nextra) ho[2 * nn + i] = extra[i];   // ||phi|| (fixed step) / the Newton state (adaptive)
    if (status && i < n_sims) hs[i] = status[i];
  }
}
__global__ void k_mul(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out, int n) {
  pdl_wait();
  pdl_launch();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] * b[i];
}

// ------------------------------------------------------------------ vhp backward top
// y = [W_L | -U]^T a read through the row-major [W_L | -U] (N x ldA) that the forward
// just streamed (L2-hot): partial sums over row chunks, threads over the M = w + n_p columns.
__global__ void k_gemv_t(const double* __restrict__ A, int ldA, int M, const double* __restrict__ x, int N,
                         int rows_per_cta, double* __restrict__ part, int nchunk) {
  pdl_wait();
  pdl_launch();
  const int chunk = blockIdx.x, sim = blockIdx.y;
  const int r0 = chunk * rows_per_cta, r1 = min(N, r0 + rows_per_cta);
  const double* xs = x + (size_t)sim * N;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 8
  for (int n = r0; n < r1; ++n) {
    const double xv = xs[n];
    const double* Ar = A + (size_t)n * ldA;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      int m = threadIdx.x + u * blockDim.x;
      if (m < M) acc[u] = fma(Ar[m], xv, acc[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    int m = threadIdx.x + u * blockDim.x;
    if (m < M) part[((size_t)sim * nchunk + chunk) * M + m] = acc[u];
  }
}

// Same product for the fused vhp chain: 256 threads = 128 column pairs (16-byte loads) x 2 row
// phases, every load of a thread issued back to back; the per-chunk partials are summed by
// the consumer (k_mlp_dual_bwd prologue), so no separate reduction launch. M even, ldA even.
__global__ void __launch_bounds__(256) k_gemv_t2(const double* __restrict__ A, int ldA, int M,
                                                 const double* __restrict__ x, int N, int rows_per_cta,
                                                 double* __restrict__ part, int nchunk) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[512];
  const int chunk = blockIdx.x, sim = blockIdx.y;
  const int r0 = chunk * rows_per_cta, r1 = min(N, r0 + rows_per_cta);
  const double* xs = x + (size_t)sim * N;
  const int cp = threadIdx.x & 127, ph = threadIdx.x >> 7;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const int c0 = 2 * cp + 256 * g;
    if (c0 < M) {
#pragma unroll 12
      for (int n = r0 + ph; n < r1; n += 2) {
        const double2 v = *reinterpret_cast<const double2*>(A + (size_t)n * ldA + c0);
        const double xv = xs[n];
        acc[g][0] = fma(v.x, xv, acc[g][0]);
        acc[g][1] = fma(v.y, xv, acc[g][1]);
      }
    }
  }
  if (ph == 1)
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int c0 = 2 * cp + 256 * g;
      if (c0 < M) {
        red[c0] = acc[g][0];
        red[c0 + 1] = acc[g][1];
      }
    }
  __syncthreads();
  if (ph == 0)
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int c0 = 2 * cp + 256 * g;
      if (c0 < M) {
        double* o = part + ((size_t)sim * nchunk + chunk) * M + c0;
        o[0] = acc[g][0] + red[c0];
        o[1] = acc[g][1] + red[c0 + 1];
      }
    }
}

// y = sum_chunks part  (grid (ceil(M/32), n_sims), block 256 = 32 outputs x 8 chunk groups)
__global__ void k_reduce_cols(const double* __restrict__ part, int nchunk, int M, double* __restrict__ y) {
  pdl_wait();
  pdl_launch();
  __shared__ double red[8][32];
  const int sim = blockIdx.y;
  const int lane = threadIdx.x & 31, gidx = threadIdx.x >> 5;
  const int m = blockIdx.x * 32 + lane;
  double acc = 0.0;
  if (m < M)
    for (int c = gidx; c < nchunk; c += 8) acc += part[((size_t)sim * nchunk + c) * M + m];
  red[gidx][lane] = acc;
  __syncthreads();
  if (gidx == 0 && m < M) {
    double s = 0.0;
#pragma unroll
    for (int g2 = 0; g2 < 8; ++g2) s += red[g2][lane];
    y[(size_t)sim * M + m] = s;
  }
}

// g = y[:w] + A_T^T y[w:]  (A_T = U^T W_L: the filter's adjoint folded into the last layer),
// Delta[p*NS + s][i] = (g_i * act'(z_{L-1}))[s] in the arithmetic of the passes
// (NS = 1 real; 2 dual (MC = 0) or complex (MC = 1)); MC = 2: z already holds act'(z) as a dual
// (the fused bundle's cache). grid (ceil(w/32), n_sims), block 256.
// Shared-real layout (EpiBwdShared): per sim [g f0 | g f1_1 .. g f1_npass] from the sin'(z) cache.
__global__ void k_bwd_delta_sh(const double* __restrict__ y, int w, int n_p, const double* __restrict__ AT,
                               const double* __restrict__ zc, int ldz, int npass, double* __restrict__ Delta) {
  pdl_wait();
  pdl_launch();
  __shared__ double g[32];
  const int sim = blockIdx.y;
  const int i0 = blockIdx.x * 32;
  const int M = w + n_p;
  const double* ys = y + (size_t)sim * M;
  {
    __shared__ double gp[8][32];
    const int il = threadIdx.x & 31, w8 = threadIdx.x >> 5;
    const int i = i0 + il;
    double acc = 0.0;
    if (i < w)
      for (int j = w8; j < n_p; j += 8) acc = fma(AT[(size_t)j * w + i], ys[w + j], acc);
    gp[w8][il] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      double s = (i < w) ? ys[i] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += gp[q][il];
      g[il] = s;
    }
  }
  __syncthreads();
  const double* Z = zc + (size_t)sim * npass * 2 * ldz;
  double* D = Delta + (size_t)sim * (npass + 1) * ldz;
  for (int t = threadIdx.x; t < (npass + 1) * 32; t += blockDim.x) {
    const int il = t & 31, s = t >> 5;
    const int i = i0 + il;
    if (i >= w) continue;
    const double f = s == 0 ? Z[i] : Z[(size_t)(2 * (s - 1) + 1) * ldz + i];
    D[(size_t)s * ldz + i] = g[il] * f;
  }
}

template <int NS, int MC>
__global__ void k_bwd_delta(const double* __restrict__ y, int w, int n_p, const double* __restrict__ AT,
                            const double* __restrict__ zc, int ldz, int npass, double* __restrict__ Delta) {
  pdl_wait();
  pdl_launch();
  __shared__ double g[32];
  const int sim = blockIdx.y;
  const int i0 = blockIdx.x * 32;
  const int M = w + n_p;
  const double* ys = y + (size_t)sim * M;
  {
    // 8 warps x 32 columns: warp w8 sums j = w8, w8+8, ... (loads independent, all in flight)
    __shared__ double gp[8][32];
    const int il = threadIdx.x & 31, w8 = threadIdx.x >> 5;
    const int i = i0 + il;
    double acc = 0.0;
    if (i < w)
      for (int j = w8; j < n_p; j += 8) acc = fma(AT[(size_t)j * w + i], ys[w + j], acc);
    gp[w8][il] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      double s = (i < w) ? ys[i] : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += gp[q][il];
      g[il] = s;
    }
  }
  __syncthreads();
  const double* Z = zc + (size_t)sim * npass * NS * ldz;
  double* D = Delta + (size_t)sim * npass * NS * ldz;
  for (int t = threadIdx.x; t < npass * 32; t += blockDim.x) {
    const int il = t & 31, p = t >> 5;
    const int i = i0 + il;
    if (i >= w) continue;
    double z[NS], f[NS], s[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) z[q] = Z[(size_t)(p * NS + q) * ldz + i];
    if (MC == 2) {  // bundle cache: sin'(z) already formed by the forward
#pragma unroll
      for (int q = 0; q < NS; ++q) f[q] = z[q];
    } else if (MC) {
      mc_sincos<NS>(z, s, f);
    } else {
      md_sincos<NS>(z, s, f);
    }
#pragma unroll
    for (int q = 0; q < NS; ++q) D[(size_t)(p * NS + q) * ldz + i] = g[il] * f[q];
  }
}

}  // namespace nlrom
