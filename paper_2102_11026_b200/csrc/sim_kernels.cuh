// Non-GEMM kernels of the reduced Newton step: seeds, wnet, StVK cubature,
// assembly, reductions, in-CTA LU with partial pivoting.
#pragma once
#include "common.cuh"
#include "mc_device.cuh"

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
  const long long total = (long long)N * npass;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int j = t % npass;
    int m = t / npass;
    out[t] = Y[((size_t)j * S + slot) * ldy + m] / div;
  }
}

// ------------------------------------------------------------------------ wnet
// Split-K GEMV: part[s][sim][m] = sum_{k in chunk s} A[m][k] x[sim][k]   (A: M x K row-major, lda)
__global__ void k_gemv_splitk(const double* __restrict__ A, int lda, const double* __restrict__ x, long long strideX,
                              int M, int K, int chunk, double* __restrict__ part, int n_sims) {
  const int s = blockIdx.x;
  const int sim = blockIdx.y;
  const int k0 = s * chunk, k1 = min(K, k0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double* xs = x + (size_t)sim * strideX;
  for (int m = warp; m < M; m += nw) {
    const double* Ar = A + (size_t)m * lda;
    double acc = 0.0;
    for (int k = k0 + lane; k < k1; k += 32) acc = fma(Ar[k], xs[k], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) part[((size_t)s * n_sims + sim) * M + m] = acc;
  }
}

// Weight-net tail (1 CTA per sim): h1 = sin(sum parts + b1), h2 = sin(W2 h1 + b2),
// h3 = sin(W3 h2 + b3), w_C = (W4[C] h3 + b4[C])^2   (PAPER.md:406 square for w >= 0)
__global__ void k_wnet_tail(const double* __restrict__ part, int n_split, int wn, const double* __restrict__ b1,
                            const double* __restrict__ W2, const double* __restrict__ b2, const double* __restrict__ W3,
                            const double* __restrict__ b3, const double* __restrict__ W4C, const double* __restrict__ b4C,
                            int n_cub, double* __restrict__ wC, int n_sims) {
  extern __shared__ double sh[];
  double* h1 = sh;
  double* h2 = sh + wn;
  const int sim = blockIdx.x;
  for (int m = threadIdx.x; m < wn; m += blockDim.x) {
    double acc = b1[m];
    for (int s = 0; s < n_split; ++s) acc += part[((size_t)s * n_sims + sim) * wn + m];
    h1[m] = sin(acc);
  }
  __syncthreads();
  for (int m = threadIdx.x; m < wn; m += blockDim.x) {
    double acc = b2[m];
    for (int k = 0; k < wn; ++k) acc = fma(W2[(size_t)m * wn + k], h1[k], acc);
    h2[m] = sin(acc);
  }
  __syncthreads();
  for (int m = threadIdx.x; m < wn; m += blockDim.x) {
    double acc = b3[m];
    for (int k = 0; k < wn; ++k) acc = fma(W3[(size_t)m * wn + k], h2[k], acc);
    h1[m] = sin(acc);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n_cub; j += blockDim.x) {
    double acc = b4C[j];
    for (int k = 0; k < wn; ++k) acc = fma(W4C[(size_t)j * wn + k], h1[k], acc);
    wC[(size_t)sim * n_cub + j] = acc * acc;
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
};

__device__ __forceinline__ void mat3_mul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) C[i * 3 + j] = A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j] + A[i * 3 + 2] * B[6 + j];
}

__global__ void k_cubature(CubArgs a) {
  extern __shared__ double sh[];
  const int n = a.n;
  const int epc = a.epc;
  double* Js = sh;                         // [epc][12][n]
  double* Gs = Js + (size_t)epc * 12 * n;  // [epc][12][n]  (w K J)
  double* Ks = Gs + (size_t)epc * 12 * n;  // [epc][12][12]
  double* Fs = Ks + (size_t)epc * 144;     // [epc][12]
  const int chunk = blockIdx.x, sim = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double* u = a.u + (size_t)sim * a.N;
  const double* Jt = a.Jt ? a.Jt + (size_t)sim * a.N * a.ldjt : nullptr;

  // gather the J~ rows of the chunk's elements
  for (int idx = threadIdx.x; Jt && idx < epc * 12 * n; idx += blockDim.x) {
    int j = idx % n;
    int l = (idx / n) % 12;
    int el = idx / (12 * n);
    int ei = chunk * epc + el;
    double val = 0.0;
    if (ei < a.n_elems) {
      int e = a.elems ? a.elems[ei] : ei;
      int row = a.elem_rows[(size_t)e * 12 + l];
      if (row >= 0) val = Jt[(size_t)row * a.ldjt + j];
    }
    Js[idx] = val;
  }
  // element physics, one warp per element
  for (int el = warp; el < epc; el += nw) {
    int ei = chunk * epc + el;
    if (ei >= a.n_elems) {
      if (lane < 12) {
        Fs[el * 12 + lane] = 0.0;
        for (int r = 0; r < 12; ++r) Ks[el * 144 + r * 12 + lane] = 0.0;
      }
      continue;
    }
    int e = a.elems ? a.elems[ei] : ei;
    double ue = 0.0;
    if (lane < 12) {
      int row = a.elem_rows[(size_t)e * 12 + lane];
      ue = row >= 0 ? u[row] : 0.0;
    }
    double uv[12];
#pragma unroll
    for (int l = 0; l < 12; ++l) uv[l] = __shfl_sync(0xffffffffu, ue, l);
    double Di[9];
#pragma unroll
    for (int l = 0; l < 9; ++l) Di[l] = a.Dm_inv[(size_t)e * 9 + l];
    const double V = a.vol[e];
    const double we = a.w ? a.w[(size_t)sim * a.n_elems + ei] : 1.0;
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
    if (lane < 12) {
      int i = lane / 3, aa = lane % 3;
      double f = V * (P[aa * 3] * G[i * 3] + P[aa * 3 + 1] * G[i * 3 + 1] + P[aa * 3 + 2] * G[i * 3 + 2]);
      Fs[el * 12 + lane] = we * f;
      a.fe_w[((size_t)sim * a.n_elems + ei) * 12 + lane] = we * f;
      // stiffness column for DOF (jv, d) = lane: dF_ab = delta_ad g_jv[b]
      int jv = lane / 3, d = lane % 3;
      double dF[9];
#pragma unroll
      for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int y = 0; y < 3; ++y) dF[x * 3 + y] = (x == d) ? G[jv * 3 + y] : 0.0;
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
        Ks[el * 144 + r * 12 + lane] = we * kv;
        if (a.Ke_out) a.Ke_out[(size_t)ei * 144 + r * 12 + lane] = we * kv;
      }
    }
  }
  __syncthreads();
  if (!Jt) return;
  if (a.fred_out) {
    for (int idx = threadIdx.x; idx < epc * n; idx += blockDim.x) {
      int el = idx / n, i = idx % n;
      int ei = chunk * epc + el;
      if (ei >= a.n_elems) continue;
      double acc = 0.0;
      for (int l = 0; l < 12; ++l) acc = fma(Js[(el * 12 + l) * n + i], Fs[el * 12 + l], acc);
      a.fred_out[(size_t)ei * n + i] = acc;
    }
    return;
  }
  // G_e = (w K_e) J~_e   (12 x n)
  for (int idx = threadIdx.x; idx < epc * 12 * n; idx += blockDim.x) {
    int j = idx % n;
    int r = (idx / n) % 12;
    int el = idx / (12 * n);
    const double* Kr = Ks + el * 144 + r * 12;
    const double* Je = Js + (size_t)el * 12 * n;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 12; ++c) acc = fma(Kr[c], Je[c * n + j], acc);
    Gs[idx] = acc;
  }
  __syncthreads();
  // partial K~ = sum_rows J~^T G ; partial f~ = sum_rows J~^T (w f)
  double* pK = a.part_K + ((size_t)sim * a.nchunk + chunk) * n * n;
  const int R = epc * 12;
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    int i = idx / n, j = idx % n;
    double acc = 0.0;
    for (int rr = 0; rr < R; ++rr) acc = fma(Js[rr * n + i], Gs[rr * n + j], acc);
    pK[idx] = acc;
  }
  double* pf = a.part_f + ((size_t)sim * a.nchunk + chunk) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double acc = 0.0;
    for (int rr = 0; rr < R; ++rr) acc = fma(Js[rr * n + i], Fs[rr], acc);
    pf[i] = acc;
  }
}

// Deterministic scatter of weighted element forces into the free-DOF vector (CSR over rows).
__global__ void k_scatter_rows(const int* __restrict__ row_ids, const int* __restrict__ row_ptr,
                               const int* __restrict__ entries, int n_rows, const double* __restrict__ fe_w,
                               int n_elems, double* __restrict__ f, int N, int n_sims) {
  const long long total = (long long)n_rows * n_sims;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int i = t % n_rows;
    int sim = t / n_rows;
    double acc = 0.0;
    for (int j = row_ptr[i]; j < row_ptr[i + 1]; ++j) acc += fe_w[(size_t)sim * n_elems * 12 + entries[j]];
    f[(size_t)sim * N + row_ids[i]] = acc;
  }
}

// -------------------------------------------------------------------- assembly
// Per chunk of rows n:  a_n = M_n (J~_n . c) + [M_n hvv_n] + dt^2 (f_n - fext_n),
//   c = (1 + alpha dt)(r - r_bar) - dt rdot_bar,
// partial P = sum_n J~_n^T [ M_n R_n | a_n ],  R_n = (1+alpha dt) J~_n + [0, dJ_n].
struct AsmArgs {
  const double* Jt; int ldjt;
  const double* dJ; int lddj;
  const double* mass;
  const double* hvv;
  const double* f;       // cubature / exact scattered force (n_sims, N)
  const double* fext;    // (n_sims, N)
  const double* r; const double* rbar; const double* rdbar;
  double* a;             // (n_sims, N)
  double* part;          // (n_sims, nchunk, n*(n+1))
  int N, n, n_p, n_q, rows_per_cta, nchunk;
  double dt, alpha;
  int drop_fict;
};

__global__ void k_assemble(AsmArgs A) {
  extern __shared__ double sh[];
  const int n = A.n, n1 = n + 1;
  const int RC = A.rows_per_cta;
  double* Js = sh;                    // [RC][n]
  double* Rs = Js + (size_t)RC * n;   // [RC][n+1]  (M R | a)
  double* cs = Rs + (size_t)RC * n1;  // [n]
  const int chunk = blockIdx.x, sim = blockIdx.y;
  const double ah = A.alpha * A.dt;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    size_t o = (size_t)sim * n + i;
    cs[i] = (1.0 + ah) * (A.r[o] - A.rbar[o]) - A.dt * A.rdbar[o];
  }
  const int row0 = chunk * RC;
  const double* Jt = A.Jt + (size_t)sim * A.N * A.ldjt;
  const double* dJ = A.dJ + (size_t)sim * A.N * A.lddj;
  for (int idx = threadIdx.x; idx < RC * n; idx += blockDim.x) {
    int rl = idx / n, j = idx % n;
    int row = row0 + rl;
    Js[idx] = row < A.N ? Jt[(size_t)row * A.ldjt + j] : 0.0;
  }
  __syncthreads();
  // a_n (one warp per row)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int rl = warp; rl < RC; rl += nw) {
    int row = row0 + rl;
    double acc = 0.0;
    for (int j = lane; j < n; j += 32) acc = fma(Js[rl * n + j], cs[j], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      double av = 0.0;
      if (row < A.N) {
        size_t o = (size_t)sim * A.N + row;
        double m = A.mass[row];
        av = m * acc + A.dt * A.dt * (A.f[o] - A.fext[o]);
        if (!A.drop_fict) av += m * A.hvv[o];
        A.a[o] = av;
      }
      Rs[rl * n1 + n] = av;
    }
  }
  for (int idx = threadIdx.x; idx < RC * n; idx += blockDim.x) {
    int rl = idx / n, j = idx % n;
    int row = row0 + rl;
    double v = 0.0;
    if (row < A.N) {
      v = (1.0 + ah) * Js[idx];
      if (j >= A.n_p) v += dJ[(size_t)row * A.lddj + (j - A.n_p)];
      v *= A.mass[row];
    }
    Rs[rl * n1 + j] = v;
  }
  __syncthreads();
  double* P = A.part + ((size_t)sim * A.nchunk + chunk) * n * n1;
  for (int idx = threadIdx.x; idx < n * n1; idx += blockDim.x) {
    int i = idx / n1, j = idx % n1;
    double acc = 0.0;
    for (int rl = 0; rl < RC; ++rl) acc = fma(Js[rl * n + i], Rs[rl * n1 + j], acc);
    P[idx] = acc;
  }
}

// phi = sum_chunks part[:, n] (one CTA per sim), ||phi||_2
__global__ void k_reduce_phi(const double* __restrict__ part, int nchunk, int n, double* __restrict__ phi,
                             double* __restrict__ norm) {
  const int sim = blockIdx.x;
  const int n1 = n + 1;
  __shared__ double red[32];
  double sq = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double acc = 0.0;
    for (int c = 0; c < nchunk; ++c) acc += part[(((size_t)sim * nchunk + c) * n + i) * n1 + n];
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
}

// S = sum part_A[:, :n] + dt^2 sum part_K + diag(0, vhp);  vhp[i][k] = G_t[2k+1][i]
__global__ void k_reduce_S(const double* __restrict__ partA, int nchA, const double* __restrict__ partK, int nchK,
                           const double* __restrict__ Gt, int ldg, int n, int n_p, int n_q, double dt,
                           double* __restrict__ S, int n_sims) {
  const long long total = (long long)n * n * n_sims;
  const int n1 = n + 1;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    int idx = t % (n * n);
    int sim = t / (n * n);
    int i = idx / n, j = idx % n;
    double acc = 0.0;
    for (int c = 0; c < nchA; ++c) acc += partA[(((size_t)sim * nchA + c) * n + i) * n1 + j];
    double k = 0.0;
    for (int c = 0; c < nchK; ++c) k += partK[((size_t)sim * nchK + c) * n * n + idx];
    acc += dt * dt * k;
    if (Gt && i >= n_p && j >= n_p) acc += Gt[((size_t)sim * 2 * n_q + 2 * (j - n_p) + 1) * ldg + (i - n_p)];
    S[(size_t)sim * n * n + idx] = acc;
  }
}

// sum of cubature partials (for cubature_integrate): f~ (n), K~ (n,n)
__global__ void k_reduce_cub(const double* __restrict__ part_f, const double* __restrict__ part_K, int nch, int n,
                             double* __restrict__ f_red, double* __restrict__ K_red) {
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
// One CTA per sim: LU with partial pivoting of S (n x n) and solve S dr = -phi
// (SPEC.md:555, 566). If `apply`, r += dr. status[sim] = 1 on a zero pivot.
__global__ void k_lu_solve(const double* __restrict__ S, const double* __restrict__ phi, double* __restrict__ dr,
                           double* __restrict__ r, int n, int apply, int* __restrict__ status) {
  extern __shared__ double sh[];
  const int sim = blockIdx.x;
  const int ld = n + 2;
  double* A = sh;  // [n][n+2], column n = rhs
  __shared__ int piv;
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) A[(idx / n) * ld + idx % n] = S[(size_t)sim * n * n + idx];
  for (int i = threadIdx.x; i < n; i += blockDim.x) A[i * ld + n] = -phi[(size_t)sim * n + i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = 0; k < n; ++k) {
    if (warp == 0) {
      double best = -1.0;
      int bi = k;
      for (int i = k + lane; i < n; i += 32) {
        double v = fabs(A[i * ld + k]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) piv = bi;
    }
    __syncthreads();
    const int p = piv;
    if (p != k)
      for (int j = threadIdx.x; j <= n; j += blockDim.x) {
        double t = A[k * ld + j];
        A[k * ld + j] = A[p * ld + j];
        A[p * ld + j] = t;
      }
    __syncthreads();
    const double akk = A[k * ld + k];
    if (akk == 0.0) {
      if (threadIdx.x == 0) status[sim] = 1;
      return;
    }
    const int rows = n - k - 1, cols = n - k;  // update rows k+1.., cols k+1..n (incl. rhs)
    for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
      int i = k + 1 + idx / cols, j = k + 1 + idx % cols;
      double l = A[i * ld + k] / akk;
      A[i * ld + j] -= l * A[k * ld + j];
    }
    __syncthreads();
  }
  // back substitution (column-oriented)
  for (int i = n - 1; i >= 0; --i) {
    double xi = A[i * ld + n] / A[i * ld + i];
    __syncthreads();
    for (int j = threadIdx.x; j < i; j += blockDim.x) A[j * ld + n] -= A[j * ld + i] * xi;
    if (threadIdx.x == 0) A[i * ld + n] = xi;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double x = A[i * ld + n];
    dr[(size_t)sim * n + i] = x;
    if (apply) r[(size_t)sim * n + i] += x;
  }
  if (threadIdx.x == 0) status[sim] = 0;
  (void)red_v; (void)red_i;
}

// r = base + t * dr ; predictor r = r_bar + dt rdot_bar ; rdot = (r - r_bar)/dt
__global__ void k_axpy(double* __restrict__ out, const double* __restrict__ base, const double* __restrict__ d,
                       double t, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = base[i] + t * d[i];
}
__global__ void k_rdot(const double* __restrict__ r, const double* __restrict__ rbar, double* __restrict__ rdot,
                       double inv_dt, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) rdot[i] = (r[i] - rbar[i]) * inv_dt;
}
__global__ void k_mul(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] * b[i];
}

// Backward top of the decoder (vhp / vjp): y = [W_L | -U]^T a (split-K partials),
// g = y[:w] + A_T^T y[w:]  (A_T = U^T W_L), then Delta = g * act'(z_{L-1}) in the
// arithmetic of the passes (NS = 1 real, 2 dual/complex), cache layout (pass*NS + slot).
template <int NS, int MC>
__global__ void k_bwd_top(const double* __restrict__ part, int n_split, int w, int n_p, const double* __restrict__ AT,
                          const double* __restrict__ zc, int ldz, int npass, double* __restrict__ Delta, int n_sims) {
  extern __shared__ double g[];
  const int sim = blockIdx.x;
  const int M = w + n_p;
  double* y = g + w;
  for (int m = threadIdx.x; m < M; m += blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < n_split; ++s) acc += part[((size_t)s * n_sims + sim) * M + m];
    y[m] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    double acc = y[i];
    for (int j = 0; j < n_p; ++j) acc = fma(AT[(size_t)j * w + i], y[w + j], acc);
    g[i] = acc;
  }
  __syncthreads();
  const double* Z = zc + (size_t)sim * npass * NS * ldz;
  double* D = Delta + (size_t)sim * npass * NS * ldz;
  for (int t = threadIdx.x; t < npass * w; t += blockDim.x) {
    int i = t % w, p = t / w;
    double z[NS], f[NS], s[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) z[q] = Z[(size_t)(p * NS + q) * ldz + i];
    if (MC) mc_sincos<NS>(z, s, f);
    else md_sincos<NS>(z, s, f);
#pragma unroll
    for (int q = 0; q < NS; ++q) D[(size_t)(p * NS + q) * ldz + i] = g[i] * f[q];
  }
}

}  // namespace nlrom
