// GEMM epilogues of the CSFD decoder passes (activation fused into the producing GEMM).
#pragma once
#include "gemm_f64.cuh"
#include "mc_device.cuh"

namespace nlrom {

enum ActKind { ACT_NONE = 0, ACT_SIN_MC = 1, ACT_SIN_MD = 2, ACT_SQUARE_MC = 3, ACT_DSIN_MD = 4 };

// Activation over passes of N = 2^order adjacent slot columns.
//  ACT_SIN_MC    : true multicomplex sin (mcx.py:63-100)
//  ACT_SIN_MD    : multi-dual sin on eps-scaled slots (SPEC.md:186 truncation)
//  ACT_SQUARE_MC : multicomplex z*z (square activation)
// Bias (FC layer) is added to the real slot only (mcx.py:333-338).
// cache (optional): pre-activation z (same layout as Y) for the backward pass.
template <int N, int ACT>
struct EpiAct {
  double* Y;
  int ldy;
  long long strideY;
  const double* bias;
  double* cache;
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    double* Yz = Y + (size_t)t.z * strideY;
    double* Cz = cache ? cache + (size_t)t.z * strideY : nullptr;
    const int npass = t.bn / N;
    for (int i = tid; i < t.bm * npass; i += nt) {
      const int p = i / t.bm, ml = i % t.bm;
      const int m = t.m0 + ml;
      const int cbase = t.c0 + p * N;
      if (m >= g.M || cbase >= g.C) continue;
      double z[N], o[N];
#pragma unroll
      for (int s = 0; s < N; ++s) z[s] = t.Cs[(p * N + s) * t.ldc + ml];
      if (bias) z[0] += bias[m];
      if (Cz) {
#pragma unroll
        for (int s = 0; s < N; ++s) Cz[(size_t)(cbase + s) * ldy + m] = z[s];
      }
      if constexpr (ACT == ACT_SIN_MC) {
        double c[N];
        mc_sincos<N>(z, o, c);
      } else if constexpr (ACT == ACT_SIN_MD) {
        md_sincos<N>(z, o, nullptr);
      } else if constexpr (ACT == ACT_SQUARE_MC) {
        mc_mul<N>(z, z, o);
      } else {
#pragma unroll
        for (int s = 0; s < N; ++s) o[s] = z[s];
      }
#pragma unroll
      for (int s = 0; s < N; ++s) Yz[(size_t)(cbase + s) * ldy + m] = o[s];
    }
  }
};

// Backward through an activation of the layer below: d_out = d_in (*) act'(z) in
// the arithmetic of the pass (N = 1 real, N = 2 complex / dual), z from the cache.
//   sin    : act'(z) = cos z      (MC: multicomplex cos, MD: multi-dual cos)
//   square : act'(z) = 2 z
template <int N, int ACT>
struct EpiBwdAct {
  double* Y;
  int ldy;
  long long strideY;
  const double* zcache;  // same layout as Y
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    double* Yz = Y + (size_t)t.z * strideY;
    const double* Zz = zcache + (size_t)t.z * strideY;
    const int npass = t.bn / N;
    for (int i = tid; i < t.bm * npass; i += nt) {
      const int p = i / t.bm, ml = i % t.bm;
      const int m = t.m0 + ml;
      const int cbase = t.c0 + p * N;
      if (m >= g.M || cbase >= g.C) continue;
      double d[N], z[N], f[N], o[N];
#pragma unroll
      for (int s = 0; s < N; ++s) {
        d[s] = t.Cs[(p * N + s) * t.ldc + ml];
        z[s] = Zz[(size_t)(cbase + s) * ldy + m];
      }
      if constexpr (ACT == ACT_SIN_MC) {
        double sn[N];
        mc_sincos<N>(z, sn, f);
      } else if constexpr (ACT == ACT_SIN_MD) {
        md_sincos<N>(z, nullptr, f);
      } else if constexpr (ACT == ACT_DSIN_MD) {  // the bundle cache already holds sin'(z) as a dual
#pragma unroll
        for (int s = 0; s < N; ++s) f[s] = z[s];
      } else if constexpr (ACT == ACT_SQUARE_MC) {
#pragma unroll
        for (int s = 0; s < N; ++s) f[s] = 2.0 * z[s];
      } else {
#pragma unroll
        for (int s = 0; s < N; ++s) f[s] = (s == 0) ? 1.0 : 0.0;
      }
      if constexpr (ACT == ACT_SIN_MD || ACT == ACT_DSIN_MD) md_mul<N>(d, f, o); else mc_mul<N>(d, f, o);
#pragma unroll
      for (int s = 0; s < N; ++s) Yz[(size_t)(cbase + s) * ldy + m] = o[s];
    }
  }
};

// vhp backward of the fused bundle at many sims with the real part shared: the real part of the
// dual cotangent is the same for every pass of a sim, so a sim's columns are [real | dual_1 ..
// dual_npass] (1 + npass instead of 2 npass). Tiles hold whole sims (GemmArgs.cstep), so the real
// column's product is in the same Cs tile: o0 = d0 f0, o_k = fma(d1_k, f0, d0 f1_k) (md_mul<2>
// order, bitwise equal to EpiBwdAct<2, ACT_DSIN_MD>). cache: per sim 2 npass columns (f0, f1_k).
struct EpiBwdShared {
  double* Y;
  int ldy;
  const double* fcache;
  int npass;
  // column-scale partials for a tcgen05 Ozaki consumer (as EpiJet::colhw): colhw[c * (M / 32) +
  // m / 32] = max over 32 rows of the high word of |Y[c][m]| (tile rows, thread counts multiples of 32)
  unsigned* colhw = nullptr;
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    const int P1 = 1 + npass;
    const double* __restrict__ fc = fcache;
    double* __restrict__ y = Y;
    // U elements per thread per round: every cache load of the round is issued before any store
    // (the compiler cannot reorder the loads past stores to Y on its own); only the two global
    // loads per element are held across the round, the tile values are read from Cs afterwards
    constexpr int U = 8;
    const int total = t.bm * t.bn;
    for (int i0 = tid; i0 < total; i0 += U * nt) {
      double f0[U], f1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * nt;
        const int cl = i / t.bm, ml = i % t.bm;
        const int c = t.c0 + cl, m = t.m0 + ml;
        const bool ok = i < total && m < g.M && c < g.C;
        const int sim = ok ? c / P1 : 0, sv = ok ? c % P1 : 0;
        const double* F = fc + (size_t)sim * 2 * npass * ldy;
        f0[u] = ok ? F[m] : 0.0;
        f1[u] = (ok && sv > 0) ? F[(size_t)(2 * (sv - 1) + 1) * ldy + m] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * nt;
        const int cl = i / t.bm, ml = i % t.bm;
        const int c = t.c0 + cl, m = t.m0 + ml;
        if (!(i < total && m < g.M && c < g.C)) continue;   // warp-uniform (bm, M multiples of 32)
        const int sv = c % P1;
        const double dv = t.Cs[(cl - sv) * t.ldc + ml];
        const double v = sv == 0 ? dv * f0[u] : fma(t.Cs[cl * t.ldc + ml], f0[u], dv * f1[u]);
        y[(size_t)c * ldy + m] = v;
        if (colhw) {
          const unsigned r = __reduce_max_sync(0xffffffffu, (unsigned)__double2hiint(fabs(v)));
          if ((tid & 31) == 0) colhw[(size_t)c * (g.M >> 5) + (m >> 5)] = r;
        }
      }
    }
  }
};

// Last layer of the shared-real vhp backward: column (sim, 0) -> G_t[sim][2k] for every k,
// column (sim, 1 + k) -> G_t[sim][2k + 1] (the reference vhp layout).
struct EpiStoreShared {
  double* Y;
  int ldy;
  int npass;
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    const int P1 = 1 + npass;
    for (int i = tid; i < t.bm * t.bn; i += nt) {
      const int cl = i / t.bm, ml = i % t.bm;
      const int c = t.c0 + cl, m = t.m0 + ml;
      if (m >= g.M || c >= g.C) continue;
      const int sim = c / P1, s = c % P1;
      const double v = t.Cs[cl * t.ldc + ml];
      double* G = Y + (size_t)sim * 2 * npass * ldy + m;
      if (s == 0)
        for (int k = 0; k < npass; ++k) G[(size_t)(2 * k) * ldy] = v;
      else
        G[(size_t)(2 * (s - 1) + 1) * ldy] = v;
    }
  }
};

// Hidden layer of the fused Newton bundle: tiles of G = BN columns laid out as
// [base jet (1, s, s^2, r) | nk tangents x (t, ts, ts^2, tr)], see mc_device.cuh.
// Writes the activated jet, and (optional) the dual cache for the vhp backward in
// the reference vhp layout (col 2k = real pre-activation z0, col 2k+1 = tangent
// t-slot pre-activation of direction k, i.e. the order-1 pass q + eps e_k i1).
struct EpiJet {
  double* Y;
  int ldy;
  long long strideY;
  const double* bias;
  double* cache;      // (n_sims * 2 n_q) x ldcache, may be null
  int ldcache;
  int group;          // columns per group (BN is a multiple of it)
  int gps;            // groups per simulation
  int n_q;            // tangent directions per simulation
  int compact;        // 1: write the output layout per sim (next layer is linear): [h_1, 2 h_ss | (h_t, 2 h_tss + h_tr) x n_q]
  // Column-scale partials for a tcgen05 Ozaki consumer (ozaki_tc.cuh), either layout:
  // colhw[c * (M / 32) + m / 32] = max over the 32 rows m of the high word of |Y[c][m]| (needs
  // M % 32 == 0 and 32-row-aligned warps: tile rows and thread counts multiples of 32).
  unsigned* colhw = nullptr;
  // the vhp cache's real parts are the same for every tangent of a sim: with the shared-real
  // backward (which reads only the first) write them once
  int real_once = 0;
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    double* Yz = Y + (size_t)t.z * strideY;
    const int nk = (group - 4) / 4;           // tangents per group
    const bool hw = colhw != nullptr && !compact;
    const bool hwc = colhw != nullptr && compact;   // compact layout: one partial per written column
    const int lane = tid & 31;
    auto note_c = [&](size_t col, int m, double v) {
      const unsigned r = __reduce_max_sync(0xffffffffu, (unsigned)__double2hiint(fabs(v)));
      if (lane == 0) colhw[col * (size_t)(g.M >> 5) + (m >> 5)] = r;
    };
    unsigned hw0 = 0u, hw1 = 0u;              // this lane's columns: lane and 32 + lane of the group
    auto note = [&](int j, double v) {        // warp max over the 32 rows of column j's |v| high word
      const unsigned r = __reduce_max_sync(0xffffffffu, (unsigned)__double2hiint(fabs(v)));
      if ((j & 31) == lane) {
        if (j < 32) hw0 = r;
        else hw1 = r;
      }
    };
    const int cs = 2 + 2 * n_q;               // output-layout columns per sim
    const int ngt = t.bn / group;             // groups in this tile
    for (int i = tid; i < t.bm * ngt; i += nt) {
      const int gt = i / t.bm, ml = i % t.bm;
      const int m = t.m0 + ml;
      const int cg = t.c0 + gt * group;       // first column of the group
      if (m >= g.M || cg >= g.C) continue;
      const int gg = cg / group;
      const int sim = gg / gps, gl = gg % gps;
      double* Cz = cache ? cache + (size_t)sim * 2 * n_q * ldcache : nullptr;
      const double* cs0 = t.Cs + (gt * group) * t.ldc + ml;
      double z[4], o[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) z[s] = cs0[s * t.ldc];
      z[0] += bias[m];
      JetCos jc;
      jet_sin_base(z, o, jc);
      if (!compact) {
#pragma unroll
        for (int s = 0; s < 4; ++s) Yz[(size_t)(cg + s) * ldy + m] = o[s];
        if (hw)
#pragma unroll
          for (int s = 0; s < 4; ++s) note(s, o[s]);
      } else if (gl == 0) {
        Yz[(size_t)(sim * cs) * ldy + m] = o[0];
        Yz[(size_t)(sim * cs + 1) * ldy + m] = 2.0 * o[2];
        if (hwc) {
          note_c((size_t)(sim * cs), m, o[0]);
          note_c((size_t)(sim * cs + 1), m, 2.0 * o[2]);
        }
      }
      for (int k = 0; k < nk; ++k) {
        const int kg = gl * nk + k;           // tangent index within the simulation
        if (compact && kg >= n_q) break;
        double y[4], yo[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) y[s] = cs0[(4 + 4 * k + s) * t.ldc];
        jet_tangent(jc, y, yo);
        if (compact) {
          const size_t col = (size_t)(sim * cs + 2 + 2 * kg);
          const double v1 = fma(2.0, yo[2], yo[3]);
          Yz[col * ldy + m] = yo[0];
          Yz[(col + 1) * ldy + m] = v1;
          if (hwc) {
            note_c(col, m, yo[0]);
            note_c(col + 1, m, v1);
          }
        } else {
          const size_t col = (size_t)(cg + 4 + 4 * k);
#pragma unroll
          for (int s = 0; s < 4; ++s) Yz[(col + s) * ldy + m] = yo[s];
          if (hw)
#pragma unroll
            for (int s = 0; s < 4; ++s) note(4 + 4 * k + s, yo[s]);
        }
        if (Cz && kg < n_q) {  // sin'(z0 + y0 e) = cos z0 - sin z0 y0 e (dual), for the vhp backward
          if (!real_once || kg == 0) Cz[(size_t)(2 * kg) * ldcache + m] = jc.c1;
          Cz[(size_t)(2 * kg + 1) * ldcache + m] = jc.ns * y[0];
        }
      }
      if (hw) {
        const int parts = g.M >> 5, rg = m >> 5;
        if (lane < group) colhw[(size_t)(cg + lane) * parts + rg] = hw0;
        if (lane + 32 < group) colhw[(size_t)(cg + 32 + lane) * parts + rg] = hw1;
      }
    }
  }
};

// Output layer over the de-replicated (compact) column layout: per sim 4 + 4 n_q columns
// [1, s, s^2, r | (t, ts, ts^2, tr) x n_q]; a tile may hold several sims / tangents.
struct EpiJetOutC {
  const double* bias;    // P b (filtered last bias), real slot only
  const double* U;       // (N, n_p) row-major
  const double* r;       // (n_sims, n): p = r[:n_p]
  double* u;             // (n_sims, N)
  double* value;         // (n_sims, N) D(q)
  double* hvv;           // (n_sims, N)
  double* Jt;            // (n_sims, N, ldjt)
  double* dJ;            // (n_sims, N, lddj)
  int ldjt, lddj, n_p, n_q;
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    const int N = g.M;
    const int cs = 2 + 2 * n_q;  // per sim: [D_1, 2 D_ss | (D_t, 2 D_tss + D_tr) x n_q] (combined upstream)
    const int ngrp = t.bn / 2;
    for (int i = tid; i < t.bm * ngrp; i += nt) {
      const int q = i / t.bm, ml = i % t.bm;
      const int m = t.m0 + ml;
      const int c = t.c0 + 2 * q;
      if (m >= N || c >= g.C) continue;
      const int sim = c / cs, rem = c % cs;
      const size_t sv = (size_t)sim * N + m;
      const double* col = t.Cs + (2 * q) * t.ldc + ml;
      if (rem == 0) {
        const double d1 = col[0] + bias[m];
        double up = 0.0;
        const double* Ur = U + (size_t)m * n_p;
        const double* pz = r + (size_t)sim * (n_p + n_q);
        for (int k = 0; k < n_p; ++k) up = fma(Ur[k], pz[k], up);
        u[sv] = up + d1;
        value[sv] = d1;
        hvv[sv] = col[t.ldc];
      } else {
        const int kg = (rem - 2) >> 1;
        Jt[sv * ldjt + n_p + kg] = col[0];
        dJ[sv * lddj + kg] = col[t.ldc];
      }
    }
  }
};

// EpiJetOutC for the tcgen05 output layer, which hands it the fp64 tile row-major (t.Cs[row * t.ldc
// + col], ozaki_tc.cuh row_major_cs): the per-sim rows of J~ and dJ are contiguous in kg, so lanes
// over the tile's column pairs store them coalesced (lanes over rows wrote 8 bytes per 256-byte J~
// row); the base columns (u, D(q), hvv, with the U p dot product) keep lanes over rows.
struct EpiJetOutCRow {
  static constexpr bool kRowMajorCs = true;
  EpiJetOutC o;
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    const int N = g.M;
    const int cs = 2 + 2 * o.n_q;
    const int ngrp = t.bn / 2;
    // base column pairs (rem == 0): at most ceil(t.bn / cs) + 1 per tile, lanes over rows
    for (int p0 = (cs - t.c0 % cs) % cs; p0 < t.bn; p0 += cs) {
      const int c = t.c0 + p0;
      if (c >= g.C) break;
      const int sim = c / cs;
      for (int ml = tid; ml < t.bm; ml += nt) {
        const int m = t.m0 + ml;
        if (m >= N) continue;
        const size_t sv = (size_t)sim * N + m;
        const double* row = t.Cs + (size_t)ml * t.ldc + p0;
        const double d1 = row[0] + o.bias[m];
        double up = 0.0;
        const double* Ur = o.U + (size_t)m * o.n_p;
        const double* pz = o.r + (size_t)sim * (o.n_p + o.n_q);
        for (int k = 0; k < o.n_p; ++k) up = fma(Ur[k], pz[k], up);
        o.u[sv] = up + d1;
        o.value[sv] = d1;
        o.hvv[sv] = row[1];
      }
    }
    // tangent column pairs: lanes over the pairs of a row
    for (int i = tid; i < t.bm * ngrp; i += nt) {
      const int q = i % ngrp, ml = i / ngrp;
      const int m = t.m0 + ml;
      const int c = t.c0 + 2 * q;
      if (m >= N || c >= g.C) continue;
      const int sim = c / cs, rem = c % cs;
      if (rem == 0) continue;
      const size_t sv = (size_t)sim * N + m;
      const double* row = t.Cs + (size_t)ml * t.ldc + 2 * q;
      const int kg = (rem - 2) >> 1;
      o.Jt[sv * o.ldjt + o.n_p + kg] = row[0];
      o.dJ[sv * o.lddj + kg] = row[1];
    }
  }
};

// Output layer of the fused bundle (linear + fused filter): from the jet columns
//   value = D_1, J e_k = D_t, hvv = H(v,v) = 2 D_ss, dJ_k = S(e_k,v,v) + H(e_k,w) = 2 D_tss + D_tr
// and u = U p + D(q). J is written into J~ = [U, J] (row-major, ldjt), dJ row-major (lddj).
struct EpiJetOut {
  const double* bias;    // P b (filtered last bias), real slot only
  const double* U;       // (N, n_p) row-major
  const double* r;       // (n_sims, n): p = r[:n_p]
  double* u;             // (n_sims, N)
  double* value;         // (n_sims, N) D(q)
  double* hvv;           // (n_sims, N)
  double* Jt;            // (n_sims, N, ldjt)
  double* dJ;            // (n_sims, N, lddj)
  int ldjt, lddj, n_p, n_q, group, gps;
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    const int gg = t.c0 / group;
    const int sim = gg / gps, gl = gg % gps;
    const int nk = (group - 4) / 4;
    const int N = g.M;
    const size_t sv = (size_t)sim * N;
    for (int ml = tid; ml < t.bm; ml += nt) {
      const int m = t.m0 + ml;
      if (m >= N) continue;
      if (gl == 0) {
        const double d1 = t.Cs[0 * t.ldc + ml] + bias[m];
        const double dss = t.Cs[2 * t.ldc + ml];
        double up = 0.0;
        const double* Ur = U + (size_t)m * n_p;
        const double* pz = r + (size_t)sim * (n_p + n_q);
        for (int i = 0; i < n_p; ++i) up = fma(Ur[i], pz[i], up);
        u[sv + m] = up + d1;
        value[sv + m] = d1;
        hvv[sv + m] = 2.0 * dss;
      }
      double* Jrow = Jt + (sv + m) * ldjt + n_p;
      double* drow = dJ + (sv + m) * lddj;
      for (int k = 0; k < nk; ++k) {
        const int kg = gl * nk + k;
        if (kg >= n_q) break;
        const double* col = t.Cs + (4 + 4 * k) * t.ldc + ml;
        Jrow[kg] = col[0];
        drow[kg] = 2.0 * col[2 * t.ldc] + col[3 * t.ldc];
      }
    }
  }
};

}  // namespace nlrom
