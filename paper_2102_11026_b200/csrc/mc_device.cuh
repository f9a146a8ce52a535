// Device-side multicomplex / multi-dual / jet arithmetic on register part stacks.
//
// Slot layout = reference bitmask layout (mcx.py:1-8): slot s is the coefficient
// of prod_{d : bit d-1 of s} i_d.
//
//  * mc_*   : TRUE multicomplex arithmetic (i_d^2 = -1), the reference algebra:
//             product by the recursive split on the top direction (mcx.py:39-49),
//             sin/cos/sinh/cosh by the angle-addition recursion (mcx.py:63-100).
//  * md_*   : multi-dual arithmetic (i_d^2 = 0) on eps-SCALED slots
//             (slot s stores part_s / eps^|s|). With eps = 1e-10 the multicomplex
//             CSFD parts equal these to relative O(eps^2) = 1e-20, far below fp64
//             roundoff, and SPEC.md:186 / PAPER.md:361 prescribe exactly
//             this truncation ("high-order terms of h are discarded").
//  * jet_*  : the collapsed Newton-bundle algebra R[t,s,r]/(t^2, s^3, r^2, s r)
//             used by the fused rdsim bundle.
#pragma once
#include <cuda_runtime.h>

namespace nlrom {

// ---------------------------------------------------------------- multicomplex
template <int N>
__device__ __forceinline__ void mc_mul(const double* a, const double* b, double* out) {
  if constexpr (N == 1) {
    out[0] = a[0] * b[0];
  } else {
    constexpr int H = N / 2;
    double t1[H], t2[H], t3[H], t4[H];
    mc_mul<H>(a, b, t1);
    mc_mul<H>(a + H, b + H, t2);
    mc_mul<H>(a, b + H, t3);
    mc_mul<H>(a + H, b, t4);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      out[i] = t1[i] - t2[i];
      out[H + i] = t3[i] + t4[i];
    }
  }
}

template <int N> __device__ void mc_sinhcosh(const double* p, double* sh, double* ch);

template <int N>
__device__ __forceinline__ void mc_sincos(const double* p, double* s, double* c) {
  if constexpr (N == 1) {
    sincos(p[0], s, c);
  } else {
    constexpr int H = N / 2;
    double su[H], cu[H], shv[H], chv[H], t[H];
    mc_sincos<H>(p, su, cu);
    mc_sinhcosh<H>(p + H, shv, chv);
    mc_mul<H>(su, chv, s);
    mc_mul<H>(cu, shv, s + H);
    mc_mul<H>(cu, chv, c);
    mc_mul<H>(su, shv, t);
#pragma unroll
    for (int i = 0; i < H; ++i) c[H + i] = -t[i];
  }
}

template <int N>
__device__ __forceinline__ void mc_sinhcosh(const double* p, double* sh, double* ch) {
  if constexpr (N == 1) {
    sh[0] = sinh(p[0]);
    ch[0] = cosh(p[0]);
  } else {
    constexpr int H = N / 2;
    double shu[H], chu[H], sv[H], cv[H];
    mc_sinhcosh<H>(p, shu, chu);
    mc_sincos<H>(p + H, sv, cv);
    mc_mul<H>(shu, cv, sh);
    mc_mul<H>(chu, sv, sh + H);
    mc_mul<H>(chu, cv, ch);
    mc_mul<H>(shu, sv, ch + H);
  }
}

// ------------------------------------------------------------------ multi-dual
template <int N>
__device__ __forceinline__ void md_mul(const double* a, const double* b, double* out) {
#pragma unroll
  for (int s = 0; s < N; ++s) {
    double acc = 0.0;
#pragma unroll
    for (int s1 = 0; s1 < N; ++s1)
      if ((s1 & s) == s1) acc = fma(a[s1], b[s ^ s1], acc);
    out[s] = acc;
  }
}

// sin / cos of a multi-dual number z = a0 + d (d nilpotent, d^(k+1) = 0, k <= 3):
//   sin z = sin a0 (1 - d^2/2) + cos a0 (d - d^3/6),  cos z = cos a0 (1 - d^2/2) - sin a0 (d - d^3/6)
template <int N>
__device__ __forceinline__ void md_sincos(const double* z, double* s, double* c) {
  double S0, C0;
  sincos(z[0], &S0, &C0);
  double d[N], d2[N], d3[N];
#pragma unroll
  for (int i = 0; i < N; ++i) d[i] = (i == 0) ? 0.0 : z[i];
  if constexpr (N >= 4) md_mul<N>(d, d, d2); else {
#pragma unroll
    for (int i = 0; i < N; ++i) d2[i] = 0.0;
  }
  if constexpr (N >= 8) md_mul<N>(d2, d, d3); else {
#pragma unroll
    for (int i = 0; i < N; ++i) d3[i] = 0.0;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double even = (i == 0 ? 1.0 : 0.0) - 0.5 * d2[i];
    const double odd = d[i] - d3[i] * (1.0 / 6.0);
    if (s) s[i] = S0 * even + C0 * odd;
    if (c) c[i] = C0 * even - S0 * odd;
  }
}

// ------------------------------------------------------------------------ jet
// Base jet z = z1 + zs s + zss s^2 + zr r ; tangent part t (yt + yts s + ytss s^2 + ytr r).
// sin(z + t y) = sin z + t cos(z) y.
struct JetCos {
  double c1, cs, css, cr;  // cos(z) coefficients
  double ns;               // -sin(z0)
};

__device__ __forceinline__ void jet_sin_base(const double z[4], double out[4], JetCos& jc) {
  double S0, C0;
  sincos(z[0], &S0, &C0);
  out[0] = S0;
  out[1] = C0 * z[1];
  out[2] = C0 * z[2] - 0.5 * S0 * z[1] * z[1];
  out[3] = C0 * z[3];
  jc.c1 = C0;
  jc.ns = -S0;
  jc.cs = -S0 * z[1];
  jc.css = -S0 * z[2] - 0.5 * C0 * z[1] * z[1];
  jc.cr = -S0 * z[3];
}

__device__ __forceinline__ void jet_tangent(const JetCos& jc, const double y[4], double out[4]) {
  out[0] = jc.c1 * y[0];
  out[1] = jc.c1 * y[1] + jc.cs * y[0];
  out[2] = jc.c1 * y[2] + jc.cs * y[1] + jc.css * y[0];
  out[3] = jc.c1 * y[3] + jc.cr * y[0];
}

}  // namespace nlrom
