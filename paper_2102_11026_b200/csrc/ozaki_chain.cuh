// Digit-chain epilogue of the tcgen05 Ozaki hidden layers (ozaki_tc.cuh, "Digit chain").
//
// EpiJetDig is EpiJet (bias + jet sin, vhp cache duals; the non-compact layout, output column =
// input column) for a layer whose consumer is another tcgen05 hidden layer. Instead of writing the
// fp64 activations it leaves them in the tile (in place), forms the column maxima of the tile's 128
// rows, exchanges them with the cluster peer that owns the other 128 rows of the same columns
// (M = 256), and converts the tile into the consumer's B stage layout -- 4 K chunks x 7 digit
// planes x (64 columns x 32 B) -- which one bulk copy stores (57 KB per tile). The digits and the
// exponents are those the consumer's converters would compute from the fp64 activations
// (oz::fixed55 / oz::digit against exp_of of the column's high-word maximum), so the chain is
// bitwise equal to the fp64 hand-off (tests/test_gpu_ozaki.py::test_digit_chain_bitwise).
#pragma once
#include "ozaki_tc.cuh"
#include "epilogues.cuh"

namespace nlrom {

struct EpiJetDig {
  static constexpr bool kDigitsOut = true;
  const double* bias;
  double* cache;   // (n_sims * 2 n_q) x ldcache, may be null
  int ldcache;
  int group, gps, n_q;
  unsigned char* dig;   // [ceil(C / 64)][M / 32][S][64 x 32 B]
  int* dexp;            // [ceil(C / 64) * 64]

  // BND = 64: a whole tile (one bulk store); BND = 32: one half tile of the consumer's 64-column B
  // tile (its 1 KB half of every (K chunk, plane) slice: 28 bulk stores).
  template <int NT, int BND>
  __device__ void dig_out(const Tile& t, const GemmArgs& g, int tid, const DigCtx& x) const {
    using namespace oz;
    double* Cs = x.Cs;
    const int ldc = t.ldc;
    if (tid < BND) x.colmax[tid] = 0u;
    // ---- phase 1: the jet epilogue in place; `split` threads share one (group, row) item's tangents
    {
    const int nk = (group - 4) / 4;
    const int ngt = BND / group;
    const int items = t.bm * ngt;
    const int split = items < NT ? NT / items : 1;
    double ob[4];
    double* obp = nullptr;   // deferred base outputs (other threads of the item still read the base)
    for (int i = tid; i < items * split; i += NT) {
      const int item = i % items, h = i / items;
      const int gt = item / t.bm, ml = item % t.bm;
      const int m = t.m0 + ml;
      const int cg = t.c0 + gt * group;
      if (m >= g.M || cg >= g.C) continue;
      const int gg = cg / group;
      const int sim = gg / gps, gl = gg % gps;
      double* Cz = cache ? cache + (size_t)sim * 2 * n_q * ldcache : nullptr;
      double* cs0 = Cs + (gt * group) * ldc + ml;
      double z[4], o[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) z[s] = cs0[s * ldc];
      z[0] += bias[m];
      JetCos jc;
      jet_sin_base(z, o, jc);
      const int k0 = (nk * h) / split, k1 = (nk * (h + 1)) / split;
      for (int k = k0; k < k1; ++k) {
        const int kg = gl * nk + k;
        double y[4], yo[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) y[s] = cs0[(4 + 4 * k + s) * ldc];
        jet_tangent(jc, y, yo);
#pragma unroll
        for (int s = 0; s < 4; ++s) cs0[(4 + 4 * k + s) * ldc] = yo[s];
        if (Cz && kg < n_q) {  // sin'(z0 + y0 e) = cos z0 - sin z0 y0 e (dual), for the vhp backward
          Cz[(size_t)(2 * kg) * ldcache + m] = jc.c1;
          Cz[(size_t)(2 * kg + 1) * ldcache + m] = jc.ns * y[0];
        }
      }
      if (h == 0) {
        if (split == 1) {
#pragma unroll
          for (int s = 0; s < 4; ++s) cs0[s * ldc] = o[s];
        } else {
#pragma unroll
          for (int s = 0; s < 4; ++s) ob[s] = o[s];
          obp = cs0;
        }
      }
    }
    named_bar_sync(2, NT);
    if (obp) {
#pragma unroll
      for (int s = 0; s < 4; ++s) obp[s * ldc] = ob[s];
    }
    }
    named_bar_sync(2, NT);
    // ---- phase 2: column maxima of the tile, the pair's exponents
    constexpr int RPU = 128 * BND / NT;   // rows per thread (16 or 32)
    static_assert(RPU % 16 == 0 && RPU <= 32, "conversion unit");
    const int c = tid % BND, r0 = (tid / BND) * RPU;
    const bool live = t.c0 + c < g.C;
    double v[RPU];
    {
      const double2* src = reinterpret_cast<const double2*>(Cs + c * ldc + r0);
#pragma unroll
      for (int q2 = 0; q2 < RPU / 2; ++q2) {
        const double2 w = src[q2];
        v[2 * q2] = live ? w.x : 0.0;
        v[2 * q2 + 1] = live ? w.y : 0.0;
      }
    }
    unsigned hw = 0u;
#pragma unroll
    for (int q = 0; q < RPU; ++q) hw = max(hw, (unsigned)__double2hiint(fabs(v[q])));
    atomicMax(x.colmax + c, hw);
    named_bar_sync(2, NT);
    if (tid < BND) {
      const unsigned mine = x.colmax[tid];
      const int slot = x.j & 1;
      const uint32_t me = cluster_rank_u32(), peer = me ^ 1u;
      st_async_b32(mapa(smem_u32(x.xslot + slot * BND + tid), peer), mine, mapa(smem_u32(x.xbar + slot), peer));
      mbar_wait(x.xbar + slot, (uint32_t)((x.j >> 1) & 1));
      const unsigned hwm = max(mine, x.xslot[slot * BND + tid]);
      const int E = hwm ? exp_of(__hiloint2double((int)hwm, (int)0xFFFFFFFFu)) : 0;
      x.colEs[tid] = E;
      if (me == 0) dexp[t.c0 + tid] = E;
      __syncwarp();
      if (tid == 0) mbar_expect_tx(x.xbar + slot, BND * 4);   // arm the slot for (half) tile j + 2
    }
    named_bar_sync(2, NT);   // also: every thread has read its Cs values (the staging overwrites them)
    // ---- phase 3: digits into the staging (the Cs region), one bulk store
    const double sc = pow2(QBITS - x.colEs[c]);
    long long qv[RPU];
#pragma unroll
    for (int q = 0; q < RPU; ++q) qv[q] = fixed55(v[q], sc);
    unsigned char* stg = reinterpret_cast<unsigned char*>(Cs);
    // staging [K chunk][plane][BND rows x 32 B] (BND = 64: exactly the consumer's stage layout)
    constexpr int PL = BND * BK;
    unsigned char* dst = stg + (r0 / BK) * (S * PL);
#pragma unroll
    for (int t2 = 0; t2 < S; ++t2) {
#pragma unroll
      for (int qb = 0; qb < RPU / 16; ++qb) {
        const long long* p = qv + 16 * qb;
        *reinterpret_cast<uint4*>(dst + t2 * PL + core_off(c, (r0 % BK) + 16 * qb)) =
            make_uint4(pack_plane(p[0], p[1], p[2], p[3], t2), pack_plane(p[4], p[5], p[6], p[7], t2),
                       pack_plane(p[8], p[9], p[10], p[11], t2), pack_plane(p[12], p[13], p[14], p[15], t2));
      }
    }
    fence_proxy_async();
    named_bar_sync(2, NT);
    const int nko = g.M / BK;
    if constexpr (BND == 64) {
      if (tid == 0) {
        bulk_s2g(dig + ((size_t)(t.c0 / 64) * nko + (t.m0 / BK)) * Cfg<64>::B_STAGE, stg, 4 * Cfg<64>::B_STAGE);
        bulk_commit();
      }
    } else {
      if (tid < 4 * S) {   // (K chunk, plane) slices of this half: 1 KB each
        const int kc4 = tid / S, t2 = tid % S;
        unsigned char* gdst = dig + (((size_t)(t.c0 / 64) * nko + (t.m0 / BK) + kc4) * S + t2) * Cfg<64>::B_SLICE +
                              (t.c0 % 64) * BK;
        bulk_s2g(gdst, stg + (kc4 * S + t2) * PL, PL);
        bulk_commit();
      }
    }
  }

};

}  // namespace nlrom
