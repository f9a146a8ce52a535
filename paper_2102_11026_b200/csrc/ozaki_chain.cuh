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
  int real_once = 0;    // vhp cache real parts once per sim (EpiJet::real_once)

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
          if (!real_once || kg == 0) Cz[(size_t)(2 * kg) * ldcache + m] = jc.c1;
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

// Seed layer of the batched decoder fused with its consumer's B operand (hidden layer 1 on tcgen05).
// The jet seed (k_seed_jet) is sparse -- per column group three base vectors (q, v, w) and unit
// tangent vectors e_kg -- so layer 0 (w = 256 rows, K = n_q) is three mat-vecs per group and copies
// of W_0's columns. One CTA per 32 columns (whole groups), one thread per row: z, the jet sin (bias,
// vhp cache duals as EpiJet) into shared memory; then one thread per (column, 32-row K chunk) holds
// its 32 values, and since the CTA has all 256 rows of its columns the column exponents need no
// exchange. DIG: the digits go straight to the consumer's B tiles (the CTA's 1 KB half of each
// (K chunk, plane) slice) plus the exponents; else the fp64 activations + EpiJet::colhw partials
// (the fp64 hand-off of the same values, bitwise equal downstream).
struct SeedLayerArgs {
  const double* r;
  const double* rbar;
  const double* rdbar;
  int n_p, n_q, n;
  double dt, alpha;
  int drop_fict;
  const double* W0;   // (256 x n_q) row-major, ld ldW0
  int ldW0;
  const double* b0;
  double* cache;      // layer-0 vhp cache, (n_sims * 2 n_q) x ldcache
  int ldcache;
  int G, gps, ncols;
  unsigned char* dig; // DIG: [ceil(ncols / 64)][8][S][64 x 32 B]
  int* dexp;          // DIG: [ceil(ncols / 64) * 64]
  double* H;          // !DIG: (ncols x ldh)
  int ldh;
  unsigned* colhw;    // !DIG: [ncols][8]
  int real_once;      // vhp cache real parts once per sim (EpiJet::real_once)
};
constexpr int SEED_LDZ = 258;
inline size_t seed_layer_smem() { return (size_t)32 * SEED_LDZ * 8 + 8 * 32 * 4 + 32 * 4; }

template <bool DIG>
__global__ void __launch_bounds__(256, 2) k_seed_layer(SeedLayerArgs a) {
  using namespace oz;
  extern __shared__ __align__(128) unsigned char sl_smem[];
  double* Zs = reinterpret_cast<double*>(sl_smem);                       // [32][SEED_LDZ]
  unsigned* part = reinterpret_cast<unsigned*>(Zs + 32 * SEED_LDZ);      // [8][32]
  int* colEs = reinterpret_cast<int*>(part + 8 * 32);                    // [32]
  pdl_wait();
  pdl_launch();
  const int m = threadIdx.x;
  const int c0 = blockIdx.x * 32;
  const int G = a.G, nk = (G - 4) / 4;
  const double* Wr = a.W0 + (size_t)m * a.ldW0;
  const double c3 = a.drop_fict ? (1.0 + a.alpha * a.dt) : (3.0 + a.alpha * a.dt);
  for (int gt = 0; gt < 32 / G; ++gt) {
    const int cg = c0 + gt * G;
    double* zc = Zs + (gt * G) * SEED_LDZ + m;
    if (cg >= a.ncols) {
      for (int j = 0; j < G; ++j) zc[j * SEED_LDZ] = 0.0;
      continue;
    }
    const int gg = cg / G, sim = gg / a.gps, gl = gg % a.gps;
    const double* rs = a.r + (size_t)sim * a.n + a.n_p;
    const double* rb = a.rbar + (size_t)sim * a.n + a.n_p;
    const double* rdb = a.rdbar + (size_t)sim * a.n + a.n_p;
    double zq = 0.0, zv = 0.0, zw = 0.0;
    for (int i = 0; i < a.n_q; ++i) {
      const double wi = Wr[i], q = rs[i], v = q - rb[i];
      zq = fma(wi, q, zq);
      zv = fma(wi, v, zv);
      zw = fma(wi, c3 * v - a.dt * rdb[i], zw);
    }
    double z[4] = {zq + a.b0[m], a.drop_fict ? 0.0 : zv, 0.0, zw}, o[4];
    JetCos jc;
    jet_sin_base(z, o, jc);
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) zc[s2 * SEED_LDZ] = o[s2];
    double* Cz = a.cache ? a.cache + (size_t)sim * 2 * a.n_q * a.ldcache : nullptr;
    for (int k = 0; k < nk; ++k) {
      const int kg = gl * nk + k;
      const double y[4] = {kg < a.n_q ? Wr[kg] : 0.0, 0.0, 0.0, 0.0};
      double yo[4];
      jet_tangent(jc, y, yo);
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) zc[(4 + 4 * k + s2) * SEED_LDZ] = yo[s2];
      if (Cz && kg < a.n_q) {
        if (!a.real_once || kg == 0) Cz[(size_t)(2 * kg) * a.ldcache + m] = jc.c1;
        Cz[(size_t)(2 * kg + 1) * a.ldcache + m] = jc.ns * y[0];
      }
    }
  }
  __syncthreads();
  const int c = m & 31, rg = m >> 5;   // column, 32-row group (= K chunk of the consumer)
  const bool live = c0 + c < a.ncols;
  double v[32];
  {
    const double2* src = reinterpret_cast<const double2*>(Zs + c * SEED_LDZ + rg * 32);
#pragma unroll
    for (int q2 = 0; q2 < 16; ++q2) {
      const double2 w = src[q2];
      v[2 * q2] = w.x;
      v[2 * q2 + 1] = w.y;
    }
  }
  unsigned hw = 0u;
#pragma unroll
  for (int q = 0; q < 32; ++q) hw = max(hw, (unsigned)__double2hiint(fabs(v[q])));
  if constexpr (!DIG) {
    if (live) a.colhw[(size_t)(c0 + c) * 8 + rg] = hw;
    for (int cc = 0; cc < 32 && c0 + cc < a.ncols; ++cc) a.H[(size_t)(c0 + cc) * a.ldh + m] = Zs[cc * SEED_LDZ + m];
  } else {
    part[rg * 32 + c] = hw;
    __syncthreads();
    if (m < 32) {
      unsigned h = 0u;
#pragma unroll
      for (int p = 0; p < 8; ++p) h = max(h, part[p * 32 + m]);
      const int E = h ? exp_of(__hiloint2double((int)h, (int)0xFFFFFFFFu)) : 0;
      colEs[m] = E;
      a.dexp[c0 + m] = E;
    }
    __syncthreads();
    const double sc = pow2(QBITS - colEs[c]);
    long long qv[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) qv[q] = fixed55(v[q], sc);
    // this CTA's 32 columns are rows (c0 % 64) .. + 31 of the 64-row plane slices (their 1 KB half)
    unsigned char* dst = a.dig + ((size_t)(c0 / 64) * 8 + rg) * Cfg<64>::B_STAGE + (c0 % 64) * BK;
#pragma unroll
    for (int t2 = 0; t2 < S; ++t2) {
#pragma unroll
      for (int qb = 0; qb < 2; ++qb) {
        const long long* q4 = qv + 16 * qb;
        *reinterpret_cast<uint4*>(dst + t2 * Cfg<64>::B_SLICE + core_off(c, 16 * qb)) =
            make_uint4(pack_plane(q4[0], q4[1], q4[2], q4[3], t2), pack_plane(q4[4], q4[5], q4[6], q4[7], t2),
                       pack_plane(q4[8], q4[9], q4[10], q4[11], t2), pack_plane(q4[12], q4[13], q4[14], q4[15], t2));
      }
    }
  }
}

// fp64 activations -> the consumer's B digit tiles, for a consumer whose producer cannot write them
// (the output layer: its input is the compact last hidden layer, and with 8 m tiles its converters
// would convert every column 8 times). Column exponents from the producer's colhw partials by the
// converters' rule, so the digits are exactly the converters'. One thread per (column, 32-row K
// chunk); ceil(C / 64) * 64 columns (padding: zero digits, exponent 0).
__global__ void __launch_bounds__(256) k_to_digits(const double* __restrict__ B, int ldb, int C, int K,
                                                   const unsigned* __restrict__ parts, int nparts,
                                                   unsigned char* __restrict__ dig, int* __restrict__ dexp) {
  using namespace oz;
  pdl_wait();
  pdl_launch();
  const int nk = K / BK;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(t % 32) + (int)(t / (32LL * nk)) * 32, kc = (int)((t / 32) % nk);
  const int Cpad = (C + 63) / 64 * 64;
  if (c >= Cpad) return;
  const bool live = c < C;
  unsigned hw = 0u;
  if (live)
    for (int p = 0; p < nparts; ++p) hw = max(hw, parts[(size_t)c * nparts + p]);
  const int E = hw ? exp_of(__hiloint2double((int)hw, (int)0xFFFFFFFFu)) : 0;
  if (kc == 0) dexp[c] = E;
  const double sc = pow2(QBITS - E);
  long long qv[32];
  const double2* src = reinterpret_cast<const double2*>(B + (size_t)(live ? c : 0) * ldb + kc * BK);
#pragma unroll
  for (int q2 = 0; q2 < 16; ++q2) {
    const double2 w = live ? src[q2] : make_double2(0.0, 0.0);
    qv[2 * q2] = fixed55(w.x, sc);
    qv[2 * q2 + 1] = fixed55(w.y, sc);
  }
  unsigned char* dst = dig + ((size_t)(c / 64) * nk + kc) * Cfg<64>::B_STAGE;
#pragma unroll
  for (int t2 = 0; t2 < S; ++t2) {
#pragma unroll
    for (int qb = 0; qb < 2; ++qb) {
      const long long* q4 = qv + 16 * qb;
      *reinterpret_cast<uint4*>(dst + t2 * Cfg<64>::B_SLICE + core_off(c % 64, 16 * qb)) =
          make_uint4(pack_plane(q4[0], q4[1], q4[2], q4[3], t2), pack_plane(q4[4], q4[5], q4[6], q4[7], t2),
                     pack_plane(q4[8], q4[9], q4[10], q4[11], t2), pack_plane(q4[12], q4[13], q4[14], q4[15], t2));
    }
  }
}

}  // namespace nlrom
