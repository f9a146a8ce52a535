// Fused hidden-layer chain of the decoder bundle on thread-block clusters.
//
// The per-layer GEMMs of the hidden chain are tiny (w x w x 16 columns per group,
// ~21 MFLOP per layer at cfg2) and latency-bound as separate kernels. Here one
// cluster of CS CTAs carries one column group [base jet | nk tangents] through ALL
// hidden layers: CTA `rank` owns output rows [rank*R, rank*R + R) of every layer
// (R = w / CS), computes them on the fp64 tensor pipe (DMMA) from the full
// activation of the previous layer held in its shared memory, applies the jet-sin
// epilogue, and broadcasts its slice into every CTA of the cluster through
// distributed shared memory; one cluster barrier per layer. The next layer's weight
// slice is prefetched with cp.async while the current layer computes.
// Columns of different groups are independent across layers (every group carries
// its own copy of the base jet), so clusters never talk to each other.
#pragma once
#include <cooperative_groups.h>
#include "common.cuh"
#include "gemm_f64.cuh"
#include "mc_device.cuh"
#include "cluster_async.cuh"

namespace nlrom {

constexpr int MLP_MAXL = 16;

// Optional phase timestamps (tools/probes/chain_probe.cu): CTA (0,0) thread 0, per layer.
#ifndef MLP_BULK
#define MLP_BULK 1   // bulk shared-memory copies + per-buffer mbarriers instead of DSMEM stores + cluster.sync
#endif
#ifdef NLROM_CHAIN_TRACE
__device__ long long g_chain_trace[MLP_MAXL][6];
__device__ long long g_bwd_trace[MLP_MAXL + 1][6];
#define CHAIN_MARK(l, p) \
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_chain_trace[l][p] = clock64();
#define BWD_MARK(s, p) \
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) g_bwd_trace[s][p] = clock64();
#else
#define CHAIN_MARK(l, p)
#define BWD_MARK(s, p)
#endif

struct MlpFwdArgs {
  // seed of the jet (same as k_seed_jet)
  const double* r;
  const double* rbar;
  const double* rdbar;
  int n_p, n_q, n;
  double dt, alpha;
  int drop_fict;
  // hidden layers l = 0 .. L1-1: W[l] (w x in[l]) row-major with ld ldW[l]; out dim w
  int L1, w;
  const double* W[MLP_MAXL];
  const double* b[MLP_MAXL];
  int ldW[MLP_MAXL];
  int in[MLP_MAXL];
  const double* Wp[MLP_MAXL];  // W[l] re-laid out (w x ldp, zero padded) so one TMA bulk copy lands a slice
  int ldp;                     // == MlpPlan::ldws(kmax)
  // outputs
  double* cache[MLP_MAXL];  // vhp caches: (n_sims * 2 n_q) x ldc per layer
  int ldc;
  double* Hout;  // last hidden layer in the output layout: (n_sims * (2 + 2 n_q)) x ldH
  int ldH;
  int G, gps;
};

// shared-memory plan (doubles): X[2][KP][LDX] | Wb[2][R][LDWS] | Bb[2][R] | Ys[G][R+1] | Os[R][LDX]
// (KP = KMAX rounded up to 16; padding rows / columns are zero)
template <int R, int G>
struct MlpPlan {
  static constexpr int LDX = ((G + 7) / 8) * 8 + 4;  // == 4 or 12 (mod 16): conflict-free fragments
  static __host__ __device__ int kp(int kmax) { return (kmax + 15) & ~15; }
  static __host__ __device__ int ldws(int kmax) { return kp(kmax) + 4; }
  static __host__ __device__ size_t bytes(int kmax) {
    return (size_t)(2 * kp(kmax) * LDX + 2 * R * ldws(kmax) + 2 * R + G * (R + 1) + R * LDX) * 8 + 32;
  }
};

// weight slice (R rows, K columns; the device weights are zero-padded to an even ld) + bias slice
template <int R>
__device__ __forceinline__ void mlp_load_w(double* Wb, double* Bb, int ldws, const double* W, int ldW,
                                           const double* b, int r0, int K, int tid, int nt) {
  const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const int Kp = (K + 15) & ~15;  // columns [K, Kp) are zero-filled (cp.async src-size 0)
  for (int rr = warp; rr < R; rr += nw)
    for (int k = 2 * lane; k < Kp; k += 64) {
      const bool ok = k < K;  // K even or the device weights are zero-padded to an even ld
      cp_async16(Wb + rr * ldws + k, ok ? W + (size_t)(r0 + rr) * ldW + k : W, ok);
    }
  for (int i = tid; i < R; i += nt) cp_async8(Bb + i, b + r0 + i);
}

template <int R, int G, int CS>
__global__ void __launch_bounds__(256) k_mlp_jet_fwd(MlpFwdArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  using P = MlpPlan<R, G>;
  extern __shared__ __align__(16) double sm[];
  const int kmax = P::kp(max(a.w, a.n_q));
  const int LDX = P::LDX;
  const int LDWS = P::ldws(kmax);
  constexpr int NTH = 256;
  // buffers addressed arithmetically (a pointer array indexed by l & 1 would live in local memory)
  auto Xb = [&](int i) { return sm + i * kmax * LDX; };
  auto Wbuf = [&](int i) { return sm + 2 * kmax * LDX + i * R * LDWS; };
  auto Bbuf = [&](int i) { return sm + 2 * kmax * LDX + 2 * R * LDWS + i * R; };
  double* Ys = sm + 2 * kmax * LDX + 2 * R * LDWS + 2 * R;  // [G][R+1]
  double* Os = Ys + G * (R + 1);                               // [R][LDX] outgoing slice
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster.block_rank();
  const int r0 = rank * R;
  const int gg = blockIdx.y;                 // global group = sim * gps + gl
  const int sim = gg / a.gps, gl = gg % a.gps;
  const int nk = (G - 4) / 4;
  const int cs = 2 + 2 * a.n_q;  // output-layer columns per sim (see EpiJetOutC)

  // weight + bias slices land by ONE TMA bulk copy each (padded global layout), on a
  // per-buffer mbarrier; issued one layer ahead by thread 0
  uint64_t* wbar = reinterpret_cast<uint64_t*>(Os + R * LDX);
  auto issue_w = [&](int l) {
    uint64_t* bar = wbar + (l & 1);
    mbar_expect_tx(bar, (uint32_t)(R * LDWS * 8 + R * 8));
    tma_g2s(Wbuf(l & 1), a.Wp[l] + (size_t)r0 * LDWS, (uint32_t)(R * LDWS * 8), bar);
    tma_g2s(Bbuf(l & 1), a.b[l] + r0, (uint32_t)(R * 8), bar);
  };
  // activation hand-off (MLP_BULK): each CTA sends its R x LDX slice of layer l's output to every
  // CTA of the cluster with ONE bulk shared-memory copy per destination, completing transaction
  // bytes on the destination's per-buffer mbarrier xbar[(l + 1) & 1]; the next layer waits on its
  // own barrier instead of a cluster-wide barrier. A buffer's next phase is armed (expect_tx) before
  // this CTA sends the slice every peer needs to produce that phase's data, so no copy can complete
  // on an unarmed phase; a peer writes buffer b only after it consumed our slice of the input held
  // there two layers ago, i.e. after we finished reading b (no write-after-read race).
  uint64_t* xbar = wbar + 2;
  constexpr uint32_t SLICE = (uint32_t)(R * P::LDX * 8);
  if (tid == 0) {
    mbar_init(wbar, 1);
    mbar_init(wbar + 1, 1);
    if (MLP_BULK) {
      mbar_init(xbar, 1);
      mbar_init(xbar + 1, 1);
    }
    fence_mbar_init();
    if (MLP_BULK && a.L1 >= 2) mbar_expect_tx(xbar + 1, CS * SLICE);   // input of layer 1
    issue_w(0);  // layer-0 weights do not depend on the producer: before the dependency wait
  }
  if (MLP_BULK) cluster_sync_all();   // every CTA's barriers exist (and are armed) before anyone sends
  pdl_wait();
  pdl_launch();
  // seed of this group: X[0][i][c], i < n_q; rows n_q .. kmax of X[0] and rows w .. kmax of X[1]
  // are zero (K padding). Rows < w of X[1] are NOT touched here: other CTAs of the cluster may
  // already be broadcasting their layer-0 slices into them.
  for (int t = tid; t < (kmax - a.n_q) * LDX; t += NTH) Xb(0)[a.n_q * LDX + t] = 0.0;
  for (int t = tid; t < (kmax - a.w) * LDX; t += NTH) Xb(1)[a.w * LDX + t] = 0.0;
  for (int t = tid; t < a.n_q * G; t += NTH) {
    const int i = t / G, cl = t % G;
    const double* rs = a.r + (size_t)sim * a.n;
    const double q = rs[a.n_p + i];
    const double v = q - a.rbar[(size_t)sim * a.n + a.n_p + i];
    const double qdb = a.rdbar[(size_t)sim * a.n + a.n_p + i];
    double val = 0.0;
    if (cl < 4) {
      if (cl == 0) val = q;
      else if (cl == 1) val = a.drop_fict ? 0.0 : v;
      else if (cl == 3) val = (a.drop_fict ? (1.0 + a.alpha * a.dt) : (3.0 + a.alpha * a.dt)) * v - a.dt * qdb;
    } else {
      const int k = (cl - 4) >> 2, s = (cl - 4) & 3;
      if (s == 0 && gl * nk + k == i) val = 1.0;
    }
    Xb(0)[i * LDX + cl] = val;
  }
  for (int l = 0; l < a.L1; ++l) {
    const int K = a.in[l];
    double* Xc = Xb(l & 1);
    double* Xn = Xb((l + 1) & 1);
    if (l + 1 < a.L1 && tid == 0) issue_w(l + 1);  // buffer (l+1)&1 was last read by layer l-1
    CHAIN_MARK(l, 0);
    if (l == 0) __syncthreads();  // seed (barrier init) visible
    if (MLP_BULK && l >= 1) mbar_wait(xbar + (l & 1), (uint32_t)(((l - 1) >> 1) & 1));   // input l complete
    mbar_wait(wbar + (l & 1), (l >> 1) & 1);  // this layer's weights have landed
    CHAIN_MARK(l, 1);
    // DMMA: warp -> 8x8 tiles of the R x G slice, 4 interleaved K chains; K padded to 16 with zeros
    const double* Ws = Wbuf(l & 1);
    constexpr int TM = R / 8, TN = G / 8, NT = TM * TN;
    const int Kp = (K + 15) & ~15;
    for (int tile = warp; tile < NT; tile += NTH / 32) {
      const int tm = tile % TM, tn = tile / TM;
      double c[4][2] = {};
      const double* wrow = Ws + (tm * 8 + (lane >> 2)) * LDWS + (lane & 3);
      const double* xcol = Xc + (lane & 3) * LDX + tn * 8 + (lane >> 2);
      // operands one 16-deep step ahead of the DMMAs (the shared-memory loads were the chain's
      // dominant stall: short scoreboard on every DMMA)
      double wa[4], xb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        wa[u] = wrow[4 * u];
        xb[u] = xcol[(4 * u) * LDX];
      }
      for (int k0 = 0; k0 < Kp; k0 += 16) {
        const int k1 = k0 + 16 < Kp ? k0 + 16 : k0;   // last step: a harmless reload
        double wn[4], xn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          wn[u] = wrow[k1 + 4 * u];
          xn[u] = xcol[(k1 + 4 * u) * LDX];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma(c[u][0], c[u][1], wa[u], xb[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          wa[u] = wn[u];
          xb[u] = xn[u];
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = tm * 8 + (lane >> 2), col = tn * 8 + 2 * (lane & 3) + e;
        Ys[col * (R + 1) + row] = (c[0][e] + c[1][e]) + (c[2][e] + c[3][e]);
      }
    }
    if (MLP_BULK && tid == 0) bulk_wait_read0();   // the previous layer's copies have read Os
    __syncthreads();
    CHAIN_MARK(l, 2);
    // jet-sin epilogue on the R rows; broadcast the activated slice to every CTA of the cluster
    const bool last = (l + 1 == a.L1);
    for (int t = tid; t < R * (1 + nk); t += NTH) {
      const int rr = t % R, unit = t / R;  // unit 0: base jet, unit 1 + k: tangent k
      const int m = r0 + rr;
      double z[4], o[4];
#pragma unroll
      for (int s = 0; s < 4; ++s) z[s] = Ys[s * (R + 1) + rr];
      z[0] += Bbuf(l & 1)[rr];
      JetCos jc;
      jet_sin_base(z, o, jc);
      int col = 0;
      int kg = -1;
      if (unit > 0) {
        const int k = unit - 1;
        kg = gl * nk + k;
        double y[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) y[s] = Ys[(4 + 4 * k + s) * (R + 1) + rr];
        if (kg < a.n_q) {
          double* Cz = a.cache[l] + (size_t)sim * 2 * a.n_q * a.ldc;
          Cz[(size_t)(2 * kg) * a.ldc + m] = jc.c1;  // sin'(z) as a dual: cos z0, -sin z0 y0
          Cz[(size_t)(2 * kg + 1) * a.ldc + m] = jc.ns * y[0];
        }
        jet_tangent(jc, y, o);
        col = 4 + 4 * k;
      }
      if (last) {
        // compact layout for the linear output layer: base once per sim, tangents by index
        if (unit == 0 && gl == 0) {
          a.Hout[(size_t)(sim * cs) * a.ldH + m] = o[0];            // value slot
          a.Hout[(size_t)(sim * cs + 1) * a.ldH + m] = 2.0 * o[2];  // 2 h_ss -> hvv
        } else if (unit > 0 && kg < a.n_q) {
          a.Hout[(size_t)(sim * cs + 2 + 2 * kg) * a.ldH + m] = o[0];                     // h_t -> J
          a.Hout[(size_t)(sim * cs + 3 + 2 * kg) * a.ldH + m] = fma(2.0, o[2], o[3]);  // 2 h_tss + h_tr -> dJ
        }
      } else {
#pragma unroll
        for (int s = 0; s < 4; ++s) Os[rr * LDX + col + s] = o[s];
      }
    }
    if (!last && MLP_BULK) {
      __syncthreads();   // Os complete
      CHAIN_MARK(l, 3);
      if (tid == 0) {
        // arm the phase of buffer l & 1 that holds input l + 2 (input l's phase completed above)
        if (l + 2 < a.L1) mbar_expect_tx(xbar + (l & 1), CS * SLICE);
        fence_proxy_async();   // Os (generic stores) visible to the bulk copies
        const uint32_t src = smem_u32(Os), dst0 = smem_u32(Xn + r0 * LDX), bar0 = smem_u32(xbar + ((l + 1) & 1));
        for (int d = 0; d < CS; ++d) {
          const int dst = (rank + d) % CS;   // staggered destinations
          bulk_s2s(mapa(dst0, dst), src, SLICE, mapa(bar0, dst));
        }
        bulk_commit();
      }
      CHAIN_MARK(l, 4);
      CHAIN_MARK(l, 5);
    } else {
      if (!last) {
        // broadcast the R x G slice to every CTA of the cluster: warp -> destination CTA,
        // 16-byte distributed-shared-memory stores of whole rows (stores straight from the
        // epilogue, 2 x 16 B per task and destination, measured slower: the cluster barrier then
        // waits on many more outstanding remote stores, 6.9k vs 6.0k cycles per layer)
        __syncthreads();
        CHAIN_MARK(l, 3);
        constexpr int C2 = G / 2;  // 16-byte chunks per row
        for (int dst = warp; dst < CS; dst += NTH / 32) {
          double* Xr = cluster.map_shared_rank(Xn, dst);
          for (int t = lane; t < R * C2; t += 32) {
            const int rr = t / C2, c2 = (t % C2) * 2;
            *reinterpret_cast<double2*>(Xr + (r0 + rr) * LDX + c2) = *reinterpret_cast<const double2*>(Os + rr * LDX + c2);
          }
        }
      }
      CHAIN_MARK(l, 4);
      cluster.sync();  // next activation complete in every CTA; Xc, Ys and Os free for reuse
      CHAIN_MARK(l, 5);
    }
  }
}


}  // namespace nlrom

namespace nlrom {

// Fused vhp backward chain (complex-step BP in dual arithmetic):
//   Delta_{L-2} = g (*) cos(z_{L-2}),  Delta_{l-1} = (W_l^T Delta_l) (*) cos(z_{l-1}),  G = W_0^T Delta_0
// per column group of 8 passes (16 columns: real / dual slot of each pass), one cluster
// per group, CTA rank owns rows [rank*R, rank*R + R) of every stage; same DSMEM
// broadcast scheme as k_mlp_jet_fwd. z are the pre-activation caches of the forward.
struct MlpBwdArgs {
  const double* g;          // (n_sims, w): W_L^T P a   (or, if gpart: chunk partials summed here)
  const double* gpart;      // (n_sims, gnch, w) partials of k_gemv_t2, may be null
  int gnch;
  int L1, w, n_q;
  const double* WT[MLP_MAXL];  // WT[l]: (in_l x ldWT[l]) = W_l^T, rows in_l (w for l >= 1, n_q for l = 0)
  int ldWT[MLP_MAXL];
  const double* WTp[MLP_MAXL];  // W_l^T re-laid out (w x ldpb, zero padded rows / columns): one TMA per slice
  int ldpb;
  const double* cache[MLP_MAXL];  // (n_sims * 2 n_q) x ldc
  int ldc;
  double* Gt;               // (n_sims * 2 n_q) x ldG
  int ldG;
  int gpb;                  // groups (of 8 passes) per sim
};

template <int R, int CS, int GB = 16>
__global__ void __launch_bounds__(256) k_mlp_dual_bwd(MlpBwdArgs a) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int G = GB, NTH = 256;  // G columns = G / 2 dual passes per group
  constexpr int PG = G / 2;
  using P = MlpPlan<R, G>;
  extern __shared__ __align__(16) double sm[];
  const int kmax = P::kp(a.w);
  const int LDX = P::LDX;
  const int LDWS = P::ldws(kmax);
  auto Xb = [&](int i) { return sm + i * kmax * LDX; };
  auto Wbuf = [&](int i) { return sm + 2 * kmax * LDX + i * R * LDWS; };
  auto Zbuf = [&](int i) { return sm + 2 * kmax * LDX + 2 * R * LDWS + i * R * G; };  // [R][G] cache slice
  constexpr int NTILE = (R / 8) * (G / 8);
  constexpr int KSPL = NTILE >= 8 ? 1 : (8 / NTILE > 4 ? 4 : 8 / NTILE);
  double* Ys = sm + 2 * kmax * LDX + 2 * R * LDWS + 2 * R * G;  // [KSPL][G][R+1] partial tiles
  double* Os = Ys + KSPL * G * (R + 1);                          // [R][LDX]
  auto ysum = [&](int col, int row) {
    double v = Ys[col * (R + 1) + row];
#pragma unroll
    for (int k2 = 1; k2 < KSPL; ++k2) v += Ys[k2 * G * (R + 1) + col * (R + 1) + row];
    return v;
  };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster.block_rank();
  const int r0 = rank * R;
  const int gg = blockIdx.y, sim = gg / a.gpb, gl = gg % a.gpb;
  const int L1 = a.L1;
  // stage s = 0 .. L1: s = 0 builds Delta_{L1-1}; stage s >= 1 multiplies by W_{L1-s}^T;
  // stages 1 .. L1-1 end with cos(z_{L1-1-s}); stage L1 writes G.
  uint64_t* wbar = reinterpret_cast<uint64_t*>(Os + R * LDX);
  auto load_w = [&](int l, int buf) {  // rows r0.. of W_l^T (zero beyond in_l), K = w: one TMA bulk copy
    if (tid == 0) {
      mbar_expect_tx(wbar + buf, (uint32_t)(R * LDWS * 8));
      tma_g2s(Wbuf(buf), a.WTp[l] + (size_t)r0 * LDWS, (uint32_t)(R * LDWS * 8), wbar + buf);
    }
  };
  if (tid == 0) {
    mbar_init(wbar, 1);
    mbar_init(wbar + 1, 1);
    fence_mbar_init();
  }
  auto load_z = [&](int l, int buf) {  // cache_l rows r0.. for the group's 16 columns
    const double* C = a.cache[l] + (size_t)sim * 2 * a.n_q * a.ldc;
    for (int t = tid; t < R * G; t += NTH) {
      const int rr = t % R, col = t / R;
      const int p = gl * PG + col / 2;
      double* dst = Zbuf(buf) + rr * G + col;
      if (p < a.n_q && r0 + rr < a.w) cp_async8(dst, C + (size_t)(2 * p + (col & 1)) * a.ldc + r0 + rr);
      else *dst = 0.0;
    }
  };
  // prologue: constants (weights of the first multiply, stage 1) before the dependency wait
  load_w(L1 - 1, 1);
  // the forward caches were written by the jet chain, which has completed when this grid starts
  // (the producer k_gemv_t2 launches dependents only after its own wait): load before ours
  load_z(L1 - 1, 0);
  cp_async_commit();
  // K padding rows w .. kmax of both X buffers: zero (the padded weight columns are zero, but
  // stale shared memory may hold NaN / Inf bit patterns, and 0 * NaN = NaN). Remote CTAs only
  // ever write rows < w.
  for (int t = tid; t < (kmax - a.w) * LDX; t += NTH) {
    Xb(0)[a.w * LDX + t] = 0.0;
    Xb(1)[a.w * LDX + t] = 0.0;
  }
  pdl_wait();
  pdl_launch();
  __shared__ double gsum[256];
  __shared__ double gval[32];
  if (a.gpart) {  // g rows of this CTA = fixed-order sum of the GEMV chunk partials
    const int rr = tid % R, grp = tid / R, ng = NTH / R;
    double acc = 0.0;
    if (r0 + rr < a.w)
      for (int c = grp; c < a.gnch; c += ng) acc += a.gpart[((size_t)sim * a.gnch + c) * a.w + r0 + rr];
    gsum[grp * R + rr] = acc;
    __syncthreads();
    if (tid < R) {
      double t2 = 0.0;
      for (int g2 = 0; g2 < ng; ++g2) t2 += gsum[g2 * R + tid];
      gval[tid] = t2;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int s = 0; s <= L1; ++s) {
    const int l = L1 - s;  // stage s >= 1 multiplies by W_l^T (l = L1 - s)
    // prefetch the next stage's weights and cache slice
    if (s + 1 <= L1 && s >= 1) load_w(l - 1, (s + 1) & 1);
    if (s + 1 <= L1 - 1) load_z(L1 - 1 - (s + 1) + 0, (s + 1) & 1);
    cp_async_commit();
    BWD_MARK(s, 0);
    if (s >= 1) {
      double* Xc = Xb(s & 1);
      const double* Ws = Wbuf(s & 1);
      constexpr int TM = R / 8, TN = G / 8, NT = TM * TN;
      const int Kp = (a.w + 15) & ~15;
      cp_async_wait<1>();
      mbar_wait(wbar + (s & 1), ((s - 1) >> 1) & 1);
      __syncthreads();
      BWD_MARK(s, 1);
      // K split over KSPL warps per tile when there are fewer tiles than warps (shorter DMMA
      // dependency chains); the partial tiles are summed in fixed order by the epilogue
      const int n16 = Kp / 16;  // K segments in units of 16 (some may be empty for small K)
      for (int tw = warp; tw < NT * KSPL; tw += NTH / 32) {
        const int tile = tw % NT, ks = tw / NT;
        const int tm = tile % TM, tn = tile / TM;
        double c[4][2] = {};
        const double* wrow = Ws + (tm * 8 + (lane >> 2)) * LDWS + (lane & 3);
        const double* xcol = Xc + (lane & 3) * LDX + tn * 8 + (lane >> 2);
        const int kb = 16 * (ks * n16 / KSPL), ke = 16 * ((ks + 1) * n16 / KSPL);
        if (kb < ke) {   // operands one step ahead of the DMMAs (as in the forward chain)
          double wa[4], xb[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            wa[u] = wrow[kb + 4 * u];
            xb[u] = xcol[(kb + 4 * u) * LDX];
          }
          for (int k0 = kb; k0 < ke; k0 += 16) {
            const int k1 = k0 + 16 < ke ? k0 + 16 : k0;
            double wn[4], xn[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              wn[u] = wrow[k1 + 4 * u];
              xn[u] = xcol[(k1 + 4 * u) * LDX];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) dmma(c[u][0], c[u][1], wa[u], xb[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              wa[u] = wn[u];
              xb[u] = xn[u];
            }
          }
        }
        double* Yp = Ys + ks * G * (R + 1);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int row = tm * 8 + (lane >> 2), col = tn * 8 + 2 * (lane & 3) + e;
          Yp[col * (R + 1) + row] = (c[0][e] + c[1][e]) + (c[2][e] + c[3][e]);
        }
      }
      __syncthreads();
      BWD_MARK(s, 2);
    }
    if (s == L1) {
      // G = W_0^T Delta_0: rows i < n_q
      for (int t = tid; t < R * G; t += NTH) {
        const int rr = t % R, col = t / R;
        const int i = r0 + rr, p = gl * PG + col / 2;
        if (i < a.n_q && p < a.n_q)
          a.Gt[((size_t)sim * 2 * a.n_q + 2 * p + (col & 1)) * a.ldG + i] = ysum(col, rr);
      }
      break;
    }
    // Delta rows of this CTA: (input (*) cos(z)) in dual arithmetic, z = cache of layer L1-1-s
    const double* Z = Zbuf(s & 1);
    for (int t = tid; t < R * PG; t += NTH) {
      const int rr = t % R, j = t / R;
      const int m = r0 + rr;
      double d0, d1;
      if (s == 0) {
        d0 = a.gpart ? gval[rr] : a.g[(size_t)sim * a.w + m];
        d1 = 0.0;
      } else {
        d0 = ysum(2 * j, rr);
        d1 = ysum(2 * j + 1, rr);
      }
      // the cache holds sin'(z) = cos(z0 + z1 e) = f0 + f1 e (formed by the forward's epilogue);
      // (d0 + d1 e)(f0 + f1 e) = d0 f0 + (d0 f1 + d1 f0) e
      const double f0 = Z[rr * G + 2 * j], f1 = Z[rr * G + 2 * j + 1];
      Os[rr * LDX + 2 * j] = d0 * f0;
      Os[rr * LDX + 2 * j + 1] = fma(d0, f1, d1 * f0);
    }
    __syncthreads();
    BWD_MARK(s, 3);
    {
      double* Xn = Xb((s + 1) & 1);
      constexpr int C2 = G / 2;
      for (int dst = warp; dst < CS; dst += NTH / 32) {
        double* Xr = cluster.map_shared_rank(Xn, dst);
        for (int t = lane; t < R * C2; t += 32) {
          const int rr = t / C2, c2 = (t % C2) * 2;
          if (r0 + rr < a.w)
            *reinterpret_cast<double2*>(Xr + (r0 + rr) * LDX + c2) =
                *reinterpret_cast<const double2*>(Os + rr * LDX + c2);
        }
      }
    }
    BWD_MARK(s, 4);
    cluster.sync();
    BWD_MARK(s, 5);
  }
}

template <int R, int G = 16>
inline size_t mlp_bwd_smem(int w) {
  using P = MlpPlan<R, G>;
  const int kp = P::kp(w);
  constexpr int NTILE = (R / 8) * (G / 8);
  constexpr int KSPL = NTILE >= 8 ? 1 : (8 / NTILE > 4 ? 4 : 8 / NTILE);
  return (size_t)(2 * kp * P::LDX + 2 * R * P::ldws(kp) + 2 * R * G + KSPL * G * (R + 1) + R * P::LDX) * 8 + 16;
}

}  // namespace nlrom
