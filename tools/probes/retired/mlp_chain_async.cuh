// Retired (measured slower at cfg2): asynchronous hand-off form of
// k_mlp_jet_fwd. Not compiled into libnlrom_b200.so; include after mlp_chain.cuh.
#pragma once
#include "../../../paper_2102_11026_b200/csrc/mlp_chain.cuh"
namespace nlrom {
// ---------------------------------------------------------------------------------------
// Same chain with asynchronous hand-off (cluster_async.cuh): per layer each CTA st.async's
// its activated R x G slice into every CTA's next X buffer, completing transaction bytes on
// the destination's per-source mbarrier; the next layer's DMMA walks the K rows source by
// source (own slice first) and waits only for the source it is about to read. Weights and
// biases land by TMA bulk copies on a per-buffer mbarrier, issued one layer ahead by one
// thread. No cluster-wide barrier inside the layer loop.
// smem: X[2][KP][LDX] | Wb[2][R][LDWS] | Bb[2][R] | Ys[G][R+1] | mbarriers wbar[2], xbar[2][CS]
template <int R, int G, int CS>
struct MlpAsyncPlan {
  static constexpr int LDX = MlpPlan<R, G>::LDX;
  static __host__ __device__ size_t doubles(int kmax) {
    const int kp = MlpPlan<R, G>::kp(kmax), ldws = MlpPlan<R, G>::ldws(kmax);
    return (size_t)2 * kp * LDX + 2 * R * ldws + 2 * R + G * (R + 1);
  }
  static __host__ __device__ size_t bytes(int kmax) { return doubles(kmax) * 8 + (2 + 2 * CS) * 8; }
};

template <int R, int G, int CS>
__global__ void __launch_bounds__(256) k_mlp_jet_fwd_async(MlpFwdArgs a) {
  using P = MlpPlan<R, G>;
  extern __shared__ __align__(16) double sm[];
  const int kmax = P::kp(max(a.w, a.n_q));
  constexpr int LDX = P::LDX;
  const int KP = kmax;
  const int LDWS = P::ldws(kmax);
  constexpr int NTH = 256;
  auto Xb = [&](int i) { return sm + i * KP * LDX; };
  auto Wbuf = [&](int i) { return sm + 2 * KP * LDX + i * R * LDWS; };
  auto Bbuf = [&](int i) { return sm + 2 * KP * LDX + 2 * R * LDWS + i * R; };
  double* Ys = sm + 2 * KP * LDX + 2 * R * LDWS + 2 * R;  // [G][R+1]
  uint64_t* wbar = reinterpret_cast<uint64_t*>(sm + MlpAsyncPlan<R, G, CS>::doubles(kmax));
  uint64_t* xbar = wbar + 2;                                  // [2][CS]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster_rank_u32();
  const int r0 = rank * R;
  const int gg = blockIdx.y;
  const int sim = gg / a.gps, gl = gg % a.gps;
  const int nk = (G - 4) / 4;
  const int cs = 2 + 2 * a.n_q;  // output-layer columns per sim (see EpiJetOutC)
  constexpr uint32_t SLICE = R * G * 8;  // bytes one source delivers per layer

  auto issue_weights = [&](int l) {  // one thread: layer l's weight + bias slices -> buffer l & 1
    uint64_t* bar = wbar + (l & 1);
    mbar_expect_tx(bar, (uint32_t)(R * LDWS * 8 + R * 8));
    tma_g2s(Wbuf(l & 1), a.Wp[l] + (size_t)r0 * LDWS, (uint32_t)(R * LDWS * 8), bar);
    tma_g2s(Bbuf(l & 1), a.b[l] + r0, R * 8, bar);
  };

  if (tid == 0) {
    mbar_init(wbar + 0, 1);
    mbar_init(wbar + 1, 1);
    for (int i = 0; i < 2 * CS; ++i) mbar_init(xbar + i, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    issue_weights(0);  // producer-independent: before the dependency wait
    // first phases of both X buffers: layer 0 outputs -> buffer 1, layer 1 outputs -> buffer 0
    for (int src = 0; src < CS; ++src) {
      if (a.L1 >= 2) mbar_expect_tx(xbar + 1 * CS + src, SLICE);
      if (a.L1 >= 3) mbar_expect_tx(xbar + 0 * CS + src, SLICE);
    }
  }
  cluster_sync_all();  // every CTA's barriers exist before anyone sends
  pdl_wait();
  pdl_launch();
  // seed of this group (layer-0 input, local): rows n_q .. KP of X[0] are zero
  for (int t = tid; t < (KP - a.n_q) * LDX; t += NTH) Xb(0)[a.n_q * LDX + t] = 0.0;
  for (int t = tid; t < a.n_q * G; t += NTH) {
    const int i = t / G, cl = t % G;
    const double q = a.r[(size_t)sim * a.n + a.n_p + i];
    const double v = q - a.rbar[(size_t)sim * a.n + a.n_p + i];
    const double qdb = a.rdbar[(size_t)sim * a.n + a.n_p + i];
    double val = 0.0;
    if (cl < 4) {
      if (cl == 0) val = q;
      else if (cl == 1) val = a.drop_fict ? 0.0 : v;
      else if (cl == 3) val = (a.drop_fict ? (1.0 + a.alpha * a.dt) : (3.0 + a.alpha * a.dt)) * v - a.dt * qdb;
    } else {
      const int k = (cl - 4) >> 2, s4 = (cl - 4) & 3;
      if (s4 == 0 && gl * nk + k == i) val = 1.0;
    }
    Xb(0)[i * LDX + cl] = val;
  }
  __syncthreads();

  constexpr int TM = R / 8, TN = G / 8, NT = TM * TN;
  for (int l = 0; l < a.L1; ++l) {
    const int b = l & 1, nb = (l + 1) & 1;
    const double* Xc = Xb(b);
    if (tid == 0 && l + 1 < a.L1) issue_weights(l + 1);  // buffer nb is free: layer l-1 is done
    CHAIN_MARK(l, 0);
    mbar_wait(wbar + b, (l >> 1) & 1);
    CHAIN_MARK(l, 1);
    const double* Ws = Wbuf(b);
    for (int tile = warp; tile < NT; tile += NTH / 32) {
      const int tm = tile % TM, tn = tile / TM;
      double c[4][2] = {};
      const double* wrow = Ws + (tm * 8 + (lane >> 2)) * LDWS + (lane & 3);
      const double* xcol = Xc + (lane & 3) * LDX + tn * 8 + (lane >> 2);
      if (l == 0) {
        const int Kp = (a.in[0] + 15) & ~15;
        for (int k0 = 0; k0 < Kp; k0 += 16) {
#pragma unroll
          for (int u = 0; u < 4; ++u) dmma(c[u][0], c[u][1], wrow[k0 + 4 * u], xcol[(k0 + 4 * u) * LDX]);
        }
      } else {
        const uint32_t par = ((l - 1) >> 1) & 1;
        for (int j = 0; j < CS; ++j) {
          int src = rank + j;
          if (src >= CS) src -= CS;
          mbar_wait(xbar + b * CS + src, par);
          if (tile == warp && tid == 0 && l + 2 < a.L1) mbar_expect_tx(xbar + b * CS + src, SLICE);
          const int k0 = src * R;
#pragma unroll
          for (int kk = 0; kk < R; kk += 16) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (kk + 4 * u < R)
                dmma(c[u][0], c[u][1], wrow[k0 + kk + 4 * u], xcol[(k0 + kk + 4 * u) * LDX]);
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = tm * 8 + (lane >> 2), col = tn * 8 + 2 * (lane & 3) + e;
        Ys[col * (R + 1) + row] = (c[0][e] + c[1][e]) + (c[2][e] + c[3][e]);
      }
    }
    __syncthreads();
    CHAIN_MARK(l, 2);
    const bool last = (l + 1 == a.L1);
    const uint32_t xn_base = smem_u32(Xb(nb));
    const uint32_t bar_local = smem_u32(xbar + nb * CS + rank);
    for (int t = tid; t < R * (1 + nk); t += NTH) {
      const int rr = t % R, unit = t / R;  // unit 0: base jet, unit 1 + k: tangent k
      const int m = r0 + rr;
      double z[4], o[4];
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) z[s4] = Ys[s4 * (R + 1) + rr];
      z[0] += Bbuf(b)[rr];
      JetCos jc;
      jet_sin_base(z, o, jc);
      int col = 0, kg = -1;
      if (unit > 0) {
        const int k = unit - 1;
        kg = gl * nk + k;
        double y[4];
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4) y[s4] = Ys[(4 + 4 * k + s4) * (R + 1) + rr];
        if (kg < a.n_q) {
          double* Cz = a.cache[l] + (size_t)sim * 2 * a.n_q * a.ldc;
          Cz[(size_t)(2 * kg) * a.ldc + m] = jc.c1;  // sin'(z) as a dual: cos z0, -sin z0 y0
          Cz[(size_t)(2 * kg + 1) * a.ldc + m] = jc.ns * y[0];
        }
        jet_tangent(jc, y, o);
        col = 4 + 4 * k;
      }
      if (last) {
        if (unit == 0 && gl == 0) {
#pragma unroll
          a.Hout[(size_t)(sim * cs) * a.ldH + m] = o[0];
          a.Hout[(size_t)(sim * cs + 1) * a.ldH + m] = 2.0 * o[2];
        } else if (unit > 0 && kg < a.n_q) {
#pragma unroll
          a.Hout[(size_t)(sim * cs + 2 + 2 * kg) * a.ldH + m] = o[0];
          a.Hout[(size_t)(sim * cs + 3 + 2 * kg) * a.ldH + m] = fma(2.0, o[2], o[3]);
        }
      } else {
        const uint32_t la = xn_base + (uint32_t)(((r0 + rr) * LDX + col) * 8);
#pragma unroll 1
        for (int d = 0; d < CS; ++d) {
          int dst = rank + d;
          if (dst >= CS) dst -= CS;
          const uint32_t ra = mapa(la, dst), rb = mapa(bar_local, dst);
          st_async_v2(ra, o[0], o[1], rb);
          st_async_v2(ra + 16, o[2], o[3], rb);
        }
      }
    }
    CHAIN_MARK(l, 4);
    __syncthreads();  // Ys is rewritten by the next layer
    CHAIN_MARK(l, 5);
  }
}

}  // namespace nlrom
