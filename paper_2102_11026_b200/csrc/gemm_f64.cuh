// fp64 tensor-core GEMM for the CSFD part-column space, with fused epilogues.
//
//   Y_t[c][m] = sum_k A[m][k] * B_t[c][k]        ("TN": both operands K-contiguous)
//
// A is a weight matrix (M x K, row-major, e.g. W_l (out,in)); B_t / Y_t hold one
// row per CSFD part-column c (a (pass, slot) pair; the MCArray slot axis of
// mcx.py:294-300 folded into the column space, slots of one pass adjacent).
// Real weights act on every slot independently (Cauchy-Riemann block rule,
// mcx.py:297-300 / PAPER.md:563), so one real GEMM serves all slots of all passes.
//
// Math: mma.sync.m8n8k4 f64 -> SASS DMMA.8x8x4 (the sm_100a fp64 tensor pipe;
// tcgen05 has no f64 kind). Operand tiles are staged with 16-byte
// cp.async (zero-filled outside [0,M) x [0,K) / [0,C) x [0,K)) in a 2-stage ring.
// After the K loop the accumulators (reduced across the WK K-split warps) land in a
// shared-memory tile Cs[c][m] and an epilogue functor turns that tile into outputs
// (bias on real slots, multicomplex / multi-dual / jet sin, caches, projections).
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace nlrom {

struct GemmArgs {
  const double* A;  // M x K, lda
  const double* B;  // C x K, ldb
  int lda, ldb;
  int M, C, K;      // K must be even; lda, ldb even; base pointers 16B aligned
  long long strideA, strideB;  // per blockIdx.z (batched), in doubles
  int cstep = 0;    // column tiles start every cstep columns (<= BN; 0: BN) -- tiles that hold whole
                    // column groups (the epilogue sees t.bn = cstep columns)
};

struct Tile {
  const double* Cs;  // [BN][LDC]
  int ldc;
  int m0, c0, bm, bn;
  int z;
};

template <int BM_, int BN_, int WM_, int WN_, int WK_, int BK_ = 16, int STAGES_ = 2>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, WK = WK_;
  static constexpr int BK = BK_;
  static constexpr int STAGES = STAGES_;
  static constexpr int NT = 32 * WM * WN * WK;
  static constexpr int TM = BM / WM, TN = BN / WN;
  static constexpr int FM = TM / 8, FN = TN / 8;
  static constexpr int KS = BK / WK;
  static constexpr int LDS = BK + 4;        // conflict-free 8-byte fragment loads
  static constexpr int LDC = BM + 2;        // conflict-free accumulator stores
  static constexpr int STAGE = (BM + BN) * LDS;
  static constexpr int PIPE = STAGES * STAGE;
  static constexpr int CT = BN * LDC;
  static constexpr int SMEM_DOUBLES = PIPE > CT ? PIPE : CT;
  static constexpr int SMEM_BYTES = SMEM_DOUBLES * 8;
  static_assert(TM % 8 == 0 && TN % 8 == 0, "warp tile must be a multiple of 8x8");
  static_assert(KS % 4 == 0, "K split must be a multiple of 4");
};

__device__ __forceinline__ void cp_async16(double* smem_dst, const double* gsrc, bool pred) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <class Cfg>
__device__ __forceinline__ void gemm_load_A(double* As, const GemmArgs& g, const double* A, int m0, int k0, int tid) {
  constexpr int CH = Cfg::BK / 2;  // 16-byte chunks per row
  for (int i = tid; i < Cfg::BM * CH; i += Cfg::NT) {
    int r = i / CH, ck = (i % CH) * 2;
    int m = m0 + r, k = k0 + ck;
    bool ok = (m < g.M) && (k < g.K);
    const double* src = ok ? (A + (size_t)m * g.lda + k) : A;
    cp_async16(As + r * Cfg::LDS + ck, src, ok);
  }
}

template <class Cfg>
__device__ __forceinline__ void gemm_load_B(double* Bs, const GemmArgs& g, const double* B, int c0, int k0, int tid) {
  constexpr int CH = Cfg::BK / 2;
  for (int i = tid; i < Cfg::BN * CH; i += Cfg::NT) {
    int r = i / CH, ck = (i % CH) * 2;
    int c = c0 + r, k = k0 + ck;
    bool ok = (c < g.C) && (k < g.K);
    const double* src = ok ? (B + (size_t)c * g.ldb + k) : B;
    cp_async16(Bs + r * Cfg::LDS + ck, src, ok);
  }
}

template <class Cfg>
__device__ __forceinline__ void gemm_load_stage(double* As, double* Bs, const GemmArgs& g, const double* A,
                                                const double* B, int m0, int c0, int k0, int tid) {
  gemm_load_A<Cfg>(As, g, A, m0, k0, tid);
  constexpr int CH = Cfg::BK / 2;
  for (int i = tid; i < Cfg::BN * CH; i += Cfg::NT) {
    int r = i / CH, ck = (i % CH) * 2;
    int c = c0 + r, k = k0 + ck;
    bool ok = (c < g.C) && (k < g.K);
    const double* src = ok ? (B + (size_t)c * g.ldb + k) : B;
    cp_async16(Bs + r * Cfg::LDS + ck, src, ok);
  }
}

template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::NT) gemm_tn_kernel(GemmArgs g, Epi epi) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wk = warp / (Cfg::WM * Cfg::WN);
  const int wmn = warp % (Cfg::WM * Cfg::WN);
  const int wm = wmn % Cfg::WM, wn = wmn / Cfg::WM;
  const int m0 = blockIdx.x * Cfg::BM, c0 = blockIdx.y * (g.cstep ? g.cstep : Cfg::BN);
  const double* A = g.A + (size_t)blockIdx.z * g.strideA;
  const double* B = g.B + (size_t)blockIdx.z * g.strideB;

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (g.K + Cfg::BK - 1) / Cfg::BK;
  // STAGES-deep cp.async ring: tiles kt+1 .. kt+STAGES-1 are in flight while tile kt is consumed.
  // The weight tiles (A) do not depend on the producer kernel: they are requested before the
  // programmatic-dependency wait, the activation tiles (B) after it.
#pragma unroll
  for (int s = 0; s < Cfg::STAGES - 1; ++s)
    if (s < nk) gemm_load_A<Cfg>(smem + s * Cfg::STAGE, g, A, m0, s * Cfg::BK, tid);
  pdl_wait();
  pdl_launch();
#pragma unroll
  for (int s = 0; s < Cfg::STAGES - 1; ++s) {
    if (s < nk) gemm_load_B<Cfg>(smem + s * Cfg::STAGE + Cfg::BM * Cfg::LDS, g, B, c0, s * Cfg::BK, tid);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<Cfg::STAGES - 2>();
    __syncthreads();
    {
      const int kn = kt + Cfg::STAGES - 1;  // refill the slot consumed at kt-1 (all warps are past it)
      if (kn < nk) {
        double* An = smem + (kn % Cfg::STAGES) * Cfg::STAGE;
        gemm_load_stage<Cfg>(An, An + Cfg::BM * Cfg::LDS, g, A, B, m0, c0, kn * Cfg::BK, tid);
      }
      cp_async_commit();
    }
    const double* As = smem + (kt % Cfg::STAGES) * Cfg::STAGE;
    const double* Bs = As + Cfg::BM * Cfg::LDS;
#pragma unroll
    for (int kk = 0; kk < Cfg::KS; kk += 4) {
      const int kc = wk * Cfg::KS + kk + (lane & 3);
      double a[Cfg::FM], b[Cfg::FN];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i) a[i] = As[(wm * Cfg::TM + i * 8 + (lane >> 2)) * Cfg::LDS + kc];
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) b[j] = Bs[(wn * Cfg::TN + j * 8 + (lane >> 2)) * Cfg::LDS + kc];
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // accumulators -> Cs[c][m] (Y_t orientation), reduced over the K-split warps
  double* Cs = smem;
#pragma unroll 1
  for (int w = 0; w < Cfg::WK; ++w) {
    if (wk == w) {
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int mm = wm * Cfg::TM + i * 8 + (lane >> 2);
            int cc = wn * Cfg::TN + j * 8 + 2 * (lane & 3) + e;
            double* dst = Cs + cc * Cfg::LDC + mm;
            *dst = (w == 0) ? acc[i][j][e] : (*dst + acc[i][j][e]);
          }
    }
    __syncthreads();
  }
  Tile t{Cs, Cfg::LDC, m0, c0, Cfg::BM, g.cstep ? g.cstep : Cfg::BN, (int)blockIdx.z};
  epi(t, g, tid, Cfg::NT);
}

template <class Cfg, class Epi>
void launch_gemm(const GemmArgs& g, const Epi& epi, cudaStream_t st, int batch = 1) {
  static bool configured = false;
  if (!configured) {
    NL_CUDA(cudaFuncSetAttribute(gemm_tn_kernel<Cfg, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::SMEM_BYTES));
    configured = true;
  }
  if (!launch_gate((const void*)gemm_tn_kernel<Cfg, Epi>)) return;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ceil_div(g.M, Cfg::BM), ceil_div(g.C, g.cstep ? g.cstep : Cfg::BN), batch);
  cfg.blockDim = dim3(Cfg::NT);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  NL_CUDA(cudaLaunchKernelEx(&cfg, gemm_tn_kernel<Cfg, Epi>, g, epi));
}

// ------------------------------------------------------------------ epilogues

// Plain store (+ bias on real slots: columns with c % bias_period == 0; bias may be null),
// optional "out = src - acc" (filter second half) when sub_src != null.
struct EpiStore {
  double* Y;
  int ldy;
  long long strideY;
  const double* bias;
  int bias_period;
  const double* sub_src;  // same layout as Y (ld = ldy), may be null
  __device__ void operator()(const Tile& t, const GemmArgs& g, int tid, int nt) const {
    double* Yz = Y + (size_t)t.z * strideY;
    const double* Sz = sub_src ? sub_src + (size_t)t.z * strideY : nullptr;
    for (int i = tid; i < t.bm * t.bn; i += nt) {
      int cl = i / t.bm, ml = i % t.bm;
      int c = t.c0 + cl, m = t.m0 + ml;
      if (c >= g.C || m >= g.M) continue;
      double v = t.Cs[cl * t.ldc + ml];
      if (bias && (c % bias_period) == 0) v += bias[m];
      if (Sz) v = Sz[(size_t)c * ldy + m] - v;
      Yz[(size_t)c * ldy + m] = v;
    }
  }
};

}  // namespace nlrom
