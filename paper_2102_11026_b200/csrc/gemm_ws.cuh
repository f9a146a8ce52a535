// Warp-specialised, persistent fp64 DMMA GEMM with a TMA + mbarrier pipeline.
//
//   Y_t[c][m] = sum_k A[m][k] * B_t[c][k]      (same "TN" contract and epilogues as gemm_f64.cuh)
//
// One producer warp streams (BM x 16) A tiles and (BN x 16) B tiles into a STAGES-deep ring of
// 128-byte-swizzled shared-memory stages with cp.async.bulk.tensor (one elected thread, no
// per-thread address math); WM x WN consumer warps wait on the stage's "full" mbarrier, run
// the DMMA.8x8x4 fragments straight from the swizzled tiles (conflict-free), and release the
// stage on its "empty" mbarrier. CTAs are persistent over the output tiles: while the
// consumers run a tile's epilogue (accumulators -> Cs -> functor) the producer is already
// loading the next tile's stages, so short-K GEMMs (K = 256 here) do not pay a pipeline
// prologue per tile. The weight (A) tiles of the first tile are requested before the
// programmatic-dependency wait. tcgen05 has no f64 kind: the tensor work stays on DMMA.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include "gemm_f64.cuh"
#include "cluster_async.cuh"

namespace nlrom {

template <int BM_, int BN_, int WM_, int WN_, int STAGES_ = 4>
struct WsCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int BK = 16;                      // 16 doubles = one 128-byte swizzle row
  static constexpr int NC = 32 * WM * WN;            // consumer threads
  static constexpr int NT = NC + 32;                 // + one producer warp
  static constexpr int TM = BM / WM, TN = BN / WN;   // warp tile
  static constexpr int FM = TM / 8, FN = TN / 8;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // multiple of 1024 (swizzle atom)
  static constexpr int LDC = BM + 2;
  static constexpr int CS_BYTES = BN * LDC * 8;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + CS_BYTES + 2 * STAGES * 8;
  static_assert(BM % 8 == 0 && BN % 8 == 0 && TM % 8 == 0 && TN % 8 == 0, "tile shape");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "swizzle-atom aligned stages");
};

// element (row, k) of a [rows][16] fp64 tile written by TMA with CU_TENSOR_MAP_SWIZZLE_128B
__device__ __forceinline__ int swz(int row, int k) { return row * 16 + ((((k >> 1) ^ (row & 7))) << 1) + (k & 1); }

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}


template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::NT) gemm_ws_kernel(const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmB, GemmArgs g,
                                                          int tiles_m, int tiles_c, int batch, Epi epi) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* Cs = reinterpret_cast<double*>(base + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::CS_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = (g.K + Cfg::BK - 1) / Cfg::BK;
  const int ntiles = tiles_m * tiles_c * batch;
  if (tid == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, Cfg::WM * Cfg::WN);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == Cfg::WM * Cfg::WN) {
    // ------------------------------------------------------------- producer warp
    if (lane == 0) {
      long long it = 0;  // stage loads issued so far; stage = it % STAGES, use = it / STAGES
      bool waited = false;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tm = t % tiles_m, tc = (t / tiles_m) % tiles_c, tz = t / (tiles_m * tiles_c);
        const int m0 = tm * Cfg::BM, c0 = tc * (g.cstep ? g.cstep : Cfg::BN);
        int kt = 0;
        if (!waited) {
          // weight tiles of the first stages do not depend on the producer kernel: request
          // them before the programmatic-dependency wait, the activation tiles after it
          const int pre = min(nk, Cfg::STAGES);
          for (int k2 = 0; k2 < pre; ++k2) {
            mbar_expect_tx(full + k2, Cfg::STAGE_BYTES);
            tma_load_3d(base + k2 * Cfg::STAGE_BYTES, &tmA, k2 * Cfg::BK, m0, tz, full + k2);
          }
          pdl_wait();
          waited = true;
          for (int k2 = 0; k2 < pre; ++k2)
            tma_load_3d(base + k2 * Cfg::STAGE_BYTES + Cfg::A_BYTES, &tmB, k2 * Cfg::BK, c0, tz, full + k2);
          kt = pre;
          it = pre;
        }
        for (; kt < nk; ++kt, ++it) {
          const int st = (int)(it % Cfg::STAGES);
          if (it >= Cfg::STAGES) mbar_wait_cta(empty + st, (uint32_t)((it / Cfg::STAGES - 1) & 1));
          mbar_expect_tx(full + st, Cfg::STAGE_BYTES);
          tma_load_3d(base + st * Cfg::STAGE_BYTES, &tmA, kt * Cfg::BK, m0, tz, full + st);
          tma_load_3d(base + st * Cfg::STAGE_BYTES + Cfg::A_BYTES, &tmB, kt * Cfg::BK, c0, tz, full + st);
        }
      }
      if (!waited) pdl_wait();
    }
    pdl_launch();
    return;
  }

  // --------------------------------------------------------------- consumer warps
  pdl_wait();
  pdl_launch();
  const int wm = warp % Cfg::WM, wn = warp / Cfg::WM;
  long long it = 0;  // stages consumed (same sequence as the producer)
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int tm = t % tiles_m, tc = (t / tiles_m) % tiles_c, tz = t / (tiles_m * tiles_c);
    double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < nk; ++kt, ++it) {
      const int s = (int)(it % Cfg::STAGES);
      mbar_wait_cta(full + s, (uint32_t)((it / Cfg::STAGES) & 1));
      const double* As = reinterpret_cast<const double*>(base + s * Cfg::STAGE_BYTES);
      const double* Bs = reinterpret_cast<const double*>(base + s * Cfg::STAGE_BYTES + Cfg::A_BYTES);
#pragma unroll
      for (int kk = 0; kk < Cfg::BK; kk += 4) {
        const int k = kk + (lane & 3);
        double a[Cfg::FM], b[Cfg::FN];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) a[i] = As[swz(wm * Cfg::TM + i * 8 + (lane >> 2), k)];
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) b[j] = Bs[swz(wn * Cfg::TN + j * 8 + (lane >> 2), k)];
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
          for (int j = 0; j < Cfg::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }
    // accumulators -> Cs[c][m]; the previous tile's epilogue must be done with Cs
    named_bar_sync(1, Cfg::NC);
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int mm = wm * Cfg::TM + i * 8 + (lane >> 2);
          const int cc = wn * Cfg::TN + j * 8 + 2 * (lane & 3) + e;
          Cs[cc * Cfg::LDC + mm] = acc[i][j][e];
        }
    named_bar_sync(1, Cfg::NC);
    const int cs = g.cstep ? g.cstep : Cfg::BN;
    Tile tile{Cs, Cfg::LDC, tm * Cfg::BM, tc * cs, Cfg::BM, cs, tz};
    epi(tile, g, tid, Cfg::NC);
  }
}

// ----------------------------------------------------------------------------- host side
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    NL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Error(NLROM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D map over a row-major (rows x K) fp64 matrix with leading dimension ld, batch stride
// zstride (doubles), box (16, box_rows, 1), 128-byte swizzle, zero fill out of bounds.
inline CUtensorMap make_tile_map(const double* ptr, int K, int rows, int ld, int batch, long long zstride,
                                 int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)std::max(1, batch)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)std::max<long long>(zstride, (long long)ld * rows) * 8};
  cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(ptr), dims, strides,
                                    box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(NLROM_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

inline int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    NL_CUDA(cudaGetDevice(&dev));
    NL_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

// Requires: lda, ldb even (16-byte strides), base pointers 16-byte aligned.
template <class Cfg, class Epi>
void launch_gemm_ws(const GemmArgs& g, const Epi& epi, cudaStream_t st, int batch = 1, int max_ctas = 0) {
  if (!launch_gate((const void*)gemm_ws_kernel<Cfg, Epi>)) return;
  static bool configured = false;
  if (!configured) {
    NL_CUDA(cudaFuncSetAttribute(gemm_ws_kernel<Cfg, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::SMEM_BYTES));
    configured = true;
  }
  const CUtensorMap tA = make_tile_map(g.A, g.K, g.M, g.lda, batch, g.strideA, Cfg::BM);
  const CUtensorMap tB = make_tile_map(g.B, g.K, g.C, g.ldb, batch, g.strideB, Cfg::BN);
  const int tiles_m = ceil_div(g.M, Cfg::BM), tiles_c = ceil_div(g.C, g.cstep ? g.cstep : Cfg::BN);
  const int ntiles = tiles_m * tiles_c * batch;
  int occ = 0;
  NL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gemm_ws_kernel<Cfg, Epi>, Cfg::NT, Cfg::SMEM_BYTES));
  int grid = std::min(ntiles, std::max(1, occ) * sm_count());
  if (max_ctas > 0) grid = std::min(grid, max_ctas);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(std::max(1, grid));
  cfg.blockDim = dim3(Cfg::NT);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  NL_CUDA(cudaLaunchKernelEx(&cfg, gemm_ws_kernel<Cfg, Epi>, tA, tB, g, tiles_m, tiles_c, batch, epi));
}

}  // namespace nlrom
