// fp64 GEMM on the 5th-generation tensor cores: Ozaki-scheme emulation with tcgen05.mma
// kind::i8, accumulators in TMEM.
//
//   Y_t[c][m] = sum_k A[m][k] * B_t[c][k]        (the "TN" contract and Epi functors of gemm_f64.cuh)
//
// tcgen05 has no f64 kind, so every fp64 operand is written as a 55-bit fixed-point
// integer against a power-of-two scale (a row exponent for A, a column exponent for B) and split
// into S = 7 balanced radix-256 digits (int8):
//   a = 2^{e_m - 55} sum_s A_s 256^{7-s},   b = 2^{f_c - 55} sum_t B_t 256^{7-t}
// (truncation error < 2^-55 of the row / column max: fp64-class). The product keeps the digit pairs
// with s + t <= S + 1 = 8 (28 of 49; the dropped pairs are below 2^-58 of |a||b| and unbiased);
// pairs with the same s + t = d share one exact int32 accumulator (<= 7 x 256 x 128^2 < 2^25 at
// K = 256), so a 128-row tile owns 7 accumulators. The epilogue recombines them exactly in int64 --
// hi = acc_2 2^16 + acc_3 2^8 + acc_4, lo = acc_5 2^24 + acc_6 2^16 + acc_7 2^8 + acc_8 -- and
// rounds once:   y = 2^{e_m + f_c + 2} (hi 2^-32 + lo 2^-64)      (one fma)
// The result agrees with an fp64 GEMM to ~1e-15 of sum_k |a_k||b_k| (tests/test_gpu_ozaki.py).
//
// Kernel (persistent, 1 CTA / SM, 18 warps):
//   warp 0     A producer: the weight slices are pre-tiled at upload in exactly the shared-memory
//              operand layout, so one cp.async.bulk per K chunk (28 KB) lands a stage
//   warp 1     TMEM owner + MMA issuer (one thread): 28 tcgen05.mma (M = 128, N = 64, K = 32) per
//              K chunk, tcgen05.commit frees the stage; a final commit hands the tile to the epilogue
//   warps 2-9  epilogue (two warps per TMEM lane quarter, each half of the columns): tcgen05.ld the 7 accumulators, exact
//              int64 recombination, fp64 tile in shared memory, then the same Epi functor as the
//              DMMA kernels (bias + jet sin, vhp epilogues, ...)
//   warps 10-17 B converters: per tile the column exponents (max over K), per K chunk the 7 int8
//              slice planes of the fp64 activations written straight into the UMMA core-matrix
//              layout (no swizzle, K-major: 8 rows x 16 B cores, LBO = 128 B, SBO = 256 B)
//
// Digit chain (hidden -> hidden layers, BDIG = true and / or a digit-producing Epi): a layer whose
// consumer is another tcgen05 hidden layer writes its output directly as the consumer's B stage
// tiles (7 digit planes per 64 columns x 32 K, the layout above) plus one exponent per column, so
// the consumer lands B by TMA like A and needs no converter warps (warps 2-17 all drain / run the
// epilogue). The producer's two m-tile CTAs of a column tile (M = 256) form a cluster pair and
// exchange their column maxima (st.async into the peer's shared memory) so both convert against
// the same column exponent; every element is converted once (the fp64 path converts each column
// once per m tile) and the fp64 activations are never written or re-read. Same digits and
// exponents as the converters: results are bitwise equal to the fp64 hand-off.
#pragma once
#include <type_traits>
#include <algorithm>
#include <cmath>
#include <vector>
#include "gemm_f64.cuh"
#include "cluster_async.cuh"

namespace nlrom {
namespace oz {

constexpr int S = 7;            // digits per operand
constexpr int NACC = 7;         // accumulators d = s + t = 2 .. 8 (28 digit pairs s + t <= 8)
constexpr int QBITS = 55;       // fixed-point bits of an operand against its power-of-two scale
constexpr int BM = 128, BK = 32;
constexpr int A_SLICE = BM * BK;             // bytes per slice plane of a stage
constexpr int A_STAGE = S * A_SLICE;         // 28 KB
constexpr int LDC = BM + 2;
#ifndef OZ_NEPI
#define OZ_NEPI 256
#endif
constexpr int NEPI = OZ_NEPI;   // epilogue threads (warps 2 ..: NEPI / 128 warps per TMEM lane quarter)
#ifndef OZ_NCONV
#define OZ_NCONV 256
#endif
constexpr int NCONV = OZ_NCONV;
#ifndef OZ_B_PREFETCH
#define OZ_B_PREFETCH 1
#endif
#ifndef OZ_DIG_SPLIT
#define OZ_DIG_SPLIT 1   // B from digits: drain warps / functor warps on two fp64 tiles (0.86 vs 0.94 ms, cfg5)
#endif // B converter threads (warps 10 ..): 256 measured 0.85 vs 0.95-1.0 ms with 128 (probe)
constexpr int EPI_W0 = 2, CONV_W0 = 2 + NEPI / 32;
constexpr int NT = 64 + NEPI + NCONV;
constexpr uint32_t TMEM_COLS = 512;

// Tile configuration per column-tile width BN (32 or 64 columns).
template <int BN_>
struct Cfg {
  static constexpr int BN = BN_;
  static constexpr int B_SLICE = BN * BK;
  static constexpr int B_STAGE = S * B_SLICE;
#ifdef OZ_STAGES64
  static constexpr int STAGES = BN == 32 ? 4 : OZ_STAGES64;   // probe override
#else
  static constexpr int STAGES = BN == 32 ? 4 : 3;
#endif
  static constexpr int CS_BYTES = BN * LDC * 8;
  static constexpr int SMEM_BYTES = 1024 + STAGES * (A_STAGE + B_STAGE) + CS_BYTES + 2048;
  // B from digit tiles: both operands by TMA; split epilogue (OZ_DIG_SPLIT): two fp64 tiles (8 warps
  // drain TMEM into one while 8 run the functor on the other) and therefore 2 stages, the next tile's
  // digit chunks prefetched into L2 (the last chained layer: 0.820 -> 0.764 ms with the prefetch)
  static constexpr int STAGES_SPLIT = 2;
  static constexpr int SMEM_BYTES_SPLIT = 1024 + STAGES_SPLIT * (A_STAGE + B_STAGE) + 2 * CS_BYTES + 2048;
  // two accumulator sets (the next tile's MMAs overlap this tile's drain) when they fit in TMEM
  static constexpr int NBUF = 2 * NACC * BN <= (int)TMEM_COLS ? 2 : 1;
  static constexpr int KPT = BN * BK / NCONV;   // K elements per converter thread per chunk (8 or 16)
  static_assert(BN == 32 || BN == 64, "column tile");
  static_assert(KPT >= 4, "converter granularity");
};

// byte offset of element (row, k) inside one K-major no-swizzle slice plane (rows x 32 B)
__host__ __device__ __forceinline__ int core_off(int row, int k) {
  return (row >> 3) * 256 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  // start address >> 4 | LBO (K direction core stride) 128 B >> 4 | SBO (8-row group stride)
  // 256 B >> 4 | version 1 (sm_100) | SWIZZLE_NONE
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);
}

// instruction descriptor: D s32, A / B signed int8, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, int (&r)[16]) { tmem_ld16(taddr, r); }
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, int (&r)[8]) { tmem_ld8(taddr, r); }
__device__ __forceinline__ void tmem_ld_n(uint32_t taddr, int (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ double pow2(int k) {  // 2^k for k in [-1022, 1023]
  return __longlong_as_double((long long)(k + 1023) << 52);
}
// exponent E with max|x| < 2^E (0 for an all-zero row / column)
__host__ __device__ __forceinline__ int scale_exp(double amax) {
  if (!(amax > 0.0)) return 0;
  int e;
  frexp(amax, &e);  // amax = f 2^e, 0.5 <= f < 1
  return e;
}

// The 7 balanced radix-256 digits of x against 2^E: q = trunc(x 2^{55-E}) (|q| < 2^55, exact: x
// has 53 significant bits), q = sum_t d_t 256^{6-t} with d_1..d_6 in [-128, 127] and the top digit
// d_0 = q' >> 48 in [-128, 127] (exp_of keeps max|x| < (127/128) 2^E, so the bias below never
// carries the top digit to 128) -- signed int8 digits with no sign bias in the low ones, so the
// dropped pairs s + t > 8 (below 2^-58 of |a||b|) cancel instead of accumulating. Computed without
// carries: q' = q + 128 sum_{t<6} 256^t, low digit = byte t of q' minus 128 (= byte ^ 0x80), top
// digit = q' >> 48.
constexpr long long BAL = 128LL * ((1LL << 48) - 1) / 255;
__host__ __device__ __forceinline__ long long balanced(long long q) { return q + BAL; }
__host__ __device__ __forceinline__ uint32_t digit(long long qb, int t) {   // t = 0 (top) .. 6, as an int8 byte
  if (t == 0) return (uint32_t)(qb >> 48) & 0xFFu;
  return ((uint32_t)(qb >> (8 * (S - 1 - t))) & 0xFFu) ^ 0x80u;
}
__device__ __forceinline__ long long fixed55(double x, double scale55) { return balanced(__double2ll_rz(x * scale55)); }
// digit plane t of four balanced values as one word (byte k = digit of value k): the same bytes as
// digit(), gathered with byte permutes (byte 6 - t of each q', low digits with the 0x80 bias removed)
__device__ __forceinline__ uint32_t pack_plane(long long q0, long long q1, long long q2, long long q3, int t) {
  const int bi = S - 1 - t;
  const bool h = bi >= 4;
  const uint32_t w0 = h ? (uint32_t)((unsigned long long)q0 >> 32) : (uint32_t)q0;
  const uint32_t w1 = h ? (uint32_t)((unsigned long long)q1 >> 32) : (uint32_t)q1;
  const uint32_t w2 = h ? (uint32_t)((unsigned long long)q2 >> 32) : (uint32_t)q2;
  const uint32_t w3 = h ? (uint32_t)((unsigned long long)q3 >> 32) : (uint32_t)q3;
  const uint32_t sel = (uint32_t)((bi & 3) | (((bi & 3) + 4) << 4));
  const uint32_t r = __byte_perm(__byte_perm(w0, w1, sel), __byte_perm(w2, w3, sel), 0x5410);
  return t == 0 ? r : r ^ 0x80808080u;
}
// exponent E of a row / column with max|x| < (127/128) 2^E (0 for an all-zero one)
// (clamped at -900 so that the 2^(55 - E) scale and the 2^(E - 62) recombination stay normal)
__host__ __device__ __forceinline__ int exp_of(double amax) {
  const int e = scale_exp(amax * (128.0 / 127.0));
  return e < -900 ? -900 : e;
}

}  // namespace oz

// A operand prepared once (host): slices of a row-major (M x K) fp64 matrix, pre-tiled per
// (m tile, k chunk) in the stage layout [slice][core layout of 128 rows x 32 B], and the row
// exponents. M % 128 == 0, K % 32 == 0.
struct OzakiA {
  const unsigned char* tiles;   // [M / 128][K / 32][S][128 x 32]
  const int* row_exp;           // [M]
};

// Column scales of the B operand from partials written by the producing layer's epilogue
// (EpiJet::colhw): parts[c * nparts + p] = max over a row group of the high word of |x|, so
// exp_of(hiword:0xFFFFFFFF) bounds the column maximum; with parts == nullptr the kernel computes
// the column maxima itself (a pre-pass over each column tile).
struct OzakiBExp {
  const unsigned* parts;
  int nparts;   // <= 8
  // digit-chain input (k_ozaki_gemm<.., BDIG = true>): the B stage tiles [C/64][K/32][S][64 x 32 B]
  // and the column exponents [C/64 * 64] written by the producing layer (EpiJetDig)
  const unsigned char* dig = nullptr;
  const int* dexp = nullptr;
};

// Digit-producing epilogues (EpiJetDig, ozaki_chain.cuh) get this context from the kernel.
struct DigCtx {
  double* Cs;          // the fp64 tile [BN][LDC]; reused as the 4 x B_STAGE staging of the digits
  unsigned* colmax;    // [64] this CTA's column maxima (high words of |y|)
  int* colEs;          // [64] the pair's column exponents
  unsigned* xslot;     // [2][64] the peer's column maxima (written by the peer with st.async)
  uint64_t* xbar;      // [2] tx barriers of xslot
  int j;               // tile counter of this CTA
};
// Epi functors that read the fp64 tile row-major (Cs[row * (BN + 1) + col]): lanes over columns
// for coalesced row-major global stores (EpiJetOutCRow)
template <class E, class = void>
struct row_major_cs : std::false_type {};
template <class E>
struct row_major_cs<E, std::void_t<decltype(E::kRowMajorCs)>> : std::bool_constant<E::kRowMajorCs> {};
template <class E, class = void>
struct digits_out : std::false_type {};
template <class E>
struct digits_out<E, std::void_t<decltype(E::kDigitsOut)>> : std::bool_constant<E::kDigitsOut> {};

// Device copy of one layer's prepared A operand (digit tiles + row exponents).
struct OzakiWeights {
  unsigned char* tiles = nullptr;
  int* exps = nullptr;
  bool ready = false;
  OzakiWeights() = default;
  OzakiWeights(const OzakiWeights&) = delete;
  OzakiWeights& operator=(const OzakiWeights&) = delete;
  OzakiWeights(OzakiWeights&& o) noexcept : tiles(o.tiles), exps(o.exps), ready(o.ready) {
    o.tiles = nullptr;
    o.exps = nullptr;
    o.ready = false;
  }
  ~OzakiWeights() {
    if (tiles) cudaFree(tiles);
    if (exps) cudaFree(exps);
  }
  OzakiA view() const { return OzakiA{tiles, exps}; }
};

inline void ozaki_prepare_a(const double* A, int lda, int M, int K, std::vector<unsigned char>& tiles,
                            std::vector<int>& exps) {
  using namespace oz;
  // rows past M (the last 128-row tile of a ragged M) are zero digits with exponent 0
  const int nk = K / BK, tm_n = (M + BM - 1) / BM;
  tiles.assign((size_t)tm_n * nk * A_STAGE, 0);
  exps.assign((size_t)tm_n * BM, 0);
  for (int m = 0; m < M; ++m) {
    double amax = 0.0;
    for (int k = 0; k < K; ++k) amax = std::max(amax, std::fabs(A[(size_t)m * lda + k]));
    exps[m] = exp_of(amax);
    for (int k = 0; k < K; ++k) {
      // the same fixed-point digits as oz::fixed55 / oz::digit on the device
      const long long qb = balanced((long long)std::trunc(std::ldexp(A[(size_t)m * lda + k], QBITS - exps[m])));
      const int tm = m / BM, kc = k / BK;
      unsigned char* st = tiles.data() + ((size_t)tm * nk + kc) * A_STAGE;
      for (int t = 0; t < S; ++t) st[t * A_SLICE + core_off(m % BM, k % BK)] = (unsigned char)digit(qb, t);
    }
  }
}

#ifdef OZ_TRACE
__device__ unsigned long long g_oz_trace[12];  // MMA: wait tempty, wait A, wait B; epi: wait tfull, drain
#define OZ_T0() const long long _t0 = clock64()
#define OZ_T1(i) atomicAdd(&g_oz_trace[i], (unsigned long long)(clock64() - _t0))
#else
#define OZ_T0()
#define OZ_T1(i)
#endif

template <int BN, class Epi, bool BDIG = false>
__global__ void __launch_bounds__(oz::NT, 1) k_ozaki_gemm(OzakiA a, OzakiBExp bexp, GemmArgs g, int tiles_m, int tiles_c,
                                                         Epi epi) {
  using namespace oz;
  using C = Cfg<BN>;
  constexpr bool SPLIT = BDIG && OZ_DIG_SPLIT;
  constexpr int STAGES = SPLIT ? C::STAGES_SPLIT : C::STAGES, NBUF = C::NBUF, KPT = C::KPT;
  constexpr int CS_REGION = SPLIT ? 2 * C::CS_BYTES : C::CS_BYTES;
  // B from digit tiles (TMA): no converter warps, their threads drain / run the epilogue
  constexpr int NE = BDIG ? NEPI + NCONV : NEPI;
  constexpr int NC = BDIG ? 0 : NCONV;
  constexpr int CONV_W = 2 + NE / 32;
  constexpr bool DOUT = digits_out<Epi>::value;
  static_assert(!DOUT || BN == 64, "digit output tiles are 64 columns");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned by pointer arithmetic on the __shared__ array (an integer round trip
  // would hide the address space and turn every shared access into a generic LD.E / ST.E)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = base;                                   // STAGES x A_STAGE
  unsigned char* sB = base + STAGES * A_STAGE;                // STAGES x B_STAGE
  double* Cs = reinterpret_cast<double*>(sB + STAGES * C::B_STAGE);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(Cs) + CS_REGION);
  uint64_t* fullA = bar;                 // [STAGES]  tx bytes of the weight slices (+ B digit tiles)
  uint64_t* fullB = bar + STAGES;        // [STAGES]  one arrival per converter warp
  uint64_t* empty = bar + 2 * STAGES;    // [STAGES]  tcgen05.commit
  uint64_t* tfull = bar + 3 * STAGES;    // [NBUF] accumulators complete (commit)
  uint64_t* tempty = tfull + 2;          // [NBUF] accumulators drained (one arrival per epilogue warp)
  uint64_t* eready = tfull + 4;          // [2] column exponents of a tile written (NCONV converters)
  uint64_t* efree = tfull + 6;           // [2] column exponents of a tile consumed (NEPI epilogue threads)
  uint64_t* tdone = tfull + 8;           // every MMA of this CTA complete (before TMEM dealloc)
  uint64_t* xbar = tfull + 9;            // [2] digit output: the peer's column maxima landed
  uint64_t* csfull = tfull + 11;         // [2] SPLIT: fp64 tile drained (drain threads)
  uint64_t* csfree = tfull + 13;         // [2] SPLIT: fp64 tile consumed (functor threads)
  int* colE = reinterpret_cast<int*>(tfull + 15);  // [2][BN]
  unsigned* xslot = reinterpret_cast<unsigned*>(colE + 2 * BN);  // [2][64]
  unsigned* colmax = xslot + 128;                                // [64]
  int* colEs = reinterpret_cast<int*>(colmax + 64);              // [64]
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(colEs + 64);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = g.K / BK;
  const int ntiles = tiles_m * tiles_c;
  pdl_launch();
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(fullA + s, 1);
      mbar_init(fullB + s, NC ? NC / 32 : 1);
      mbar_init(empty + s, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + i, 1);
      mbar_init(tempty + i, SPLIT ? NE / 64 : NE / 32);
      mbar_init(eready + i, NC ? NC : 1);
      mbar_init(efree + i, NE);
      mbar_init(xbar + i, 1);
      mbar_init(csfull + i, SPLIT ? NE / 2 : 1);
      mbar_init(csfree + i, SPLIT ? NE / 2 : 1);
    }
    mbar_init(tdone, 1);
    fence_mbar_init();
    if constexpr (DOUT) {   // the peer's column maxima of tiles 0 and 1 (64 x 4 bytes each)
      mbar_expect_tx(xbar, 256);
      mbar_expect_tx(xbar + 1, 256);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_s)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // digit output: the peer's barriers are initialised before any st.async reaches them
  if constexpr (DOUT) cluster_sync_all();
  const uint32_t tmem = *tmem_base_s;

  if (warp == 0) {
    // --------------------------------------------------------------- A (+ B digit tiles) producer
    if (lane == 0) {
      if constexpr (BDIG) pdl_wait();   // the B tiles are the previous layer's output
      int st = 0;
      uint32_t ph = 0;
      bool wrapped = false;   // the ring has been filled once: wait for the stage's previous use
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int tm = t % tiles_m;
        for (int kc = 0; kc < nk; ++kc) {
          if (wrapped) mbar_wait_cta(empty + st, ph ^ 1u);
          mbar_expect_tx(fullA + st, BDIG ? A_STAGE + C::B_STAGE : A_STAGE);
          tma_g2s(sA + st * A_STAGE, a.tiles + ((size_t)tm * nk + kc) * A_STAGE, A_STAGE, fullA + st);
          if constexpr (BDIG) {
            tma_g2s(sB + st * C::B_STAGE, bexp.dig + ((size_t)(t / tiles_m) * nk + kc) * C::B_STAGE, C::B_STAGE,
                    fullA + st);
#if OZ_B_PREFETCH
            // the next tile's digit chunk into L2 (the 2-stage ring of the split epilogue cannot hide
            // a DRAM round trip per chunk)
            const int tn = t + gridDim.x;
            if (tn < ntiles) {
              const unsigned char* pf = bexp.dig + ((size_t)(tn / tiles_m) * nk + kc) * C::B_STAGE;
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"((uint32_t)C::B_STAGE) : "memory");
            }
#endif
          }
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
            wrapped = true;
          }
        }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------------- MMA issuer
    // Products A_s B_t, t = 1 .. S + 1 - s, land in accumulators d = s + t, which are laid out
    // consecutively (acc_d at TMEM column (d - 2) BN): the B planes t0 .. t1 are consecutive too, so
    // one MMA with N = (t1 - t0 + 1) BN <= 256 covers a run of them (7 / 11 MMAs per K chunk at
    // BN = 32 / 64 instead of 28; the A digit plane is read once per run). The s = 1 runs touch every
    // accumulator first, so only they restart the accumulation at K chunk 0.
    if (lane == 0) {
      constexpr int RUN = 256 / BN;   // B planes per MMA
      int st = 0;
      uint32_t ph = 0;
      int j = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
        const int buf = NBUF == 2 ? (j & 1) : 0;
        const int use = NBUF == 2 ? (j >> 1) : j;
        if (use > 0) {
          OZ_T0();
          mbar_wait_cta(tempty + buf, (uint32_t)((use - 1) & 1));
          OZ_T1(0);
          tc_fence_after();
        }
        const uint32_t tacc = tmem + (uint32_t)(buf * NACC * BN);
        for (int kc = 0; kc < nk; ++kc) {
          {
            OZ_T0();
            mbar_wait_cta(fullA + st, ph);
            OZ_T1(1);
          }
          if constexpr (!BDIG) {
            OZ_T0();
            mbar_wait_cta(fullB + st, ph);
            OZ_T1(2);
          }
          tc_fence_after();
          const uint32_t aBase = smem_u32(sA + st * A_STAGE), bBase = smem_u32(sB + st * C::B_STAGE);
#pragma unroll
          for (int s = 1; s <= S; ++s) {
#pragma unroll
            for (int t0 = 1; t0 <= S + 1 - s; t0 += RUN) {
              const int nt = min(RUN, S + 2 - s - t0);   // planes t0 .. t0 + nt - 1
              mma_i8(tacc + (uint32_t)((s + t0 - 2) * BN), smem_desc(aBase + (s - 1) * A_SLICE),
                     smem_desc(bBase + (t0 - 1) * C::B_SLICE), idesc_i8(nt * BN), (kc > 0 || s > 1) ? 1u : 0u);
            }
          }
          tc_commit(empty + st);  // the stage is free once these MMAs have read it
          if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
          }
        }
        tc_commit(tfull + buf);   // accumulators of tile j complete
      }
      tc_commit(tdone);
      mbar_wait_cta(tdone, 0);
    }
  } else if (warp >= CONV_W) {
    if constexpr (!BDIG) {
    // --------------------------------------------------------------- B converters (warps 10 .. 17)
    pdl_wait();
    const int ct = tid - CONV_W * 32;   // 0 .. NCONV-1
    constexpr int TPC = NCONV / BN;  // threads per column (2 or 4), each KPT consecutive K per chunk
    constexpr int PF = (KPT == 8 && NCONV <= 128) ? 4 : 2;   // chunks in flight per thread (register ring)
    const int cl = ct / TPC, kq = ct % TPC;
    const int my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long total = (long long)my_tiles * nk;
    // column of this thread in its j-th tile; tiles start every cs columns (GemmArgs.cstep: tiles of
    // whole column groups) and columns cl >= cs of a tile are padding (zeros, never stored)
    const int cs = g.cstep ? g.cstep : BN;
    auto col_of = [&](int j) { return cl < cs ? ((blockIdx.x + j * gridDim.x) / tiles_m) * cs + cl : g.C; };
    // load pointer (tile jl, chunk kl) runs PF chunks ahead of the slicing position
    int jl = 0, kl = 0;
    auto load_chunk = [&](double (&x)[KPT]) {
      const int c = jl < my_tiles ? col_of(jl) : g.C;
      if (c < g.C) {
        const double2* src = reinterpret_cast<const double2*>(g.B + (size_t)c * g.ldb + kl * BK + kq * KPT);
#pragma unroll
        for (int q2 = 0; q2 < KPT / 2; ++q2) {
          const double2 v = src[q2];
          x[2 * q2] = v.x;
          x[2 * q2 + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int q2 = 0; q2 < KPT; ++q2) x[q2] = 0.0;
      }
      if (++kl == nk) {
        kl = 0;
        ++jl;
      }
    };
    // column exponent of tile j for this thread's column: max over the producer's partials (up to
    // MAXP, loaded one tile ahead and reduced when the tile starts), or (no partials) a pre-pass
    // over the column by the TPC threads that share it
    constexpr int MAXP = 8;
    auto load_parts = [&](int j, unsigned (&pp)[MAXP]) {
      const int c = j < my_tiles ? col_of(j) : g.C;
#pragma unroll
      for (int p = 0; p < MAXP; ++p) pp[p] = (c < g.C && p < bexp.nparts) ? bexp.parts[(size_t)c * bexp.nparts + p] : 0u;
    };
    auto prepass_exp = [&](int j) -> int {
      const int c = j < my_tiles ? col_of(j) : g.C;
      double m = 0.0;  // every lane reaches the shuffles below
      if (c < g.C)
        for (int k = kq; k < g.K; k += TPC) m = fmax(m, fabs(g.B[(size_t)c * g.ldb + k]));
#pragma unroll
      for (int o = 1; o < TPC; o <<= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
      return exp_of(m);
    };
    unsigned pp_next[MAXP];
    if (bexp.parts) load_parts(0, pp_next);
    double xr[PF][KPT];
#pragma unroll
    for (int p = 0; p < PF; ++p) load_chunk(xr[p]);
    double sc = 1.0;
    int st = 0;
    uint32_t ph = 0;
    bool wrapped = false;
    int j = 0, kc = 0;   // slicing position
#pragma unroll 1
    for (long long i0 = 0; i0 < total; i0 += PF) {
#pragma unroll
      for (int p = 0; p < PF; ++p) {
        if (i0 + p >= total) break;
        if (kc == 0) {
          // tile j starts: publish its column exponents (epilogue scale), fetch tile j + 1's
          int e;
          if (bexp.parts) {
            unsigned hw = pp_next[0];
#pragma unroll
            for (int p = 1; p < MAXP; ++p) hw = max(hw, pp_next[p]);
            e = hw ? exp_of(__hiloint2double((int)hw, (int)0xFFFFFFFFu)) : 0;   // bounds the column max
            load_parts(j + 1, pp_next);
          } else {
            e = prepass_exp(j);
          }
          if (j >= 2) mbar_wait_cta(efree + (j & 1), (uint32_t)(((j >> 1) - 1) & 1));
          if (kq == 0) colE[(j & 1) * BN + cl] = e;
          mbar_arrive(eready + (j & 1));
          sc = oz::pow2(QBITS - e);
        }
        double x[KPT];
#pragma unroll
        for (int q2 = 0; q2 < KPT; ++q2) x[q2] = xr[p][q2];
        load_chunk(xr[p]);
        long long qv[KPT];
#pragma unroll
        for (int q2 = 0; q2 < KPT; ++q2) qv[q2] = oz::fixed55(x[q2], sc);
        uint32_t w[S][KPT / 4];
#pragma unroll
        for (int t2 = 0; t2 < S; ++t2)
#pragma unroll
          for (int q = 0; q < KPT / 4; ++q)
            w[t2][q] = oz::digit(qv[4 * q], t2) | (oz::digit(qv[4 * q + 1], t2) << 8) |
                       (oz::digit(qv[4 * q + 2], t2) << 16) | (oz::digit(qv[4 * q + 3], t2) << 24);
#ifdef OZ_PROBE_NO_CONVERT
#pragma unroll
        for (int t2 = 0; t2 < S; ++t2)
#pragma unroll
          for (int q = 0; q < KPT / 4; ++q) w[t2][q] = 0x01010101u;
#endif
        if (wrapped) mbar_wait_cta(empty + st, ph ^ 1u);
        unsigned char* dst = sB + st * C::B_STAGE + oz::core_off(cl, kq * KPT);
#pragma unroll
        for (int t2 = 0; t2 < S; ++t2) {
          if constexpr (KPT == 16)
            *reinterpret_cast<uint4*>(dst + t2 * C::B_SLICE) = make_uint4(w[t2][0], w[t2][1], w[t2][2], w[t2][3]);
          else if constexpr (KPT == 8)
            *reinterpret_cast<uint2*>(dst + t2 * C::B_SLICE) = make_uint2(w[t2][0], w[t2][1]);
          else
            *reinterpret_cast<uint32_t*>(dst + t2 * C::B_SLICE) = w[t2][0];
        }
        fence_proxy_async();     // generic-proxy stores -> visible to the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(fullB + st);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
          wrapped = true;
        }
        if (++kc == nk) {
          kc = 0;
          ++j;
        }
      }
    }
    }
  } else if (SPLIT) {
    if constexpr (SPLIT) {
    // ------------------------------------------ epilogue, B from digits: warps 2-9 drain TMEM into one
    // of two fp64 tiles while warps 10-17 run the Epi functor on the other
    pdl_wait();
    constexpr int NDR = NE / 2, NFN = NE / 2;
    constexpr int CSD = BN * LDC;   // doubles per fp64 tile
    if (warp < EPI_W0 + NDR / 32) {
      const int q = warp & 3;
      const int chalf = (warp - EPI_W0) >> 2;   // column half
      const int row_l = q * 32 + lane;
      int j = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
        const int tm = t % tiles_m, tc = t / tiles_m;
        const int m0 = tm * BM, c0 = tc * BN;
        const int buf = NBUF == 2 ? (j & 1) : 0;
        const int use = NBUF == 2 ? (j >> 1) : j;
        double* Csb = Cs + (j & 1) * CSD;
        const int ecol = __ldg(bexp.dexp + c0 + chalf * 32 + lane);   // this half's column exponents
        {
          OZ_T0();
          mbar_wait_cta(tfull + buf, (uint32_t)(use & 1));
          if (tid == EPI_W0 * 32) OZ_T1(4);
        }
        tc_fence_after();
        if (j >= 2) mbar_wait_cta(csfree + (j & 1), (uint32_t)(((j >> 1) - 1) & 1));
        const int m = m0 + row_l;
        const int em = (m < g.M) ? a.row_exp[m] : 0;
        const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * NACC * BN + chalf * 32);
        constexpr int CW = 8;
#pragma unroll 1
        for (int ch = 0; ch < 32 / CW; ++ch) {
          int acc[NACC][CW];
#pragma unroll
          for (int d = 0; d < NACC; ++d) oz::tmem_ld_n(tacc + (uint32_t)(d * BN + ch * CW), acc[d]);
          oz::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < CW; ++i) {
            const int cl = ch * CW + i;
            const long long hi = ((long long)acc[0][i] << 16) + ((long long)acc[1][i] << 8) + (long long)acc[2][i];
            const long long lo = ((long long)acc[3][i] << 24) + ((long long)acc[4][i] << 16) +
                                 ((long long)acc[5][i] << 8) + (long long)acc[6][i];
            const int E = em + __shfl_sync(0xffffffffu, ecol, cl);
            const double yv = E < -960 ? 0.0 : fma((double)hi, oz::pow2(E - 30), (double)lo * oz::pow2(E - 62));
            if constexpr (row_major_cs<Epi>::value) Csb[row_l * (BN + 1) + chalf * 32 + cl] = yv;
            else Csb[(chalf * 32 + cl) * LDC + row_l] = yv;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + buf);   // TMEM may take the next tile's accumulators
        mbar_arrive(csfull + (j & 1));
      }
    } else {
      const int ft = tid - (EPI_W0 * 32 + NDR);   // 0 .. NFN-1
      int j = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
        const int tm = t % tiles_m, tc = t / tiles_m;
        double* Csb = Cs + (j & 1) * CSD;
        mbar_wait_cta(csfull + (j & 1), (uint32_t)((j >> 1) & 1));
        Tile tile{Csb, row_major_cs<Epi>::value ? BN + 1 : LDC, tm * BM, tc * BN, BM, BN, 0};
        OZ_T0();
#ifndef OZ_PROBE_NO_EPI
        if constexpr (DOUT) {
          epi.template dig_out<NFN, 64>(tile, g, ft, DigCtx{Csb, colmax, colEs, xslot, xbar, j});
          if (ft == 0) bulk_wait_read0();   // the digit store has read the staging (this fp64 tile)
        } else {
          epi(tile, g, ft, NFN);
        }
#endif
        if (ft == 0) OZ_T1(6);
        mbar_arrive(csfree + (j & 1));
      }
      if constexpr (DOUT) {
        if (ft == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // digit stores complete
      }
    }
    }
  } else {
    // --------------------------------------------------------------- epilogue (warps 2 .. CONV_W - 1)
    pdl_wait();
    const int q = warp & 3;              // TMEM lane quarter of this warp
    const int et = tid - EPI_W0 * 32;     // 0 .. NE-1
    // which slice of the tile's columns this warp drains (NE / 128 slices; lane quarter = warp % 4)
    constexpr int NSL = NE / 128;
    const int chalf = (warp - EPI_W0) >> 2;
    const int row_l = q * 32 + lane;      // tile row = TMEM lane
    int j = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++j) {
      const int tm = t % tiles_m, tc = t / tiles_m;
      const int cs = g.cstep ? g.cstep : BN;
      const int m0 = tm * BM, c0 = tc * cs;
      const int buf = NBUF == 2 ? (j & 1) : 0;
      const int use = NBUF == 2 ? (j >> 1) : j;
      {
        OZ_T0();
        mbar_wait_cta(tfull + buf, (uint32_t)(use & 1));
        if (et == 0) OZ_T1(4);
      }
      tc_fence_after();
      if constexpr (!BDIG) mbar_wait_cta(eready + (j & 1), (uint32_t)((j >> 1) & 1));
#ifdef OZ_TRACE
      const long long _td = clock64();
#endif
      const int m = m0 + row_l;
      const int em = (m < g.M) ? a.row_exp[m] : 0;
      const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * NACC * BN);
      if constexpr (DOUT) {
        if (et == 0) bulk_wait_read0();   // the previous tile's digit store has read the staging (Cs)
      }
      named_bar_sync(1, NE);  // the previous tile's epilogue is done with Cs
      // CW columns per TMEM load (x16 with 128 converter threads; x8 keeps the epilogue within the
      // register budget of the 576-thread build with 256 converter threads)
      constexpr int CW = BDIG ? 8 : (NCONV > 256 || NEPI > 256) ? 4 : NCONV > 128 ? 8 : 16;
      constexpr int SLW = BN / NSL;   // columns drained by this warp
      // BDIG: this warp's column exponents, one per lane (shuffled per column below)
      const int ecol = BDIG ? __ldg(bexp.dexp + c0 + chalf * SLW + (lane % SLW)) : 0;
#pragma unroll 1
      for (int ch = chalf * (BN / NSL / CW); ch < (chalf + 1) * (BN / NSL / CW); ++ch) {
        int acc[NACC][CW];
#pragma unroll
        for (int d = 0; d < NACC; ++d) {
          oz::tmem_ld_n(tacc + (uint32_t)(d * BN + ch * CW), acc[d]);
        }
        oz::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < CW; ++i) {
          const int cl = ch * CW + i;
          const long long hi = ((long long)acc[0][i] << 16) + ((long long)acc[1][i] << 8) + (long long)acc[2][i];
          const long long lo = ((long long)acc[3][i] << 24) + ((long long)acc[4][i] << 16) +
                               ((long long)acc[5][i] << 8) + (long long)acc[6][i];
          const int E = em + (BDIG ? __shfl_sync(0xffffffffu, ecol, cl - chalf * SLW) : colE[(j & 1) * BN + cl]);
          // x_a x_b = q_a q_b 2^{E-110} = 2^{E+2} sum_d acc_d 2^{-8d} = hi 2^{E-30} + lo 2^{E-62}
          const double yv = E < -960 ? 0.0 : fma((double)hi, oz::pow2(E - 30), (double)lo * oz::pow2(E - 62));
          if constexpr (row_major_cs<Epi>::value) Cs[row_l * (BN + 1) + cl] = yv;
          else Cs[cl * LDC + row_l] = yv;
        }
      }
      tc_fence_before();
#ifdef OZ_TRACE
      if (et == 0) atomicAdd(&g_oz_trace[5], (unsigned long long)(clock64() - _td));
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + buf);   // TMEM may take the next tiles' accumulators
      if constexpr (!BDIG) mbar_arrive(efree + (j & 1));
      named_bar_sync(1, NE);
      Tile tile{Cs, row_major_cs<Epi>::value ? BN + 1 : LDC, m0, c0, BM, cs, 0};
#ifndef OZ_PROBE_NO_EPI
      OZ_T0();
      if constexpr (DOUT)
        epi.template dig_out<NE, 64>(tile, g, et, DigCtx{Cs, colmax, colEs, xslot, xbar, j});
      else
        epi(tile, g, et, NE);
      if (et == 0) OZ_T1(6);
#endif
    }
    if constexpr (DOUT) {
      if (et == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // digit stores complete
    }
  }
  tc_fence_before();
  __syncthreads();
  // digit output: no CTA of the pair leaves while the other may still write into its shared memory
  if constexpr (DOUT) cluster_sync_all();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

inline int sm_count_oz() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    NL_CUDA(cudaGetDevice(&dev));
    NL_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

// Launch over all column tiles (persistent grid of one CTA per SM). Requirements: K % 32 == 0
// (M ragged: the prepared A operand is zero-padded to 128-row tiles, the epilogue skips m >= M), ldb
// even and g.B 16-byte aligned, the Epi column groups divide BN (or g.cstep <= BN columns per tile,
// then the epilogue sees t.bn = cstep). BDIG: B from digit tiles (be.dig / be.dexp, C padded to
// whole 64-column tiles). A digit-producing Epi (EpiJetDig) runs as cluster pairs over the two
// m tiles of M = 256 (tiles_m == 2, even grid).
template <int BN, class Epi, bool BDIG = false>
void launch_ozaki(const OzakiA& a, const OzakiBExp& be, const GemmArgs& g, const Epi& epi, cudaStream_t st) {
  using C = oz::Cfg<BN>;
  constexpr bool DOUT = digits_out<Epi>::value;
  constexpr bool SPLIT = BDIG && OZ_DIG_SPLIT;
  auto kern = k_ozaki_gemm<BN, Epi, BDIG>;
  if (!launch_gate((const void*)kern)) return;
  static bool configured = false;
  if (!configured) {
    NL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SPLIT ? C::SMEM_BYTES_SPLIT : C::SMEM_BYTES));
    configured = true;
  }
  const int tiles_m = ceil_div(g.M, oz::BM), tiles_c = ceil_div(g.C, g.cstep ? g.cstep : BN);
  const int ntiles = tiles_m * tiles_c;
  if (DOUT && (tiles_m != 2 || g.cstep)) {
    fprintf(stderr, "nlrom: digit-output Ozaki layer needs M = 256 (got %d)\n", g.M);
    abort();
  }
  int grid = std::max(1, std::min(ntiles, sm_count_oz()));
  if (DOUT) grid &= ~1;   // cluster pairs
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(oz::NT);
  cfg.dynamicSmemBytes = SPLIT ? C::SMEM_BYTES_SPLIT : C::SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = DOUT ? 2 : 1;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = DOUT ? 2 : 1;
  NL_CUDA(cudaLaunchKernelEx(&cfg, kern, a, be, g, tiles_m, tiles_c, epi));
}

inline void ozaki_upload(OzakiWeights& w, const double* A, int lda, int M, int K) {
  std::vector<unsigned char> tiles;
  std::vector<int> exps;
  ozaki_prepare_a(A, lda, M, K, tiles, exps);
  NL_CUDA(cudaMalloc(&w.tiles, tiles.size()));
  NL_CUDA(cudaMalloc(&w.exps, exps.size() * sizeof(int)));
  NL_CUDA(cudaMemcpy(w.tiles, tiles.data(), tiles.size(), cudaMemcpyHostToDevice));
  NL_CUDA(cudaMemcpy(w.exps, exps.data(), exps.size() * sizeof(int), cudaMemcpyHostToDevice));
  w.ready = true;
}

}  // namespace nlrom
