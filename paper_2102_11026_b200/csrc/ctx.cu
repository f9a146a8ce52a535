// Reduced simulator context: the per-Newton-iteration hot path of arXiv 2102.11026
// (rdsim.step) as a CUDA-graph of sm_100a kernels.
//
// One Newton iteration = E (evaluate at r) + J (Jacobian + solve):
//   E: seed jet -> decoder bundle forward (L fp64-DMMA GEMMs with fused jet-sin
//      epilogues; last layer fused with the filter) -> weight net -> StVK cubature
//      (+ J~ projection) -> assembly of a and [J~^T M R | J~^T a] partials -> phi, ||phi||
//   J: vhp = H~^T a by complex-step backprop (dual arithmetic) -> S = reduce + vhp
//      -> in-CTA LU with partial pivoting -> dr (r += dr in fixed-iteration mode)
#include <vector>
#include <cstring>
#include <cstdio>
#include <string>
#include <map>
#include <algorithm>
#include <cmath>
#include <functional>
#include "common.cuh"
#include "epilogues.cuh"
#include "sim_kernels.cuh"
#include "solve_kernels.cuh"
#include "mlp_chain.cuh"
#include "coupled_kernels.cuh"
#include "gemm_ws.cuh"
#include "ozaki_tc.cuh"
#include "ozaki_chain.cuh"
#ifndef OZ_OUT_DIG
#define OZ_OUT_DIG 1
#endif
#include "newton_kernels.cuh"

namespace nlrom {
void fc_forward(int order, int act, const GemmArgs& g, double* Y, int ldy, const double* bias, double* cache,
                cudaStream_t st);
}

using namespace nlrom;

namespace {

// hidden / backward layers (K = 256): 16-row tiles, 4 warps split K, 32-wide K tiles,
// deep cp.async ring so the whole K extent is in flight (latency-bound regime)
using CfgBwd = GemmCfg<16, 16, 1, 1, 4, 32, 8>;
template <int G> using CfgHid = GemmCfg<16, G, 1, 1, 4, 32, (G <= 32 ? 8 : 4)>;
template <int G> using CfgOut = GemmCfg<64, G, 4, 1, 1, 32, 4>;
// batched (many sims): 64 x 128 tiles, 8 warps, 16-wide K tiles, 3 stages: 90 KB smem so two
// CTAs share an SM and one's epilogue overlaps the other's DMMA loop (tools/probes/gemm_probe.cu:
// 26.7 TFLOP/s vs 22.1 for 32-wide K tiles at one CTA per SM, M = K = 256, 393k columns)
using CfgBig = GemmCfg<64, 128, 2, 4, 1, 16, 3>;
// the last shared-real vhp backward layer (M = n_q <= 24 output rows): 24-row tiles, K split over
// two warps (CfgBig's 64-row tiles left 69% of the DMMA work on padding rows at n_q = 20)
using CfgBwdLast = GemmCfg<24, 128, 1, 4, 2, 16, 3>;

struct CubSet {
  IBuf elems;
  IBuf rows_g;       // (n, 12) DOF rows of the set's elements, gathered once (no id indirection)
  DBuf Dm_g, vol_g;  // (n, 9) Dm^-1 and (n) volumes of the set's elements
  int n = 0;
  IBuf row_ids, row_ptr, entries;
  IBuf rowptr_full;  // (N + 1) CSR over all free-DOF rows (same entries), gathered by k_assemble_a
  int n_rows = 0;
  int epc = 1, nchunk = 0;  // elements per chunk; partials per sim (CTAs along x)
  int nech = 0, cpc = 1;     // element chunks; element chunks per CTA (nchunk = ceil(nech / cpc))
  DBuf fe_w, part_f, part_K, f;
  // many sims: k_cub_sims (one CTA per sim, B-projected 9-row Gram) with the B columns of the
  // constant U block precomputed per set element (n, 9, n_p); ti = Gram row tiles (n < 8 ti)
  bool sims = false;
  int ti = 0;
  DBuf BU;
};

int gemm_launch_count = 0;

// Code-path overrides for tests: NLROM_PATH = comma-separated tokens, read once per context.
// Every token selects a correct, tested path that the size heuristics would otherwise pick only
// at other problem sizes (so small tests can cover the cfg5-scale kernels):
//   batched         many-sims big-tile per-layer GEMMs (default when n_sims (4 + 4 n_q) >= 2048)
//   unfused         per-layer GEMMs instead of the cluster-fused hidden / vhp chains
//   hid_cp          cp.async big-tile hidden layers instead of the warp-specialised TMA kernel
//   bwd_cp          cp.async big-tile shared-real vhp layers instead of the TMA kernel
//   shared_real     shared-real vhp backward even below 4 waves of CTAs
//   no_shared_real  2 n_q dual columns per sim in the batched vhp backward
//   cpc=K, cpm=K    element / mass row chunks walked per CTA (many sims)
//   tangents=K      jet tangents per column group (1, 3, 5, 7 or 15)
//   dmma_hidden     batched hidden jet layers on the fp64 DMMA kernels instead of the tcgen05
//                   Ozaki-int8 GEMM (ozaki_tc.cuh)
//   cub_chunked     many sims: the element-chunk cubature kernel (k_cubature, 12-row Gram) instead
//                   of the per-sim B-projected kernel (k_cub_sims)
//   dmma_bwd        batched shared-real vhp backward layers on the fp64 DMMA kernel instead of the
//                   tcgen05 Ozaki GEMM
//   dmma_out        batched output layer on the fp64 DMMA kernel instead of the tcgen05 Ozaki GEMM
//   oz_fp64_chain   tcgen05 hidden layers hand their activations to the next one in fp64 (the
//                   consumer converts) instead of as digit tiles (ozaki_chain.cuh)
struct PathOpts {
  bool batched = false, unfused = false, hid_cp = false, bwd_cp = false, shared_real = false,
       no_shared_real = false, dmma_hidden = false, cub_chunked = false, dmma_bwd = false, dmma_out = false,
       oz_fp64_chain = false;
  int cpc = 0, cpm = 0, tangents = 0;
  static PathOpts from_env() {
    PathOpts o;
    const char* env = getenv("NLROM_PATH");
    if (!env) return o;
    std::string list(env);
    size_t pos = 0;
    while (pos <= list.size()) {
      size_t e = list.find(',', pos);
      if (e == std::string::npos) e = list.size();
      const std::string tok = list.substr(pos, e - pos);
      const size_t eq = tok.find('=');
      const std::string key = tok.substr(0, eq);
      const int val = eq == std::string::npos ? 1 : atoi(tok.c_str() + eq + 1);
      if (key == "batched") o.batched = true;
      else if (key == "unfused") o.unfused = true;
      else if (key == "hid_cp") o.hid_cp = true;
      else if (key == "bwd_cp") o.bwd_cp = true;
      else if (key == "shared_real") o.shared_real = true;
      else if (key == "no_shared_real") o.no_shared_real = true;
      else if (key == "dmma_hidden") o.dmma_hidden = true;
      else if (key == "cub_chunked") o.cub_chunked = true;
      else if (key == "dmma_bwd") o.dmma_bwd = true;
      else if (key == "dmma_out") o.dmma_out = true;
      else if (key == "oz_fp64_chain") o.oz_fp64_chain = true;
      else if (key == "cpc") o.cpc = val;
      else if (key == "cpm") o.cpm = val;
      else if (key == "tangents") o.tangents = val;
      else if (!key.empty()) throw Error(NLROM_ERR_ARG, "unknown NLROM_PATH token: " + key);
      pos = e + 1;
    }
    return o;
  }
};

}  // namespace

struct nlrom_ctx {
  int device = 0;
  PathOpts opt;
  cudaStream_t st = nullptr, st2 = nullptr, st3 = nullptr;
  cudaEvent_t evFork = nullptr, evJoin = nullptr, evFork2 = nullptr, evJoin2 = nullptr;
  cudaEvent_t evWf = nullptr, evW = nullptr;  // early weight net: fork after the hidden chain, join before the cubature
  cudaEvent_t evK = nullptr, evM = nullptr;    // split cubature: stiffness branch fork; mass block (st3) done
  cudaEvent_t evP = nullptr;                   // phi reduced (st3)
  DBuf wA1;        // weight-net layer 1 folded onto the decoder: [W1 P W_L | W1 U | W1 P b_L] (wn x wA1ld)
  int wA1ld = 0;
  std::string err;
  double last_norm = 0.0;
  int N = 0, n_p = 0, n_q = 0, n = 0, L = 0, n_sims = 1, T = 0, V = 0;
  std::vector<int> widths;
  // decoder
  std::vector<DBuf> W, WT, b;
  std::vector<int> ldW, ldWT;
  std::vector<DBuf> Wp, WTp;  // fused chains: padded copies (one TMA bulk copy per CTA slice)
  std::vector<OzakiWeights> ozW;  // batched hidden layers on tcgen05: int8 digit tiles of W_l (ozaki_tc.cuh)
  std::vector<OzakiWeights> ozWT;  // batched shared-real vhp backward layers: digit tiles of W_l^T
  OzakiWeights ozWL;               // batched output layer: digit tiles of P W_L (N rows, zero-padded to 128)
  unsigned* ozBHW[2] = {nullptr, nullptr};  // ping-pong column-scale partials between backward layers
  unsigned* ozHW[2] = {nullptr, nullptr};  // ping-pong column-scale partials between hidden layers
  int* ozDE[2] = {nullptr, nullptr};        // ping-pong column exponents of the digit chain (ozaki_chain.cuh)
  int ldpf = 0, ldpb = 0;
  DBuf Alast, AT, Pb, U, mass;
  int ldlast = 0, wL1 = 0, next = 0;
  bool batched = false;  // many sims: big-tile per-layer GEMMs instead of the latency kernels
  DBuf AlastT;           // (P W_L)^T (w x ldAT), batched backward top
  int ldAT = 0;  // next: K-extension of the output layer (0: filter folded)
  // mesh
  IBuf elem_rows;
  DBuf Dm_inv, vol;
  double mu = 0, lam = 0, alpha = 0;
  CubSet setC, setAll;
  CubSet setCF;  // split phase E: the cubature set chunked for the force-only launch (2 elements per CTA)
  // wnet
  int wn = 0, n_cub = 0;
  DBuf W1, b1, W2, b2, W3, b3, W4C, b4C;
  int wsplit = 0, wchunk = 0;
  DBuf wpart, wC;
  // bundle
  int G = 0, gps = 0, Cb = 0, Cc = 0, ldq = 0, ldjt = 0, lddj = 0;
  DBuf X0;
  std::vector<DBuf> H, cache;
  std::vector<int> ldH, ldc;
  DBuf u, value, hvv, Jt, dJ;
  // assembly / solve
  int rpc = 128, nchA = 0;
  int nchAa = 0, nphi = 0;     // k_assemble_a chunks (32 rows) when it also forms the vhp seed; partPhi chunks
  bool agemv = false;          // the last assemble_phase produced the vhp-chain seed partials
  int rpcM = 128, nchM = 0;  // row chunking of the mass block (finer: more CTAs for its Gram)
  int cpmM = 1;              // mass-block row chunks per CTA (nchM = partials per sim)
  DBuf a, partA, partPhi, phi, norm, S, dr, r, rbar, rdbar, fext, rsave, rdot, tmpN;
  IBuf status;
  // backward
  int brows = 32, bnch = 0;
  DBuf bpart, ybuf, Delta0, Delta1, Gt;
  int ldGt = 0;
  // graphs
  cudaGraphExec_t gE = nullptr, gJ = nullptr, gIter = nullptr;
  cudaGraphExec_t gStep = nullptr;  // whole fixed-iteration step incl. pinned H2D / D2H (nlrom_step)
  cudaGraphExec_t gAdapt = nullptr; // whole adaptive step: conditional while nodes (newton_kernels.cuh)
  std::string adapt_key;
  DBuf ad;                          // adaptive Newton state (NT_SIZE doubles)
  DBuf wsk;                         // batched weight-net layer 1: split-K partials [sim][split][wn]
  std::string step_key;
  std::string graph_key;
  int launches_E = 0, launches_J = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  DBuf flush;
  HBuf hin, hout;  // pinned staging of nlrom_step's host inputs / outputs
  // substructured scene (coupled_kernels.cuh): strings of this rank + replicated core
  bool coupled = false;
  DBuf cpR, cpFloc, cpFsum, cpCore, cpBlocks, cpCb, cpX, cpFcore;
  double cp_m_core = 0, cp_k_core = 0, cp_m_string = 0, cp_m_total = 0;
  cudaGraphExec_t gC[2] = {nullptr, nullptr};
  std::string cp_key[2];
  int launches_C[2] = {0, 0};
};

namespace {

int fail(nlrom_ctx* c, const Error& e) {
  if (c) c->err = e.what();
  return e.code;
}

template <class... KArgs, class... Args>
void launch(nlrom_ctx* c, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  if (!launch_gate((const void*)kernel)) return;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL edges in the captured graph
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  NL_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
  ++gemm_launch_count;
}

int grid1(long long n, int bs = 256) { return (int)std::max(1LL, std::min(2048LL, (n + bs - 1) / bs)); }

// ---------------------------------------------------------------- GEMM dispatch
// tcgen05 Ozaki GEMMs only with >= 3 waves of 128 x 64 tiles over the SMs: the persistent kernel
// balances poorly on fewer (cfg3 at 256 sims, n_q = 5: 192 tiles, 71.5k vs 77.5k sim-iterations/s
// on the DMMA kernels)
inline bool oz_enough_tiles(int M, int C, int cstep = 64) {
  return (long long)ceil_div(M, 128) * ceil_div(C, cstep) >= 3LL * 148;
}
template <class Epi>
void hid_gemm(int G, const GemmArgs& g, const Epi& e, cudaStream_t st, bool big = false, bool cp_async = false,
              const OzakiWeights* oz = nullptr, OzakiBExp be = OzakiBExp{nullptr, 0}) {
  // big-tile hidden layers on the 5th-gen tensor cores: Ozaki-scheme fp64 on tcgen05.mma kind::i8
  // (ozaki_tc.cuh; 1.75x the DMMA kernel at the cfg5 shape, ~1e-16 of sum |w||x|)
  if (big && oz && oz->ready && 64 % G == 0 && g.M % oz::BM == 0 && g.K % oz::BK == 0 && g.ldb % 2 == 0 &&
      !g.cstep && oz_enough_tiles(g.M, g.C)) {
    launch_ozaki<64>(oz->view(), be, g, e, st);
    ++gemm_launch_count;
    return;
  }
  // big-tile hidden layers on the warp-specialised TMA pipeline (16 consumer warps, 4 stages):
  // cfg5 hidden layers 14.76 -> 14.51 ms vs the cp.async CfgBig kernel (NLROM_PATH=hid_cp)
  if (big && 128 % G == 0 && !cp_async && g.K % 16 == 0 && g.lda % 2 == 0 && g.ldb % 2 == 0) {
    launch_gemm_ws<WsCfg<64, 128, 4, 4, 4>>(g, e, st);
    ++gemm_launch_count;
    return;
  }
  if (big && 128 % G == 0) {
    launch_gemm<CfgBig>(g, e, st);
    ++gemm_launch_count;
    return;
  }
  switch (G) {
    case 8: launch_gemm<CfgHid<8>>(g, e, st); break;
    case 16: launch_gemm<CfgHid<16>>(g, e, st); break;
    case 24: launch_gemm<CfgHid<24>>(g, e, st); break;
    case 32: launch_gemm<CfgHid<32>>(g, e, st); break;
    case 64: launch_gemm<CfgHid<64>>(g, e, st); break;
    default: throw Error(NLROM_ERR_ARG, "unsupported jet group size");
  }
  ++gemm_launch_count;
}
template <class Epi>
void out_gemm(int G, const GemmArgs& g, const Epi& e, cudaStream_t st) {
  switch (G) {
    case 8: launch_gemm<CfgOut<8>>(g, e, st); break;
    case 16: launch_gemm<CfgOut<16>>(g, e, st); break;
    case 24: launch_gemm<CfgOut<24>>(g, e, st); break;
    case 32: launch_gemm<CfgOut<32>>(g, e, st); break;
    case 64: launch_gemm<CfgOut<64>>(g, e, st); break;
    default: throw Error(NLROM_ERR_ARG, "unsupported jet group size");
  }
  ++gemm_launch_count;
}

void choose_groups(int n_q, int width, bool batched, int forced, int& G, int& gps) {
  const int cand[5] = {1, 3, 5, 7, 15};
  int g = 3;
  if (forced > 0) g = forced;
  else if (batched) {
    // big 128-column tiles: G | 128, fewest executed columns G * ceil(n_q / g)
    int best = 1 << 30;
    for (int c : {1, 3, 7, 15}) {
      const int cols = (4 + 4 * c) * ((n_q + c - 1) / c);
      if (cols < best) { best = cols; g = c; }
    }
  } else if (width > 64) {
    g = 3;  // wide decoders: G = 16 is the fused hidden chain that fits in shared memory
  } else if (n_q <= 15) {
    for (int c : cand)
      if (c >= n_q) { g = c; break; }
  } else {
    g = 3;
  }
  bool ok = false;
  for (int c : cand) ok |= (c == g);
  if (!ok) throw Error(NLROM_ERR_ARG, "jet tangents per group must be one of 1,3,5,7,15");
  G = 4 + 4 * g;
  gps = (n_q + g - 1) / g;
  (void)width;
}

void upload(DBuf& d, const double* h, size_t n);

void build_set(nlrom_ctx* c, CubSet& s, const std::vector<int>& elems, const std::vector<int>& rows_host,
               int epc, const double* Dm_host, const double* vol_host, const double* U_host = nullptr) {
  s.n = (int)elems.size();
  s.elems.upload(elems.data(), elems.size());
  {
    std::vector<int> rg((size_t)std::max(s.n, 1) * 12, -1);
    std::vector<double> dg((size_t)std::max(s.n, 1) * 9, 0.0), vg((size_t)std::max(s.n, 1), 0.0);
    for (int i = 0; i < s.n; ++i) {
      for (int l = 0; l < 12; ++l) rg[(size_t)i * 12 + l] = rows_host[(size_t)elems[i] * 12 + l];
      for (int l = 0; l < 9; ++l) dg[(size_t)i * 9 + l] = Dm_host[(size_t)elems[i] * 9 + l];
      vg[i] = vol_host[elems[i]];
    }
    s.rows_g.upload(rg.data(), rg.size());
    upload(s.Dm_g, dg.data(), dg.size());
    upload(s.vol_g, vg.data(), vg.size());
  }
  // CSR: unique rows -> (element slot * 12 + l)
  std::map<int, std::vector<int>> m;
  for (int i = 0; i < s.n; ++i)
    for (int l = 0; l < 12; ++l) {
      int row = rows_host[(size_t)elems[i] * 12 + l];
      if (row >= 0) m[row].push_back(i * 12 + l);
    }
  std::vector<int> ids, ptr{0}, ent;
  for (auto& kv : m) {
    ids.push_back(kv.first);
    for (int e : kv.second) ent.push_back(e);
    ptr.push_back((int)ent.size());
  }
  s.n_rows = (int)ids.size();
  {
    std::vector<int> full((size_t)c->N + 1, 0);
    for (size_t k = 0; k < ids.size(); ++k) full[(size_t)ids[k] + 1] = ptr[k + 1] - ptr[k];
    for (int r = 0; r < c->N; ++r) full[(size_t)r + 1] += full[r];
    s.rowptr_full.upload(full.data(), full.size());
  }
  s.row_ids.upload(ids.data(), ids.size());
  s.row_ptr.upload(ptr.data(), ptr.size());
  s.entries.upload(ent.data(), ent.size());
  const int n = c->n;
  s.epc = epc;
  while (s.epc > 1 && (size_t)(2 * s.epc * 12 * gram_ld(n) + s.epc * 162) * 8 > 200 * 1024) s.epc /= 2;
  s.nech = std::max(1, ceil_div(std::max(s.n, 1), s.epc));
  // Many sims: a CTA walks several element chunks of its sim and accumulates the Gram in shared
  // memory, so the partial K~ traffic (n^2 doubles per CTA, written and re-read by the
  // reduction) shrinks by cpc; keep >= ~2 waves of 3 CTAs per SM.
  s.cpc = 1;
  if (c->n_sims > 1 && n <= 256 &&
      (size_t)(2 * s.epc * 12 * gram_ld(n) + s.epc * 162 + n * n + n) * 8 <= 200 * 1024) {
    const long long ctas = (long long)c->n_sims * s.nech;
    s.cpc = (int)std::max(1LL, std::min<long long>(s.nech, ctas / (148 * 3 * 2)));
    if (c->opt.cpc > 0) s.cpc = std::max(1, std::min(s.nech, c->opt.cpc));
  }
  s.nchunk = ceil_div(s.nech, s.cpc);
  // many sims with a small reduced space: one CTA per sim (k_cub_sims), one partial per sim
  const int np = c->n_p;
  s.ti = std::max(1, ceil_div(n + 1, 8));
  s.sims = U_host && c->n_sims > 1 && s.ti <= 4 && s.n > 0 && !c->opt.cub_chunked &&
           cub_sims_smem(n, np, s.ti) <= 110 * 1024;
  if (s.sims) {
    s.nchunk = 1;
    // BU[(i, a * 3 + y), j] = sum_v G[v][y] U[row(v, a)][j],  G[v] = row v - 1 of Dm^-1, G[0] = -sum
    std::vector<double> bu((size_t)s.n * 9 * std::max(np, 1), 0.0);
    for (int i = 0; i < s.n; ++i) {
      const double* Di = Dm_host + (size_t)elems[i] * 9;
      for (int aa = 0; aa < 3; ++aa)
        for (int y = 0; y < 3; ++y)
          for (int j = 0; j < np; ++j) {
            double acc = 0.0;
            for (int v = 0; v < 4; ++v) {
              const int row = rows_host[(size_t)elems[i] * 12 + 3 * v + aa];
              if (row < 0) continue;
              const double g = v == 0 ? -(Di[y] + Di[3 + y] + Di[6 + y]) : Di[(v - 1) * 3 + y];
              acc += g * U_host[(size_t)row * np + j];
            }
            bu[((size_t)i * 9 + aa * 3 + y) * np + j] = acc;
          }
    }
    upload(s.BU, bu.data(), bu.size());
  }
  s.fe_w.alloc((size_t)c->n_sims * std::max(s.n, 1) * 12);
  s.part_f.alloc((size_t)c->n_sims * s.nchunk * n);
  s.part_K.alloc((size_t)c->n_sims * s.nchunk * n * n);
  s.f.alloc((size_t)c->n_sims * c->N);
}

// ----------------------------------------------------------------- E and J phases
// Decoder output layer + fused filter over the compact columns: D = [W_L | -U][h; U^T W_L h] + P b.
// The dominant kernel of one Newton iteration (fp64 DMMA, 8 warps, 48 x 128 tiles, one wave).
using CfgOutC = GemmCfg<48, 128, 2, 4, 1, 32, 3>;
// same tiling on the warp-specialised TMA pipeline (gemm_ws.cuh): 6 swizzled stages, one
// producer warp; 13% faster on this shape (tools/probes/gemm_ws_probe.cu), bitwise identical
using CfgOutWs = WsCfg<48, 128, 3, 4, 6>;  // 12 consumer warps (16 x 32 warp tiles): best of the probe
// <= 64 output columns (one sim at n_q <= 31: 2 + 2 n_q columns): half-width tiles, so no DMMA
// work is spent on padding columns
// (16 x 64 tiles, 420 CTAs: fastest of 48x128 / 48x64 / 24x64 / 16x64 / 8x64 in the cfg2 graph)
using CfgOutWs64c = WsCfg<16, 64, 2, 2, 6>;

// the output layer on tcgen05: the compact last hidden layer writes its column scales for it
bool out_on_tc(nlrom_ctx* c) {
  // (>= 8192 columns: below that the persistent 1-CTA/SM kernel costs the step more than it saves
  // in the GEMM -- it cannot share SMs with the side-branch kernels: cfg3 at 256 sims, n_q = 5,
  // 3072 columns, 71k vs 78k sim-iterations/s; n_q = 30, 15872 columns, 46k vs 43k)
  return c->batched && c->ozWL.ready && c->ozHW[0] && c->wL1 % 32 == 0 && c->ldlast % 2 == 0 && !c->next &&
         c->Cc % 2 == 0 && oz_enough_tiles(c->N, c->n_sims * c->Cc) && c->n_sims * c->Cc >= 8192;
}

void output_layer(nlrom_ctx* c) {
  GemmArgs g{c->Alast.p, c->H[c->L - 2].p, c->ldlast, c->ldlast, c->N, c->n_sims * c->Cc, c->wL1 + c->next, 0, 0};
  EpiJetOutC e{c->Pb.p, c->U.p, c->r.p, c->u.p, c->value.p, c->hvv.p, c->Jt.p, c->dJ.p, c->ldjt, c->lddj,
               c->n_p, c->n_q};
  // batched: tcgen05 Ozaki GEMM over the compact columns (their column scales from the last hidden
  // layer's epilogue), else the cp.async big-tile kernel (the warp-specialised pipeline measured
  // slower here: 3.38 vs 3.06 ms at cfg5, the EpiJetOutC scatter dominates the tile)
  if (c->batched && out_on_tc(c)) {
    // row-major fp64 tile: coalesced J~ / dJ row stores (EpiJetOutCRow)
    const OzakiBExp hw{c->ozHW[(c->L - 2) & 1], c->wL1 / 32};
    const int C = g.C, Cpad = round_up(C, 64);
    const bool dig = OZ_OUT_DIG && !c->opt.oz_fp64_chain && c->L >= 4 && c->ozDE[0] && g.K == 256 && c->wL1 == 256 &&
                     (size_t)Cpad * 7 * 256 <= (size_t)c->n_sims * c->Cb * c->ldH[c->L - 3] * 8 &&
                     Cpad <= round_up(c->n_sims * c->Cb, 64);
    if (dig) {
      // 8 m tiles per column: the input converted once (k_to_digits) into digit tiles landed by TMA
      unsigned char* buf = reinterpret_cast<unsigned char*>(c->H[c->L - 3].p);   // consumed by the last hidden layer
      int* dexp = c->ozDE[(c->L - 2) & 1];
      launch(c, k_to_digits, ceil_div(Cpad * (g.K / 32), 256), 256, 0, (const double*)g.B, g.ldb, C, g.K, hw.parts,
             hw.nparts, buf, dexp);
      OzakiBExp be{nullptr, 0};
      be.dig = buf;
      be.dexp = dexp;
      launch_ozaki<64, EpiJetOutCRow, true>(c->ozWL.view(), be, g, EpiJetOutCRow{e}, c->st);
    } else {
      launch_ozaki<64>(c->ozWL.view(), hw, g, EpiJetOutCRow{e}, c->st);
    }
  } else if (c->batched) launch_gemm<CfgBig>(g, e, c->st);
  else if (c->ldlast % 2 == 0 && g.C <= 64) launch_gemm_ws<CfgOutWs64c>(g, e, c->st);
  else if (c->ldlast % 2 == 0) launch_gemm_ws<CfgOutWs>(g, e, c->st);
  else launch_gemm<CfgOutC>(g, e, c->st);
  ++gemm_launch_count;
}

// Fused hidden chain (mlp_chain.cuh): one cluster of CS CTAs per column group.
template <int R, int G, int CS>
bool launch_mlp_fwd(nlrom_ctx* c, const MlpFwdArgs& a) {
  // DSMEM stores + cluster barrier per layer (the st.async / per-source mbarrier variant measured
  // slower at cfg2: tools/probes/retired/mlp_chain_async.cuh)
  const int kmax = std::max(c->wL1, c->n_q);
  const size_t smem = MlpPlan<R, G>::bytes(kmax);
  if (smem > 227 * 1024) return false;
  auto kern = k_mlp_jet_fwd<R, G, CS>;
  static bool configured = false;
  if (!configured) {
    NL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (CS > 8) NL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, c->n_sims * c->gps, 1);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (!launch_gate((const void*)kern)) return true;
  NL_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  ++gemm_launch_count;
  return true;
}

bool fused_hidden_forward(nlrom_ctx* c, double dt, int drop_fict) {
  if (c->opt.unfused || c->batched) return false;
  const int L1 = c->L - 1, w = c->wL1;
  if (L1 < 1 || L1 > MLP_MAXL) return false;
  for (int l = 1; l <= L1; ++l)
    if (c->widths[l] != w) return false;
  MlpFwdArgs a{};
  a.r = c->r.p; a.rbar = c->rbar.p; a.rdbar = c->rdbar.p;
  a.n_p = c->n_p; a.n_q = c->n_q; a.n = c->n; a.dt = dt; a.alpha = c->alpha; a.drop_fict = drop_fict;
  a.L1 = L1; a.w = w;
  for (int l = 0; l < L1; ++l) {
    a.W[l] = c->W[l].p; a.b[l] = c->b[l].p; a.ldW[l] = c->ldW[l]; a.in[l] = c->widths[l];
    a.Wp[l] = c->Wp[l].p;
    a.cache[l] = c->cache[l].p;
  }
  a.ldc = c->ldc[0];
  a.ldp = c->ldpf;
  if (c->ldpf != round_up(std::max(w, c->n_q), 16) + 4) return false;  // padded layout == smem slice layout
  a.Hout = c->H[L1 - 1].p;
  a.ldH = c->ldH[L1 - 1];
  a.G = c->G; a.gps = c->gps;
  const int G = c->G;
  if (w == 256 && G == 16) return launch_mlp_fwd<32, 16, 8>(c, a);
  if (w == 256 && G == 24) return launch_mlp_fwd<32, 24, 8>(c, a);
  if (w == 64 && G == 24) return launch_mlp_fwd<8, 24, 8>(c, a);
  if (w == 64 && G == 16) return launch_mlp_fwd<8, 16, 8>(c, a);
  if (w == 40 && G == 24) return launch_mlp_fwd<8, 24, 5>(c, a);
  if (w == 8 && G == 16) return launch_mlp_fwd<8, 16, 1>(c, a);
  return false;
}

bool shared_real_bwd(nlrom_ctx* c, int npass_per_sim);

// with_output = false: hidden layers only (stage timing of nlrom_bench_kernels).
void bundle_forward(nlrom_ctx* c, double dt, int drop_fict, bool with_output = true) {
  if (fused_hidden_forward(c, dt, drop_fict)) {
    if (with_output) output_layer(c);
    return;
  }
  const int ncols = c->n_sims * c->Cb;
  const int nq = c->n_q;
  const double* in = c->X0.p;
  int ldin = c->ldq;
  // hidden layer l runs on the tcgen05 Ozaki GEMM (the dispatch rule of hid_gemm)
  auto oz_runs = [&](int l) {
    if (!c->batched || l < 0 || l >= (int)c->ozW.size() || !c->ozW[l].ready) return false;
    const int ldb = l == 0 ? c->ldq : c->ldH[l - 1];
    return 64 % c->G == 0 && c->widths[l + 1] % oz::BM == 0 && c->widths[l] % oz::BK == 0 && ldb % 2 == 0 &&
           oz_enough_tiles(c->widths[l + 1], ncols);
  };
  // digit chain: a tcgen05 layer of width 256 whose consumer is a tcgen05 hidden layer hands over
  // digit tiles (ozaki_chain.cuh); its buffer H[l] holds them (7 of the 8 bytes per element)
  // the seed layer fused with layer 1's B operand (k_seed_layer: layer 0 = three mat-vecs per group)
  const bool seed_fused = c->L >= 3 && c->G >= 8 && 32 % c->G == 0 && c->widths[1] == 256 && c->ozDE[0] &&
                          c->ldH[0] % 2 == 0 && c->ozHW[0] && oz_runs(1) &&
                          (size_t)round_up(ncols, 64) * 7 <= (size_t)ncols * c->ldH[0] * 8;
  auto dig_out = [&](int l) {
    if (l == 0) return seed_fused && !c->opt.oz_fp64_chain;
    return !c->opt.oz_fp64_chain && c->ozDE[0] && 32 % c->G == 0 && l + 1 <= c->L - 2 && oz_runs(l) && oz_runs(l + 1) &&
           c->widths[l + 1] == 256 && (size_t)round_up(ncols, 64) * 7 <= (size_t)ncols * c->ldH[l] * 8;
  };
  // the shared-real vhp backward reads one real part per sim and layer (EpiJet::real_once)
  const bool real_once = shared_real_bwd(c, nq);
  if (seed_fused) {
    SeedLayerArgs sa{(const double*)c->r.p, (const double*)c->rbar.p, (const double*)c->rdbar.p, c->n_p, nq, c->n,
                     dt, c->alpha, drop_fict, (const double*)c->W[0].p, c->ldW[0], (const double*)c->b[0].p,
                     c->cache[0].p, c->ldc[0], c->G, c->gps, ncols, reinterpret_cast<unsigned char*>(c->H[0].p),
                     c->ozDE[0], c->H[0].p, c->ldH[0], c->ozHW[0], real_once ? 1 : 0};
    const bool dig = dig_out(0);
    // whole 64-column digit tiles: the CTAs past ncols write the padding half's zero digits
    if (dig) launch(c, k_seed_layer<true>, round_up(ncols, 64) / 32, 256, seed_layer_smem(), sa);
    else launch(c, k_seed_layer<false>, ceil_div(ncols, 32), 256, seed_layer_smem(), sa);
    in = c->H[0].p;
    ldin = c->ldH[0];
  } else {
    launch(c, k_seed_jet, grid1((long long)ncols * nq), 256, 0, (const double*)c->r.p, (const double*)c->rbar.p,
           (const double*)c->rdbar.p, c->X0.p, c->ldq, c->n_p, nq, c->n, c->G, c->gps, c->n_sims, dt, c->alpha,
           drop_fict);
  }
  for (int l = seed_fused ? 1 : 0; l + 1 < c->L; ++l) {
    // the last hidden layer writes the de-replicated layout (its consumer is linear)
    const int compact = (l == c->L - 2) ? 1 : 0;
    GemmArgs g{c->W[l].p, in, c->ldW[l], ldin, c->widths[l + 1], ncols, c->widths[l], 0, 0};
    EpiJet e{c->H[l].p, c->ldH[l], 0, c->b[l].p, c->cache[l].p, c->ldc[l], c->G, c->gps, nq, compact};
    e.real_once = real_once ? 1 : 0;
    // tcgen05 Ozaki layers read their input's column scales from the previous layer's epilogue
    const bool oz_here = c->batched && l < (int)c->ozW.size() && c->ozW[l].ready;
    const bool oz_next = (c->batched && l + 1 < (int)c->ozW.size() && c->ozW[l + 1].ready && !compact &&
                          c->widths[l + 1] % 32 == 0 && c->ozHW[0] && oz_enough_tiles(c->widths[l + 2], ncols)) ||
                         (compact && out_on_tc(c));
    if (oz_next) e.colhw = c->ozHW[l & 1];
    const bool din = dig_out(l - 1), dout = dig_out(l);
    if (din || dout) {
      OzakiBExp be = OzakiBExp{nullptr, 0};
      if (din) {
        be.dig = reinterpret_cast<const unsigned char*>(c->H[l - 1].p);
        be.dexp = c->ozDE[(l - 1) & 1];
      } else if (l >= 1 && c->ozHW[0]) {
        be = OzakiBExp{c->ozHW[(l - 1) & 1], c->widths[l] / 32};
      }
      if (dout) {
        EpiJetDig ed{c->b[l].p, c->cache[l].p, c->ldc[l], c->G, c->gps, nq, reinterpret_cast<unsigned char*>(c->H[l].p),
                     c->ozDE[l & 1], real_once ? 1 : 0};
        if (din) launch_ozaki<64, EpiJetDig, true>(c->ozW[l].view(), be, g, ed, c->st);
        else launch_ozaki<64, EpiJetDig, false>(c->ozW[l].view(), be, g, ed, c->st);
      } else {
        launch_ozaki<64, EpiJet, true>(c->ozW[l].view(), be, g, e, c->st);
      }
      ++gemm_launch_count;
    } else {
      const OzakiBExp be = (oz_here && l >= 1 && c->ozHW[0]) ? OzakiBExp{c->ozHW[(l - 1) & 1], c->widths[l] / 32}
                                                            : OzakiBExp{nullptr, 0};
      hid_gemm(c->G, g, e, c->st, c->batched, c->opt.hid_cp, oz_here ? &c->ozW[l] : nullptr, be);
    }
    in = c->H[l].p;
    ldin = c->ldH[l];
  }
  if (c->next) {  // T = (U^T W_L) h -> columns wL1.. of the last hidden buffer (filter as K-extension)
    GemmArgs g{c->AT.p, in, round_up(c->wL1, 2), ldin, c->n_p, c->n_sims * c->Cc, c->wL1, 0, 0};
    EpiStore e{c->H[c->L - 2].p + c->wL1, c->ldlast, 0, nullptr, 1, nullptr};
    hid_gemm(c->G, g, e, c->st);
  }
  if (with_output) output_layer(c);
}

void wnet_phase(nlrom_ctx* c) {
  int nsplit = c->wsplit;
  if (c->batched) {
    // layer 1 for all sims as one GEMM: part (n_sims x wn) = u (n_sims x N) W1^T; few output tiles
    // (M = wn) and K = N long: split K over blockIdx.z into [sim][split][wn] partials, then a
    // fixed-order reduction (cfg5: 32 CTAs, 95 us unsplit)
    const int M = c->wn, tiles = ceil_div(M, CfgBig::BM) * ceil_div(c->n_sims, CfgBig::BN);
    int split = 1;
    for (int sp : {16, 12, 10, 8, 6, 5, 4, 3, 2})
      if (tiles * sp <= 2 * 148 * 2 && c->N % sp == 0 && (c->N / sp) % 2 == 0 && c->N / sp >= 64 &&
          (size_t)c->n_sims * sp * M <= c->wsk.n) {
        split = sp;
        break;
      }
    if (split == 1) {
      GemmArgs g{c->W1.p, c->u.p, round_up(c->N, 2), c->N, M, c->n_sims, c->N, 0, 0};
      launch_gemm<CfgBig>(g, EpiStore{c->wpart.p, M, 0, nullptr, 1, nullptr}, c->st);
    } else {
      const int Kc = c->N / split;
      GemmArgs g{c->W1.p, c->u.p, round_up(c->N, 2), c->N, M, c->n_sims, Kc, Kc, Kc};
      launch_gemm<CfgBig>(g, EpiStore{c->wsk.p, split * M, M, nullptr, 1, nullptr}, c->st, split);
      launch(c, k_reduce_cols, dim3(ceil_div(M, 32), c->n_sims), 256, 0, (const double*)c->wsk.p, split, M,
             c->wpart.p);
    }
    ++gemm_launch_count;
    nsplit = 1;
  } else {
    if (c->wchunk == 64)
      launch(c, k_gemv_splitk_t<2>, dim3(c->wsplit, c->n_sims), 256, 0, (const double*)c->W1.p, round_up(c->N, 2),
             (const double*)c->u.p, (long long)c->N, c->wn, c->N, c->wpart.p, c->n_sims);
    else if (c->wchunk == 32)
      launch(c, k_gemv_splitk_t<1>, dim3(c->wsplit, c->n_sims), 256, 0, (const double*)c->W1.p, round_up(c->N, 2),
             (const double*)c->u.p, (long long)c->N, c->wn, c->N, c->wpart.p, c->n_sims);
    else
      launch(c, k_gemv_splitk, dim3(c->wsplit, c->n_sims), 256, 0, (const double*)c->W1.p, round_up(c->N, 2),
             (const double*)c->u.p, (long long)c->N, c->wn, c->N, c->wchunk, c->wpart.p, c->n_sims);
  }
  const size_t wsm = (size_t)(5 * c->wn + 64 + 2 * c->wn * c->wn + 64 * c->wn + nsplit * c->wn) * 8;
  if (c->wn % 2 == 0 && 256 % c->wn == 0 && c->wn >= 16 && (c->n_sims == 1 || nsplit == 1)) {
    launch(c, k_wnet_tail2, dim3(std::max(1, ceil_div(c->n_cub, 64)), c->n_sims), 256, wsm + 16,
           (const double*)c->wpart.p, nsplit, c->wn, (const double*)c->b1.p, (const double*)c->W2.p,
           (const double*)c->b2.p, (const double*)c->W3.p, (const double*)c->b3.p, (const double*)c->W4C.p,
           (const double*)c->b4C.p, c->n_cub, c->wC.p, c->n_sims);
    return;
  }
  launch(c, k_wnet_tail, dim3(std::max(1, ceil_div(c->n_cub, 64)), c->n_sims), 256, wsm, (const double*)c->wpart.p, nsplit, c->wn,
         (const double*)c->b1.p, (const double*)c->W2.p, (const double*)c->b2.p, (const double*)c->W3.p,
         (const double*)c->b3.p, (const double*)c->W4C.p, (const double*)c->b4C.p, c->n_cub, c->wC.p, c->n_sims);
}

// part: 0 forces + stiffness, 1 weighted element forces only (fe_w), 2 stiffness / Gram only
void cubature_phase(nlrom_ctx* c, CubSet& s, bool weighted, bool scatter = true, bool early = true, int part = 0) {
  if (s.sims && part == 0) {
    CubSimsArgs a{s.rows_g.p, s.Dm_g.p, s.vol_g.p, s.BU.p, s.n, weighted ? c->wC.p : nullptr, c->u.p, c->Jt.p,
                  c->N, c->n, c->n_p, c->ldjt, c->mu, c->lam, s.fe_w.p, s.part_f.p, s.part_K.p, 0};
    const size_t smem = cub_sims_smem(c->n, c->n_p, s.ti);
    // two CTAs per SM (128 registers): the 3-CTA / 80-register build spills and measured 2x slower
    switch (s.ti) {
      case 1: launch(c, k_cub_sims<1, 2>, dim3(c->n_sims), 256, smem, a); break;
      case 2: launch(c, k_cub_sims<2, 2>, dim3(c->n_sims), 256, smem, a); break;
      case 3: launch(c, k_cub_sims<3, 2>, dim3(c->n_sims), 256, smem, a); break;
      default: launch(c, k_cub_sims<4, 2>, dim3(c->n_sims), 256, smem, a); break;
    }
    if (scatter)
      launch(c, k_scatter_rows, grid1((long long)s.n_rows * c->n_sims), 256, 0, (const int*)s.row_ids.p,
             (const int*)s.row_ptr.p, (const int*)s.entries.p, s.n_rows, (const double*)s.fe_w.p, s.n, s.f.p, c->N,
             c->n_sims);
    return;
  }
  CubArgs a{s.elems.p, s.n, c->elem_rows.p, c->Dm_inv.p, c->vol.p, weighted ? c->wC.p : nullptr, c->u.p,
            part == 1 ? nullptr : c->Jt.p, c->N, c->n, c->ldjt, c->mu, c->lam, s.epc, s.fe_w.p, s.part_f.p,
            s.part_K.p, s.nchunk, nullptr, nullptr};
  a.skip_fe = part == 2 ? 1 : 0;
  a.rows_g = s.rows_g.p;
  a.Dm_g = s.Dm_g.p;
  a.vol_g = s.vol_g.p;
  a.cpc = part == 1 ? 1 : s.cpc;  // the force-only launch writes no partials: one chunk per CTA
  // early: the weight-net tail (the only producer) launches dependents only after its own wait,
  // so J~ / u are complete at launch; not when the output layer itself is a direct producer
  a.early = (weighted && early) ? 1 : 0;
  size_t smem = (size_t)(2 * s.epc * 12 * gram_ld(c->n) + s.epc * 162 + (a.cpc > 1 ? c->n * c->n + c->n : 0)) * 8;
  // many sims: 3 resident CTAs per SM (80 registers) when the shared memory allows it
  const bool three = c->n_sims > 1 && smem <= 74 * 1024;
  launch(c, three ? k_cubature<3> : k_cubature<2>, dim3(a.cpc > 1 ? s.nchunk : s.nech, c->n_sims), 256, smem, a);
  if (scatter)
  launch(c, k_scatter_rows, grid1((long long)s.n_rows * c->n_sims), 256, 0, (const int*)s.row_ids.p,
         (const int*)s.row_ptr.p, (const int*)s.entries.p, s.n_rows, (const double*)s.fe_w.p, s.n, s.f.p, c->N,
         c->n_sims);
}

// S = mass-block partials + dt^2 (cubature K~ partials) (+ the vhp block Gt)
void reduce_S_launch(nlrom_ctx* c, CubSet& s, const double* Gt, double dt) {
  const int n = c->n;
  if (c->n_sims > 1)
    launch(c, k_reduce_S_flat, grid1((long long)c->n_sims * n * n), 256, 0, (const double*)c->partA.p, c->nchM,
           (const double*)s.part_K.p, s.nchunk, Gt, c->ldGt, n, c->n_p, c->n_q, dt, c->S.p, c->n_sims);
  else
    launch(c, k_reduce_S, dim3(ceil_div(n * n, 32), c->n_sims), 256, 0, (const double*)c->partA.p, c->nchM,
           (const double*)s.part_K.p, s.nchunk, Gt, c->ldGt, n, c->n_p, c->n_q, dt, c->S.p);
}

void assemble_launch(nlrom_ctx* c, CubSet& s, double dt, int drop_fict, int mode) {
  AsmArgs A{c->Jt.p, c->ldjt, c->dJ.p, c->lddj, c->mass.p, c->hvv.p, s.f.p, c->fext.p, c->r.p, c->rbar.p,
            c->rdbar.p, c->a.p, c->partA.p, c->partPhi.p, c->N, c->n, c->n_p, c->n_q, c->rpc, c->nchA, dt,
            c->alpha, drop_fict, mode};
  size_t smem = (size_t)(2 * c->rpc * gram_ld(c->n) + 2 * c->rpc + c->n) * 8;
  launch(c, k_assemble, dim3(c->nchA, c->n_sims), 256, smem, A);
}

// The mass block J~^T M [(1+alpha dt)U, (1+alpha dt)J + dJ] depends only on the decoder bundle:
// it runs on a side stream (a parallel graph branch) while the weight net, the cubature and
// the a-vector -- the critical path -- run on the main stream.
size_t mass_smem(nlrom_ctx* c) {
  return (size_t)(2 * c->rpcM * c->ldjt + c->rpcM * c->lddj + c->rpcM) * 8 + 16 +
         (c->cpmM > 1 ? (size_t)c->n * c->n * 8 : 0);
}

void mass_block_launch(nlrom_ctx* c, CubSet& s, double dt, int drop_fict) {
  if (c->rpcM != c->rpc || (c->ldjt == gram_ld(c->n) && c->lddj % 2 == 0 && mass_smem(c) <= 220 * 1024)) {
    launch(c, k_assemble_mass, dim3(c->nchM, c->n_sims), 256, mass_smem(c), (const double*)c->Jt.p, c->ldjt,
           (const double*)c->dJ.p, c->lddj, (const double*)c->mass.p, c->N, c->n, c->n_p, c->rpcM, c->nchM,
           c->alpha * dt, c->partA.p, c->cpmM);
  } else {
    assemble_launch(c, s, dt, drop_fict, 1);
  }
}

void mass_block_fork(nlrom_ctx* c, CubSet& s, double dt, int drop_fict) {
  NL_CUDA(cudaEventRecord(c->evFork, c->st));
  NL_CUDA(cudaStreamWaitEvent(c->st2, c->evFork, 0));
  std::swap(c->st, c->st2);
  mass_block_launch(c, s, dt, drop_fict);
  std::swap(c->st, c->st2);
  NL_CUDA(cudaEventRecord(c->evJoin, c->st2));
}

// a and the J~^T a partials on the critical path; phi = sum of partials and S_base = mass block
// + dt^2 K~ (no vhp) on the side branch (after the mass block), joined where they are consumed.
bool fused_vhp_backward(nlrom_ctx* c, bool check_only);

void assemble_phase(nlrom_ctx* c, CubSet& s, double dt, int drop_fict) {
  c->agemv = false;
  c->nphi = c->nchA;
  if (c->rpc <= 128 && c->n <= 128) {
    // with the fused vhp chain: 32-row chunks that also form the chain's seed (P W_L)^T a
    const bool g = fused_vhp_backward(c, true) && c->wL1 <= 256 && c->ldlast % 2 == 0;
    const int rc = g ? ASMA_GROWS : c->rpc, nch = g ? c->nchAa : c->nchA;
    AsmAArgs A{c->Jt.p, c->ldjt, c->mass.p, c->hvv.p, c->fext.p, c->r.p, c->rbar.p, c->rdbar.p,
               s.rowptr_full.p, s.entries.p, s.fe_w.p, std::max(s.n, 1), c->a.p, c->partPhi.p,
               c->N, c->n, rc, nch, dt, c->alpha, drop_fict,
               (const double*)c->Alast.p, c->ldlast, c->wL1, g ? c->bpart.p : nullptr};
    if (g) launch(c, k_assemble_a<true>, dim3(nch, c->n_sims), 256, 0, A);
    else launch(c, k_assemble_a<false>, dim3(nch, c->n_sims), 256, 0, A);
    c->agemv = g;
    c->nphi = nch;
  } else {
    launch(c, k_scatter_rows, grid1((long long)s.n_rows * c->n_sims), 256, 0, (const int*)s.row_ids.p,
           (const int*)s.row_ptr.p, (const int*)s.entries.p, s.n_rows, (const double*)s.fe_w.p, s.n, s.f.p, c->N,
           c->n_sims);
    assemble_launch(c, s, dt, drop_fict, 2);
  }
  NL_CUDA(cudaEventRecord(c->evFork2, c->st));
  NL_CUDA(cudaStreamWaitEvent(c->st2, c->evFork2, 0));
  std::swap(c->st, c->st2);
  launch(c, k_reduce_phi, c->n_sims, 256, (size_t)8 * c->n * 8, (const double*)c->partPhi.p, c->nphi, c->n,
         c->phi.p, c->norm.p);
  reduce_S_launch(c, s, nullptr, dt);
  std::swap(c->st, c->st2);
  NL_CUDA(cudaEventRecord(c->evJoin2, c->st2));
}

// join_side = false leaves the phi / S_base branch open for phase_J (one-graph Newton iteration)
// Early weight net: the net's layer 1 is folded onto the hidden chain's output (k_wnet_head), so
// head + tail run on a side branch concurrently with the output layer instead of after it.
// CTAs per sim of k_wnet_head: 8 output rows each (32 threads per row)
int wnet_head_split(nlrom_ctx* c) { return c->wn % 8 == 0 && c->wn >= 8 ? c->wn / 8 : 1; }

bool early_wnet_ok(nlrom_ctx* c) {
  return c->wA1.p && !c->batched && c->wn >= 16 && c->wn % 2 == 0 && 256 % c->wn == 0 &&
         c->wL1 + c->n_p + 1 <= 1024 && c->n_cub > 0 && wnet_head_smem(c->wn, c->wA1ld) <= 220 * 1024;
}

// Split phase E (early weight net + mass block on st3 + cubature split into a force-only launch
// on the critical path and the stiffness / Gram launch on a side branch):
//   st : jet chain -> output layer -> [wait W] -> k_cubature(forces) -> k_assemble_a
//   st2: wnet head -> tail (W) -> [wait K] k_cubature(stiffness) -> [wait M] k_reduce_S
//   st3: [after the output layer] k_assemble_mass (M) -> [wait A] k_reduce_phi (P)
//   (st2 and st3 joined before the LU)
// resid_only: the residual and ||phi|| alone (the step's final convergence evaluation): no mass
// block, no stiffness / Gram launch, no S_base reduction, no vhp seed partials
void phase_E_split(nlrom_ctx* c, const nlrom_simcfg& cfg, CubSet& s, bool resid_only = false) {
  auto on = [&](cudaStream_t& other, auto fn) {
    std::swap(c->st, other);
    fn();
    std::swap(c->st, other);
  };
  NL_CUDA(cudaEventRecord(c->evWf, c->st));
  NL_CUDA(cudaStreamWaitEvent(c->st2, c->evWf, 0));
  on(c->st2, [&] {
    launch(c, k_wnet_head, dim3(wnet_head_split(c), c->n_sims), 256,
           wnet_head_smem(c->wn / wnet_head_split(c), c->wA1ld), (const double*)c->H[c->L - 2].p,
           c->ldH[c->L - 2], c->Cc, (const double*)c->r.p, c->n, c->n_p, c->wL1, (const double*)c->wA1.p, c->wA1ld,
           c->wn, c->wpart.p);
    const size_t wsm = (size_t)(5 * c->wn + 64 + 2 * c->wn * c->wn + 64 * c->wn + c->wn) * 8;
    launch(c, k_wnet_tail2, dim3(std::max(1, ceil_div(c->n_cub, 64)), c->n_sims), 256, wsm + 16,
           (const double*)c->wpart.p, 1, c->wn, (const double*)c->b1.p, (const double*)c->W2.p,
           (const double*)c->b2.p, (const double*)c->W3.p, (const double*)c->b3.p, (const double*)c->W4C.p,
           (const double*)c->b4C.p, c->n_cub, c->wC.p, c->n_sims);
  });
  NL_CUDA(cudaEventRecord(c->evW, c->st2));
  output_layer(c);
  if (!resid_only) {
    NL_CUDA(cudaEventRecord(c->evFork, c->st));
    NL_CUDA(cudaStreamWaitEvent(c->st3, c->evFork, 0));
    on(c->st3, [&] { mass_block_launch(c, s, cfg.dt, cfg.drop_fict); });
    NL_CUDA(cudaEventRecord(c->evM, c->st3));
  }
  NL_CUDA(cudaStreamWaitEvent(c->st, c->evW, 0));
  if (!resid_only) {
    NL_CUDA(cudaEventRecord(c->evK, c->st));
    NL_CUDA(cudaStreamWaitEvent(c->st2, c->evK, 0));
    on(c->st2, [&] { cubature_phase(c, s, true, false, false, 2); });
  }
  CubSet& sf = c->setCF.n ? c->setCF : s;
  cubature_phase(c, sf, true, false, false, 1);
  // a (+ the vhp seed partials) on the critical path; phi and S_base on st2
  c->agemv = false;
  const bool g = !resid_only && fused_vhp_backward(c, true) && c->wL1 <= 256 && c->ldlast % 2 == 0;
  const int rc = g ? ASMA_GROWS : c->rpc, nch = g ? c->nchAa : c->nchA;
  AsmAArgs A{c->Jt.p, c->ldjt, c->mass.p, c->hvv.p, c->fext.p, c->r.p, c->rbar.p, c->rdbar.p,
             sf.rowptr_full.p, sf.entries.p, sf.fe_w.p, std::max(sf.n, 1), c->a.p, c->partPhi.p,
             c->N, c->n, rc, nch, cfg.dt, c->alpha, cfg.drop_fict,
             (const double*)c->Alast.p, c->ldlast, c->wL1, g ? c->bpart.p : nullptr};
  if (g) launch(c, k_assemble_a<true>, dim3(nch, c->n_sims), 256, 0, A);
  else launch(c, k_assemble_a<false>, dim3(nch, c->n_sims), 256, 0, A);
  c->agemv = g;
  c->nphi = nch;
  // phi on st3 (after the mass block), S_base on st2 (after the stiffness launch and the mass
  // block): the two reductions run concurrently; evJoin2 covers both
  NL_CUDA(cudaEventRecord(c->evFork2, c->st));
  NL_CUDA(cudaStreamWaitEvent(c->st3, c->evFork2, 0));
  on(c->st3, [&] {
    launch(c, k_reduce_phi, c->n_sims, 256, (size_t)8 * c->n * 8, (const double*)c->partPhi.p, c->nphi, c->n,
           c->phi.p, c->norm.p);
  });
  NL_CUDA(cudaEventRecord(c->evP, c->st3));
  if (!resid_only) {
    NL_CUDA(cudaStreamWaitEvent(c->st2, c->evM, 0));  // the mass block partials
    on(c->st2, [&] { reduce_S_launch(c, s, nullptr, cfg.dt); });
  }
  NL_CUDA(cudaStreamWaitEvent(c->st2, c->evP, 0));
  NL_CUDA(cudaEventRecord(c->evJoin2, c->st2));
}

bool split_phase_ok(nlrom_ctx* c) {
  return c->rpc <= 128 && c->n <= 128;
}

void phase_E(nlrom_ctx* c, const nlrom_simcfg& cfg, bool join_side = true, bool resid_only = false) {
  CubSet& s = cfg.integration == 1 ? c->setAll : c->setC;
  bool early_w = cfg.integration == 0 && early_wnet_ok(c) && fused_hidden_forward(c, cfg.dt, cfg.drop_fict);
  if (early_w && split_phase_ok(c)) {
    phase_E_split(c, cfg, s, resid_only);
    if (join_side) NL_CUDA(cudaStreamWaitEvent(c->st, c->evJoin2, 0));
    return;
  }
  if (early_w) {
    NL_CUDA(cudaEventRecord(c->evWf, c->st));
    NL_CUDA(cudaStreamWaitEvent(c->st2, c->evWf, 0));
    std::swap(c->st, c->st2);
    launch(c, k_wnet_head, dim3(wnet_head_split(c), c->n_sims), 256, wnet_head_smem(c->wn / wnet_head_split(c), c->wA1ld),
           (const double*)c->H[c->L - 2].p, c->ldH[c->L - 2], c->Cc,
           (const double*)c->r.p, c->n, c->n_p, c->wL1, (const double*)c->wA1.p, c->wA1ld, c->wn, c->wpart.p);
    const size_t wsm = (size_t)(5 * c->wn + 64 + 2 * c->wn * c->wn + 64 * c->wn + c->wn) * 8;
    launch(c, k_wnet_tail2, dim3(std::max(1, ceil_div(c->n_cub, 64)), c->n_sims), 256, wsm + 16,
           (const double*)c->wpart.p, 1, c->wn, (const double*)c->b1.p, (const double*)c->W2.p,
           (const double*)c->b2.p, (const double*)c->W3.p, (const double*)c->b3.p, (const double*)c->W4C.p,
           (const double*)c->b4C.p, c->n_cub, c->wC.p, c->n_sims);
    std::swap(c->st, c->st2);
    NL_CUDA(cudaEventRecord(c->evW, c->st2));
    output_layer(c);
  } else {
    bundle_forward(c, cfg.dt, cfg.drop_fict);
  }
  if (early_w) {
    NL_CUDA(cudaStreamWaitEvent(c->st, c->evW, 0));
    cubature_phase(c, s, true, false, /*early=*/false);
  } else {
    if (cfg.integration == 0) wnet_phase(c);
    cubature_phase(c, s, cfg.integration == 0, false);  // forces gathered per row by the assembly
  }
  mass_block_fork(c, s, cfg.dt, cfg.drop_fict);
  assemble_phase(c, s, cfg.dt, cfg.drop_fict);
  if (join_side) NL_CUDA(cudaStreamWaitEvent(c->st, c->evJoin2, 0));  // phi, S_base (and the mass block)
}

// vhp backward: dual (NS = 2) passes, cache written by the bundle forward.
// dcache: the caches hold sin'(z) as duals (the fused bundle's forward), not z.
// the batched vhp backward with the real part shared across a sim's passes (EpiBwdShared): only
// when the GEMMs are throughput-bound (>= 4 waves of CTAs in the 2 npass layout): with few CTAs
// (cfg4: 25 per layer) fewer, longer tiles are slower (0.92 vs 0.85 ms)
bool shared_real_bwd(nlrom_ctx* c, int npass_per_sim) {
  const long long ctas2 = (long long)ceil_div(c->n_sims * 2 * npass_per_sim, CfgBig::BN) * ceil_div(c->wL1, CfgBig::BM);
  return c->batched && 1 + npass_per_sim <= CfgBig::BN && (ctas2 >= 4 * 148 || c->opt.shared_real) &&
         !c->opt.no_shared_real;
}

void decoder_backward(nlrom_ctx* c, const double* a_vec, int NS, bool mc, int npass_per_sim, std::vector<DBuf>& caches,
                      std::vector<int>& ldcs, DBuf& D0, DBuf& D1, DBuf& Gout, int ldG, bool dcache = false) {
  const int ncols = c->n_sims * npass_per_sim * NS;
  const int M = c->wL1 + c->next;
  if (c->batched && c->AlastT.p && !c->next) {
    // y (n_sims x w) = a (n_sims x N) (P W_L): one GEMM for all sims. Few output tiles (K = N
    // long): split K over blockIdx.z into [sim][split][M] partials, then a fixed-order reduction.
    const int tiles = ceil_div(M, CfgBig::BM) * ceil_div(c->n_sims, CfgBig::BN);
    int split = 1;
    for (int sp : {16, 12, 10, 8, 6, 5, 4, 3, 2})
      if (tiles * sp <= 2 * 148 * 2 && c->N % sp == 0 && (c->N / sp) % 2 == 0 && c->N / sp >= 64 &&
          (size_t)c->n_sims * sp * M <= c->bpart.n) {
        split = sp;
        break;
      }
    if (tiles >= 148) split = 1;
    if (split == 1) {
      GemmArgs g{c->AlastT.p, a_vec, c->ldAT, c->N, M, c->n_sims, c->N, 0, 0};
      launch_gemm<CfgBig>(g, EpiStore{c->ybuf.p, M, 0, nullptr, 1, nullptr}, c->st);
    } else {
      const int Kc = c->N / split;
      GemmArgs g{c->AlastT.p, a_vec, c->ldAT, c->N, M, c->n_sims, Kc, Kc, Kc};
      launch_gemm<CfgBig>(g, EpiStore{c->bpart.p, split * M, M, nullptr, 1, nullptr}, c->st, split);
      launch(c, k_reduce_cols, dim3(ceil_div(M, 32), c->n_sims), 256, 0, (const double*)c->bpart.p, split, M,
             c->ybuf.p);
    }
    ++gemm_launch_count;
  } else {
    launch(c, k_gemv_t, dim3(c->bnch, c->n_sims), 128, 0, (const double*)c->Alast.p, c->ldlast, M, a_vec, c->N,
           c->brows, c->bpart.p, c->bnch);
    launch(c, k_reduce_cols, dim3(ceil_div(M, 32), c->n_sims), 256, 0, (const double*)c->bpart.p, c->bnch, M,
           c->ybuf.p);
  }
  const int l_top = c->L - 2;
  dim3 gd(ceil_div(c->wL1, 32), c->n_sims);
  const int P1 = 1 + npass_per_sim;
  if (NS == 2 && !mc && dcache && shared_real_bwd(c, npass_per_sim)) {
    // shared real part (EpiBwdShared): 1 + npass columns per sim instead of 2 npass, tiles of
    // whole sims
    const int cstep = (CfgBig::BN / P1) * P1, ncs = c->n_sims * P1;
    launch(c, k_bwd_delta_sh, gd, 256, 0, (const double*)c->ybuf.p, c->wL1, c->next, (const double*)c->AT.p,
           (const double*)caches[l_top].p, ldcs[l_top], npass_per_sim, D0.p);
    DBuf* cur = &D0;
    DBuf* nxt = &D1;
    // tcgen05 Ozaki layers (ozaki_tc.cuh): 64-column tiles of whole sims; each layer's epilogue
    // writes the next Ozaki layer's column-scale partials (the first one scans its input)
    const int ocs = (64 / P1) * P1;
    auto oz_bwd = [&](int l) {
      return l >= 1 && l < (int)c->ozWT.size() && c->ozWT[l].ready && ocs >= P1 && ldcs[l] % 2 == 0 &&
             c->ozBHW[0] != nullptr && oz_enough_tiles(c->widths[l], ncs, ocs);
    };
    for (int l = c->L - 2; l >= 1; --l) {
      if (oz_bwd(l)) {
        GemmArgs g{c->WT[l].p, cur->p, c->ldWT[l], ldcs[l], c->widths[l], ncs, c->widths[l + 1], 0, 0, ocs};
        const bool from_oz = oz_bwd(l + 1) && l + 1 <= c->L - 2;
        const OzakiBExp be = from_oz ? OzakiBExp{c->ozBHW[(l + 1) & 1], c->widths[l + 1] / 32} : OzakiBExp{nullptr, 0};
        EpiBwdShared e{nxt->p, ldcs[l - 1], caches[l - 1].p, npass_per_sim};
        if (oz_bwd(l - 1) && c->widths[l] % 32 == 0) e.colhw = c->ozBHW[l & 1];
        launch_ozaki<64>(c->ozWT[l].view(), be, g, e, c->st);
        ++gemm_launch_count;
        std::swap(cur, nxt);
        continue;
      }
      GemmArgs g{c->WT[l].p, cur->p, c->ldWT[l], ldcs[l], c->widths[l], ncs, c->widths[l + 1], 0, 0, cstep};
      // warp-specialised TMA pipeline with sim-aligned column tiles: cfg5 vhp 5.14 -> 4.77 ms
      if (!c->opt.bwd_cp && c->widths[l + 1] % 16 == 0 && c->ldWT[l] % 2 == 0 && ldcs[l] % 2 == 0)
        launch_gemm_ws<WsCfg<64, 128, 4, 4, 4>>(g, EpiBwdShared{nxt->p, ldcs[l - 1], caches[l - 1].p, npass_per_sim},
                                                c->st);
      else
        launch_gemm<CfgBig>(g, EpiBwdShared{nxt->p, ldcs[l - 1], caches[l - 1].p, npass_per_sim}, c->st);
      ++gemm_launch_count;
      std::swap(cur, nxt);
    }
    GemmArgs g{c->WT[0].p, cur->p, c->ldWT[0], ldcs[0], c->widths[0], ncs, c->widths[1], 0, 0, cstep};
    if (c->widths[0] <= 24 && c->widths[1] % 16 == 0) launch_gemm<CfgBwdLast>(g, EpiStoreShared{Gout.p, ldG, npass_per_sim}, c->st);
    else launch_gemm<CfgBig>(g, EpiStoreShared{Gout.p, ldG, npass_per_sim}, c->st);
    ++gemm_launch_count;
    return;
  }
  if (NS == 2) {
    if (mc)
      launch(c, k_bwd_delta<2, 1>, gd, 256, 0, (const double*)c->ybuf.p, c->wL1, c->next, (const double*)c->AT.p,
             (const double*)caches[l_top].p, ldcs[l_top], npass_per_sim, D0.p);
    else if (dcache)
      launch(c, k_bwd_delta<2, 2>, gd, 256, 0, (const double*)c->ybuf.p, c->wL1, c->next, (const double*)c->AT.p,
             (const double*)caches[l_top].p, ldcs[l_top], npass_per_sim, D0.p);
    else
      launch(c, k_bwd_delta<2, 0>, gd, 256, 0, (const double*)c->ybuf.p, c->wL1, c->next, (const double*)c->AT.p,
             (const double*)caches[l_top].p, ldcs[l_top], npass_per_sim, D0.p);
  } else {
    launch(c, k_bwd_delta<1, 1>, gd, 256, 0, (const double*)c->ybuf.p, c->wL1, c->next, (const double*)c->AT.p,
           (const double*)caches[l_top].p, ldcs[l_top], npass_per_sim, D0.p);
  }
  DBuf* cur = &D0;
  DBuf* nxt = &D1;
  for (int l = c->L - 2; l >= 1; --l) {
    // delta_{l-1} = (W_l^T Delta_l) * act'(z_{l-1})
    GemmArgs g{c->WT[l].p, cur->p, c->ldWT[l], ldcs[l], c->widths[l], ncols, c->widths[l + 1], 0, 0};
    if (NS == 2) {
      if (mc) launch_gemm<CfgBwd>(g, EpiBwdAct<2, ACT_SIN_MC>{nxt->p, ldcs[l - 1], 0, caches[l - 1].p}, c->st);
      else if (dcache && c->batched)
        launch_gemm<CfgBig>(g, EpiBwdAct<2, ACT_DSIN_MD>{nxt->p, ldcs[l - 1], 0, caches[l - 1].p}, c->st);
      else if (dcache)
        launch_gemm<CfgBwd>(g, EpiBwdAct<2, ACT_DSIN_MD>{nxt->p, ldcs[l - 1], 0, caches[l - 1].p}, c->st);
      else if (c->batched) launch_gemm<CfgBig>(g, EpiBwdAct<2, ACT_SIN_MD>{nxt->p, ldcs[l - 1], 0, caches[l - 1].p}, c->st);
      else launch_gemm<CfgBwd>(g, EpiBwdAct<2, ACT_SIN_MD>{nxt->p, ldcs[l - 1], 0, caches[l - 1].p}, c->st);
    } else {
      launch_gemm<CfgBwd>(g, EpiBwdAct<1, ACT_SIN_MC>{nxt->p, ldcs[l - 1], 0, caches[l - 1].p}, c->st);
    }
    ++gemm_launch_count;
    std::swap(cur, nxt);
  }
  GemmArgs g{c->WT[0].p, cur->p, c->ldWT[0], ldcs[0], c->widths[0], ncols, c->widths[1], 0, 0};
  if (c->batched) launch_gemm<CfgBig>(g, EpiStore{Gout.p, ldG, 0, nullptr, 1, nullptr}, c->st);
  else launch_gemm<CfgBwd>(g, EpiStore{Gout.p, ldG, 0, nullptr, 1, nullptr}, c->st);
  ++gemm_launch_count;
}

// Fused vhp backward chain (mlp_chain.cuh): g = (P W_L)^T a, then one cluster per 8 passes.
template <int R, int CS, int G = 16>
bool launch_mlp_bwd(nlrom_ctx* c, MlpBwdArgs a, int dry) {
  a.gpb = ceil_div(c->n_q, G / 2);
  const int groups = c->n_sims * a.gpb;
  const size_t smem = mlp_bwd_smem<R, G>(c->wL1);
  if (smem > 227 * 1024) return false;
  if (dry) return true;
  static bool configured = false;
  if (!configured) {
    NL_CUDA(cudaFuncSetAttribute(k_mlp_dual_bwd<R, CS, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (CS > 8)
      NL_CUDA(cudaFuncSetAttribute(k_mlp_dual_bwd<R, CS, G>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    configured = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, groups, 1);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  if (!launch_gate((const void*)k_mlp_dual_bwd<R, CS, G>)) return true;
  NL_CUDA(cudaLaunchKernelEx(&cfg, k_mlp_dual_bwd<R, CS, G>, a));
  ++gemm_launch_count;
  return true;
}

// check_only: report whether the fused chain applies (nothing launched)
bool fused_vhp_backward(nlrom_ctx* c, bool check_only) {
  if (c->opt.unfused || c->next || c->batched) return false;
  const int L1 = c->L - 1, w = c->wL1;
  if (L1 < 1 || L1 > MLP_MAXL) return false;
  for (int l = 1; l <= L1; ++l)
    if (c->widths[l] != w) return false;
  const int M = w;
  MlpBwdArgs a{};
  a.g = c->ybuf.p; a.L1 = L1; a.w = w; a.n_q = c->n_q;
  for (int l = 0; l < L1; ++l) {
    a.WT[l] = c->WT[l].p; a.ldWT[l] = c->ldWT[l]; a.cache[l] = c->cache[l].p;
    a.WTp[l] = c->WTp[l].p;
  }
  a.ldc = c->ldc[0]; a.Gt = c->Gt.p; a.ldG = c->ldGt;
  a.ldpb = c->ldpb;
  if (c->ldpb != round_up(w, 16) + 4) return false;
  auto go = [&](bool dry) -> bool {
    if (w == 256) {
      // 4 dual passes (8 columns) per 8-CTA cluster halve the DSMEM bytes each CTA broadcasts per
      // stage relative to 8 passes on 16-CTA clusters (the stage is broadcast-bound)
      return launch_mlp_bwd<32, 8, 8>(c, a, dry);
    }
    if (w == 64) return launch_mlp_bwd<8, 8>(c, a, dry);
    if (w == 40) return launch_mlp_bwd<8, 5>(c, a, dry);
    if (w == 8) return launch_mlp_bwd<8, 1>(c, a, dry);
    return false;
  };
  if (!go(true)) return false;
  if (check_only) return true;
  if (c->agemv) {
    // seed partials already formed by k_assemble_a (32-row chunks)
    a.gpart = c->bpart.p;
    a.gnch = c->nchAa;
  } else if (M % 2 == 0 && c->ldlast % 2 == 0 && M <= 512) {
    // 24-row chunks over ~280 CTAs; the chain's prologue sums the partials (no reduce launch)
    const int rows = 24, nch = ceil_div(c->N, rows);
    launch(c, k_gemv_t2, dim3(nch, c->n_sims), 256, 0, (const double*)c->Alast.p, c->ldlast, M,
           (const double*)c->a.p, c->N, rows, c->bpart.p, nch);
    a.gpart = c->bpart.p;
    a.gnch = nch;
  } else {
    launch(c, k_gemv_t, dim3(c->bnch, c->n_sims), 128, 0, (const double*)c->Alast.p, c->ldlast, M,
           (const double*)c->a.p, c->N, c->brows, c->bpart.p, c->bnch);
    launch(c, k_reduce_cols, dim3(ceil_div(M, 32), c->n_sims), 256, 0, (const double*)c->bpart.p, c->bnch, M,
           c->ybuf.p);
  }
  return go(false);
}

// In-CTA LU-pp solve of every sim's Eq. 11 system; register block sized to n + 1.
// Extra right-hand sides (xrhs, nx columns of n per sim) are solved alongside -phi into xout.
void launch_lu(nlrom_ctx* c, bool apply, const double* xrhs = nullptr, int nx = 0, double* xout = nullptr,
               bool add_vhp = false) {
  const int n = c->n;
  const double* Gt = add_vhp ? (const double*)c->Gt.p : nullptr;
  auto go = [&](auto kern) {
    launch(c, kern, c->n_sims, 256, lu_lookahead_smem_bytes(n + nx, c->n_q), (const double*)c->S.p,
           (const double*)c->phi.p, c->dr.p, c->r.p, n, apply ? 1 : 0, c->status.p, xrhs, nx, xout, Gt, c->ldGt,
           c->n_p);
  };
  // One warp owns the pivot chain (4-column panels in registers, the next panel brought up to date
  // by the same warp), 7 warps apply the trailing updates: bitwise equal to the one-barrier-per-pivot
  // k_lu_solve; as fast at n = 60, 10-35% faster at n = 70..124 (tools/probes/lu_blocked_probe.cu,
  // profiles/r02_lu_probe.txt). Retired variants (warp-register, column-cyclic, rank-2, look-ahead
  // pivot, split front/back, k_lu_blocked): DESIGN.md §8b, tools/probes/retired/
  if (c->n_sims > 1 && nx == 0 && n <= 32) {   // many small systems: a warp per system (k_lu_warp)
    launch(c, k_lu_warp, ceil_div(c->n_sims, 8), 256, 0, (const double*)c->S.p, (const double*)c->phi.p, c->dr.p,
           c->r.p, n, apply ? 1 : 0, c->status.p, Gt, c->ldGt, c->n_p, c->n_sims);
    return;
  }
  switch (lu_nb(n + nx)) {
    case 4: go(k_lu_lookahead<4>); break;
    case 6: go(k_lu_lookahead<6>); break;
    default: go(k_lu_lookahead<8>); break;
  }
}

// side_open: phase E left its phi / S_base branch unjoined (captured in the same graph)
void phase_J(nlrom_ctx* c, const nlrom_simcfg& cfg, bool apply, const double* xrhs = nullptr, int nx = 0,
             double* xout = nullptr, bool side_open = false) {
  if (!fused_vhp_backward(c, false))
    decoder_backward(c, c->a.p, 2, false, c->n_q, c->cache, c->ldc, c->Delta0, c->Delta1, c->Gt, c->ldGt, true);
  if (side_open) NL_CUDA(cudaStreamWaitEvent(c->st, c->evJoin2, 0));  // S_base, phi from phase E's branch
  launch_lu(c, apply, xrhs, nx, xout, true);  // S = S_base + diag(0, vhp) while staging
}

// S with the vhp block (system_jacobian API; the Newton iteration adds it inside the LU)
void full_S(nlrom_ctx* c, const nlrom_simcfg& cfg) {
  CubSet& s = cfg.integration == 1 ? c->setAll : c->setC;
  reduce_S_launch(c, s, c->Gt.p, cfg.dt);
}

std::string cfg_key(const nlrom_simcfg& cfg) {
  char buf[128];
  snprintf(buf, sizeof buf, "%.17g|%d|%d", cfg.dt, cfg.drop_fict, cfg.integration);
  return buf;
}

cudaGraphExec_t capture(nlrom_ctx* c, const std::function<void()>& body, int* count) {
  gemm_launch_count = 0;
  cudaGraph_t g;
  NL_CUDA(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaStreamEndCapture(c->st, &g);
    throw;
  }
  NL_CUDA(cudaStreamEndCapture(c->st, &g));
  cudaGraphExec_t ex;
  NL_CUDA(cudaGraphInstantiate(&ex, g, 0));
  cudaGraphDestroy(g);
  if (count) *count = gemm_launch_count;
  return ex;
}

void ensure_graphs(nlrom_ctx* c, const nlrom_simcfg& cfg) {
  std::string key = cfg_key(cfg);
  if (key == c->graph_key && c->gE) return;
  if (c->gE) cudaGraphExecDestroy(c->gE);
  if (c->gJ) cudaGraphExecDestroy(c->gJ);
  if (c->gIter) cudaGraphExecDestroy(c->gIter);
  if (c->gStep) cudaGraphExecDestroy(c->gStep);
  c->gE = c->gJ = c->gIter = c->gStep = nullptr;
  c->step_key.clear();
  // eager warm-up (sets kernel attributes outside of capture)
  phase_E(c, cfg);
  phase_J(c, cfg, false);
  NL_CUDA(cudaStreamSynchronize(c->st));
  c->gE = capture(c, [&] { phase_E(c, cfg); }, &c->launches_E);
  c->gJ = capture(c, [&] { phase_J(c, cfg, false); }, &c->launches_J);
  c->gIter = capture(c, [&] { phase_E(c, cfg, false); phase_J(c, cfg, true, nullptr, 0, nullptr, true); }, nullptr);
  c->graph_key = key;
}

void upload(DBuf& d, const double* h, size_t n) {
  d.alloc(n);
  if (n) {
    NL_CUDA(cudaMemcpy(d.p, h, n * 8, cudaMemcpyHostToDevice));
    // a pageable H2D returns once staged; the legacy stream does not order against the contexts'
    // non-blocking streams, so wait for the DMA before kernels there may read the buffer
    NL_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
  }
}

void h2d(nlrom_ctx* c, DBuf& d, const double* h, size_t n) {
  NL_CUDA(cudaMemcpyAsync(d.p, h, n * 8, cudaMemcpyHostToDevice, c->st));
}
void d2h(nlrom_ctx* c, double* h, const DBuf& d, size_t n) {
  NL_CUDA(cudaMemcpyAsync(h, d.p, n * 8, cudaMemcpyDeviceToHost, c->st));
}

void set_state(nlrom_ctx* c, const double* r, const double* rbar, const double* rdbar, const double* fext) {
  const size_t nn = (size_t)c->n_sims * c->n;
  if (r) h2d(c, c->r, r, nn);
  if (rbar) h2d(c, c->rbar, rbar, nn);
  if (rdbar) h2d(c, c->rdbar, rdbar, nn);
  if (fext) h2d(c, c->fext, fext, (size_t)c->n_sims * c->N);
}

void check_status(nlrom_ctx* c) {
  std::vector<int> st(c->n_sims);
  NL_CUDA(cudaMemcpyAsync(st.data(), c->status.p, c->n_sims * sizeof(int), cudaMemcpyDeviceToHost, c->st));
  NL_CUDA(cudaStreamSynchronize(c->st));
  for (int s : st)
    if (s) throw Error(NLROM_ERR_NONFINITE, "singular system Jacobian (zero pivot in LU)");
}

}  // namespace

// =========================================================================== C ABI

extern "C" int nlrom_create(nlrom_ctx** out, int device, const nlrom_model_desc* d) {
  nlrom_ctx* c = nullptr;
  try {
    if (!out || !d) throw Error(NLROM_ERR_ARG, "null argument");
    if (d->n_fc < 2) throw Error(NLROM_ERR_ARG, "decoder needs >= 2 FC layers");
    if (d->widths[0] != d->n_q || d->widths[d->n_fc] != d->N) throw Error(NLROM_ERR_DIM, "decoder widths do not match (n_q, N)");
    NL_CUDA(cudaSetDevice(device));
    c = new nlrom_ctx();
    c->device = device;
    c->opt = PathOpts::from_env();
    NL_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    NL_CUDA(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
    NL_CUDA(cudaStreamCreateWithFlags(&c->st3, cudaStreamNonBlocking));
    NL_CUDA(cudaEventCreateWithFlags(&c->evFork, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreateWithFlags(&c->evJoin, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreateWithFlags(&c->evFork2, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreateWithFlags(&c->evJoin2, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreateWithFlags(&c->evWf, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreateWithFlags(&c->evW, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreateWithFlags(&c->evK, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreateWithFlags(&c->evM, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreateWithFlags(&c->evP, cudaEventDisableTiming));
    NL_CUDA(cudaEventCreate(&c->ev0));
    NL_CUDA(cudaEventCreate(&c->ev1));
    c->n_sims = d->n_sims > 0 ? d->n_sims : 1;
    c->N = d->N; c->n_p = d->n_p; c->n_q = d->n_q; c->n = d->n_p + d->n_q; c->L = d->n_fc;
    c->T = d->n_tets; c->V = d->n_verts;
    c->mu = d->mu; c->lam = d->lambda; c->alpha = d->alpha;
    c->widths.assign(d->widths, d->widths + d->n_fc + 1);
    const int N = c->N, n_p = c->n_p, n_q = c->n_q, L = c->L;
    c->wL1 = c->widths[L - 1];
    // hidden FC layers 0..L-2 and their transposes
    c->W.resize(L); c->WT.resize(L); c->b.resize(L); c->ldW.resize(L); c->ldWT.resize(L);
    for (int l = 0; l < L - 1; ++l) {
      int in = c->widths[l], o = c->widths[l + 1];
      c->ldW[l] = round_up(in, 2);
      c->ldWT[l] = round_up(o, 2);
      upload_matrix(c->W[l], d->W[l], o, in, c->ldW[l]);
      std::vector<double> wt((size_t)in * o);
      for (int r = 0; r < o; ++r)
        for (int k = 0; k < in; ++k) wt[(size_t)k * o + r] = d->W[l][(size_t)r * in + k];
      upload_matrix(c->WT[l], wt.data(), in, o, c->ldWT[l]);
      upload(c->b[l], d->b[l], o);
    }
    {  // padded copies for the fused chains: W_l as (w x ldpf), W_l^T as (w x ldpb), zero padded
      int kmax = n_q;
      for (int l = 1; l < L; ++l) kmax = std::max(kmax, c->widths[l]);
      c->ldpf = round_up(kmax, 16) + 4;
      c->ldpb = round_up(c->wL1, 16) + 4;
      c->Wp.resize(L - 1);
      c->WTp.resize(L - 1);
      for (int l = 0; l < L - 1; ++l) {
        const int in = c->widths[l], o = c->widths[l + 1];
        const int rows = std::max(o, kmax);
        std::vector<double> wp((size_t)rows * c->ldpf, 0.0), wtp((size_t)std::max(rows, in) * c->ldpb, 0.0);
        for (int r = 0; r < o; ++r)
          for (int k = 0; k < in; ++k) {
            wp[(size_t)r * c->ldpf + k] = d->W[l][(size_t)r * in + k];
            if (o <= c->ldpb - 4) wtp[(size_t)k * c->ldpb + r] = d->W[l][(size_t)r * in + k];
          }
        upload(c->Wp[l], wp.data(), wp.size());
        upload(c->WTp[l], wtp.data(), wtp.size());
      }
    }
    std::vector<double> PWL_host, PbL_host;  // P W_L (N x w), P b_L (N): also fold the weight net's layer 1
    // last layer fused with the filter: D = P (W_L h + b_L) = (P W_L) h + P b_L with
    // P = I - U U^T folded into the weights once at upload (no filter GEMM per iteration).
    const double* WL = d->W[L - 1];
    const double* bL = d->b[L - 1];
    const int w = c->wL1;
    c->next = 0;
    c->ldlast = round_up(w, 2);
    {
      std::vector<double>& Pbh = PbL_host;
      std::vector<double>& A = PWL_host;
      Pbh.assign(N, 0.0);
      A.assign((size_t)N * w, 0.0);
      std::vector<double> ATh((size_t)n_p * w, 0.0), Utb(n_p, 0.0);
      for (int r = 0; r < N; ++r)
        for (int j = 0; j < n_p; ++j) {
          const double ur = d->U[(size_t)r * n_p + j];
          Utb[j] += ur * bL[r];
          for (int k = 0; k < w; ++k) ATh[(size_t)j * w + k] += ur * WL[(size_t)r * w + k];
        }
      for (int r = 0; r < N; ++r) {
        double s = bL[r];
        for (int j = 0; j < n_p; ++j) s -= d->U[(size_t)r * n_p + j] * Utb[j];
        Pbh[r] = s;
        for (int k = 0; k < w; ++k) {
          double a = WL[(size_t)r * w + k];
          for (int j = 0; j < n_p; ++j) a -= d->U[(size_t)r * n_p + j] * ATh[(size_t)j * w + k];
          A[(size_t)r * w + k] = a;
        }
      }
      upload_matrix(c->Alast, A.data(), N, w, c->ldlast);
      // (K = w >= 128: at cfg4's w = 64 the two-chunk K loop leaves the Ozaki tile overhead-bound,
      // 0.94 vs 0.82 ms per coupled iteration with the DMMA output layer)
      if ((c->n_sims * (4 + 4 * n_q) >= 2048 || c->opt.batched) && !c->opt.dmma_hidden && !c->opt.dmma_out &&
          w % oz::BK == 0 && w >= 128 && w <= 256)
        ozaki_upload(c->ozWL, A.data(), w, N, w);
      if (c->n_sims > 1) {
        std::vector<double> At((size_t)w * N);
        for (int r = 0; r < N; ++r)
          for (int k = 0; k < w; ++k) At[(size_t)k * N + r] = A[(size_t)r * w + k];
        c->ldAT = round_up(N, 2);
        upload_matrix(c->AlastT, At.data(), w, N, c->ldAT);
      }
      upload_matrix(c->AT, ATh.data(), n_p, w, round_up(w, 2));
      upload(c->Pb, Pbh.data(), N);
      upload(c->U, d->U, (size_t)N * n_p);
      upload(c->mass, d->mass, N);
    }
    // mesh
    {
      std::vector<int> rows((size_t)c->T * 12);
      for (int e = 0; e < c->T; ++e)
        for (int v = 0; v < 4; ++v) {
          int dv = d->vert_dof[d->tets[(size_t)e * 4 + v]];
          for (int a = 0; a < 3; ++a) rows[(size_t)e * 12 + v * 3 + a] = dv >= 0 ? 3 * dv + a : -1;
        }
      c->elem_rows.upload(rows.data(), rows.size());
      upload(c->Dm_inv, d->Dm_inv, (size_t)c->T * 9);
      upload(c->vol, d->vol, c->T);
      std::vector<int> cub(d->cub_elems, d->cub_elems + d->n_cub), all(c->T);
      for (int e = 0; e < c->T; ++e) all[e] = e;
      // cubature set: 2 elements per CTA (250 CTAs for |C| = 500); the all-element set of the
      // exact-sum mode (not the hot path): 8, keeping its per-chunk partials small
      // many sims (batched): 8 elements per CTA keeps the per-chunk partials (and their reduction) small
      const bool many = c->n_sims * (4 + 4 * c->n_q) >= 2048 || c->opt.batched;
      // split phase E (default): the stiffness / Gram launch is off the critical path, where fewer,
      // longer chunks win (12 elements per CTA: fewer K~ partials to reduce); the force-only launch
      // on the critical path keeps 2 per CTA (setCF)
      const bool split = !many;
      build_set(c, c->setC, cub, rows, many ? 8 : 12,
                d->Dm_inv, d->vol, many ? d->U : nullptr);
      if (split)
        build_set(c, c->setCF, cub, rows, 6, d->Dm_inv, d->vol);
      build_set(c, c->setAll, all, rows, 8, d->Dm_inv, d->vol, many ? d->U : nullptr);
    }
    // weight net (rows of the last layer restricted to C)
    {
      c->wn = d->wnet_width;
      c->n_cub = d->n_cub;
      const int wn = c->wn;
      upload_matrix(c->W1, d->wnet_W[0], wn, N, round_up(N, 2));
      upload(c->b1, d->wnet_b[0], wn);
      upload(c->W2, d->wnet_W[1], (size_t)wn * wn);
      upload(c->b2, d->wnet_b[1], wn);
      upload(c->W3, d->wnet_W[2], (size_t)wn * wn);
      upload(c->b3, d->wnet_b[2], wn);
      std::vector<double> w4((size_t)std::max(1, c->n_cub) * wn), b4(std::max(1, c->n_cub));
      for (int j = 0; j < c->n_cub; ++j) {
        int e = d->cub_elems[j];
        if (e < 0 || e >= c->T) throw Error(NLROM_ERR_ARG, "cubature element id out of range");
        for (int k = 0; k < wn; ++k) w4[(size_t)j * wn + k] = d->wnet_W[3][(size_t)e * wn + k];
        b4[j] = d->wnet_b[3][e];
      }
      upload(c->W4C, w4.data(), w4.size());
      upload(c->b4C, b4.data(), b4.size());
      // layer 1 of the weight net on u = U p + P (W_L h + b_L) folded onto the
      // last hidden activation h and p: W1 u = (W1 P W_L) h + (W1 U) p + W1 P b_L, a wn x (w + n_p + 1)
      // matrix formed once -- the weight net then needs only the hidden chain, not the output layer
      if (!PWL_host.empty()) {
        const int wL = c->wL1;
        c->wA1ld = round_up(wL + n_p + 1, 2);
        std::vector<double> F((size_t)wn * c->wA1ld, 0.0);
        for (int o = 0; o < wn; ++o) {
          double* Fo = F.data() + (size_t)o * c->wA1ld;
          const double* W1o = d->wnet_W[0] + (size_t)o * N;
          for (int r = 0; r < N; ++r) {
            const double wv = W1o[r];
            const double* Ar = PWL_host.data() + (size_t)r * wL;
            for (int k = 0; k < wL; ++k) Fo[k] += wv * Ar[k];
            for (int j = 0; j < n_p; ++j) Fo[wL + j] += wv * d->U[(size_t)r * n_p + j];
            Fo[wL + n_p] += wv * PbL_host[r];
          }
        }
        upload(c->wA1, F.data(), F.size());
      }
      c->wchunk = round_up(std::max(32, ceil_div(N, 148)), 32);
      c->wsplit = ceil_div(N, c->wchunk);
      c->wpart.alloc((size_t)c->wsplit * c->n_sims * wn);
      if (c->n_sims * (4 + 4 * n_q) >= 2048 || c->opt.batched)   // the batched path (c->batched, below)
        c->wsk.alloc((size_t)16 * c->n_sims * wn);
      c->wC.alloc((size_t)c->n_sims * std::max(1, c->n_cub));
    }
    // bundle buffers
    c->Cc = 2 + 2 * n_q;  // output-layer columns per sim: [D_1, 2 D_ss | (D_t, 2 D_tss + D_tr) x n_q]
    c->batched = c->n_sims * (4 + 4 * n_q) >= 2048 || c->opt.batched;
    choose_groups(n_q, w, c->batched, c->opt.tangents, c->G, c->gps);
    c->Cb = c->G * c->gps;
    if (c->batched && !c->opt.dmma_hidden) {
      // hidden layers 1 .. L-2 (K = w) as int8 digit tiles for the tcgen05 Ozaki GEMM
      c->ozW.resize(L - 1);
      int maxw = 0;
      for (int l = 1; l < L - 1; ++l) {
        const int in = c->widths[l], o = c->widths[l + 1];
        if (o % oz::BM == 0 && in % oz::BK == 0 && in <= 256) ozaki_upload(c->ozW[l], d->W[l], in, o, in);
        maxw = std::max(maxw, in);
      }
      const size_t hwn = (size_t)c->n_sims * c->Cb * (size_t)ceil_div(std::max(maxw, c->wL1), 32);
      for (auto& p : c->ozHW) NL_CUDA(cudaMalloc(&p, std::max<size_t>(hwn, 1) * sizeof(unsigned)));
      for (auto& p : c->ozDE) NL_CUDA(cudaMalloc(&p, (size_t)round_up(c->n_sims * c->Cb, 64) * sizeof(int)));
      if (!c->opt.dmma_bwd) {
        // shared-real vhp backward layers 1 .. L-2: W_l^T (widths[l] x widths[l+1]) as digit tiles
        c->ozWT.resize(L - 1);
        for (int l = 1; l < L - 1; ++l) {
          const int in = c->widths[l], o = c->widths[l + 1];   // W_l^T: M = in, K = o
          if (in % oz::BM == 0 && o % oz::BK == 0 && o <= 256) {
            std::vector<double> wt((size_t)in * o);
            for (int r = 0; r < o; ++r)
              for (int k = 0; k < in; ++k) wt[(size_t)k * o + r] = d->W[l][(size_t)r * in + k];
            ozaki_upload(c->ozWT[l], wt.data(), o, in, o);
          }
        }
        const size_t bhw = (size_t)c->n_sims * (1 + n_q) * (size_t)ceil_div(maxw, 32);
        for (auto& p : c->ozBHW) NL_CUDA(cudaMalloc(&p, std::max<size_t>(bhw, 1) * sizeof(unsigned)));
      }
    }
    c->ldq = round_up(n_q, 2);
    const int ncols = c->n_sims * c->Cb;
    c->X0.alloc((size_t)ncols * c->ldq);
    c->H.resize(L - 1); c->cache.resize(L - 1); c->ldH.resize(L - 1); c->ldc.resize(L - 1);
    for (int l = 0; l < L - 1; ++l) {
      c->ldH[l] = (l == L - 2) ? c->ldlast : round_up(c->widths[l + 1], 2);
      c->ldc[l] = round_up(c->widths[l + 1], 2);
      c->H[l].alloc((size_t)std::max(ncols, c->n_sims * c->Cc) * c->ldH[l]);
      c->cache[l].alloc((size_t)c->n_sims * 2 * n_q * c->ldc[l]);
    }
    c->ldjt = gram_ld(c->n);  // J~ rows pitched like the Gram panels: one TMA copy per row chunk
    c->lddj = n_q;
    c->u.alloc((size_t)c->n_sims * N);
    c->value.alloc((size_t)c->n_sims * N);
    c->hvv.alloc((size_t)c->n_sims * N);
    c->Jt.alloc((size_t)c->n_sims * N * c->ldjt);
    c->dJ.alloc((size_t)c->n_sims * N * c->lddj);
    {  // constant U block of J~
      std::vector<double> jt((size_t)N * c->ldjt, 0.0);
      for (int r = 0; r < N; ++r)
        for (int j = 0; j < n_p; ++j) jt[(size_t)r * c->ldjt + j] = d->U[(size_t)r * n_p + j];
      for (int s = 0; s < c->n_sims; ++s)
        NL_CUDA(cudaMemcpy(c->Jt.p + (size_t)s * N * c->ldjt, jt.data(), jt.size() * 8, cudaMemcpyHostToDevice));
    }
    // assembly / solve
    while (c->rpc > 16 && (size_t)(2 * c->rpc * gram_ld(c->n) + 2 * c->rpc + c->n) * 8 > 200 * 1024) c->rpc /= 2;
    c->nchA = ceil_div(N, c->rpc);
    c->rpcM = c->rpc;
    if (c->ldjt == gram_ld(c->n) && c->lddj % 2 == 0) {
      c->rpcM = 64;
      while (c->rpcM > 16 && mass_smem(c) > 200 * 1024) c->rpcM /= 2;
    }
    c->nchM = ceil_div(N, c->rpcM);
    if (c->ldjt == gram_ld(c->n) && c->lddj % 2 == 0 && (c->n_sims > 1 || c->opt.cpm > 0)) {
      // many sims: a CTA walks several row chunks of its sim (>= ~2 waves of 2 CTAs per SM)
      const int rows_ch = c->nchM;
      // (at most a third of a sim's chunks per CTA: cfg5 0.574 -> 0.547 ms with 5 of 15)
      c->cpmM = (int)std::max(1LL, std::min<long long>(ceil_div(rows_ch, 3), (long long)c->n_sims * rows_ch / (148 * 2 * 2)));
      if (c->opt.cpm > 0) c->cpmM = std::max(1, std::min(rows_ch, c->opt.cpm));
      if (mass_smem(c) > 200 * 1024) c->cpmM = 1;
      c->nchM = ceil_div(rows_ch, c->cpmM);
    }
    const int n = c->n, S = c->n_sims;
    c->a.alloc((size_t)S * N);
    c->partA.alloc((size_t)S * std::max(c->nchA, c->nchM) * n * n);
    c->nchAa = ceil_div(N, ASMA_GROWS);
    c->partPhi.alloc((size_t)S * std::max(c->nchA, c->nchAa) * n);
    c->phi.alloc((size_t)S * n);
    c->norm.alloc(S);
    c->S.alloc((size_t)S * n * n);
    c->dr.alloc((size_t)S * n);
    c->r.alloc((size_t)S * n);
    c->rbar.alloc((size_t)S * n);
    c->rdbar.alloc((size_t)S * n);
    c->rsave.alloc((size_t)S * n);
    c->rdot.alloc((size_t)S * n);
    c->fext.alloc((size_t)S * N);
    c->tmpN.alloc((size_t)S * N);
    c->status.alloc(S);
    // backward
    if (w + n_p > 512) throw Error(NLROM_ERR_ARG, "last hidden width + n_p must be <= 512");
    c->bnch = ceil_div(N, c->brows);
    c->bpart.alloc((size_t)std::max(c->bnch, ceil_div(N, 8)) * S * (w + n_p));
    c->ybuf.alloc((size_t)S * (w + n_p));
    int maxw = 0;
    for (int l = 1; l < L; ++l) maxw = std::max(maxw, round_up(c->widths[l], 2));
    c->Delta0.alloc((size_t)S * 2 * n_q * maxw);
    c->Delta1.alloc((size_t)S * 2 * n_q * maxw);
    c->ldGt = round_up(n_q, 2);
    c->Gt.alloc((size_t)S * 2 * n_q * c->ldGt);
    // kernel attributes for large dynamic shared memory
    NL_CUDA(cudaFuncSetAttribute(k_cubature<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_cubature<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_seed_layer<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_seed_layer<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_cub_sims<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_cub_sims<2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_cub_sims<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_cub_sims<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_wnet_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_wnet_tail2, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_assemble_mass, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_lu_lookahead<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_lu_lookahead<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_lu_lookahead<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_lu_solve<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_lu_solve<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_lu_solve<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    NL_CUDA(cudaFuncSetAttribute(k_wnet_head, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    if (c->n + 4 > 128) throw Error(NLROM_ERR_ARG, "n_p + n_q must be <= 124");
    NL_CUDA(cudaDeviceSynchronize());
    *out = c;
    return NLROM_OK;
  } catch (const Error& e) {
    int code = e.code;
    if (c) nlrom_destroy(c);
    return code;
  }
}

extern "C" void nlrom_destroy(nlrom_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  if (c->gE) cudaGraphExecDestroy(c->gE);
  if (c->gJ) cudaGraphExecDestroy(c->gJ);
  if (c->gIter) cudaGraphExecDestroy(c->gIter);
  if (c->gStep) cudaGraphExecDestroy(c->gStep);
  if (c->gAdapt) cudaGraphExecDestroy(c->gAdapt);
  for (auto g : c->gC)
    if (g) cudaGraphExecDestroy(g);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->st) cudaStreamDestroy(c->st);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->st3) cudaStreamDestroy(c->st3);
  if (c->evFork) cudaEventDestroy(c->evFork);
  if (c->evJoin) cudaEventDestroy(c->evJoin);
  if (c->evFork2) cudaEventDestroy(c->evFork2);
  if (c->evJoin2) cudaEventDestroy(c->evJoin2);
  if (c->evWf) cudaEventDestroy(c->evWf);
  if (c->evW) cudaEventDestroy(c->evW);
  if (c->evK) cudaEventDestroy(c->evK);
  if (c->evM) cudaEventDestroy(c->evM);
  if (c->evP) cudaEventDestroy(c->evP);
  for (auto p : c->ozBHW)
    if (p) cudaFree(p);
  for (auto p : c->ozHW)
    if (p) cudaFree(p);
  for (auto p : c->ozDE)
    if (p) cudaFree(p);
  delete c;
}

extern "C" const char* nlrom_last_error(const nlrom_ctx* c) { return c ? c->err.c_str() : "null handle"; }

#define CTX_TRY(c)          \
  if (!(c)) return NLROM_ERR_ARG; \
  try {                     \
    NL_CUDA(cudaSetDevice((c)->device));
#define CTX_END(c)              \
  return NLROM_OK;              \
  }                             \
  catch (const Error& e) {      \
    return fail((c), e);        \
  }

// ---------------------------------------------------------------- diffops (reference passes)
extern "C" int nlrom_diffop(nlrom_ctx* c, int op, const double* q, const double* vec, double eps, int mode, double* out) {
  CTX_TRY(c)
  if (c->n_sims != 1) throw Error(NLROM_ERR_ARG, "diffop requires a single-sim context");
  if (op < 0 || op > NLROM_OP_VHP) throw Error(NLROM_ERR_ARG, "unknown op");
  if (mode == 1 && !(eps > 0)) throw Error(NLROM_ERR_ARG, "eps must be > 0 (SPEC.md:206)");
  const int nq = c->n_q, N = c->N, L = c->L;
  int order = 0, npass = 1;
  switch (op) {
    case NLROM_OP_VALUE: case NLROM_OP_VJP: order = 0; npass = 1; break;
    case NLROM_OP_JVP: order = 1; npass = 1; break;
    case NLROM_OP_JACOBIAN: case NLROM_OP_VHP: order = 1; npass = nq; break;
    case NLROM_OP_HVV: order = 2; npass = 1; break;
    case NLROM_OP_HV: order = 2; npass = nq; break;
    case NLROM_OP_SVV: order = 3; npass = nq; break;
  }
  const int S = 1 << order, ncols = npass * S;
  const double scale = mode == 1 ? eps : 1.0;
  const int act = mode == 1 ? ACT_SIN_MC : ACT_SIN_MD;
  const bool bwd = (op == NLROM_OP_VJP || op == NLROM_OP_VHP);
  DBuf dq(nq), dv(std::max(nq, N));
  h2d(c, dq, q, nq);
  if (vec) h2d(c, dv, vec, (op == NLROM_OP_VJP || op == NLROM_OP_VHP) ? N : nq);
  DBuf X0((size_t)ncols * c->ldq);
  launch(c, k_seed_ref, grid1((long long)ncols * nq), 256, 0, (const double*)dq.p,
         (const double*)(vec && !bwd ? dv.p : nullptr), X0.p, c->ldq, nq, op, S, npass, scale);
  std::vector<DBuf> Hs(L - 1), caches(L - 1);
  std::vector<int> ldcs(L - 1);
  const double* in = X0.p;
  int ldin = c->ldq;
  for (int l = 0; l < L - 1; ++l) {
    int ldo = (l == L - 2) ? c->ldlast : round_up(c->widths[l + 1], 2);
    ldcs[l] = ldo;
    Hs[l].alloc((size_t)ncols * ldo);
    if (bwd) caches[l].alloc((size_t)ncols * ldo);
    GemmArgs g{c->W[l].p, in, c->ldW[l], ldin, c->widths[l + 1], ncols, c->widths[l], 0, 0};
    fc_forward(order, act, g, Hs[l].p, ldo, c->b[l].p, bwd ? caches[l].p : nullptr, c->st);
    in = Hs[l].p;
    ldin = ldo;
  }
  if (!bwd) {
    if (c->next) {
      GemmArgs gT{c->AT.p, in, round_up(c->wL1, 2), ldin, c->n_p, ncols, c->wL1, 0, 0};
      fc_forward(0, ACT_NONE, gT, Hs[L - 2].p + c->wL1, c->ldlast, nullptr, nullptr, c->st);
    }
    const int ldy = round_up(N, 2);
    DBuf Y((size_t)ncols * ldy);
    GemmArgs g{c->Alast.p, in, c->ldlast, ldin, N, ncols, c->wL1 + c->next, 0, 0};
    // linear output layer: bias P b on the real slot of every pass (period S)
    launch_gemm<GemmCfg<64, 64, 2, 2, 1>>(g, EpiStore{Y.p, ldy, 0, c->Pb.p, S, nullptr}, c->st);
    int slot = (op == NLROM_OP_VALUE) ? 0 : (op == NLROM_OP_JVP || op == NLROM_OP_JACOBIAN) ? 1
             : (op == NLROM_OP_SVV) ? 7 : 3;
    double div = std::pow(scale, __builtin_popcount(slot));
    DBuf o((size_t)N * npass);
    launch(c, k_extract_slot, grid1((long long)N * npass), 256, 0, (const double*)Y.p, ldy, N, S, npass, slot, div, o.p);
    d2h(c, out, o, (size_t)N * npass);
  } else {
    // caches hold layer pre-activations with ld of their output buffers; the backward
    // writes Delta with the same ld per layer.
    int maxld = 0;
    for (int l = 0; l < L - 1; ++l) maxld = std::max(maxld, ldcs[l]);
    DBuf D0((size_t)ncols * maxld), D1((size_t)ncols * maxld), Gout((size_t)ncols * c->ldq);
    DBuf da(N);
    h2d(c, da, vec, N);
    decoder_backward(c, da.p, S, mode == 1, npass, caches, ldcs, D0, D1, Gout, c->ldq);
    if (op == NLROM_OP_VJP) {
      NL_CUDA(cudaMemcpyAsync(out, Gout.p, nq * 8, cudaMemcpyDeviceToHost, c->st));
    } else {
      // vhp[i][k] = Im(G_t[pass k])[i] / eps
      DBuf o((size_t)nq * nq);
      launch(c, k_extract_slot, grid1((long long)nq * nq), 256, 0, (const double*)Gout.p, c->ldq, nq, 2, nq, 1, scale,
             o.p);
      d2h(c, out, o, (size_t)nq * nq);
    }
  }
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

// ---------------------------------------------------------------- fused-path queries
static void eval_point(nlrom_ctx* c, const nlrom_simcfg& cfg) {
  ensure_graphs(c, cfg);
  NL_CUDA(cudaGraphLaunch(c->gE, c->st));
}

static nlrom_simcfg default_cfg(double dt, int drop_fict, int integration) {
  nlrom_simcfg s{};
  s.dt = dt; s.newton_tol = 1e-8; s.max_iters = 20; s.drop_fict = drop_fict; s.integration = integration;
  s.line_search = 1; s.fixed_iters = 0;
  return s;
}

extern "C" int nlrom_residual(nlrom_ctx* c, const double* r, const double* rbar, const double* rdbar,
                              const double* fext, const nlrom_simcfg* cfg, double* phi) {
  CTX_TRY(c)
  set_state(c, r, rbar, rdbar, fext);
  eval_point(c, *cfg);
  d2h(c, phi, c->phi, (size_t)c->n_sims * c->n);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_system_jacobian(nlrom_ctx* c, const double* r, const double* rbar, const double* rdbar,
                                     const double* fext, const nlrom_simcfg* cfg, double* S) {
  CTX_TRY(c)
  set_state(c, r, rbar, rdbar, fext);
  eval_point(c, *cfg);
  NL_CUDA(cudaGraphLaunch(c->gJ, c->st));
  full_S(c, *cfg);
  d2h(c, S, c->S, (size_t)c->n_sims * c->n * c->n);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

static void bundle_only(nlrom_ctx* c, const double* q, const double* qbar, const double* qdbar, double dt, int drop_fict,
                        const double* p) {
  std::vector<double> r(c->n, 0.0), rb(c->n, 0.0), rd(c->n, 0.0);
  for (int i = 0; i < c->n_q; ++i) {
    r[c->n_p + i] = q[i];
    rb[c->n_p + i] = qbar ? qbar[i] : q[i];
    rd[c->n_p + i] = qdbar ? qdbar[i] : 0.0;
  }
  if (p)
    for (int i = 0; i < c->n_p; ++i) r[i] = p[i];
  h2d(c, c->r, r.data(), c->n);
  h2d(c, c->rbar, rb.data(), c->n);
  h2d(c, c->rdbar, rd.data(), c->n);
  bundle_forward(c, dt, drop_fict);
}

extern "C" int nlrom_delta_j(nlrom_ctx* c, const double* q, const double* qbar, const double* qdbar, double dt,
                             int drop_fict, double* dJ) {
  CTX_TRY(c)
  bundle_only(c, q, qbar, qdbar, dt, drop_fict, nullptr);
  d2h(c, dJ, c->dJ, (size_t)c->N * c->n_q);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_fictitious_force(nlrom_ctx* c, const double* q, const double* qbar, double* f) {
  CTX_TRY(c)
  bundle_only(c, q, qbar, nullptr, 1.0, 0, nullptr);
  launch(c, k_mul, grid1(c->N), 256, 0, (const double*)c->mass.p, (const double*)c->hvv.p, c->tmpN.p, c->N);
  d2h(c, f, c->tmpN, c->N);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_full_displacement(nlrom_ctx* c, const double* r, double* u) {
  CTX_TRY(c)
  bundle_only(c, r + c->n_p, nullptr, nullptr, 1.0, 0, r);
  d2h(c, u, c->u, c->N);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_jtilde(nlrom_ctx* c, const double* q, double* Jt) {
  CTX_TRY(c)
  bundle_only(c, q, nullptr, nullptr, 1.0, 0, nullptr);
  NL_CUDA(cudaMemcpy2DAsync(Jt, (size_t)c->n * 8, c->Jt.p, (size_t)c->ldjt * 8, (size_t)c->n * 8, c->N,
                            cudaMemcpyDeviceToHost, c->st));
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_wnet_forward(nlrom_ctx* c, const double* r, double* w, int64_t w_len) {
  CTX_TRY(c)
  if (w_len != c->n_cub) throw Error(NLROM_ERR_DIM, "wnet_forward: output length must equal |C|");
  bundle_only(c, r + c->n_p, nullptr, nullptr, 1.0, 0, r);
  wnet_phase(c);
  d2h(c, w, c->wC, c->n_cub);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_cubature_integrate(nlrom_ctx* c, const double* r, int integration, double* f_red, double* K_red) {
  CTX_TRY(c)
  bundle_only(c, r + c->n_p, nullptr, nullptr, 1.0, 0, r);
  CubSet& s = integration == 1 ? c->setAll : c->setC;
  if (integration == 0) wnet_phase(c);
  cubature_phase(c, s, integration == 0);
  DBuf fr(c->n), Kr((size_t)c->n * c->n);
  launch(c, k_reduce_cub, grid1((long long)c->n * c->n + c->n), 256, 0, (const double*)s.part_f.p,
         (const double*)s.part_K.p, s.nchunk, c->n, fr.p, Kr.p);
  d2h(c, f_red, fr, c->n);
  d2h(c, K_red, Kr, (size_t)c->n * c->n);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

// ---------------------------------------------------------------- adaptive step graph
// Adds a conditional while node after the current capture dependencies of c->st and returns its
// body graph (to be captured after the enclosing capture ends).
static cudaGraph_t add_while_node(nlrom_ctx* c, cudaGraphConditionalHandle h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t graph;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  NL_CUDA(cudaStreamGetCaptureInfo(c->st, &cs, nullptr, &graph, &deps, &nd));
  if (cs != cudaStreamCaptureStatusActive) throw Error(NLROM_ERR_CUDA, "adaptive graph: stream not capturing");
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  NL_CUDA(cudaGraphAddNode(&node, graph, deps, nd, &p));
  NL_CUDA(cudaStreamUpdateCaptureDependencies(c->st, &node, 1, cudaStreamSetCaptureDependencies));
  return p.conditional.phGraph_out[0];
}

static cudaGraph_t capture_graph_of(nlrom_ctx* c) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t graph;
  NL_CUDA(cudaStreamGetCaptureInfo(c->st, &cs, nullptr, &graph, nullptr, nullptr));
  return graph;
}

// The whole adaptive timestep as ONE graph (single sim): pinned H2D of r_bar, rdot_bar, f_ext,
// predictor, E, then the Newton / line-search loops as nested conditional while nodes, rdot and
// the pinned D2H of r, rdot and the Newton state -- one launch and one host sync per step.
static void ensure_adaptive_graph(nlrom_ctx* c, const nlrom_simcfg& cfg, double* hi, double* ho) {
  ensure_graphs(c, cfg);
  char kb[256];
  snprintf(kb, sizeof kb, "%s|%.17g|%d|%d|%p|%p", c->graph_key.c_str(), cfg.newton_tol, cfg.max_iters,
           cfg.line_search, (void*)hi, (void*)ho);
  if (c->gAdapt && c->adapt_key == kb) return;
  if (c->gAdapt) cudaGraphExecDestroy(c->gAdapt);
  c->gAdapt = nullptr;
  if (!c->ad.p) c->ad.alloc(NT_SIZE);
  const int n = c->n;
  const size_t N = (size_t)c->N;
  const int nb = std::min(256, round_up(n, 32));
  cudaGraph_t G = nullptr, bodyO = nullptr, bodyI = nullptr;
  cudaGraphConditionalHandle hO, hI;
  gemm_launch_count = 0;
  // prologue + outer while node + epilogue
  NL_CUDA(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
  try {
    NL_CUDA(cudaGraphConditionalHandleCreate(&hO, capture_graph_of(c), 0, 0));
    // the host hand-off by kernels on the pinned staging (as nlrom_step's fixed-iteration graph)
    launch(c, k_step_in, grid1((long long)std::max<size_t>(N, n)), 256, 0, (const double*)hi, c->rbar.p, c->rdbar.p,
           c->fext.p, c->r.p, cfg.dt, n, (long long)N);
    phase_E(c, cfg);
    launch(c, k_nt_init, 1, 1, 0, hO, (const double*)c->norm.p, c->ad.p, cfg.newton_tol, cfg.max_iters);
    bodyO = add_while_node(c, hO);
    launch(c, k_step_out, grid1(std::max(n, (int)NT_SIZE)), 256, 0, (const double*)c->r.p, (const double*)c->rbar.p,
           c->rdot.p, 1.0 / cfg.dt, n, (const double*)c->ad.p, (int)NT_SIZE, (const int*)nullptr, 1, ho, (int*)nullptr);
  } catch (...) {
    cudaStreamEndCapture(c->st, &G);
    if (G) cudaGraphDestroy(G);
    throw;
  }
  NL_CUDA(cudaStreamEndCapture(c->st, &G));
  try {
    // Newton iteration: J -> dr, then the line search while node, then the convergence test
    NL_CUDA(cudaStreamBeginCaptureToGraph(c->st, bodyO, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    NL_CUDA(cudaGraphConditionalHandleCreate(&hI, bodyO, 0, 0));
    phase_J(c, cfg, false);
    launch(c, k_nt_ls_begin, 1, nb, 0, hI, (const int*)c->status.p, (const double*)c->r.p, c->rsave.p, c->ad.p, n);
    bodyI = add_while_node(c, hI);
    launch(c, k_nt_check, 1, 1, 0, hO, c->ad.p, cfg.newton_tol, cfg.max_iters);
    NL_CUDA(cudaStreamEndCapture(c->st, &bodyO));
    // one line-search trial: r = rsave + t dr, E(r)
    NL_CUDA(cudaStreamBeginCaptureToGraph(c->st, bodyI, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    launch(c, k_nt_axpy, 1, nb, 0, c->r.p, (const double*)c->rsave.p, (const double*)c->dr.p,
           (const double*)c->ad.p, n);
    phase_E(c, cfg);
    launch(c, k_nt_ls_check, 1, 1, 0, hI, (const double*)c->norm.p, c->ad.p, cfg.line_search);
    NL_CUDA(cudaStreamEndCapture(c->st, &bodyI));
    NL_CUDA(cudaGraphInstantiate(&c->gAdapt, G, 0));
  } catch (...) {
    cudaStreamCaptureStatus cs;
    if (cudaStreamIsCapturing(c->st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
      cudaGraph_t tmp;
      cudaStreamEndCapture(c->st, &tmp);
    }
    cudaGraphDestroy(G);
    throw;
  }
  cudaGraphDestroy(G);
  c->adapt_key = kb;
}

// ---------------------------------------------------------------- step
extern "C" int nlrom_step(nlrom_ctx* c, const double* rbar, const double* rdbar, const double* fext,
                          const nlrom_simcfg* cfg, double* r_out, double* rdot_out, nlrom_step_info* info) {
  CTX_TRY(c)
  const int nn = c->n_sims * c->n;
  const size_t nf = (size_t)c->n_sims * c->N;
  if (cfg->fixed_iters > 0) {
    // fixed-iteration mode: inputs through pinned staging, every launch enqueued, ONE host sync
    // at the end for r, rdot, the status flags and the final residual norm
    c->hin.alloc(2 * (size_t)nn + nf);
    c->hout.alloc(2 * (size_t)nn + 2 + c->n_sims);
    double* hi = c->hin.p;
    memcpy(hi, rbar, (size_t)nn * 8);
    memcpy(hi + nn, rdbar, (size_t)nn * 8);
    memcpy(hi + 2 * nn, fext, nf * 8);
    double* ho = c->hout.p;
    int* hs = reinterpret_cast<int*>(ho + 2 * nn + 2);
    ensure_graphs(c, *cfg);
    char kb[96];
    const bool want_norm = info != nullptr;   // the final residual only when the caller reads it
    snprintf(kb, sizeof kb, "|%d|%p|%p|%d", cfg->fixed_iters, (void*)hi, (void*)ho, (int)want_norm);
    const std::string key = c->graph_key + kb;
    if (!c->gStep || c->step_key != key) {
      // the whole step as ONE graph: pinned H2D, predictor, the Newton iterations, the final
      // residual, rdot and the pinned D2H of r, rdot, ||phi|| and the pivot status
      if (c->gStep) cudaGraphExecDestroy(c->gStep);
      c->gStep = capture(c, [&] {
        // the host hand-off by two kernels on the pinned staging (k_step_in / k_step_out): the
        // copy-engine nodes cost ~5 us each per step call at cfg2
        launch(c, k_step_in, grid1((long long)std::max<size_t>(nf, nn)), 256, 0, (const double*)hi, c->rbar.p,
               c->rdbar.p, c->fext.p, c->r.p, cfg->dt, nn, (long long)nf);
        for (int it = 0; it < cfg->fixed_iters; ++it) {
          phase_E(c, *cfg, false);
          phase_J(c, *cfg, true, nullptr, 0, nullptr, true);
        }
        if (want_norm) phase_E(c, *cfg, true, /*resid_only=*/true);   // ||phi|| of the final iterate
        launch(c, k_step_out, grid1(std::max(nn, c->n_sims)), 256, 0, (const double*)c->r.p, (const double*)c->rbar.p,
               c->rdot.p, 1.0 / cfg->dt, nn, (const double*)c->norm.p, want_norm ? 1 : 0, (const int*)c->status.p,
               c->n_sims, ho, hs);
      }, nullptr);
      c->step_key = key;
    }
    NL_CUDA(cudaGraphLaunch(c->gStep, c->st));
    NL_CUDA(cudaStreamSynchronize(c->st));
    for (int s2 = 0; s2 < c->n_sims; ++s2)
      if (hs[s2]) throw Error(NLROM_ERR_NONFINITE, "singular system Jacobian (zero pivot in LU)");
    memcpy(r_out, ho, (size_t)nn * 8);
    memcpy(rdot_out, ho + nn, (size_t)nn * 8);
    c->last_norm = ho[2 * nn];
    if (info) { info->iters = cfg->fixed_iters; info->res_norm = ho[2 * nn]; info->status = 0; }
  } else {
    if (c->n_sims != 1) throw Error(NLROM_ERR_ARG, "adaptive Newton requires a single-sim context");
    const int n = c->n;
    c->hin.alloc(2 * (size_t)n + c->N);
    c->hout.alloc(2 * (size_t)n + NT_SIZE);
    double* hi = c->hin.p;
    double* ho = c->hout.p;
    memcpy(hi, rbar, (size_t)n * 8);
    memcpy(hi + n, rdbar, (size_t)n * 8);
    memcpy(hi + 2 * n, fext, (size_t)c->N * 8);
    ensure_adaptive_graph(c, *cfg, hi, ho);
    NL_CUDA(cudaGraphLaunch(c->gAdapt, c->st));
    NL_CUDA(cudaStreamSynchronize(c->st));
    const double* st = ho + 2 * n;
    const int status = (int)st[NT_STATUS], it = (int)st[NT_IT];
    const double nrm = st[NT_NORM];
    c->last_norm = nrm;
    if (status == NT_SINGULAR) throw Error(NLROM_ERR_NONFINITE, "singular system Jacobian (zero pivot in LU)");
    if (status == NT_NONFINITE) throw Error(NLROM_ERR_NONFINITE, "non-finite residual");
    if (status == NT_MAXITER) {
      char buf[160];
      snprintf(buf, sizeof buf, "Newton did not converge in %d iterations; last residual norm %.17g", cfg->max_iters, nrm);
      throw Error(NLROM_ERR_NEWTON, buf);
    }
    memcpy(r_out, ho, (size_t)n * 8);
    memcpy(rdot_out, ho + n, (size_t)n * 8);
    if (info) { info->iters = it; info->res_norm = nrm; info->status = 0; }
  }
  CTX_END(c)
}

extern "C" int nlrom_step_device(nlrom_ctx* c, const double* rbar, const double* rdbar, const double* fext,
                                 const nlrom_simcfg* cfg, double* r_out, double* rdot_out, void* stream) {
  CTX_TRY(c)
  if (cfg->fixed_iters <= 0) throw Error(NLROM_ERR_ARG, "nlrom_step_device needs fixed_iters > 0");
  cudaStream_t us = (cudaStream_t)stream;
  const int nn = c->n_sims * c->n;
  // order the context stream after the caller's stream, copy inputs in
  NL_CUDA(cudaEventRecord(c->ev0, us));
  NL_CUDA(cudaStreamWaitEvent(c->st, c->ev0, 0));
  NL_CUDA(cudaMemcpyAsync(c->rbar.p, rbar, nn * 8, cudaMemcpyDeviceToDevice, c->st));
  NL_CUDA(cudaMemcpyAsync(c->rdbar.p, rdbar, nn * 8, cudaMemcpyDeviceToDevice, c->st));
  NL_CUDA(cudaMemcpyAsync(c->fext.p, fext, (size_t)c->n_sims * c->N * 8, cudaMemcpyDeviceToDevice, c->st));
  ensure_graphs(c, *cfg);
  launch(c, k_axpy, grid1(nn), 256, 0, c->r.p, (const double*)c->rbar.p, (const double*)c->rdbar.p, cfg->dt, nn);
  for (int it = 0; it < cfg->fixed_iters; ++it) NL_CUDA(cudaGraphLaunch(c->gIter, c->st));
  launch(c, k_rdot, grid1(nn), 256, 0, (const double*)c->r.p, (const double*)c->rbar.p, c->rdot.p, 1.0 / cfg->dt, nn);
  NL_CUDA(cudaMemcpyAsync(r_out, c->r.p, nn * 8, cudaMemcpyDeviceToDevice, c->st));
  NL_CUDA(cudaMemcpyAsync(rdot_out, c->rdot.p, nn * 8, cudaMemcpyDeviceToDevice, c->st));
  NL_CUDA(cudaEventRecord(c->ev1, c->st));
  NL_CUDA(cudaStreamWaitEvent(us, c->ev1, 0));
  CTX_END(c)
}

__global__ void k_flush(double* p, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void k_poison_smem(int n) {
  extern __shared__ double ps[];
  const double nan = __longlong_as_double(0x7ff8dead0000beefLL);
  for (int i = threadIdx.x; i < n; i += blockDim.x) ps[i] = nan;
  __syncthreads();
  if (threadIdx.x == 0 && ps[n - 1] == 0.0) ps[0] = 1.0;  // keep the stores
}

extern "C" int nlrom_debug_poison_shared_memory(int device) {
  try {
    NL_CUDA(cudaSetDevice(device));
    int smem = 0, sms = 0;
    NL_CUDA(cudaDeviceGetAttribute(&smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    NL_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    NL_CUDA(cudaFuncSetAttribute(k_poison_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int rep = 0; rep < 4; ++rep) k_poison_smem<<<sms * 2, 1024, smem>>>(smem / 8);
    NL_CHECK_LAUNCH();
    NL_CUDA(cudaDeviceSynchronize());
    return NLROM_OK;
  } catch (const Error& e) {
    return e.code;
  }
}

extern "C" int nlrom_bench_iterations(nlrom_ctx* c, int n_iters, int flush_l2, float* ms_total, float* ms_dom) {
  CTX_TRY(c)
  if (c->graph_key.empty()) throw Error(NLROM_ERR_ARG, "run nlrom_step first (captures the graphs)");
  if (flush_l2 && !c->flush.p) c->flush.alloc((size_t)32 << 20);  // 256 MB > 126 MB L2
  float tot = 0.f;
  for (int i = 0; i < n_iters; ++i) {
    if (flush_l2) {
      k_flush<<<1184, 256, 0, c->st>>>(c->flush.p, c->flush.n, (double)i);
      NL_CHECK_LAUNCH();
    }
    NL_CUDA(cudaEventRecord(c->ev0, c->st));
    NL_CUDA(cudaGraphLaunch(c->gIter, c->st));
    NL_CUDA(cudaEventRecord(c->ev1, c->st));
    NL_CUDA(cudaEventSynchronize(c->ev1));
    float ms = 0.f;
    NL_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    tot += ms;
  }
  *ms_total = tot;
  // dominant kernel (output decoder layer + fused filter) timed alone on the same stream
  if (ms_dom) {
    float dom = 0.f;
    for (int i = 0; i < n_iters; ++i) {
      if (flush_l2) {
        k_flush<<<1184, 256, 0, c->st>>>(c->flush.p, c->flush.n, (double)i);
        NL_CHECK_LAUNCH();
      }
      NL_CUDA(cudaEventRecord(c->ev0, c->st));
      output_layer(c);
      NL_CUDA(cudaEventRecord(c->ev1, c->st));
      NL_CUDA(cudaEventSynchronize(c->ev1));
      float ms = 0.f;
      NL_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
      dom += ms;
    }
    *ms_dom = dom / std::max(1, n_iters);
  }
  CTX_END(c)
}

extern "C" int nlrom_bench_replays(nlrom_ctx* c, int n_iters, int flush_l2, float* ms_each) {
  CTX_TRY(c)
  if (c->graph_key.empty()) throw Error(NLROM_ERR_ARG, "run nlrom_step first (captures the graphs)");
  if (n_iters <= 0 || !ms_each) throw Error(NLROM_ERR_ARG, "n_iters > 0 and ms_each required");
  if (flush_l2 && !c->flush.p) c->flush.alloc((size_t)32 << 20);  // 256 MB > 126 MB L2
  std::vector<cudaEvent_t> ev(2 * (size_t)n_iters);
  for (auto& e : ev) NL_CUDA(cudaEventCreate(&e));
  try {
    for (int i = 0; i < n_iters; ++i) {
      if (flush_l2) {
        k_flush<<<1184, 256, 0, c->st>>>(c->flush.p, c->flush.n, (double)i);
        NL_CHECK_LAUNCH();
      }
      NL_CUDA(cudaEventRecord(ev[2 * i], c->st));
      NL_CUDA(cudaGraphLaunch(c->gIter, c->st));
      NL_CUDA(cudaEventRecord(ev[2 * i + 1], c->st));
    }
    NL_CUDA(cudaStreamSynchronize(c->st));
    for (int i = 0; i < n_iters; ++i) NL_CUDA(cudaEventElapsedTime(&ms_each[i], ev[2 * i], ev[2 * i + 1]));
  } catch (...) {
    for (auto& e : ev) cudaEventDestroy(e);
    throw;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  CTX_END(c)
}

extern "C" int nlrom_iterate(nlrom_ctx* c, int n_iters) {
  CTX_TRY(c)
  if (c->graph_key.empty()) throw Error(NLROM_ERR_ARG, "run nlrom_step first (captures the graphs)");
  for (int i = 0; i < n_iters; ++i) NL_CUDA(cudaGraphLaunch(c->gIter, c->st));
  check_status(c);
  CTX_END(c)
}

extern "C" int nlrom_get_iterate(nlrom_ctx* c, double* r, double* phi, double* norm) {
  CTX_TRY(c)
  const size_t nn = (size_t)c->n_sims * c->n;
  if (r) d2h(c, r, c->r, nn);
  if (phi) d2h(c, phi, c->phi, nn);
  if (norm) d2h(c, norm, c->norm, c->n_sims);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_set_iterate(nlrom_ctx* c, const double* r) {
  CTX_TRY(c)
  if (!r) throw Error(NLROM_ERR_ARG, "null argument");
  h2d(c, c->r, r, (size_t)c->n_sims * c->n);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

// Per-stage device time (CUDA events on the context stream, L2 optionally flushed before
// each launch), averaged over n_iters: [0] hidden jet chain (fused cluster kernel),
// [1] decoder output layer, [2] vhp backward chain, [3] LU solve.
extern "C" int nlrom_bench_kernels(nlrom_ctx* c, int n_iters, int flush_l2, float* ms4) {
  CTX_TRY(c)
  if (c->graph_key.empty()) throw Error(NLROM_ERR_ARG, "run nlrom_step first (captures the graphs)");
  if (flush_l2 && !c->flush.p) c->flush.alloc((size_t)32 << 20);
  const double dt = 1.0 / 60.0;
  auto stage = [&](int which) {
    switch (which) {
      case 0:
        if (!fused_hidden_forward(c, dt, 0)) bundle_forward(c, dt, 0, false);  // hidden layers only
        break;
      case 1: output_layer(c); break;
      case 2:
        if (!fused_vhp_backward(c, false))
          decoder_backward(c, c->a.p, 2, false, c->n_q, c->cache, c->ldc, c->Delta0, c->Delta1, c->Gt, c->ldGt, true);
        break;
      default: {
        const int n = c->n;
        (void)n;
        launch_lu(c, false);
      }
    }
  };
  for (int w = 0; w < 4; ++w) {
    float acc = 0.f;
    for (int i = 0; i < n_iters; ++i) {
      if (flush_l2) {
        k_flush<<<1184, 256, 0, c->st>>>(c->flush.p, c->flush.n, (double)i);
        NL_CHECK_LAUNCH();
      }
      NL_CUDA(cudaEventRecord(c->ev0, c->st));
      stage(w);
      NL_CUDA(cudaEventRecord(c->ev1, c->st));
      NL_CUDA(cudaEventSynchronize(c->ev1));
      float ms = 0.f;
      NL_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
      acc += ms;
    }
    ms4[w] = acc / std::max(1, n_iters);
  }
  CTX_END(c)
}

// Device time of one cubature launch (the context's cubature set: weighted element forces,
// element stiffness, G_e = w_e K_e J~_e and the J~_C^T G / J~_C^T f partials, the kernel of the
// batched step), L2 flushed before each launch; *bytes = SURVEY.md 8d's algorithmic bytes
// B_cub = |C| (96 n + 200) + 8 (n + n^2) per sim, times n_sims.
extern "C" int nlrom_bench_cubature(nlrom_ctx* c, int n_iters, int flush_l2, float* ms, double* bytes) {
  CTX_TRY(c)
  if (c->graph_key.empty()) throw Error(NLROM_ERR_ARG, "run nlrom_step first (captures the graphs)");
  if (flush_l2 && !c->flush.p) c->flush.alloc((size_t)32 << 20);
  int integ = 0;
  {
    double dt;
    int drop;
    sscanf(c->graph_key.c_str(), "%lf|%d|%d", &dt, &drop, &integ);
  }
  CubSet& s = integ == 1 ? c->setAll : c->setC;
  float acc = 0.f;
  for (int i = 0; i < n_iters; ++i) {
    if (flush_l2) {
      k_flush<<<1184, 256, 0, c->st>>>(c->flush.p, c->flush.n, (double)i);
      NL_CHECK_LAUNCH();
    }
    NL_CUDA(cudaEventRecord(c->ev0, c->st));
    cubature_phase(c, s, integ == 0, false, false, 0);
    NL_CUDA(cudaEventRecord(c->ev1, c->st));
    NL_CUDA(cudaEventSynchronize(c->ev1));
    float t = 0.f;
    NL_CUDA(cudaEventElapsedTime(&t, c->ev0, c->ev1));
    acc += t;
  }
  *ms = acc / std::max(1, n_iters);
  const double n = c->n;
  *bytes = (double)c->n_sims * ((double)s.n * (96.0 * n + 200.0) + 8.0 * (n + n * n));
  CTX_END(c)
}

extern "C" int nlrom_launches_per_iteration(nlrom_ctx* c) { return c ? c->launches_E + c->launches_J : 0; }
extern "C" int nlrom_tc_info(nlrom_ctx* c, int* out) {
  if (!c || !out) return NLROM_ERR_ARG;
  out[0] = out[1] = out[2] = 0;
  for (int l = 0; l < (int)c->ozW.size(); ++l)
    out[0] += (c->ozW[l].ready && oz_enough_tiles(c->widths[l + 1], c->n_sims * c->Cb)) ? 1 : 0;
  out[1] = out_on_tc(c) ? 1 : 0;
  // backward layers on tcgen05: the shared-real path with whole sims in a 64-column tile
  const int P1 = 1 + c->n_q, ocs = (64 / P1) * P1;
  if (shared_real_bwd(c, c->n_q) && ocs >= P1)
    for (int l = 0; l < (int)c->ozWT.size(); ++l)
      out[2] += (c->ozWT[l].ready && oz_enough_tiles(c->widths[l], c->n_sims * P1, ocs)) ? 1 : 0;
  return NLROM_OK;
}
extern "C" int nlrom_tc_layers(nlrom_ctx* c) {
  int k = 0;
  if (c)
    for (auto& w : c->ozW) k += w.ready ? 1 : 0;
  return k;
}

// Prefix-graph timing: for k = 1 .. n, capture the first k launches of one Newton iteration
// (E + J + update) as a graph and time n_iters replays (L2 flushed before each); ms[k-1] is the
// mean device time of prefix k, so ms[k-1] - ms[k-2] is launch k's marginal in-graph cost
// (PDL overlap included). names: '\n'-separated kernel names of the n launches.
extern "C" int nlrom_bench_prefix(nlrom_ctx* c, int n_iters, int flush_l2, int cap, float* ms, char* names,
                                  int names_len, int* n_launches) {
  CTX_TRY(c)
  if (c->graph_key.empty()) throw Error(NLROM_ERR_ARG, "run nlrom_step first (captures the graphs)");
  if (flush_l2 && !c->flush.p) c->flush.alloc((size_t)32 << 20);
  nlrom_simcfg cfg = default_cfg(1.0 / 60.0, 0, 0);
  {
    const std::string& key = c->graph_key;  // dt | drop_fict | integration of the captured graphs
    double dt;
    int drop, integ;
    if (sscanf(key.c_str(), "%lf|%d|%d", &dt, &drop, &integ) == 3) cfg = default_cfg(dt, drop, integ);
  }
  const int total = c->launches_E + c->launches_J;
  const int n = std::min(cap, total);
  std::string nm;
  NL_CUDA(cudaMemcpyAsync(c->rsave.p, c->r.p, (size_t)c->n_sims * c->n * 8, cudaMemcpyDeviceToDevice, c->st));
  for (int k = 1; k <= n; ++k) {
    launch_budget() = k;
    launch_log().clear();
    cudaGraphExec_t g = nullptr;
    try {
      g = capture(c, [&] { phase_E(c, cfg, false); phase_J(c, cfg, true, nullptr, 0, nullptr, true); }, nullptr);
    } catch (...) {
      launch_budget() = kNoBudget;
      throw;
    }
    launch_budget() = kNoBudget;
    if (k == n)
      for (const void* f : launch_log()) {
        const char* s = nullptr;
        if (cudaFuncGetName(&s, f) == cudaSuccess && s) nm += s;
        nm += "\n";
      }
    float acc = 0.f;
    for (int i = 0; i < n_iters + 1; ++i) {
      NL_CUDA(cudaMemcpyAsync(c->r.p, c->rsave.p, (size_t)c->n_sims * c->n * 8, cudaMemcpyDeviceToDevice, c->st));
      if (flush_l2) {
        k_flush<<<1184, 256, 0, c->st>>>(c->flush.p, c->flush.n, (double)i);
        NL_CHECK_LAUNCH();
      }
      NL_CUDA(cudaEventRecord(c->ev0, c->st));
      NL_CUDA(cudaGraphLaunch(g, c->st));
      NL_CUDA(cudaEventRecord(c->ev1, c->st));
      NL_CUDA(cudaEventSynchronize(c->ev1));
      float t = 0.f;
      NL_CUDA(cudaEventElapsedTime(&t, c->ev0, c->ev1));
      if (i) acc += t;  // first replay warms the instantiated graph
    }
    cudaGraphExecDestroy(g);
    ms[k - 1] = acc / std::max(1, n_iters);
  }
  NL_CUDA(cudaMemcpyAsync(c->r.p, c->rsave.p, (size_t)c->n_sims * c->n * 8, cudaMemcpyDeviceToDevice, c->st));
  NL_CUDA(cudaStreamSynchronize(c->st));
  if (names && names_len > 0) {
    const size_t m = std::min(nm.size(), (size_t)names_len - 1);
    memcpy(names, nm.data(), m);
    names[m] = 0;
  }
  if (n_launches) *n_launches = n;
  CTX_END(c)
}

extern "C" int nlrom_element_forces(nlrom_ctx* c, const double* u, int want_K, double* f_int, double* K_elems) {
  CTX_TRY(c)
  CubSet& s = c->setAll;
  h2d(c, c->u, u, c->N);
  DBuf Ke(want_K ? (size_t)c->T * 144 : 0);
  CubArgs a{s.elems.p, s.n, c->elem_rows.p, c->Dm_inv.p, c->vol.p, nullptr, c->u.p, nullptr,
            c->N, c->n, c->ldjt, c->mu, c->lam, s.epc, s.fe_w.p, s.part_f.p, s.part_K.p, s.nchunk,
            want_K ? Ke.p : nullptr, nullptr};
  size_t smem = (size_t)(2 * s.epc * 12 * gram_ld(c->n) + s.epc * 162) * 8;
  launch(c, k_cubature<2>, dim3(s.nech, 1), 256, smem, a);  // force-only: no partials
  launch(c, k_scatter_rows, grid1((long long)s.n_rows), 256, 0, (const int*)s.row_ids.p, (const int*)s.row_ptr.p,
         (const int*)s.entries.p, s.n_rows, (const double*)s.fe_w.p, s.n, s.f.p, c->N, 1);
  d2h(c, f_int, s.f, c->N);
  if (want_K) d2h(c, K_elems, Ke, (size_t)c->T * 144);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_element_reduced_forces(nlrom_ctx* c, const double* r, const int* elems, int n_elems, double* out) {
  CTX_TRY(c)
  if (n_elems <= 0) return NLROM_OK;
  for (int i = 0; i < n_elems; ++i)
    if (elems[i] < 0 || elems[i] >= c->T) throw Error(NLROM_ERR_ARG, "element id out of range");
  bundle_only(c, r + c->n_p, nullptr, nullptr, 1.0, 0, r);
  IBuf de;
  de.upload(elems, n_elems);
  const int epc = c->setAll.epc;
  const int nch = ceil_div(n_elems, epc);
  DBuf few((size_t)n_elems * 12), pf((size_t)nch * c->n), pK((size_t)nch * c->n * c->n), fo((size_t)n_elems * c->n);
  CubArgs a{de.p, n_elems, c->elem_rows.p, c->Dm_inv.p, c->vol.p, nullptr, c->u.p, c->Jt.p,
            c->N, c->n, c->ldjt, c->mu, c->lam, epc, few.p, pf.p, pK.p, nch, nullptr, fo.p};
  size_t smem = (size_t)(2 * epc * 12 * gram_ld(c->n) + epc * 162) * 8;
  launch(c, k_cubature<2>, dim3(nch, 1), 256, smem, a);
  d2h(c, out, fo, (size_t)n_elems * c->n);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

// Training-set builder: per-element reduced forces of ALL elements at
// n_poses poses, buffers allocated once, one decoder bundle + one cubature launch per pose.
extern "C" int nlrom_train_forces(nlrom_ctx* c, const double* rs, int n_poses, double* F_out, double* u_out) {
  CTX_TRY(c)
  if (n_poses <= 0) return NLROM_OK;
  CubSet& s = c->setAll;
  const int T = c->T, n = c->n, epc = s.epc, nch = ceil_div(T, epc);
  DBuf few((size_t)T * 12), pf((size_t)nch * n), pK((size_t)nch * n * n), fo((size_t)T * n);
  CubArgs a{nullptr, T, c->elem_rows.p, c->Dm_inv.p, c->vol.p, nullptr, c->u.p, c->Jt.p,
            c->N, n, c->ldjt, c->mu, c->lam, epc, few.p, pf.p, pK.p, nch, nullptr, fo.p};
  a.rows_g = s.rows_g.p;
  a.Dm_g = s.Dm_g.p;
  a.vol_g = s.vol_g.p;
  const size_t smem = (size_t)(2 * epc * 12 * gram_ld(n) + epc * 162) * 8;
  for (int k = 0; k < n_poses; ++k) {
    const double* r = rs + (size_t)k * n;
    bundle_only(c, r + c->n_p, nullptr, nullptr, 1.0, 0, r);
    launch(c, k_cubature<2>, dim3(nch, 1), 256, smem, a);
    d2h(c, F_out + (size_t)k * T * n, fo, (size_t)T * n);
    if (u_out) d2h(c, u_out + (size_t)k * c->N, c->u, c->N);
  }
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

// =========================================================================== substructured scene
// this context's sims are strings [lo, hi) of a scene of k_total strings
// on a translating core; the host drives one Newton iteration as
//   nlrom_coupled_eval(jacobian=1) -> allreduce(partial, 16 doubles) -> nlrom_coupled_update(mode 1)
// (model: oracle/coupled.py; kernels: coupled_kernels.cuh).

namespace {

void coupled_body(nlrom_ctx* c, const nlrom_simcfg& cfg, int jac, double* partial) {
  const double h = cfg.dt, ah = c->alpha * cfg.dt;
  const int S = c->n_sims, n = c->n;
  launch(c, k_cp_fext, grid1((long long)S * c->N), 256, 0, (const double*)c->cpFloc.p, (const double*)c->cpR.p,
         (const double*)c->cpCore.p, (const double*)c->mass.p, c->N, S, h, ah, c->fext.p);
  phase_E(c, cfg);
  launch(c, k_cp_blocks, S, 256, 0, (const double*)c->Jt.p, c->ldjt, (const double*)c->dJ.p, c->lddj,
         (const double*)c->hvv.p, (const double*)c->mass.p, (const double*)c->cpR.p, c->N, n, c->n_q, cfg.drop_fict,
         ah, c->cpBlocks.p, c->cpCb.p);
  if (jac) phase_J(c, cfg, false, c->cpCb.p, 3, c->cpX.p);
  CpPartialArgs A{c->cpR.p, c->cpBlocks.p, c->cpFsum.p, c->cpCore.p, c->r.p, c->rbar.p, c->rdbar.p, c->phi.p,
                  c->cpX.p, c->dr.p, S, n, c->n_p, c->n_q, h, ah, c->cp_m_string, jac, partial};
  launch(c, k_cp_partial, 1, 256, 0, A);
}

void coupled_graph(nlrom_ctx* c, const nlrom_simcfg& cfg, int jac, double* partial) {
  char buf[64];
  snprintf(buf, sizeof buf, "|%p", (void*)partial);
  const std::string key = cfg_key(cfg) + buf;
  if (c->gC[jac] && c->cp_key[jac] == key) return;
  if (c->gC[jac]) cudaGraphExecDestroy(c->gC[jac]);
  c->gC[jac] = nullptr;
  coupled_body(c, cfg, jac, partial);  // eager warm-up (kernel attributes outside capture)
  NL_CUDA(cudaStreamSynchronize(c->st));
  c->gC[jac] = capture(c, [&] { coupled_body(c, cfg, jac, partial); }, &c->launches_C[jac]);
  c->cp_key[jac] = key;
}

void require_coupled(nlrom_ctx* c) {
  if (!c->coupled) throw Error(NLROM_ERR_ARG, "call nlrom_coupled_setup first");
}

}  // namespace

extern "C" int nlrom_stream(nlrom_ctx* c, void** stream) {
  CTX_TRY(c)
  if (!stream) throw Error(NLROM_ERR_ARG, "null argument");
  *stream = (void*)c->st;
  CTX_END(c)
}

extern "C" int nlrom_coupled_setup(nlrom_ctx* c, const double* R, const double* f_world, int k_total, double m_core,
                                   double k_core, const double* f_core) {
  CTX_TRY(c)
  if (!R || !f_world || !f_core) throw Error(NLROM_ERR_ARG, "null argument");
  if (k_total < c->n_sims) throw Error(NLROM_ERR_DIM, "k_total must cover this context's strings");
  const int S = c->n_sims, N = c->N, n = c->n;
  std::vector<double> mass(N), floc((size_t)S * N), fsum((size_t)S * 3, 0.0);
  NL_CUDA(cudaMemcpy(mass.data(), c->mass.p, N * 8, cudaMemcpyDeviceToHost));
  double ms = 0.0;
  for (int i = 0; i < N; i += 3) ms += mass[i];
  for (int s = 0; s < S; ++s) {
    const double* Rs = R + (size_t)s * 9;
    for (int v = 0; v < N / 3; ++v) {
      const double* fw = f_world + (size_t)s * N + 3 * v;
      for (int d = 0; d < 3; ++d) {
        floc[(size_t)s * N + 3 * v + d] = Rs[0 * 3 + d] * fw[0] + Rs[1 * 3 + d] * fw[1] + Rs[2 * 3 + d] * fw[2];
        fsum[(size_t)s * 3 + d] += fw[d];
      }
    }
  }
  upload(c->cpR, R, (size_t)S * 9);
  upload(c->cpFloc, floc.data(), floc.size());
  upload(c->cpFsum, fsum.data(), fsum.size());
  upload(c->cpFcore, f_core, 3);
  c->cpCore.alloc(CORE_SIZE);
  c->cpBlocks.alloc((size_t)S * (3 * (n + c->n_q) + 3));
  c->cpCb.alloc((size_t)S * 3 * n);
  c->cpX.alloc((size_t)S * 3 * n);
  c->cp_m_core = m_core;
  c->cp_k_core = k_core;
  c->cp_m_string = ms;
  c->cp_m_total = m_core + (double)k_total * ms;
  c->coupled = true;
  CTX_END(c)
}

extern "C" int nlrom_coupled_begin(nlrom_ctx* c, const double* r_bar, const double* rdot_bar, const double* c_bar,
                                   const double* cdot_bar, const nlrom_simcfg* cfg) {
  CTX_TRY(c)
  require_coupled(c);
  const int nn = c->n_sims * c->n;
  set_state(c, nullptr, r_bar, rdot_bar, nullptr);
  double core[CORE_SIZE] = {};
  for (int a = 0; a < 3; ++a) {
    core[CORE_C + a] = c_bar[a] + cfg->dt * cdot_bar[a];
    core[CORE_CBAR + a] = c_bar[a];
    core[CORE_CDBAR + a] = cdot_bar[a];
  }
  NL_CUDA(cudaMemcpyAsync(c->cpCore.p, core, sizeof core, cudaMemcpyHostToDevice, c->st));
  launch(c, k_axpy, grid1(nn), 256, 0, c->r.p, (const double*)c->rbar.p, (const double*)c->rdbar.p, cfg->dt, nn);
  NL_CUDA(cudaStreamSynchronize(c->st));
  CTX_END(c)
}

extern "C" int nlrom_coupled_eval(nlrom_ctx* c, const nlrom_simcfg* cfg, int jacobian, double* partial_dev) {
  CTX_TRY(c)
  require_coupled(c);
  if (!partial_dev) throw Error(NLROM_ERR_ARG, "null partial buffer");
  const int j = jacobian ? 1 : 0;
  coupled_graph(c, *cfg, j, partial_dev);
  NL_CUDA(cudaGraphLaunch(c->gC[j], c->st));
  CTX_END(c)
}

extern "C" int nlrom_coupled_update(nlrom_ctx* c, const nlrom_simcfg* cfg, const double* total_dev, int mode, double t,
                                    double* norm_host) {
  CTX_TRY(c)
  require_coupled(c);
  const double h = cfg->dt, ah = c->alpha * cfg->dt;
  const int nn = c->n_sims * c->n;
  if (mode == 0 || mode == 1)
    launch(c, k_cp_update, 1, 32, 0, total_dev, c->cpCore.p, h, ah, c->cp_m_core, c->cp_m_total, c->cp_k_core,
           (const double*)c->cpFcore.p, mode);
  if (mode == 1) NL_CUDA(cudaMemcpyAsync(c->rsave.p, c->r.p, (size_t)nn * 8, cudaMemcpyDeviceToDevice, c->st));
  if (mode == 1 || mode == 2)
    launch(c, k_cp_apply, grid1(nn), 256, 0, c->r.p, (const double*)c->rsave.p, (const double*)c->dr.p,
           (const double*)c->cpX.p, c->cpCore.p, c->n_sims, c->n, t);
  if (norm_host) {
    check_status(c);
    NL_CUDA(cudaMemcpyAsync(norm_host, c->cpCore.p + CORE_NORM, 8, cudaMemcpyDeviceToHost, c->st));
    NL_CUDA(cudaStreamSynchronize(c->st));
  }
  CTX_END(c)
}

extern "C" int nlrom_coupled_read(nlrom_ctx* c, double dt, double* r, double* rdot, double* core_c, double* core_cdot) {
  CTX_TRY(c)
  require_coupled(c);
  const int nn = c->n_sims * c->n;
  launch(c, k_rdot, grid1(nn), 256, 0, (const double*)c->r.p, (const double*)c->rbar.p, c->rdot.p, 1.0 / dt, nn);
  double core[CORE_SIZE];
  check_status(c);
  d2h(c, r, c->r, nn);
  d2h(c, rdot, c->rdot, nn);
  NL_CUDA(cudaMemcpyAsync(core, c->cpCore.p, sizeof core, cudaMemcpyDeviceToHost, c->st));
  NL_CUDA(cudaStreamSynchronize(c->st));
  for (int a = 0; a < 3; ++a) {
    core_c[a] = core[CORE_C + a];
    core_cdot[a] = (core[CORE_C + a] - core[CORE_CBAR + a]) / dt;
  }
  CTX_END(c)
}

extern "C" int nlrom_coupled_launches(nlrom_ctx* c) {
  return c ? c->launches_C[1] + 2 : 0;
}
