// Generic dense network over real / multicomplex scalars on the GPU:
// densenet.forward and densenet.backward.
//
// Device layout: part-column space, X_t[c][d] with c = b * 2^order + s (the slots
// of one batch member adjacent), row length ld = round_up(dim, 2). Host part
// stacks (2^order, dim, batch) (mcx.py:294-300) are permuted on the device.
#include <vector>
#include <string>
#include <cstring>
#include "common.cuh"
#include "epilogues.cuh"

namespace nlrom {

void upload_matrix(DBuf& dst, const double* h, int rows, int cols, int ld, int rows_alloc) {
  if (rows_alloc < rows) rows_alloc = rows;
  dst.alloc((size_t)rows_alloc * ld);
  if (rows && cols) {
    NL_CUDA(cudaMemcpy2D(dst.p, (size_t)ld * 8, h, (size_t)cols * 8, (size_t)cols * 8, rows, cudaMemcpyHostToDevice));
    NL_CUDA(cudaStreamSynchronize(cudaStreamLegacy));   // (as upload: pageable H2D vs non-blocking streams)
  }
}

// (S, D, B) host-layout -> X_t[(b*S+s)][d] (ld)
__global__ void k_parts_to_cols(const double* __restrict__ in, double* __restrict__ out, int S, int D, int B, int ld) {
  long long n = (long long)S * D * B;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int b = i % B;
    long long r = i / B;
    int d = r % D;
    int s = r / D;
    out[((size_t)b * S + s) * ld + d] = in[i];
  }
}
__global__ void k_cols_to_parts(const double* __restrict__ in, double* __restrict__ out, int S, int D, int B, int ld) {
  long long n = (long long)S * D * B;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int b = i % B;
    long long r = i / B;
    int d = r % D;
    int s = r / D;
    out[i] = in[((size_t)b * S + s) * ld + d];
  }
}
// X_t[(b*S+s)][d] -> slot-major K=b layout P[(s*D+d)][b] (ldp)
__global__ void k_cols_to_slotmajor(const double* __restrict__ in, double* __restrict__ out, int S, int D, int B,
                                    int ld, int ldp) {
  long long n = (long long)S * D * B;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int b = i % B;
    long long r = i / B;
    out[r * ldp + b] = in[((size_t)b * S + (r / D)) * ld + (r % D)];
  }
}
// Combine slot products P[(s2,i)][(s1,o)] into multicomplex dW[s][o][i] (order 0/1),
// and db[s][o] = sum_b d[s][o][b].
__global__ void k_param_combine(const double* __restrict__ P, int ldp, const double* __restrict__ dS, int ldd,
                                double* __restrict__ dW, double* __restrict__ db, int S, int O, int I, int B) {
  long long n = (long long)S * O * I;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    int i = t % I;
    int o = (t / I) % O;
    int s = t / ((long long)I * O);
    auto Pv = [&](int s1, int s2) { return P[((size_t)s2 * I + i) * ldp + (size_t)s1 * O + o]; };
    double v;
    if (S == 1) v = Pv(0, 0);
    else if (s == 0) v = Pv(0, 0) - Pv(1, 1);
    else v = Pv(0, 1) + Pv(1, 0);
    dW[t] = v;
  }
  long long nb = (long long)S * O;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nb; t += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < B; ++b) acc += dS[t * ldd + b];
    db[t] = acc;
  }
}

using CfgBig = GemmCfg<64, 64, 2, 2, 1>;
using CfgSmall = GemmCfg<16, 16, 1, 1, 4>;

template <class Epi>
static void gemm_auto(const GemmArgs& g, const Epi& e, cudaStream_t st) {
  if ((long long)g.M * g.C >= 64LL * 64 * 64) launch_gemm<CfgBig>(g, e, st);
  else launch_gemm<CfgSmall>(g, e, st);
}

template <int N>
static void act_gemm(int act, const GemmArgs& g, double* Y, int ldy, const double* bias, double* cache,
                     cudaStream_t st) {
  switch (act) {
    case ACT_SIN_MC: gemm_auto(g, EpiAct<N, ACT_SIN_MC>{Y, ldy, 0, bias, cache}, st); break;
    case ACT_SIN_MD: gemm_auto(g, EpiAct<N, ACT_SIN_MD>{Y, ldy, 0, bias, cache}, st); break;
    case ACT_SQUARE_MC: gemm_auto(g, EpiAct<N, ACT_SQUARE_MC>{Y, ldy, 0, bias, cache}, st); break;
    default: gemm_auto(g, EpiAct<N, ACT_NONE>{Y, ldy, 0, bias, cache}, st); break;
  }
}

void fc_forward(int order, int act, const GemmArgs& g, double* Y, int ldy, const double* bias, double* cache,
                cudaStream_t st) {
  switch (order) {
    case 0: act_gemm<1>(act, g, Y, ldy, bias, cache, st); break;
    case 1: act_gemm<2>(act, g, Y, ldy, bias, cache, st); break;
    case 2: act_gemm<4>(act, g, Y, ldy, bias, cache, st); break;
    case 3: act_gemm<8>(act, g, Y, ldy, bias, cache, st); break;
    default: throw Error(NLROM_ERR_ORDER, "order out of range 0..3");
  }
}

template <int N>
static void bwd_gemm_n(int act, const GemmArgs& g, double* Y, int ldy, const double* z, cudaStream_t st) {
  switch (act) {
    case ACT_SIN_MC: gemm_auto(g, EpiBwdAct<N, ACT_SIN_MC>{Y, ldy, 0, z}, st); break;
    case ACT_SIN_MD: gemm_auto(g, EpiBwdAct<N, ACT_SIN_MD>{Y, ldy, 0, z}, st); break;
    case ACT_SQUARE_MC: gemm_auto(g, EpiBwdAct<N, ACT_SQUARE_MC>{Y, ldy, 0, z}, st); break;
    default: gemm_auto(g, EpiStore{Y, ldy, 0, nullptr, 1, nullptr}, st); break;
  }
}

void fc_backward(int order, int act, const GemmArgs& g, double* Y, int ldy, const double* zcache, cudaStream_t st) {
  if (order == 0) bwd_gemm_n<1>(act, g, Y, ldy, zcache, st);
  else if (order == 1) bwd_gemm_n<2>(act, g, Y, ldy, zcache, st);
  else throw Error(NLROM_ERR_ORDER, "backward supports real or order-1 complex scalars (SPEC.md:149)");
}

}  // namespace nlrom

using namespace nlrom;

struct NetLayer {
  int kind = 0, in = 0, out = 0, nb = 0;
  int act_after = ACT_NONE;  // for FC: activation of the following layer (fused)
  DBuf W, WT, b, U, Ut;
  int ldw = 0, ldwt = 0, ldu = 0, ldut = 0;
};

struct nlrom_net {
  int device = 0;
  std::vector<NetLayer> L;
  std::string err;
  cudaStream_t st = nullptr;
};

static int fail(nlrom_net* n, const Error& e) {
  if (n) n->err = e.what();
  return e.code;
}

extern "C" int nlrom_net_create(nlrom_net** out, int device, int n_layers, const nlrom_layer_desc* layers) {
  nlrom_net* n = nullptr;
  try {
    if (!out || n_layers < 1 || !layers) throw Error(NLROM_ERR_ARG, "bad arguments");
    NL_CUDA(cudaSetDevice(device));
    n = new nlrom_net();
    n->device = device;
    NL_CUDA(cudaStreamCreateWithFlags(&n->st, cudaStreamNonBlocking));
    for (int i = 0; i < n_layers; ++i) {
      const nlrom_layer_desc& d = layers[i];
      NetLayer l;
      l.kind = d.kind;
      l.in = d.in_dim;
      l.out = d.out_dim;
      if (i > 0 && n->L.back().out != l.in) throw Error(NLROM_ERR_DIM, "layer dims do not chain");
      if (d.kind == NLROM_LAYER_FC) {
        l.ldw = round_up(l.in, 2);
        l.ldwt = round_up(l.out, 2);
        upload_matrix(l.W, d.W, l.out, l.in, l.ldw);
        std::vector<double> wt((size_t)l.in * l.out);
        for (int o = 0; o < l.out; ++o)
          for (int k = 0; k < l.in; ++k) wt[(size_t)k * l.out + o] = d.W[(size_t)o * l.in + k];
        upload_matrix(l.WT, wt.data(), l.in, l.out, l.ldwt);
        l.b.alloc(l.out);
        NL_CUDA(cudaMemcpy(l.b.p, d.b, l.out * 8, cudaMemcpyHostToDevice));
        NL_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
      } else if (d.kind == NLROM_LAYER_FILTER) {
        if (l.in != l.out) throw Error(NLROM_ERR_DIM, "filter layers are square (SPEC.md:114)");
        l.nb = d.n_basis;
        l.ldu = round_up(l.nb, 2);
        l.ldut = round_up(l.in, 2);
        upload_matrix(l.U, d.W, l.in, l.nb, l.ldu);
        std::vector<double> ut((size_t)l.nb * l.in);
        for (int r = 0; r < l.in; ++r)
          for (int k = 0; k < l.nb; ++k) ut[(size_t)k * l.in + r] = d.W[(size_t)r * l.nb + k];
        upload_matrix(l.Ut, ut.data(), l.nb, l.in, l.ldut);
      } else if (d.kind == NLROM_LAYER_SIN || d.kind == NLROM_LAYER_SQUARE) {
        if (l.in != l.out) throw Error(NLROM_ERR_DIM, "activation layers are square");
      } else {
        throw Error(NLROM_ERR_ARG, "unsupported layer kind (softmax is out of scope)");
      }
      n->L.push_back(std::move(l));
    }
    // fuse activation layers into the preceding FC
    for (size_t i = 0; i + 1 < n->L.size(); ++i)
      if (n->L[i].kind == NLROM_LAYER_FC) {
        int k = n->L[i + 1].kind;
        n->L[i].act_after = (k == NLROM_LAYER_SIN) ? ACT_SIN_MC : (k == NLROM_LAYER_SQUARE) ? ACT_SQUARE_MC : ACT_NONE;
      }
    *out = n;
    return NLROM_OK;
  } catch (const Error& e) {
    int c = e.code;
    delete n;
    return c;
  }
}

extern "C" void nlrom_net_destroy(nlrom_net* n) {
  if (!n) return;
  cudaSetDevice(n->device);
  if (n->st) cudaStreamDestroy(n->st);
  delete n;
}

extern "C" const char* nlrom_net_last_error(const nlrom_net* n) { return n ? n->err.c_str() : "null handle"; }

// Elementwise activation over a column buffer (activation layer not preceded by an FC).
template <int N, int ACT>
__global__ void k_act_cols(const double* in, double* out, double* cache, int ncols, int dim, int ld) {
  long long n = (long long)(ncols / N) * dim;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    int d = t % dim;
    int p = t / dim;
    double z[N], o[N], c[N];
#pragma unroll
    for (int s = 0; s < N; ++s) z[s] = in[(size_t)(p * N + s) * ld + d];
    if (cache)
#pragma unroll
      for (int s = 0; s < N; ++s) cache[(size_t)(p * N + s) * ld + d] = z[s];
    if constexpr (ACT == ACT_SIN_MC) mc_sincos<N>(z, o, c);
    else mc_mul<N>(z, z, o);
#pragma unroll
    for (int s = 0; s < N; ++s) out[(size_t)(p * N + s) * ld + d] = o[s];
  }
}
template <int N, int ACT>
__global__ void k_act_bwd_cols(const double* d_in, const double* zc, double* out, int ncols, int dim, int ld) {
  long long n = (long long)(ncols / N) * dim;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    int d = t % dim;
    int p = t / dim;
    double z[N], g[N], f[N], o[N], sn[N];
#pragma unroll
    for (int s = 0; s < N; ++s) {
      z[s] = zc[(size_t)(p * N + s) * ld + d];
      g[s] = d_in[(size_t)(p * N + s) * ld + d];
    }
    if constexpr (ACT == ACT_SIN_MC) mc_sincos<N>(z, sn, f);
    else
#pragma unroll
      for (int s = 0; s < N; ++s) f[s] = 2.0 * z[s];
    mc_mul<N>(g, f, o);
#pragma unroll
    for (int s = 0; s < N; ++s) out[(size_t)(p * N + s) * ld + d] = o[s];
  }
}

template <int N>
static void act_cols(int act, const double* in, double* out, double* cache, int ncols, int dim, int ld, cudaStream_t st) {
  int blocks = std::min(4096, ceil_div((ncols / N) * dim, 256));
  if (act == ACT_SIN_MC) k_act_cols<N, ACT_SIN_MC><<<blocks, 256, 0, st>>>(in, out, cache, ncols, dim, ld);
  else k_act_cols<N, ACT_SQUARE_MC><<<blocks, 256, 0, st>>>(in, out, cache, ncols, dim, ld);
  NL_CHECK_LAUNCH();
}
template <int N>
static void act_bwd_cols(int act, const double* d, const double* zc, double* out, int ncols, int dim, int ld,
                         cudaStream_t st) {
  int blocks = std::min(4096, ceil_div((ncols / N) * dim, 256));
  if (act == ACT_SIN_MC) k_act_bwd_cols<N, ACT_SIN_MC><<<blocks, 256, 0, st>>>(d, zc, out, ncols, dim, ld);
  else k_act_bwd_cols<N, ACT_SQUARE_MC><<<blocks, 256, 0, st>>>(d, zc, out, ncols, dim, ld);
  NL_CHECK_LAUNCH();
}

static void act_cols_any(int order, int act, const double* in, double* out, double* cache, int ncols, int dim, int ld,
                         cudaStream_t st) {
  switch (order) {
    case 0: act_cols<1>(act, in, out, cache, ncols, dim, ld, st); break;
    case 1: act_cols<2>(act, in, out, cache, ncols, dim, ld, st); break;
    case 2: act_cols<4>(act, in, out, cache, ncols, dim, ld, st); break;
    case 3: act_cols<8>(act, in, out, cache, ncols, dim, ld, st); break;
  }
}

// Runs the forward; if `caches` is non-null, records every layer input (index i = input of layer i)
// and the pre-activation of fused FC+act layers (stored at index i+1's "pre" slot).
struct FwdRecord {
  std::vector<DBuf> inputs;  // input of layer i, (ncols x ld_i)
  std::vector<DBuf> pre;     // pre-activation of activation layer i (if any)
};

static void net_forward_dev(nlrom_net* n, int order, DBuf& X0, int ncols, DBuf& out, int& ld_out, FwdRecord* rec) {
  cudaStream_t st = n->st;
  const int S = 1 << order;
  DBuf cur = std::move(X0);
  int dim = n->L[0].in;
  int ld = round_up(dim, 2);
  size_t nL = n->L.size();
  if (rec) {
    rec->inputs.resize(nL);
    rec->pre.resize(nL);
  }
  for (size_t i = 0; i < nL; ++i) {
    NetLayer& l = n->L[i];
    const int ldo = round_up(l.out, 2);
    if (l.kind == NLROM_LAYER_FC) {
      DBuf y((size_t)ncols * ldo);
      double* cache = nullptr;
      if (rec && l.act_after != ACT_NONE) {
        rec->pre[i + 1].alloc((size_t)ncols * ldo);
        cache = rec->pre[i + 1].p;
      }
      GemmArgs g{l.W.p, cur.p, l.ldw, ld, l.out, ncols, l.in, 0, 0};
      fc_forward(order, l.act_after, g, y.p, ldo, l.b.p, cache, st);
      if (rec) rec->inputs[i] = std::move(cur);
      cur = std::move(y);
      if (l.act_after != ACT_NONE) {
        ++i;  // activation consumed
        if (rec) rec->inputs[i].alloc(0);
      }
    } else if (l.kind == NLROM_LAYER_FILTER) {
      // T_t = X_t U ; Y = X - U T (factored delta_ij - sum_k U_ik U_jk)
      DBuf T((size_t)ncols * l.ldu);
      GemmArgs g1{l.Ut.p, cur.p, l.ldut, ld, l.nb, ncols, l.in, 0, 0};
      gemm_auto(g1, EpiStore{T.p, l.ldu, 0, nullptr, 1, nullptr}, st);
      DBuf y((size_t)ncols * ldo);
      GemmArgs g2{l.U.p, T.p, l.ldu, l.ldu, l.out, ncols, l.nb, 0, 0};
      gemm_auto(g2, EpiStore{y.p, ldo, 0, nullptr, 1, cur.p}, st);
      if (rec) rec->inputs[i] = std::move(cur);
      cur = std::move(y);
    } else {
      int act = (l.kind == NLROM_LAYER_SIN) ? ACT_SIN_MC : ACT_SQUARE_MC;
      DBuf y((size_t)ncols * ldo);
      double* cache = nullptr;
      if (rec) {
        rec->pre[i].alloc((size_t)ncols * ldo);
        cache = rec->pre[i].p;
      }
      act_cols_any(order, act, cur.p, y.p, cache, ncols, l.in, ld, st);
      if (rec) rec->inputs[i] = std::move(cur);
      cur = std::move(y);
    }
    dim = l.out;
    ld = ldo;
  }
  out = std::move(cur);
  ld_out = ld;
  (void)S;
}

extern "C" int nlrom_net_forward(nlrom_net* n, int order, const double* parts_in, int batch, double* parts_out) {
  try {
    if (!n) return NLROM_ERR_ARG;
    if (order < 0 || order > 3) throw Error(NLROM_ERR_ORDER, "order out of range 0..3");
    NL_CUDA(cudaSetDevice(n->device));
    const int S = 1 << order, ncols = S * batch;
    const int din = n->L[0].in, dout = n->L.back().out;
    DBuf hin((size_t)S * din * batch), X0((size_t)ncols * round_up(din, 2));
    NL_CUDA(cudaMemcpyAsync(hin.p, parts_in, hin.n * 8, cudaMemcpyHostToDevice, n->st));
    k_parts_to_cols<<<std::min(4096, ceil_div((int)hin.n, 256)), 256, 0, n->st>>>(hin.p, X0.p, S, din, batch,
                                                                                round_up(din, 2));
    NL_CHECK_LAUNCH();
    DBuf y;
    int ldy = 0;
    net_forward_dev(n, order, X0, ncols, y, ldy, nullptr);
    DBuf hout((size_t)S * dout * batch);
    k_cols_to_parts<<<std::min(4096, ceil_div((int)hout.n, 256)), 256, 0, n->st>>>(y.p, hout.p, S, dout, batch, ldy);
    NL_CHECK_LAUNCH();
    NL_CUDA(cudaMemcpyAsync(parts_out, hout.p, hout.n * 8, cudaMemcpyDeviceToHost, n->st));
    NL_CUDA(cudaStreamSynchronize(n->st));
    return NLROM_OK;
  } catch (const Error& e) {
    return fail(n, e);
  }
}

extern "C" int nlrom_net_backward(nlrom_net* n, int order, const double* x_parts, const double* up_parts, int batch,
                                  double* in_cot, double* param_cot) {
  try {
    if (!n) return NLROM_ERR_ARG;
    if (order < 0 || order > 1)
      throw Error(NLROM_ERR_ORDER, "backward supports real or order-1 complex scalars (SPEC.md:149)");
    NL_CUDA(cudaSetDevice(n->device));
    cudaStream_t st = n->st;
    const int S = 1 << order, ncols = S * batch;
    const int din = n->L[0].in, dout = n->L.back().out;
    DBuf hx((size_t)S * din * batch), X0((size_t)ncols * round_up(din, 2));
    NL_CUDA(cudaMemcpyAsync(hx.p, x_parts, hx.n * 8, cudaMemcpyHostToDevice, st));
    k_parts_to_cols<<<std::min(4096, ceil_div((int)hx.n, 256)), 256, 0, st>>>(hx.p, X0.p, S, din, batch, round_up(din, 2));
    NL_CHECK_LAUNCH();
    FwdRecord rec;
    DBuf y;
    int ldy = 0;
    net_forward_dev(n, order, X0, ncols, y, ldy, &rec);
    // upstream
    DBuf hu((size_t)S * dout * batch);
    int ld = round_up(dout, 2);
    DBuf d((size_t)ncols * ld);
    NL_CUDA(cudaMemcpyAsync(hu.p, up_parts, hu.n * 8, cudaMemcpyHostToDevice, st));
    k_parts_to_cols<<<std::min(4096, ceil_div((int)hu.n, 256)), 256, 0, st>>>(hu.p, d.p, S, dout, batch, ld);
    NL_CHECK_LAUNCH();
    std::vector<DBuf> pgW, pgB;  // per FC layer (in reverse order)
    std::vector<int> fc_idx;
    for (int i = (int)n->L.size() - 1; i >= 0; --i) {
      NetLayer& l = n->L[i];
      const int ldi = round_up(l.in, 2);
      if (l.kind == NLROM_LAYER_FC) {
        if (param_cot) {
          // dW[s] = sum_b d (x) x in (multi)complex arithmetic, via slot-major GEMM over K = batch
          const int ldp = round_up(batch, 2);
          DBuf Dm((size_t)S * l.out * ldp), Xm((size_t)S * l.in * ldp), P((size_t)S * l.in * round_up(S * l.out, 2));
          k_cols_to_slotmajor<<<std::min(4096, ceil_div(S * l.out * batch, 256)), 256, 0, st>>>(d.p, Dm.p, S, l.out,
                                                                                              batch, ld, ldp);
          k_cols_to_slotmajor<<<std::min(4096, ceil_div(S * l.in * batch, 256)), 256, 0, st>>>(
              rec.inputs[i].p, Xm.p, S, l.in, batch, ldi, ldp);
          NL_CHECK_LAUNCH();
          GemmArgs gp{Dm.p, Xm.p, ldp, ldp, S * l.out, S * l.in, batch, 0, 0};
          gemm_auto(gp, EpiStore{P.p, round_up(S * l.out, 2), 0, nullptr, 1, nullptr}, st);
          DBuf dW((size_t)S * l.out * l.in), db((size_t)S * l.out);
          k_param_combine<<<std::min(4096, ceil_div(S * l.out * l.in, 256)), 256, 0, st>>>(
              P.p, round_up(S * l.out, 2), Dm.p, ldp, dW.p, db.p, S, l.out, l.in, batch);
          NL_CHECK_LAUNCH();
          pgW.push_back(std::move(dW));
          pgB.push_back(std::move(db));
          fc_idx.push_back(i);
        }
        // d_in = W^T d, times act'(z) of an activation layer directly below (fused)
        int act_below = ACT_NONE;
        const double* zc = nullptr;
        if (i >= 1 && (n->L[i - 1].kind == NLROM_LAYER_SIN || n->L[i - 1].kind == NLROM_LAYER_SQUARE)) {
          act_below = n->L[i - 1].kind == NLROM_LAYER_SIN ? ACT_SIN_MC : ACT_SQUARE_MC;
          zc = rec.pre[i - 1].p;
        }
        DBuf dn((size_t)ncols * ldi);
        GemmArgs g{l.WT.p, d.p, l.ldwt, ld, l.in, ncols, l.out, 0, 0};
        fc_backward(order, act_below, g, dn.p, ldi, zc, st);
        d = std::move(dn);
        if (act_below != ACT_NONE) {
          --i;  // activation consumed
        }
      } else if (l.kind == NLROM_LAYER_FILTER) {
        DBuf T((size_t)ncols * l.ldu);
        GemmArgs g1{l.Ut.p, d.p, l.ldut, ld, l.nb, ncols, l.in, 0, 0};
        gemm_auto(g1, EpiStore{T.p, l.ldu, 0, nullptr, 1, nullptr}, st);
        DBuf dn((size_t)ncols * ldi);
        GemmArgs g2{l.U.p, T.p, l.ldu, l.ldu, l.out, ncols, l.nb, 0, 0};
        gemm_auto(g2, EpiStore{dn.p, ldi, 0, nullptr, 1, d.p}, st);
        d = std::move(dn);
      } else {
        int act = (l.kind == NLROM_LAYER_SIN) ? ACT_SIN_MC : ACT_SQUARE_MC;
        DBuf dn((size_t)ncols * ldi);
        if (order == 0) act_bwd_cols<1>(act, d.p, rec.pre[i].p, dn.p, ncols, l.in, ldi, st);
        else act_bwd_cols<2>(act, d.p, rec.pre[i].p, dn.p, ncols, l.in, ldi, st);
        d = std::move(dn);
      }
      ld = ldi;
    }
    DBuf hout((size_t)S * din * batch);
    k_cols_to_parts<<<std::min(4096, ceil_div((int)hout.n, 256)), 256, 0, st>>>(d.p, hout.p, S, din, batch, ld);
    NL_CHECK_LAUNCH();
    NL_CUDA(cudaMemcpyAsync(in_cot, hout.p, hout.n * 8, cudaMemcpyDeviceToHost, st));
    if (param_cot) {
      size_t off = 0;
      for (int j = (int)fc_idx.size() - 1; j >= 0; --j) {  // forward layer order
        NL_CUDA(cudaMemcpyAsync(param_cot + off, pgW[j].p, pgW[j].n * 8, cudaMemcpyDeviceToHost, st));
        off += pgW[j].n;
        NL_CUDA(cudaMemcpyAsync(param_cot + off, pgB[j].p, pgB[j].n * 8, cudaMemcpyDeviceToHost, st));
        off += pgB[j].n;
      }
    }
    NL_CUDA(cudaStreamSynchronize(st));
    return NLROM_OK;
  } catch (const Error& e) {
    return fail(n, e);
  }
}
