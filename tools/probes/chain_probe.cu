// Probe: where the time of one layer of the fused hidden jet chain goes (cfg2 shape:
// w = 256, 9 hidden layers, G = 16 columns per group, 10 groups, 8-CTA clusters).
// Phase timestamps from CTA (0,0): weights landed | DMMA done | epilogue done |
// broadcast done | cluster barrier done.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DNLROM_CHAIN_TRACE \
//        -I../../paper_2102_11026_b200/csrc chain_probe.cu -o chain_probe
#include <cstdio>
#include <vector>
#include <random>
#include "mlp_chain.cuh"

using namespace nlrom;

int main() {
  const int w = 256, nq = 30, np = 30, n = np + nq, L1 = 9, G = 16, gps = 10;
  constexpr int R = 32, CS = 8;
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> U(-0.06, 0.06);
  MlpFwdArgs a{};
  std::vector<double> h;
  auto dev = [&](size_t cnt, bool rnd) {
    h.assign(cnt, 0.0);
    if (rnd)
      for (auto& x : h) x = U(rng);
    double* d;
    cudaMalloc(&d, cnt * 8);
    cudaMemcpy(d, h.data(), cnt * 8, cudaMemcpyHostToDevice);
    return d;
  };
  a.r = dev(n, true);
  a.rbar = dev(n, true);
  a.rdbar = dev(n, true);
  a.n_p = np; a.n_q = nq; a.n = n; a.dt = 1.0 / 60; a.alpha = 0.1; a.drop_fict = 0;
  a.L1 = L1; a.w = w;
  const int ldp = 256 + 4;
  a.ldp = ldp;
  for (int l = 0; l < L1; ++l) {
    const int in = l ? w : nq;
    a.W[l] = dev((size_t)w * in, true);
    {
      std::vector<double> wp((size_t)w * ldp, 0.0);
      for (int r = 0; r < w; ++r)
        for (int k = 0; k < in; ++k) wp[(size_t)r * ldp + k] = h[(size_t)r * in + k];
      double* d;
      cudaMalloc(&d, wp.size() * 8);
      cudaMemcpy(d, wp.data(), wp.size() * 8, cudaMemcpyHostToDevice);
      a.Wp[l] = d;
    }
    a.b[l] = dev(w, true);
    a.ldW[l] = in;
    a.in[l] = in;
    a.cache[l] = dev((size_t)2 * nq * w, false);
  }
  a.ldc = w;
  a.Hout = dev((size_t)(4 + 4 * nq) * w, false);
  a.ldH = w;
  a.G = G; a.gps = gps;
  auto run = [&](bool async_chain) {
    (void)async_chain;   // the st.async variant is retired (tools/probes/retired/mlp_chain_async.cuh)
    auto kern = k_mlp_jet_fwd<R, G, CS>;
    const size_t smem = MlpPlan<R, G>::bytes(w);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS, gps, 1);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 5; ++it) cudaLaunchKernelEx(&cfg, kern, a);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) cudaLaunchKernelEx(&cfg, kern, a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s: %.2f us per launch (back-to-back, smem %zu B) err=%s\n",
           async_chain ? "k_mlp_jet_fwd_async<32,16,8>" : "k_mlp_jet_fwd<32,16,8>", ms / 20 * 1e3, smem,
           cudaGetErrorString(cudaGetLastError()));
    long long tr[MLP_MAXL][6];
    cudaMemcpyFromSymbol(tr, g_chain_trace, sizeof tr);
    printf("layer  wait_w  dmma  epi+send  barrier  total (cycles)\n");
    for (int l = 0; l < L1; ++l) {
      long long prev = (l == 0) ? tr[0][0] : tr[l - 1][5];
      printf("%5d %7lld %5lld %9lld %8lld %6lld\n", l, tr[l][1] - prev, tr[l][2] - tr[l][1], tr[l][4] - tr[l][2],
             tr[l][5] - tr[l][4], tr[l][5] - prev);
    }
    std::vector<double> out((size_t)(4 + 4 * nq) * w);
    cudaMemcpy(out.data(), a.Hout, out.size() * 8, cudaMemcpyDeviceToHost);
    double cs = 0;
    for (double v : out) cs += v;
    std::vector<double> cache((size_t)2 * nq * w);
    cudaMemcpy(cache.data(), a.cache[4], cache.size() * 8, cudaMemcpyDeviceToHost);
    for (double v : cache) cs += v;
    printf("checksum %.17g\n", cs);
  };
  run(false);
  // ---- vhp backward chain <32, 8, 8> on the caches of the forward run
  {
    constexpr int RB = 32, CSB = 8, GB = 8;
    MlpBwdArgs b{};
    std::vector<double> gh(w);
    for (auto& x : gh) x = U(rng);
    double* gd;
    cudaMalloc(&gd, w * 8);
    cudaMemcpy(gd, gh.data(), w * 8, cudaMemcpyHostToDevice);
    b.g = gd; b.gpart = nullptr; b.L1 = L1; b.w = w; b.n_q = nq;
    const int ldpb = 256 + 4;
    for (int l = 0; l < L1; ++l) {
      const int in = l ? w : nq;
      std::vector<double> wtp((size_t)w * ldpb, 0.0);
      std::vector<double> wl((size_t)w * in);
      cudaMemcpy(wl.data(), a.W[l], wl.size() * 8, cudaMemcpyDeviceToHost);
      for (int r = 0; r < w; ++r)
        for (int k = 0; k < in; ++k) wtp[(size_t)k * ldpb + r] = wl[(size_t)r * in + k];
      double* d;
      cudaMalloc(&d, wtp.size() * 8);
      cudaMemcpy(d, wtp.data(), wtp.size() * 8, cudaMemcpyHostToDevice);
      b.WTp[l] = d;
      b.cache[l] = a.cache[l];
    }
    b.ldpb = ldpb; b.ldc = w;
    double* Gt;
    cudaMalloc(&Gt, (size_t)2 * nq * w * 8);
    b.Gt = Gt; b.ldG = w;
    b.gpb = (nq + GB / 2 - 1) / (GB / 2);
    const size_t smem = mlp_bwd_smem<RB, GB>(w);
    cudaFuncSetAttribute(k_mlp_dual_bwd<RB, CSB, GB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CSB, b.gpb, 1);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CSB;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 5; ++it) cudaLaunchKernelEx(&cfg, k_mlp_dual_bwd<RB, CSB, GB>, b);
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) cudaLaunchKernelEx(&cfg, k_mlp_dual_bwd<RB, CSB, GB>, b);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("k_mlp_dual_bwd<32,8,8>: %.2f us per launch (smem %zu B) err=%s\n", ms / 20 * 1e3, smem,
           cudaGetErrorString(cudaGetLastError()));
    long long tr[MLP_MAXL + 1][6];
    cudaMemcpyFromSymbol(tr, g_bwd_trace, sizeof tr);
    printf("stage  wait   dmma  epilogue  bcast  barrier  total (cycles)\n");
    for (int st = 1; st <= L1; ++st) {
      long long prev = tr[st - 1][5];
      printf("%5d %6lld %6lld %9lld %6lld %8lld %6lld\n", st, tr[st][1] - tr[st][0], tr[st][2] - tr[st][1],
             tr[st][3] - tr[st][2], tr[st][4] - tr[st][3], tr[st][5] - tr[st][4], tr[st][5] - prev);
    }
  }
  return 0;
}
