// Shared helpers for the nlrom_b200 sm_100a kernels.
#pragma once
#include <vector>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <stdexcept>

#include "../../include/nlrom_b200.h"

namespace nlrom {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define NL_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      throw ::nlrom::Error(NLROM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define NL_CHECK_LAUNCH() NL_CUDA(cudaGetLastError())

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Launch gate for prefix-graph profiling (nlrom_bench_prefix): while a budget is set, only the
// first `budget` kernel launches are issued and their entry points are logged.
constexpr int kNoBudget = 1 << 30;
inline int& launch_budget() { static int b = kNoBudget; return b; }
inline std::vector<const void*>& launch_log() { static std::vector<const void*> v; return v; }
// Timing experiments only, compiled in with -DNLROM_TIMING_EXPERIMENTS (never in the release
// library): NLROM_DEBUG_SKIP=name1,name2 drops every launch whose kernel name contains one of
// the substrings (results are then wrong; used to find the critical path).
inline bool launch_skipped(const void* fn) {
#ifndef NLROM_TIMING_EXPERIMENTS
  (void)fn;
  return false;
#else
  static const char* env = getenv("NLROM_DEBUG_SKIP");
  if (!env || !*env) return false;
  const char* name = nullptr;
  if (cudaFuncGetName(&name, fn) != cudaSuccess || !name) return false;
  std::string list(env), nm(name);
  size_t pos = 0;
  while (pos <= list.size()) {
    size_t e = list.find(',', pos);
    if (e == std::string::npos) e = list.size();
    const std::string tok = list.substr(pos, e - pos);
    if (!tok.empty() && nm.find(tok) != std::string::npos) return true;
    pos = e + 1;
  }
  return false;
#endif
}
inline bool launch_gate(const void* fn) {
  if (launch_skipped(fn)) return false;
  int& b = launch_budget();
  if (b >= kNoBudget) return true;
  if (b <= 0) return false;
  --b;
  launch_log().push_back(fn);
  return true;
}
inline int round_up(int a, int b) { return ceil_div(a, b) * b; }

// Device buffer (owning). Zero-initialised so padded rows / columns read as 0.
struct DBuf {
  double* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    free();
    n = count;
    if (count) {
      NL_CUDA(cudaMalloc(&p, count * sizeof(double)));
      // the zero fill runs on the legacy stream, which does not order against the contexts'
      // non-blocking streams: wait for it, or a kernel enqueued next on a context stream could
      // write the buffer before the fill lands (a per-call diffop output read back as zeros)
      NL_CUDA(cudaMemset(p, 0, count * sizeof(double)));
      NL_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { free(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept { free(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; return *this; }
};

// pinned host staging buffer (fast async host<->device copies for the host-buffer API)
struct HBuf {
  double* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    if (count <= n) return;
    free();
    NL_CUDA(cudaHostAlloc(&p, count * sizeof(double), cudaHostAllocDefault));
    n = count;
  }
  void free() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
  ~HBuf() { free(); }
};

struct IBuf {
  int* p = nullptr;
  size_t n = 0;
  IBuf() = default;
  void alloc(size_t count) {
    free();
    n = count;
    if (count) {
      NL_CUDA(cudaMalloc(&p, count * sizeof(int)));
      NL_CUDA(cudaMemset(p, 0, count * sizeof(int)));
      NL_CUDA(cudaStreamSynchronize(cudaStreamLegacy));   // (as DBuf::alloc)
    }
  }
  void upload(const int* h, size_t count) {
    alloc(count);
    if (count) {
      NL_CUDA(cudaMemcpy(p, h, count * sizeof(int), cudaMemcpyHostToDevice));
      NL_CUDA(cudaStreamSynchronize(cudaStreamLegacy));   // pageable H2D: the DMA may still be in flight
    }
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~IBuf() { free(); }
  IBuf(const IBuf&) = delete;
  IBuf& operator=(const IBuf&) = delete;
};

// Programmatic dependent launch (kernels are captured with programmatic stream
// serialisation): wait for the producer grid before touching its outputs; allow the
// next grid to start its independent prologue (e.g. weight prefetch) early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// 8-byte async global->shared copy: staging loops issue every load before any
// result is needed (a plain load->st.shared loop serialises on memory latency).
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_all_wait() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// Upload a (rows, cols) row-major host matrix into a device matrix with leading
// dimension ld (>= cols); padding is zero.
void upload_matrix(DBuf& dst, const double* h, int rows, int cols, int ld, int rows_alloc = -1);

}  // namespace nlrom
