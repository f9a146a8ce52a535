// Shared helpers for the nlrom_b200 sm_100a kernels.
#pragma once
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
      NL_CUDA(cudaMemset(p, 0, count * sizeof(double)));
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
    }
  }
  void upload(const int* h, size_t count) {
    alloc(count);
    if (count) NL_CUDA(cudaMemcpy(p, h, count * sizeof(int), cudaMemcpyHostToDevice));
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

// Upload a (rows, cols) row-major host matrix into a device matrix with leading
// dimension ld (>= cols); padding is zero.
void upload_matrix(DBuf& dst, const double* h, int rows, int cols, int ld, int rows_alloc = -1);

}  // namespace nlrom
