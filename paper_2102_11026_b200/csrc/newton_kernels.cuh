// Adaptive Newton on the device (rdsim.step): the convergence test, the
// backtracking line search (<= 10 halvings) and the max_iters limit run inside ONE CUDA graph
// as two nested conditional while nodes (CUDA 12.4+), set by the single-thread kernels below:
//
//   prologue:  inputs H2D, predictor r = r_bar + dt rdot_bar, E(r) -> ||phi||, k_nt_init
//   while (outer):                        Newton iterations
//     J(r) -> dr (vhp + LU-pp), k_nt_ls_begin (rsave = r, t = 1)
//     while (inner):                      line search
//       k_nt_axpy (r = rsave + t dr), E(r) -> ||phi||, k_nt_ls_check
//     k_nt_check                          converged / max_iters / keep going
//   epilogue:  rdot = (r - r_bar) / dt, outputs + state D2H
//
// State (device doubles): [0] ||phi|| of the accepted iterate, [1] t, [2] iterations, [3] line-search
// trial, [4] status (0 ok, 1 singular LU, 2 non-finite residual, 3 max_iters reached).
// Same decisions as the host loop it replaces: iterate while ||phi|| > tol; a trial is accepted
// when the line search is off, the norm decreased, or after the 11th trial.
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace nlrom {

enum { NT_NORM = 0, NT_T = 1, NT_IT = 2, NT_K = 3, NT_STATUS = 4, NT_SIZE = 8 };
enum { NT_OK = 0, NT_SINGULAR = 1, NT_NONFINITE = 2, NT_MAXITER = 3 };

__global__ void k_nt_init(cudaGraphConditionalHandle outer, const double* __restrict__ norm, double* __restrict__ ad,
                          double tol, int max_iters) {
  pdl_wait();
  pdl_launch();
  const double nv = norm[0];
  ad[NT_NORM] = nv;
  ad[NT_T] = 1.0;
  ad[NT_IT] = 0.0;
  ad[NT_K] = 0.0;
  int status = isfinite(nv) ? NT_OK : NT_NONFINITE;
  const bool go = status == NT_OK && nv > tol;
  if (go && max_iters <= 0) status = NT_MAXITER;
  ad[NT_STATUS] = status;
  cudaGraphSetConditional(outer, (go && status == NT_OK) ? 1u : 0u);
}

__global__ void k_nt_ls_begin(cudaGraphConditionalHandle inner, const int* __restrict__ lu_status,
                              const double* __restrict__ r, double* __restrict__ rsave, double* __restrict__ ad, int n) {
  pdl_wait();
  pdl_launch();
  for (int i = threadIdx.x; i < n; i += blockDim.x) rsave[i] = r[i];
  if (threadIdx.x == 0) {
    ad[NT_T] = 1.0;
    ad[NT_K] = 0.0;
    const bool singular = lu_status[0] != 0;
    if (singular) ad[NT_STATUS] = NT_SINGULAR;
    cudaGraphSetConditional(inner, singular ? 0u : 1u);
  }
}

__global__ void k_nt_axpy(double* __restrict__ r, const double* __restrict__ rsave, const double* __restrict__ dr,
                          const double* __restrict__ ad, int n) {
  pdl_wait();
  pdl_launch();
  const double t = ad[NT_T];
  for (int i = threadIdx.x; i < n; i += blockDim.x) r[i] = fma(t, dr[i], rsave[i]);
}

__global__ void k_nt_ls_check(cudaGraphConditionalHandle inner, const double* __restrict__ norm, double* __restrict__ ad,
                              int line_search) {
  pdl_wait();
  pdl_launch();
  const double nt = norm[0];
  if (!isfinite(nt)) {
    ad[NT_STATUS] = NT_NONFINITE;
    cudaGraphSetConditional(inner, 0u);
    return;
  }
  if (!line_search || nt < ad[NT_NORM] || ad[NT_K] >= 10.0) {
    ad[NT_NORM] = nt;
    cudaGraphSetConditional(inner, 0u);
  } else {
    ad[NT_T] *= 0.5;
    ad[NT_K] += 1.0;
    cudaGraphSetConditional(inner, 1u);
  }
}

__global__ void k_nt_check(cudaGraphConditionalHandle outer, double* __restrict__ ad, double tol, int max_iters) {
  pdl_wait();
  pdl_launch();
  if (ad[NT_STATUS] != NT_OK) {
    cudaGraphSetConditional(outer, 0u);
    return;
  }
  ad[NT_IT] += 1.0;
  if (ad[NT_NORM] <= tol) {
    cudaGraphSetConditional(outer, 0u);
  } else if (ad[NT_IT] >= max_iters) {
    ad[NT_STATUS] = NT_MAXITER;
    cudaGraphSetConditional(outer, 0u);
  } else {
    cudaGraphSetConditional(outer, 1u);
  }
}

}  // namespace nlrom
