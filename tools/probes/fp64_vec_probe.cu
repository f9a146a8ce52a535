// Probe: vector (non-tensor) fp64 throughput on one B200: DFMA / DMUL issue rate per SM and the
// cost of the fp64 <-> int64 conversions the Ozaki epilogues use (F2I.S64.F64, I2F.F64.S64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probes/fp64_vec_probe.cu -o tools/probes/fp64_vec_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void loop(double* out, int iters) {
  double a[8];
  long long q[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; q[i] = threadIdx.x + i; }
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fma(a[i], b, c);
      if (OP == 1) a[i] = a[i] * b;
      if (OP == 2) { q[i] = __double2ll_rz(a[i] * 1.5) + q[i]; a[i] = a[i] + 1.0; }
      if (OP == 3) { a[i] = (double)q[i] + a[i]; q[i] += 3; }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + (double)q[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int sms, double* out, int ops_per_iter) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int grid = sms * 4, block = 512, iters = 4096;
  loop<OP><<<grid, block>>>(out, 16);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    loop<OP><<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double n = (double)grid * block * iters * 8 * ops_per_iter;
  const double per_sm_clk = n / (best * 1e-3) / sms / 1.965e9;
  printf("%-28s %.1f G/s  = %.1f per SM per clock (at 1965 MHz)\n", name, n / best / 1e6, per_sm_clk);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, (size_t)p.multiProcessorCount * 4 * 512 * 8);
  run<0>("DFMA", p.multiProcessorCount, out, 1);
  run<1>("DMUL", p.multiProcessorCount, out, 1);
  run<2>("DMUL+F2I.S64 (+IADD64,DADD)", p.multiProcessorCount, out, 1);
  run<3>("I2F.F64.S64 (+DADD,IADD64)", p.multiProcessorCount, out, 1);
  printf("err=%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
