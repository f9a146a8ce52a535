// Probe: cost of the per-step building blocks of an in-CTA LU on B200.
#include <cstdio>
__global__ void k_sync(int steps, double* out, int nthreads_active) {
  __shared__ double s[256];
  double acc = threadIdx.x;
  for (int k = 0; k < steps; ++k) {
    s[threadIdx.x] = acc;
    __syncthreads();
    acc += s[(threadIdx.x + k) & 255] * 1e-9;
    __syncthreads();
  }
  out[threadIdx.x] = acc;
}
__global__ void k_shfl(int steps, double* out) {
  double acc = threadIdx.x;
  for (int k = 0; k < steps; ++k) {
#pragma unroll
    for (int o = 8; o; o >>= 1) acc = fmax(acc, __shfl_xor_sync(0xffffffffu, acc, o)) + 1e-9;
  }
  out[threadIdx.x] = acc;
}
__global__ void k_div(int steps, double* out) {
  double acc = threadIdx.x + 1.5;
  for (int k = 0; k < steps; ++k) acc = 1.0 / acc + 0.5;
  out[threadIdx.x] = acc;
}
__global__ void k_fma(int steps, double* out) {
  double acc = threadIdx.x + 1.5;
  for (int k = 0; k < steps; ++k) acc = fma(acc, 0.999, 1e-3);
  out[threadIdx.x] = acc;
}
int main() {
  double* out; cudaMalloc(&out, 4096 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  const int steps = 10000;
  for (int bs : {64, 128, 256}) {
    k_sync<<<1, bs>>>(10, out, bs);
    cudaEventRecord(a); k_sync<<<1, bs>>>(steps, out, bs); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("2x syncthreads+lds/sts per step, %d threads: %.1f ns/step\n", bs, ms * 1e6 / steps);
  }
  k_shfl<<<1, 32>>>(10, out);
  cudaEventRecord(a); k_shfl<<<1, 32>>>(steps, out); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("4 dependent fp64 shfl+fmax: %.1f ns/step\n", ms * 1e6 / steps);
  cudaEventRecord(a); k_div<<<1, 32>>>(steps, out); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("dependent fp64 div: %.1f ns\n", ms * 1e6 / steps);
  cudaEventRecord(a); k_fma<<<1, 32>>>(steps, out); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b); printf("dependent DFMA: %.2f ns\n", ms * 1e6 / steps);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock %d kHz\n", clk);
}
