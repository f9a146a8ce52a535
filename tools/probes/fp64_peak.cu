// Probe: measured fp64 throughput on B200 (DFMA vector pipe vs DMMA tensor pipe)
// and cross-check of the mma.sync f64 fragment layout. Used to pick the fp64
// roofline denominator recorded in profiles/.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 * i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSM : {2, 4, 8}) {
    int grid = p.multiProcessorCount * blocksPerSM, block = 256, iters = 4096;
    dfma_loop<<<grid, block>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)grid * block;
    printf("DFMA  bps=%d  %.2f TFLOP/s\n", blocksPerSM, fl / ms / 1e9);
    dmma_loop<<<grid, block>>>(out, 16);
    cudaEventRecord(e0);
    dmma_loop<<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * grid * (block / 32);
    printf("DMMA.m8n8k4  bps=%d  %.2f TFLOP/s\n", blocksPerSM, fl / ms / 1e9);
    dmma16_loop<<<grid, block>>>(out, 16);
    cudaEventRecord(e0);
    dmma16_loop<<<grid, block>>>(out, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 4 * (double)(iters / 4) * grid * (block / 32);
    printf("DMMA.m16n8k16  bps=%d  %.2f TFLOP/s\n", blocksPerSM, fl / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
