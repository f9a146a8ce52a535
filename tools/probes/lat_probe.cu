// Probe: dependent-chain latencies (clock64) of the operations on the LU pivot-step critical
// path on B200: DFMA, DMUL, REDUX.MAX, SHFL, MUFU RCP64H, fp64 compare+select, LDS, bar.sync.
#include <cstdio>
#include <cstdint>
__device__ long long g_out[32];
__device__ double g_sink;
__global__ void lat(double x0, int n) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  double x = x0 + lane * 1e-3;
  unsigned u = lane;
  long long t0, t1;
  sm[threadIdx.x] = x;
  __syncthreads();
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999, 1e-3);
  t1 = clock64();
  if (threadIdx.x == 0) g_out[0] = (t1 - t0);
  // DMUL
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0001;
  t1 = clock64();
  if (threadIdx.x == 0) g_out[1] = (t1 - t0);
  // REDUX max
  t0 = clock64();
  for (int i = 0; i < n; ++i) u = __reduce_max_sync(0xffffffffu, u + lane);
  t1 = clock64();
  if (threadIdx.x == 0) g_out[2] = (t1 - t0);
  // SHFL double
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64();
  if (threadIdx.x == 0) g_out[3] = (t1 - t0);
  // rcp.approx.f64
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r;
  }
  t1 = clock64();
  if (threadIdx.x == 0) g_out[4] = (t1 - t0);
  // fabs + compare + select
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = fabs(x); x = (v > 0.5) ? v - 0.25 : v + 0.25; }
  t1 = clock64();
  if (threadIdx.x == 0) g_out[5] = (t1 - t0);
  // LDS dependent (pointer chase through an index)
  int* si = reinterpret_cast<int*>(sm + 512);
  si[threadIdx.x] = (threadIdx.x + 1) & 255;
  __syncthreads();
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) idx = si[idx];
  t1 = clock64();
  if (threadIdx.x == 0) g_out[6] = (t1 - t0);
  // bar.sync 256 threads
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (threadIdx.x == 0) g_out[7] = (t1 - t0);
  // full division
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.5);
  t1 = clock64();
  if (threadIdx.x == 0) g_out[8] = (t1 - t0);
  g_sink = x + u + idx;
}
int main() {
  const int n = 256;
  lat<<<1, 256, 8192>>>(1.0, n);
  cudaDeviceSynchronize();
  lat<<<1, 256, 8192>>>(1.0, n);
  long long h[32];
  cudaMemcpyFromSymbol(h, g_out, sizeof h);
  const char* names[] = {"DFMA", "DMUL", "REDUX.MAX", "SHFL.f64", "RCP64 approx", "fabs+cmp+sel f64", "LDS chase",
                         "bar.sync(256)", "1/x IEEE"};
  for (int i = 0; i < 9; ++i) printf("%-18s %6.1f cycles\n", names[i], (double)h[i] / n);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
