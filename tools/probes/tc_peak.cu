// Probe: measured tensor-pipe peaks on one B200, the roofline denominators bench.py reports
// against (profiles/r02_tc_peaks.json, written by tools/tc_peaks.py, which samples SM clocks
// with nvidia-smi while this runs).
//   * fp64 DMMA (mma.sync m8n8k4 / m16n8k16): the decoder's DMMA kernels.
//   * tcgen05.mma kind::i8 (M = 128, K = 32, N = 64 and 256, operands resident in shared
//     memory, accumulators in TMEM): the Ozaki hidden-layer GEMM (csrc/ozaki_tc.cuh) issues
//     M = 128, N = 64 (BN) instructions, so its ceiling is the N = 64 rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//          tools/probes/tc_peak.cu -o tools/probes/tc_peak
#include <cstdio>
#include <cstdint>
#include "../../paper_2102_11026_b200/csrc/ozaki_tc.cuh"
using namespace nlrom;

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// One CTA per SM. Thread 0 issues `iters` kind::i8 MMAs round-robin over NACCUM TMEM
// accumulators (independent chains), then one commit; the CTA waits on it.
template <int N, int NACCUM>
__global__ void __launch_bounds__(128, 1) i8_loop(int iters, int* out) {
  __shared__ __align__(1024) unsigned char sa[oz::BM * oz::BK];
  __shared__ __align__(1024) unsigned char sb[N * oz::BK];
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < oz::BM * oz::BK; i += 128) sa[i] = (unsigned char)(i * 7 + 1);
  for (int i = tid; i < N * oz::BK; i += 128) sb[i] = (unsigned char)(i * 5 + 3);
  if (tid == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  // TMEM allocations are a power of two >= 32 columns
  constexpr uint32_t COLS = N * NACCUM <= 32 ? 32 : N * NACCUM <= 64 ? 64 : N * NACCUM <= 128 ? 128
                          : N * NACCUM <= 256 ? 256 : 512;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                 "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  oz::tc_fence_before();
  __syncthreads();
  oz::tc_fence_after();
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint64_t ad = oz::smem_desc(smem_u32(sa)), bd = oz::smem_desc(smem_u32(sb));
    const uint32_t idesc = oz::idesc_i8(N);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int a = 0; a < NACCUM; ++a) oz::mma_i8(tmem + a * N, ad, bd, idesc, it > 0 ? 1u : 0u);
    }
    oz::tc_commit(&done);
  }
  __syncwarp();
  mbar_wait_cta(&done, 0);
  oz::tc_fence_after();
  if (warp == 0) {  // read one accumulator row back so the work is observable
    int r[16];
    oz::tmem_ld16(tmem, r);
    oz::tmem_wait_ld();
    if (blockIdx.x == 0) out[tid] = r[0] + r[15];
  }
  oz::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    oz::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(COLS));
  }
}

template <int N, int NACCUM>
static double run_i8(int sms, int* out, cudaEvent_t e0, cudaEvent_t e1, int iters) {
  i8_loop<N, NACCUM><<<sms, 128>>>(16, out);
  NL_CUDA(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    i8_loop<N, NACCUM><<<sms, 128>>>(iters, out);
    cudaEventRecord(e1);
    NL_CUDA(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * oz::BM * N * oz::BK * (double)iters * NACCUM * sms;
  const double tops = ops / best / 1e9;
  printf("I8 N=%d accum=%d  %.1f TOP/s  (%.3f ms)\n", N, NACCUM, tops, best);
  return tops;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  cudaDeviceProp p;
  NL_CUDA(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  printf("device %s SMs %d\n", p.name, sms);
  double* dout;
  int* iout;
  NL_CUDA(cudaMalloc(&dout, (size_t)sms * 8 * 256 * sizeof(double)));
  NL_CUDA(cudaMalloc(&iout, 128 * sizeof(int)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // fp64 DMMA: 8 CTAs of 256 threads per SM, several long launches (the clock sampler needs
  // a sustained load), best of 5
  {
    const int grid = sms * 8, block = 256, iters = 65536;
    dmma_loop<<<grid, block>>>(dout, 16);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dmma_loop<<<grid, block>>>(dout, iters);
      cudaEventRecord(e1);
      NL_CUDA(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double fl = 2.0 * 8 * 8 * 4 * 8 * (double)iters * grid * (block / 32);
    printf("DMMA.m8n8k4 %.2f TFLOP/s  (%.3f ms)\n", fl / best / 1e9, best);
  }
  const int it = 1 << 17;
  run_i8<64, 1>(sms, iout, e0, e1, it);
  run_i8<64, 4>(sms, iout, e0, e1, it / 4);
  run_i8<64, 7>(sms, iout, e0, e1, it / 7);
  run_i8<128, 2>(sms, iout, e0, e1, it / 4);
  run_i8<256, 1>(sms, iout, e0, e1, it / 4);
  run_i8<256, 2>(sms, iout, e0, e1, it / 8);
  cudaError_t err = cudaDeviceSynchronize();
  printf("err=%s\n", cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
