// Probe: per-kernel overhead of dependent launches in a CUDA graph on B200, with and without
// programmatic dependent launch (PDL), for tiny and 148-CTA kernels.
#include <cstdio>
__global__ void k_tiny(double* p, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) p[blockIdx.x] += 1.0;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}
int main() {
  double* p; cudaMalloc(&p, 4096 * 8); cudaMemset(p, 0, 4096 * 8);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(k_tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int grid : {1, 148}) for (int pdl : {0, 1}) for (int smem : {0, 64 * 1024}) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 32; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid; cfg.blockDim = 256; cfg.dynamicSmemBytes = smem; cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = pdl;
      cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_tiny, p, pdl);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, st);
    cudaEventRecord(a, st);
    for (int r = 0; r < 100; ++r) cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid %3d pdl %d smem %6d: %.2f us per kernel (graph of 32)\n", grid, pdl, smem, ms * 1000 / 100 / 32);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
