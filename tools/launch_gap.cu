// Launch-gap probe: a CUDA graph of K dependent small kernels, with and
// without programmatic dependent launch (PDL).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void small(double* a, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = a[i] * 1.0000001 + 1.0;
  if (pdl) asm volatile("griddepcontrol.launch_dependents;");
}
int main() {
  const int n = 1 << 16, K = 200;
  double* a;
  cudaMalloc(&a, n * sizeof(double));
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int blocks : {1, 64, 256}) {
      cudaGraph_t g;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = blocks; cfg.blockDim = 256; cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
        cudaLaunchKernelEx(&cfg, small, a, blocks * 256 < n ? blocks * 256 : n, pdl);
      }
      cudaStreamEndCapture(s, &g);
      cudaGraphExec_t e;
      if (cudaGraphInstantiate(&e, g, 0) != cudaSuccess) { printf("inst fail\n"); return 1; }
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(e, s);
      cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
      cudaEventRecord(t0, s);
      for (int r = 0; r < 10; ++r) cudaGraphLaunch(e, s);
      cudaEventRecord(t1, s);
      cudaEventSynchronize(t1);
      float ms; cudaEventElapsedTime(&ms, t0, t1);
      printf("pdl=%d blocks=%d: %.2f us per kernel (%s)\n", pdl, blocks, ms * 1e3 / (10 * K),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
