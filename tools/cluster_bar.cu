// Microbenchmark: cost of barrier.cluster (arrive.release + wait.acquire) for
// one cluster of C CTAs x T threads, K barriers per launch, with and without a
// DSMEM broadcast of one double per thread before each barrier.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void kbar(int K, int bc, double* out) {
  extern __shared__ double sm[];
  const int ctas = gridDim.x;
  double v = threadIdx.x;
  for (int k = 0; k < K; ++k) {
    if (bc) {
      const unsigned a = (unsigned)__cvta_generic_to_shared(sm + threadIdx.x);
      for (int r = 0; r < ctas; ++r) {
        unsigned ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
      }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    v += sm[(threadIdx.x + 1) % blockDim.x];
  }
  if (v == -1.0) out[0] = v;
}
__global__ void kempty(double* out) { if (threadIdx.x == 12345) out[0] = 1; }

int main() {
  double* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(kbar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(kbar, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int C : {2, 4, 8, 16})
    for (int T : {128, 512})
      for (int bc : {0, 1})
        for (int K : {1, 101}) {
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = C;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cudaLaunchConfig_t cfg{};
          cfg.gridDim = dim3(C);
          cfg.blockDim = dim3(T);
          cfg.dynamicSmemBytes = 64 * 1024;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, kbar, K, bc, out);
          cudaEventRecord(a);
          for (int r = 0; r < 20; ++r) cudaLaunchKernelEx(&cfg, kbar, K, bc, out);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          printf("cluster %2d x %3d thr bcast %d: %3d barriers %8.2f us/launch  %s\n", C, T, bc, K,
                 ms * 1e3 / 20, cudaGetErrorString(cudaGetLastError()));
        }
  cudaEventRecord(a);
  for (int r = 0; r < 100; ++r) kempty<<<1, 32>>>(out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("empty kernel: %.2f us/launch\n", ms * 1e3 / 100);
  return 0;
}
