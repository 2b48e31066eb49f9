// Do FP64 and shared-memory (LSU) work overlap on one SM?  16 warps per SM
// (4 CTAs x 128 threads) run F DFMAs and/or S LDS.64+STS.64 pairs per
// iteration; cycles per iteration for FP64 only, LSU only, both in every warp,
// and split (even warps FP64, odd warps LSU).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_overlap tools/pipe_overlap.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(128, 4) k(double* out, long long* clk, int iters) {
  __shared__ double sm[128 * 16];
  double a[8], s[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; s[i] = i; }
  for (int i = threadIdx.x; i < 128 * 16; i += 128) sm[i] = i;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const bool do_f = MODE == 0 || MODE == 2 || (MODE == 3 && (warp & 1) == 0);
  const bool do_s = MODE == 1 || MODE == 2 || (MODE == 3 && (warp & 1) == 1);
  const double c = 1.0000001, d = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (do_f) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[i]) : "d"(c), "d"(d));
    }
    if (do_s) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double t;
        const unsigned ad = (unsigned)__cvta_generic_to_shared(sm + threadIdx.x + 128 * i);
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(t) : "r"(ad));
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(ad + 8 * 128 * 8), "d"(s[i]));
        s[i] = t;
      }
    }
  }
  long long t1 = clock64();
  double acc = 0;
  for (int i = 0; i < 8; ++i) acc += a[i] + s[i];
  if (acc == 1.2345) out[0] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int MODE>
double run(double* out, long long* clk, int iters) {
  k<MODE><<<148 * 4, 128>>>(out, clk, iters);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<148 * 4, 128>>>(out, clk, iters);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  printf("[%.1f us total, %.2f ns/iter] ", ms * 1e3, ms * 1e6 / iters);
  static long long h[592];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 592; ++i) s += h[i];
  return s / 592 / iters;
}
int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 8); cudaMalloc(&clk, 8 * 1024);
  const int iters = 20000;
  printf("per iteration (64 DFMA and/or 8 LDS.64 + 8 STS.64 per thread, 16 warps/SM):\n");
  printf("  FP64 only : %.1f clk (pipe floor 16 warps x 64 / 2 per clk = 512)\n", run<0>(out, clk, iters));
  printf("  LSU only  : %.1f clk (floor 16 warps x 16 x 2 wavefronts = 512)\n", run<1>(out, clk, iters));
  printf("  both/warp : %.1f clk\n", run<2>(out, clk, iters));
  printf("  split     : %.1f clk (8 warps FP64, 8 warps LSU: floor 256 each)\n", run<3>(out, clk, iters));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
