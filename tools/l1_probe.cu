// L1 capacity probe under a given shared-memory carveout: 4 CTAs/SM of 128
// threads read a W-byte table (coalesced 16-byte read-only loads, serialised
// through the loaded value) over and over; the time per load shows whether the
// table stays in L1 (~35 cycles) or comes from L2 (~250+).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l1_probe tools/l1_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128, 4) probe(const double2* tab, int entries, int reps, double* out, long long* clk) {
  extern __shared__ double sm[];
  int idx = threadIdx.x;
  double acc = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < entries; i += 128) {
      double2 v;
      asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(tab + i + idx - threadIdx.x));
      acc += v.x;
      idx = threadIdx.x + (int)v.y;  // table holds zeros: serialises the loads
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  if (acc == 123.0) out[0] = acc + sm[0];
}
int main() {
  double2* tab; double* out; long long* clk;
  cudaMalloc(&tab, 1 << 20); cudaMemset(tab, 0, 1 << 20);
  cudaMalloc(&out, 8); cudaMalloc(&clk, 8 * 1024);
  for (int smem_kb : {32, 40, 48}) {
    int smem = smem_kb * 1024 - 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int carve : {-1, 60, 72, 86, 100}) {
      cudaFuncSetAttribute(probe, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
      printf("smem/CTA %d KB carveout %d:", smem_kb, carve);
      for (int kb : {8, 16, 24, 32, 40, 48, 56, 64, 80, 96, 128}) {
        int entries = kb * 1024 / 16, reps = 40;
        probe<<<148 * 4, 128, smem>>>(tab, entries, reps, out, clk);
        cudaDeviceSynchronize();
        long long h[592]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0; for (int i = 0; i < 592; ++i) s += h[i];
        printf(" %dK:%.0f", kb, s / 592 / (double(reps) * (entries / 128)));
      }
      printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
