// Shared device/host helpers for the B200 CN-WSGD hot path.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace fde_b200 {

// Error classes of the C-ABI (include/fde_b200.h) -- the reference throws
// std::invalid_argument / std::runtime_error; we carry the same distinction.
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
// Kernels launched by this library since load (fde_kernel_launches()).
extern std::atomic<unsigned long long> g_kernel_launches;

#define FDE_CUDA(call) ::fde_b200::cuda_check((call), #call)
#define FDE_LAUNCH_CHECK()                                                  \
  do {                                                                      \
    ::fde_b200::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
    ::fde_b200::cuda_check(cudaGetLastError(), "kernel launch");            \
  } while (0)

// ---- complex helpers on double2 (x = re, y = im) ---------------------------
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 conjg(double2 a) { return make_double2(a.x, -a.y); }

}  // namespace fde_b200
