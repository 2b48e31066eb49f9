// Shared device/host helpers for the B200 CN-WSGD hot path.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

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

// ---- tracing -------------------------------------------------------------
// NVTX range over a host-side phase (time step, Krylov solve, V-cycle,
// operator apply): shows up in Nsight timelines, a no-op without a tool
// attached (header-only NVTX 3).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- one-time per-device setup --------------------------------------------
// Kernel attributes (opt-in shared memory, carveout) and occupancy-derived
// grids belong to a device, not to the process: a second GPU touched by the
// same process needs its own setup.  DeviceCache<T> maps the current device
// to a value built on first use.
inline int current_device() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  return dev;
}
template <class T>
class DeviceCache {
 public:
  template <class Make>
  T& get(Make&& make) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu_);
    auto it = vals_.find(dev);
    if (it == vals_.end()) it = vals_.emplace(dev, make(dev)).first;
    return it->second;
  }

 private:
  std::mutex mu_;
  std::map<int, T> vals_;
};

// ---- programmatic dependent launch ---------------------------------------
// Every kernel is launched with programmatic stream serialization and opens
// with pdl_enter(): it lets the next kernel in the stream (or captured graph)
// be launched as soon as all of this grid's CTAs are running, then waits for
// the previous kernel to complete and flush before touching memory.  Kernel
// boundaries then overlap launch processing and CTA dispatch with the tail of
// the previous grid (the V-cycle's coarse levels are chains of short kernels).
// FDE_PDL=0 in the environment launches plainly (the waits become no-ops).
__device__ __forceinline__ void pdl_enter() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_launch_dependents() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
bool pdl_enabled();
// Plain (fully serialised) launches while a PdlOff is alive on this thread.
// The multi-GPU path interleaves kernels with copy-engine nodes (virtual-rank
// device copies, small host<->device scalar copies): a kernel launched with
// programmatic serialization right after such a node was observed to start
// before the copy had landed (GMRES coefficients read stale; FDE_PDL=0 or
// this scope removes it), and NCCL kernels never trigger early anyway.
inline int& pdl_off_depth() {
  static thread_local int depth = 0;
  return depth;
}
struct PdlOff {
  PdlOff() { ++pdl_off_depth(); }
  ~PdlOff() { --pdl_off_depth(); }
  PdlOff(const PdlOff&) = delete;
  PdlOff& operator=(const PdlOff&) = delete;
};

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t s, Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl_enabled() && pdl_off_depth() == 0) ? 1 : 0;
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "kernel launch");
}

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
