// RAII device buffer (owned HBM allocation).
#pragma once
#include <utility>

#include "common.cuh"

namespace fde_b200 {

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
    }
    return *this;
  }
  void alloc(size_t n) {
    release();
    if (n == 0) return;
    // 16 bytes of slack: the line kernels' bulk copies move whole 16-byte
    // chunks and may read up to 8 bytes past the last element of an array
    FDE_CUDA(cudaMalloc(&p_, n * sizeof(T) + 16));
    n_ = n;
  }
  void upload(const T* h, size_t n) {
    if (n != n_) alloc(n);
    if (n) FDE_CUDA(cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void zero(cudaStream_t s = nullptr) const {
    if (n_) FDE_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace fde_b200
