#include "stencil.cuh"

namespace fde_b200 {
namespace {

__global__ void k_stencil(int n1, int n2, const double* __restrict__ coef,
                          const double* __restrict__ x, double* out, int epi,
                          const double* __restrict__ b, const double* __restrict__ dinv,
                          double omega) {
  pdl_enter();
  const size_t n = (size_t)n1 * n2;
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(p % n1), j = (int)(p / n1);
    double s = 0.0;  // CSR row order: increasing column index (sparse.cpp:42-49)
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj) {
      const int jj = j + dj;
      if (jj < 0 || jj >= n2) continue;
#pragma unroll
      for (int di = -1; di <= 1; ++di) {
        const int ii = i + di;
        if (ii < 0 || ii >= n1) continue;
        const double c = coef[(size_t)((dj + 1) * 3 + di + 1) * n + p];
        if (c != 0.0) s += c * x[(size_t)jj * n1 + ii];
      }
    }
    const double xv = x[p];
    switch (epi) {
      case EPI_RESID: out[p] = b[p] - s; break;
      case EPI_JACOBI: out[p] = xv + omega * dinv[p] * (b[p] - s); break;
      default: out[p] = s; break;
    }
  }
}

}  // namespace

StencilOp::StencilOp(size_t n1, size_t n2, std::vector<double> coef)
    : n1_(n1), n2_(n2), coef_(std::move(coef)) {
  const size_t n = n1_ * n2_;
  if (n == 0 || coef_.size() != 9 * n) throw InvalidArgument("stencil size mismatch");
  diag_.assign(coef_.begin() + 4 * n, coef_.begin() + 5 * n);
  d_coef_.upload(coef_.data(), coef_.size());
}

void StencilOp::run(const double* x, double* out, int epi, const EpiArgs& e,
                    cudaStream_t s) const {
  if (epi == EPI_JACOBI && x == out) {
    // the stencil reads neighbours: in-place Jacobi needs a copy of x
    throw InvalidArgument("stencil Jacobi update cannot run in place");
  }
  const size_t n = size();
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(k_stencil, blocks, 256, 0, s, (int)n1_, (int)n2_, d_coef_.get(), x, out, epi, e.b, e.dinv,
                                   e.omega);
  FDE_LAUNCH_CHECK();
}

}  // namespace fde_b200
