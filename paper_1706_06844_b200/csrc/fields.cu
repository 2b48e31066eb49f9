// Device sampling of coefficient fields and sources for the reference's
// manufactured examples (examples.cuh), and the generic path that samples the
// problem's host callbacks and uploads them.  Compiled with -fmad=false
// (Makefile) so the formulas round like their host evaluation.
#include <vector>

#include "problem.cuh"

namespace fde_b200 {

namespace {

constexpr int kThreads = 256;

int blocks_for(size_t n) {
  const size_t b = (n + kThreads - 1) / kThreads;
  return (int)(b < 148 * 16 ? b : 148 * 16);
}

// Grid::x / y (problem.hpp:48-49): ax + hx (i + 1)
__global__ void k_example_fields(ExampleSpec e, int n1, int n2, double gx0, double hx,
                                 double gy0, double hy, double t, double* __restrict__ dp,
                                 double* __restrict__ dm, double* __restrict__ ep,
                                 double* __restrict__ em) {
  pdl_enter();
  const size_t n = (size_t)n1 * n2;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % n1), j = (int)(q / n1);
    const double x = gx0 + hx * (double)(i + 1), y = gy0 + hy * (double)(j + 1);
    dp[q] = example_coeff(e, 0, x, y, t);
    dm[q] = example_coeff(e, 1, x, y, t);
    ep[q] = example_coeff(e, 2, x, y, t);
    em[q] = example_coeff(e, 3, x, y, t);
  }
}

__global__ void k_example_source(ExampleSpec e, int n1, int n2, double gx0, double hx,
                                 double gy0, double hy, double t, double* __restrict__ v) {
  pdl_enter();
  const size_t n = (size_t)n1 * n2;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n;
       q += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(q % n1), j = (int)(q / n1);
    const double x = gx0 + hx * (double)(i + 1), y = gy0 + hy * (double)(j + 1);
    v[q] = example_source(e, x, y, t);
  }
}

constexpr int kSumBlocks = 296;

// per-block sums of a+b and c+d over contiguous chunks (fixed launch shape:
// deterministic partials, summed in block order on the host)
__global__ void k_pair_sums(size_t n, const double* __restrict__ a, const double* __restrict__ b,
                            const double* __restrict__ c, const double* __restrict__ d,
                            double* __restrict__ part) {
  pdl_enter();
  __shared__ double s1[kThreads], s2[kThreads];
  const size_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const size_t lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
  double x = 0.0, y = 0.0;
  for (size_t p = lo + threadIdx.x; p < hi; p += blockDim.x) {
    x += a[p] + b[p];
    y += c[p] + d[p];
  }
  s1[threadIdx.x] = x;
  s2[threadIdx.x] = y;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      s1[threadIdx.x] += s1[threadIdx.x + w];
      s2[threadIdx.x] += s2[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s1[0];
    part[2 * blockIdx.x + 1] = s2[0];
  }
}

void check_flag(FieldScratch& f, cudaStream_t s) {
  int flag = 0;
  FDE_CUDA(cudaMemcpyAsync(&flag, f.flag.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  FDE_CUDA(cudaStreamSynchronize(s));
  if (flag & 1) throw InvalidArgument("negative diffusion coefficient sample");
  if (flag & 2) throw InvalidArgument("operator diagonal must be strictly positive");
}

}  // namespace

void FieldScratch::ensure(size_t n) {
  if (dp.size() < n) {
    dp.alloc(n);
    dm.alloc(n);
    ep.alloc(n);
    em.alloc(n);
  }
  if (!partial.size()) partial.alloc(2 * kSumBlocks);
  if (!flag.size()) flag.alloc(1);
}

double anisotropy_ratio_device(FieldScratch& f, size_t n, double s_over_r, double alpha,
                               double beta, cudaStream_t s) {
  launch_k(k_pair_sums, kSumBlocks, kThreads, 0, s, n, f.dp.get(), f.dm.get(), f.ep.get(), f.em.get(),
                                              f.partial.get());
  FDE_LAUNCH_CHECK();
  std::vector<double> part(2 * kSumBlocks);
  FDE_CUDA(cudaMemcpyAsync(part.data(), f.partial.get(), part.size() * sizeof(double),
                           cudaMemcpyDeviceToHost, s));
  FDE_CUDA(cudaStreamSynchronize(s));
  double sx = 0.0, sy = 0.0;
  for (int b = 0; b < kSumBlocks; ++b) {
    sx += part[2 * b];
    sy += part[2 * b + 1];
  }
  const double nn = static_cast<double>(n);
  const double cx = sx / nn * q_gamma_pi(alpha);  // multigrid.cpp:116-128
  const double cy = s_over_r * (sy / nn) * q_gamma_pi(beta);
  return cy / cx;
}

void refresh_step_operator(StructuredOp& op, const Problem& p, const Grid& g, size_t m,
                           FieldScratch& f, cudaStream_t s) {
  f.ensure(g.size());
  f.flag.zero(s);
  sample_fields_device(p, g, m, f.dp.get(), f.dm.get(), f.ep.get(), f.em.get(), s);
  op.refresh(f.dp.get(), f.dm.get(), f.ep.get(), f.em.get(), nullptr, f.flag.get(), s);
  check_flag(f, s);
}

bool refresh_geometric_hierarchy(Hierarchy& h, const Problem& p, const Grid& g, size_t m,
                                 FieldScratch& f, cudaStream_t s) {
  f.ensure(g.size());
  for (size_t l = 0; l < h.depth(); ++l)
    if (!h.level(l).sop) throw InvalidArgument("refresh needs a geometric (structured) hierarchy");
  // the step-m plan (build_geometric_hierarchy: ratio of the fine operator)
  sample_fields_device(p, g, m, f.dp.get(), f.dm.get(), f.ep.get(), f.em.get(), s);
  const double ratio = anisotropy_ratio_device(f, g.size(), g.s_over_r, p.alpha, p.beta, s);
  const auto dims = plan_level_dims(g.n1, g.n2, ratio, p.alpha, p.beta);
  if (dims.size() != h.depth()) return false;
  for (size_t l = 0; l < dims.size(); ++l)
    if (dims[l] != h.dims(l)) return false;
  f.flag.zero(s);
  for (size_t l = 0; l < h.depth(); ++l) {
    if (l > 0) {
      const Grid lg(p, dims[l].first, dims[l].second, g.steps);
      sample_fields_device(p, lg, m, f.dp.get(), f.dm.get(), f.ep.get(), f.em.get(), s);
    }
    h.level(l).sop->refresh(f.dp.get(), f.dm.get(), f.ep.get(), f.em.get(), h.dinv_dev(l),
                            f.flag.get(), s);
  }
  check_flag(f, s);
  h.refactor_coarse(s);
  return true;
}

void sample_fields_device(const Problem& p, const Grid& g, size_t m, double* dp, double* dm,
                          double* ep, double* em, cudaStream_t s) {
  const double t = static_cast<double>(m) * g.dt;  // problem.cpp:52
  const size_t n = g.size();
  if (p.example.which) {
    launch_k(k_example_fields, blocks_for(n), kThreads, 0, s, p.example, (int)g.n1, (int)g.n2, g.ax,
                                                        g.hx, g.ay, g.hy, t, dp, dm, ep, em);
    FDE_LAUNCH_CHECK();
    return;
  }
  if (!p.d_plus || !p.d_minus || !p.e_plus || !p.e_minus)
    throw InvalidArgument("problem is missing a coefficient field");
  std::vector<double> h(4 * n);
  for (size_t j = 0; j < g.n2; ++j) {
    const double y = g.y(j);
    for (size_t i = 0; i < g.n1; ++i) {
      const double x = g.x(i);
      const size_t q = i + j * g.n1;
      h[q] = p.d_plus(x, y, t);
      h[n + q] = p.d_minus(x, y, t);
      h[2 * n + q] = p.e_plus(x, y, t);
      h[3 * n + q] = p.e_minus(x, y, t);
    }
  }
  double* dst[4] = {dp, dm, ep, em};
  for (int f = 0; f < 4; ++f)
    FDE_CUDA(cudaMemcpyAsync(dst[f], h.data() + f * n, n * sizeof(double),
                             cudaMemcpyHostToDevice, s));
  FDE_CUDA(cudaStreamSynchronize(s));  // h is released on return
}

void example_source_device(const Problem& p, const Grid& g, size_t m, double* v,
                           cudaStream_t s) {
  if (!p.example.which) throw InvalidArgument("not an example problem");
  const double t_half = (static_cast<double>(m) - 0.5) * g.dt;  // problem.cpp:81
  launch_k(k_example_source, blocks_for(g.size()), kThreads, 0, s, 
      p.example, (int)g.n1, (int)g.n2, g.ax, g.hx, g.ay, g.hy, t_half, v);
  FDE_LAUNCH_CHECK();
}

}  // namespace fde_b200
