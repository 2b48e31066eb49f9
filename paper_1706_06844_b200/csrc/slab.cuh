// y-slab piece of a level operator for the multi-GPU path:
// rank r owns grid rows [r0, r1) for the row (x) pass and, after the
// all-to-all transpose, columns [c0, c1) for the column (y) pass.  Same
// kernels as StructuredOp; the slab only samples the coefficients it needs.
#pragma once
#include <vector>

#include "problem.cuh"

namespace fde_b200 {

class SlabOp {
 public:
  // Level grid (d1 x d2) of problem p at step m; fine dims (nf1, nf2) give the
  // rediscretisation scale (hx_fine / hx_level)^alpha (multigrid.cpp:421-427).
  SlabOp(const Problem& p, size_t nf1, size_t nf2, size_t d1, size_t d2, size_t steps, size_t m,
         size_t r0, size_t r1, size_t c0, size_t c1);
  size_t n1() const { return n1_; }
  size_t n2() const { return n2_; }
  // QT[c * n2 + j] = sign s/r (ep T_b x + em T_b^T x) for local columns c (global c0 + c);
  // xT[c * n2 + j] = x[c0 + c, j].
  void ypass(const double* xT, double* QT, double sign, cudaStream_t s) const;
  // rows [r0, r1): out = epilogue(inv_r x + sign (dp T_a x + dm T_a^T x) + Q)
  void xpass(const double* x, const double* Q, double* out, double sign, int epi,
             const EpiArgs& e, cudaStream_t s) const;
  const std::vector<double>& diagonal() const { return diag_; }  // local rows
  double inv_r() const { return inv_r_; }
  double s_over_r() const { return s_over_r_; }

 private:
  size_t n1_, n2_, r0_, r1_, c0_, c1_;
  double inv_r_, s_over_r_;
  ToeplitzDev ax_, ay_;
  std::vector<double> diag_;
  DevBuf<double> d_dp_, d_dm_, d_epT_, d_emT_;
};

}  // namespace fde_b200
