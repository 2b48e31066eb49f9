// Variable-coefficient 9-point stencil operator: the B200 form of the
// reference's CSR levels on the P2 path (build_p2 5-point fine level,
// Galerkin R A P coarse levels; proj/src/precond.cpp:50-88,
// proj/src/sparse.cpp:42-49,131-140).  Stored as 9 coefficient planes
// (DIA layout, x fastest) instead of CSR -- coalesced, no index traffic.
#pragma once
#include <vector>

#include "devbuf.cuh"
#include "operator.cuh"

namespace fde_b200 {

class StencilOp {
 public:
  // coef[k * N + p], k = (dj + 1) * 3 + (di + 1): weight of x[(i+di) + (j+dj) n1]
  // in row p = i + j n1.  Entries reaching outside the grid must be zero.
  StencilOp(size_t n1, size_t n2, std::vector<double> coef);
  size_t size() const { return n1_ * n2_; }
  size_t n1() const { return n1_; }
  size_t n2() const { return n2_; }
  const std::vector<double>& coef() const { return coef_; }
  const std::vector<double>& diagonal() const { return diag_; }
  void run(const double* x, double* out, int epi, const EpiArgs& e, cudaStream_t s) const;

 private:
  size_t n1_, n2_;
  std::vector<double> coef_, diag_;
  DevBuf<double> d_coef_;
};

}  // namespace fde_b200
