// Device-resident ToeplitzBlock / StructuredFdeOperator
// (reference: proj/include/fde/structured.hpp:19-97, proj/src/structured.cpp).
#pragma once
#include <memory>
#include <vector>

#include "devbuf.cuh"
#include "line_conv.cuh"

namespace fde_b200 {

// weights.cpp:21-28 -- g_0 = 1, g_k = g_{k-1} (1 - (gamma+1)/k)
std::vector<double> binom_coeffs(double gamma, size_t K);
// weights.cpp:30-51 for pq = 0 ((p,q) = (1,0)); pq = 1 is the (1,-1) WSGD
// table (not in the reference; SURVEY.md 8(a')): w_k = l1 g_k + l2 g_{k-2},
// l1 = (gamma+2)/4, l2 = (2-gamma)/4.
std::vector<double> wsgd_weights(double gamma, size_t K, int pq);
size_t next_pow2(size_t n);  // fft.cpp:11-15

// Fused-epilogue operands of one operator application (see line_conv.cuh).
struct EpiArgs {
  const double* b = nullptr;
  const double* dinv = nullptr;
  double omega = 0.0;
  const double* src = nullptr;
  double src_scale = 0.0;
};

class ToeplitzDev {
 public:
  // structured.cpp:34-45 validation: sizes match, corner entries agree.
  ToeplitzDev(std::vector<double> first_col, std::vector<double> first_row);
  // structured.cpp:47-55: col = -w_{1..n}, row = (-w_1, -w_0, 0, ...)
  static ToeplitzDev fractional(double gamma, size_t n, int pq);

  size_t size() const { return n_; }
  size_t circulant_length() const { return L_; }
  const std::vector<double>& first_col() const { return col_; }
  const std::vector<double>& first_row() const { return row_; }
  double entry(size_t i, size_t j) const { return i >= j ? col_[i - j] : row_[j - i]; }
  LineBlockDev dev() const;

 private:
  size_t n_ = 0, L_ = 0;
  int logM_ = 0;
  std::vector<double> col_, row_;
  std::shared_ptr<DevBuf<double2>> spec_;  // per-k spectral constants
  std::shared_ptr<DevBuf<double>> dcol_, drow_;
};

class StructuredOp {
 public:
  // structured.cpp:99-123: validation + diagonal (host, reference order).
  StructuredOp(size_t n1, size_t n2, double inv_r, double s_over_r, ToeplitzDev ax,
               ToeplitzDev ay, std::vector<double> dp, std::vector<double> dm,
               std::vector<double> ep, std::vector<double> em);

  size_t size() const { return n1_ * n2_; }
  size_t n1() const { return n1_; }
  size_t n2() const { return n2_; }
  double inv_r() const { return inv_r_; }
  double s_over_r() const { return s_over_r_; }
  const ToeplitzDev& block_x() const { return ax_; }
  const ToeplitzDev& block_y() const { return ay_; }
  const std::vector<double>& dp() const { return dp_; }
  const std::vector<double>& dm() const { return dm_; }
  const std::vector<double>& ep() const { return ep_; }
  const std::vector<double>& em() const { return em_; }
  const std::vector<double>& diagonal() const { return diag_; }
  const double* diagonal_dev() const { return d_diag_.get(); }
  // device coefficient fields (ep/em transposed: i * n2 + j)
  const double* dp_dev() const { return d_dp_.get(); }
  const double* dm_dev() const { return d_dm_.get(); }
  const double* epT_dev() const { return d_epT_.get(); }
  const double* emT_dev() const { return d_emT_.get(); }

  // out = epilogue(A~ x) with A~ = apply (sign +1) or apply_rhs (sign -1).
  // Two launches (y-pass, x-pass) on stream s.  out may alias x only for
  // EPI_JACOBI.  Not re-entrant across streams (one Q scratch per operator).
  void run(const double* x, double* out, double sign, int epi, const EpiArgs& e,
           cudaStream_t s) const;
  // Whether run_mapped is available: the column pass reads a transposed copy
  // of x, so the input map rides on that transpose.
  bool maps_input() const;
  // x = in(.) is formed (and stored to x, which may alias in.a) by the column
  // transpose, then out = epi(A x) as in run().
  void run_mapped(const InMap& in, double* x, double* out, double sign, int epi,
                  const EpiArgs& e, cudaStream_t s) const;
  void apply(const double* x, double* y, cudaStream_t s) const {
    run(x, y, 1.0, EPI_STORE, EpiArgs{}, s);
  }
  void apply_rhs(const double* x, double* y, cudaStream_t s) const {
    run(x, y, -1.0, EPI_STORE, EpiArgs{}, s);
  }
  // structured.cpp:154-162.  Rejected once a hierarchy holds the operator:
  // its one-launch coarse tail and the captured V-cycle graphs bake in inv_r,
  // s/r and 1/diag, so a later scale() would leave them silently stale.
  void scale(double s);
  void freeze() const { frozen_ = true; }

  // Per-step re-assembly for time-dependent coefficients (driver.cpp:37-41,
  // problem.cpp:50-71): new UNSCALED samples (device arrays) replace the
  // coefficients, the scale() factors applied so far are re-applied in order,
  // and the diagonal is recomputed on the device in the reference's order
  // (structured.cpp:119-122 then 154-162); dinv = 1/diag when dinv is set
  // (MgHierarchy ctor, multigrid.cpp:306-312).  flag (device int) gets bit 0
  // for a negative coefficient sample, bit 1 for a nonpositive diagonal.
  // Host copies (dp(), diagonal(), ...) are stale until sync_host().
  void refresh(const double* dp, const double* dm, const double* ep, const double* em,
               double* dinv, int* flag, cudaStream_t s);
  void sync_host(cudaStream_t s);

 private:
  void run_impl(const InMap* in, const double* x, double* out, double sign, int epi,
                const EpiArgs& e, cudaStream_t s) const;
  void upload();
  size_t n1_, n2_;
  double inv_r_, s_over_r_;
  double inv_r0_, s_over_r0_;  // as constructed (before scale())
  std::vector<double> scales_;  // scale() factors in order
  ToeplitzDev ax_, ay_;
  std::vector<double> dp_, dm_, ep_, em_, diag_;
  DevBuf<double> d_dp_, d_dm_, d_epT_, d_emT_, d_diag_;
  mutable DevBuf<double> d_q_, d_xT_;
  bool transpose_columns_ = true;
  bool host_stale_ = false;
  mutable bool frozen_ = false;
};

}  // namespace fde_b200
