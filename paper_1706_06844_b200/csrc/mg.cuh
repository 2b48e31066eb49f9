// Device-resident multigrid hierarchy (reference: proj/include/fde/multigrid.hpp,
// proj/src/multigrid.cpp:114-441).  Level operators keep the diag x Toeplitz
// form (no level is stored densely); the V-cycle is a host-ordered sequence of
// fused kernels on one stream: apply+Jacobi, apply+residual, restriction,
// prolongation+correction.
#pragma once
#include <memory>
#include <utility>
#include <vector>

#include "operator.cuh"
#include "csr.cuh"
#include "stencil.cuh"
#include "tail.cuh"
#include "vec_kernels.cuh"

namespace fde_b200 {

enum CoarseSolve : int { COARSE_LU = 0, COARSE_SWEEPS = 1, COARSE_NONE = 2 };
enum CoarseningMode : int { MODE_GEOMETRIC = 0, MODE_GALERKIN = 1 };

size_t coarse_size(size_t n);  // multigrid.cpp:114
// eval_q_gamma(gamma, pi) (symbols.cpp:23-33) with the reference's complex
// evaluation of (1 - e^{i pi})^gamma.
double q_gamma_pi(double gamma);
// multigrid.cpp:116-128
double anisotropy_ratio(const StructuredOp& op, double alpha, double beta);
// multigrid.cpp:130-158 (semicoarsening when the tracked ratio leaves [1/5, 5])
std::vector<std::pair<size_t, size_t>> plan_level_dims(size_t n1, size_t n2, double ratio0,
                                                       double alpha, double beta);
// multigrid.cpp:98-110 (full coarsening down to <= 8 x 8, Galerkin default)
std::vector<std::pair<size_t, size_t>> level_dims(size_t n1, size_t n2);

// A level operator: the structured (diag x Toeplitz) operator, a Galerkin
// 9-point stencil (P2 path) or a CSR matrix (Galerkin levels on the full
// operator, `mgm-galerkin`).
struct LevelOp {
  std::shared_ptr<StructuredOp> sop;
  std::shared_ptr<StencilOp> stencil;
  std::shared_ptr<CsrOp> csr;
  size_t size() const { return sop ? sop->size() : stencil ? stencil->size() : csr->size(); }
  const std::vector<double>& diagonal() const {
    return sop ? sop->diagonal() : stencil ? stencil->diagonal() : csr->diagonal();
  }
  void run(const double* x, double* out, int epi, const EpiArgs& e, cudaStream_t s) const {
    if (sop) sop->run(x, out, 1.0, epi, e, s);
    else if (stencil) stencil->run(x, out, epi, e, s);
    else csr->run(x, out, epi, e, s);
  }
};

class Hierarchy {
 public:
  // MgHierarchy ctor (multigrid.cpp:301-316): dinv = 1/diag (throws on <= 0),
  // dense LU of the coarsest level when coarse == COARSE_LU.
  Hierarchy(std::vector<LevelOp> levels, std::vector<std::pair<size_t, size_t>> dims,
            int mode, double omega, int coarse, size_t coarse_sweeps);

  size_t depth() const { return levels_.size(); }
  const std::pair<size_t, size_t>& dims(size_t l) const { return dims_[l]; }
  const LevelOp& level(size_t l) const { return levels_[l]; }
  double omega() const { return omega_; }
  int coarse() const { return coarse_; }

  // MgHierarchy::vcycle (multigrid.cpp:385-394); the caller states whether x
  // is all-zero instead of the reference's scan.
  void vcycle(const double* b, double* x, bool zero_guess, cudaStream_t s) const;

  // Per-step refresh of time-dependent levels (refresh_geometric_hierarchy):
  // the level's dinv buffer (rewritten in place, so captured V-cycle graphs
  // stay valid) and re-factoring of the dense coarsest level.
  double* dinv_dev(size_t l) const { return dinv_[l].get(); }
  void refactor_coarse(cudaStream_t s);

 private:
  // prescaled: x already holds the zero-guess smoothing omega dinv b (fused
  // into the restriction that produced b)
  void cycle(size_t l, const double* b, double* x, bool zero, cudaStream_t s,
             bool prescaled = false) const;
  bool zero_guess_is_diag_scale(size_t l) const;
  void plan_tail();
  std::vector<LevelOp> levels_;
  std::vector<std::pair<size_t, size_t>> dims_;
  std::vector<Xfer> xfer_;
  std::vector<DevBuf<double>> dinv_, r_, bc_, xc_;
  int mode_;
  double omega_;
  int coarse_;
  size_t coarse_sweeps_;
  int fuse_ = 3;
  DevBuf<double> lu_;
  DevBuf<int> perm_;
  // levels tail_..depth-1 run as one cluster launch (tail.cuh); 0 = none
  size_t tail_ = 0;
  TailDesc tail_desc_{};
};

}  // namespace fde_b200
