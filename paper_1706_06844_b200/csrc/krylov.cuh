// Preconditioners and Krylov solvers (reference: proj/include/fde/krylov.hpp,
// proj/src/krylov.cpp:12-166, proj/src/precond.cpp:22-26,103-157).
//
// GMRES keeps the reference control flow exactly (left preconditioning, MGS
// with conditional re-orthogonalisation, Givens rotations, "estimate <= tol
// => verify with the true residual", restart semantics, zero initial guess)
// so iteration counts match the CPU oracle.  Vectors, the Arnoldi basis and
// all N-length work live on the device; the (restart+1) x restart Hessenberg
// column, the rotations and the control decisions are scalar host work fed
// by one small device->host copy per iteration.
#pragma once
#include <memory>
#include <vector>

#include "mg.cuh"

namespace fde_b200 {

// PrecondKind (precond.hpp:18); numbering of the C ABI (p2-exact and
// mgm-galerkin appended after the reference's default kinds)
enum PrecondKind : int { PC_NONE = 0, PC_P2 = 1, PC_MGM = 2, PC_P2_EXACT = 3, PC_MGM_GALERKIN = 4 };

class Precond {
 public:
  Precond(int kind, std::shared_ptr<Hierarchy> h, size_t n, size_t cycles);
  // PC_P2_EXACT: the exact banded solve (P2ExactPrecond, precond.cpp:90-101)
  Precond(std::shared_ptr<BandedLu> lu, size_t n);
  ~Precond();
  Precond(const Precond&) = delete;
  Precond& operator=(const Precond&) = delete;
  int kind() const { return kind_; }
  size_t size() const { return n_; }
  const Hierarchy* hierarchy() const { return h_.get(); }
  // in-place refresh of time-dependent levels (captured graphs stay valid)
  Hierarchy* mutable_hierarchy() const { return h_.get(); }
  // z = cycles V-cycles from z = 0 (precond.cpp:22-26); PC_NONE copies.
  // The whole cycle (~7 launches per level) is captured once per (r, z)
  // pair into a CUDA graph and replayed (FDE_NO_GRAPH=1 disables).
  void apply(const double* r, double* z, cudaStream_t s) const;

 private:
  void record(const double* r, double* z, cudaStream_t s) const;
  int kind_;
  std::shared_ptr<Hierarchy> h_;
  std::shared_ptr<BandedLu> lu_;
  size_t n_, cycles_;
  bool use_graphs_ = true;
  mutable cudaStream_t cap_ = nullptr;
  struct Entry {
    const double* r;
    double* z;
    cudaGraphExec_t exec;
    unsigned long long kernels;  // kernel nodes, for fde_kernel_launches()
  };
  mutable std::vector<Entry> graphs_;
};

struct SolverConfig {  // krylov.hpp:16-21
  double tol = 1e-7;
  size_t restart = 20;
  size_t max_outer = 100;
};

struct KrylovResult {  // krylov.hpp:23-30 (solution stays on the device)
  size_t total_iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
};

// Linear operator as the Krylov layer sees it (linop.hpp:10-15 + fused
// residual epilogue).
struct KrylovOp {
  std::shared_ptr<StructuredOp> op;
  size_t size() const { return op->size(); }
};

class KrylovWorkspace {
 public:
  explicit KrylovWorkspace(size_t n, size_t restart);
  ~KrylovWorkspace();
  KrylovWorkspace(const KrylovWorkspace&) = delete;
  KrylovWorkspace& operator=(const KrylovWorkspace&) = delete;
  size_t n() const { return n_; }
  size_t restart() const { return rst_; }

  // gmres (krylov.cpp:34-166); x receives the solution (device).
  KrylovResult gmres(const StructuredOp& a, const Precond* m, const SolverConfig& cfg,
                     const double* b, double* x, cudaStream_t s);
  // Left-preconditioned BiCGSTAB (NOT in the reference; see oracle/fde_oracle.c
  // bicgstab for the restated definition this mirrors).  max_it =
  // restart * max_outer.
  KrylovResult bicgstab(const StructuredOp& a, const Precond* m, const SolverConfig& cfg,
                        const double* b, double* x, cudaStream_t s);

 private:
  void precondition(const Precond* m, const double* r, double* z, cudaStream_t s);
  double nrm2_host(const double* v, cudaStream_t s);
  double dot_host(const double* x, const double* y, cudaStream_t s);
  void fetch(size_t count, cudaStream_t s);  // device scalars -> host mirror
  double true_rel(const StructuredOp& a, const Precond* m, const double* b, const double* x,
                  double norm_b, cudaStream_t s);

  size_t n_, rst_;
  std::vector<DevBuf<double>> v_;
  DevBuf<double> t_, r_, z_, w_, w2_, trial_, p_, s_, rh_, vv_, tt_;
  DevBuf<double> dsc_;         // device scalar slots
  DevBuf<double> dcoef_;       // lincomb coefficients
  DevBuf<const double*> dptr_; // lincomb basis pointers
  double* hsc_ = nullptr;      // pinned host mirror of dsc_
  // GMRES step staging: two pinned slots of the Hessenberg column + norms,
  // each completed by an event (the next step may be enqueued meanwhile)
  double* hstep_ = nullptr;
  size_t hstride_ = 0;
  cudaEvent_t ev_step_[2] = {nullptr, nullptr};
  bool speculate_ = true;  // FDE_GMRES_SPECULATE=0 disables
  Reducer red_;
};

}  // namespace fde_b200
