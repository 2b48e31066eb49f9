// Drop-in check at the reference's plugin boundary (TEST INFRASTRUCTURE ONLY).
//
// The reference's OWN solver code -- fde::gmres (proj/src/krylov.cpp:12-166)
// and its per-step loop over fde::assemble_rhs (driver.cpp:34-52) -- drives
// the B200 library through the C ABI (include/fde_b200.h), via the two
// adapters INTEGRATION.md describes:
//   B200Op  : fde::LinOp  (proj/include/fde/linop.hpp:10-15)  -> fde_op_*
//   B200Mgm : fde::Precond (proj/include/fde/krylov.hpp:11-14) -> fde_mg_*
// Both are built FROM reference objects (a StructuredFdeOperator and an
// mg::MgHierarchy), so nothing about the problem is re-derived here: the GPU
// sees exactly the coefficients, blocks and level plan the reference built.
// Host buffers cross the boundary on every call (LinOp/Precond take host
// pointers), which is what a maintainer's first integration would do.
//
// Built by oracle/Makefile (`make adapter`) into _ref/libfde_adapter.so,
// linked against _ref/libfde_ref.so and ../paper_1706_06844_b200/libfde_b200.so.
#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fde_b200.h"
#include "ref_setup.hpp"

using namespace refh;

namespace {

thread_local std::string g_err;

void ck(int rc, const char* what) {
  if (rc != FDE_OK) throw std::runtime_error(std::string(what) + ": " + fde_last_error());
}
void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct DevVec {
  double* p = nullptr;
  explicit DevVec(std::size_t n) { ckc(cudaMalloc(&p, n * sizeof(double)), "cudaMalloc"); }
  ~DevVec() { cudaFree(p); }
  DevVec(const DevVec&) = delete;
  DevVec& operator=(const DevVec&) = delete;
};

fde_op make_op(const fde::StructuredFdeOperator& op) {
  fde_op h = nullptr;
  ck(fde_op_create(op.n1(), op.n2(), op.inv_r(), op.s_over_r(), op.block_x().first_col().data(),
                   op.block_x().first_row().data(), op.block_y().first_col().data(),
                   op.block_y().first_row().data(), op.dp().data(), op.dm().data(),
                   op.ep().data(), op.em().data(), &h),
     "fde_op_create");
  return h;
}

// fde::LinOp over a B200 operator handle.
class B200Op final : public fde::LinOp {
 public:
  explicit B200Op(const fde::StructuredFdeOperator& op)
      : n_(op.size()), diag_(op.diagonal()), h_(make_op(op)), x_(n_), y_(n_) {}
  ~B200Op() override { fde_op_destroy(h_); }
  std::size_t size() const override { return n_; }
  void apply(const double* x, double* y) const override {
    ckc(cudaMemcpy(x_.p, x, n_ * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    ck(fde_op_apply(h_, x_.p, y_.p, nullptr), "fde_op_apply");
    ckc(cudaMemcpy(y, y_.p, n_ * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  }
  const std::vector<double>& diagonal() const override { return diag_; }

 private:
  std::size_t n_;
  std::vector<double> diag_;
  fde_op h_;
  DevVec x_, y_;
};

// fde::Precond running `cycles` V-cycles from z = 0 (precond.cpp:22-26) on a
// B200 hierarchy mirroring a reference mg::MgHierarchy level by level.
class B200Mgm final : public fde::Precond {
 public:
  // coarse_sweeps: MgHierarchy keeps it private (multigrid.hpp:133), so the
  // caller passes the value it built the hierarchy with
  B200Mgm(const fde::mg::MgHierarchy& h, std::size_t cycles, std::size_t coarse_sweeps)
      : n_(h.level(0).op->size()), cycles_(cycles), r_(n_), z_(n_) {
    std::vector<fde_op> ops;
    for (std::size_t l = 0; l < h.depth(); ++l) {
      const auto* sop = dynamic_cast<const fde::StructuredFdeOperator*>(h.level(l).op.get());
      if (!sop) throw std::invalid_argument("B200Mgm mirrors structured (geometric) levels only");
      ops.push_back(make_op(*sop));
    }
    const int coarse = h.coarse_solve() == fde::mg::CoarseSolve::lu
                           ? FDE_COARSE_LU
                           : (h.coarse_solve() == fde::mg::CoarseSolve::sweeps ? FDE_COARSE_SWEEPS
                                                                               : FDE_COARSE_NONE);
    const int rc = fde_mg_create(ops.data(), ops.size(), h.omega(), coarse, coarse_sweeps, &mg_);
    for (fde_op o : ops) fde_op_destroy(o);  // retained by the hierarchy
    ck(rc, "fde_mg_create");
  }
  ~B200Mgm() override { fde_mg_destroy(mg_); }
  void apply(const double* r, double* z) const override {
    ckc(cudaMemcpy(r_.p, r, n_ * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    ckc(cudaMemset(z_.p, 0, n_ * sizeof(double)), "memset");
    for (std::size_t c = 0; c < cycles_; ++c)
      ck(fde_mg_vcycle(mg_, r_.p, z_.p, c == 0 ? 1 : 0, nullptr), "fde_mg_vcycle");
    ckc(cudaMemcpy(z, z_.p, n_ * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  }

 private:
  std::size_t n_, cycles_;
  fde_mg mg_ = nullptr;
  DevVec r_, z_;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

fde::SolverConfig solver_config(const ref_spec& s, const fde::Precond* pc) {
  fde::SolverConfig c;
  c.tol = s.tol;
  c.restart = static_cast<std::size_t>(s.restart);
  c.max_outer = static_cast<std::size_t>(s.max_outer);
  c.preconditioner = pc;
  return c;
}

// The reference operator and V-cycle for a spec, plus their B200 mirrors.
struct Pair {
  Setup st;
  fde::StructuredFdeOperator op;
  std::unique_ptr<fde::Precond> ref_pc;
  std::unique_ptr<B200Op> gpu_op;
  std::unique_ptr<B200Mgm> gpu_pc;
};

std::unique_ptr<Pair> build(const ref_spec& s) {
  if (s.precond != 2) throw std::invalid_argument("adapter: precond must be mgm (2)");
  auto p = std::make_unique<Pair>(Pair{make_setup(s), {}, nullptr, nullptr, nullptr});
  p->op = step_op(p->st.p, p->st.g, 1, p->st.pq);
  const fde::mg::MgHierarchy h = geometric(p->st.p, p->st.g, 1, p->st.pq, s.omega,
                                           coarse_of(s.coarse),
                                           static_cast<std::size_t>(s.coarse_sweeps));
  p->gpu_op = std::make_unique<B200Op>(p->op);
  p->gpu_pc = std::make_unique<B200Mgm>(h, static_cast<std::size_t>(s.cycles),
                                          static_cast<std::size_t>(s.coarse_sweeps));
  p->ref_pc = make_pc(s, p->st, p->op);
  return p;
}

}  // namespace

extern "C" {

const char* adapter_last_error() { return g_err.c_str(); }

// fde::gmres on the step system with b given.  which_op / which_pc: 0 = the
// reference's own object, 1 = the B200 adapter.
int adapter_gmres(const ref_spec* s, int which_op, int which_pc, const double* b, double* x,
                  int* iterations, int* converged, double* history, int max_history,
                  int* n_history) {
  return guarded([&] {
    auto p = build(*s);
    const fde::LinOp& a = which_op ? static_cast<const fde::LinOp&>(*p->gpu_op)
                                   : static_cast<const fde::LinOp&>(p->op);
    const fde::Precond* pc = which_pc ? static_cast<const fde::Precond*>(p->gpu_pc.get())
                                      : p->ref_pc.get();
    const fde::KrylovResult r =
        fde::gmres(a, solver_config(*s, pc), std::vector<double>(b, b + p->st.g.size()));
    std::copy(r.solution.begin(), r.solution.end(), x);
    *iterations = static_cast<int>(r.total_iterations);
    *converged = r.converged ? 1 : 0;
    const int nh = static_cast<int>(r.residual_history.size());
    *n_history = nh;
    for (int k = 0; k < nh && k < max_history; ++k) history[k] = r.residual_history[k];
  });
}

// The reference's step loop (driver.cpp:34-52: assemble_rhs, zero-guess
// gmres, u <- solution) with the B200 operator and V-cycle plugged in.
int adapter_march(const ref_spec* s, double* u_out, int* its, double* res) {
  return guarded([&] {
    auto p = build(*s);
    std::vector<double> u = fde::sample_initial(p->st.p, p->st.g);
    const fde::SolverConfig c = solver_config(*s, p->gpu_pc.get());
    for (std::size_t m = 1; m <= p->st.g.steps; ++m) {
      const std::vector<double> b = fde::assemble_rhs(p->st.p, p->st.g, m, u, p->op);
      fde::KrylovResult r = fde::gmres(*p->gpu_op, c, b);
      its[m - 1] = static_cast<int>(r.total_iterations);
      res[m - 1] = r.residual_history.back();
      u = std::move(r.solution);
    }
    std::copy(u.begin(), u.end(), u_out);
  });
}

}  // extern "C"
