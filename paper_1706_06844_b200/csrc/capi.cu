// extern "C" boundary (include/fde_b200.h) over the B200 host classes.
#include <chrono>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "../../include/fde_b200.h"
#include "krylov.cuh"
#include "problem.cuh"
#include "slab.cuh"
#include "dist.cuh"
#include <thread>

namespace fde_b200 {
std::atomic<unsigned long long> g_kernel_launches{0};
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FDE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
}

using namespace fde_b200;

struct fde_op_s {
  std::shared_ptr<StructuredOp> op;
  std::unique_ptr<KrylovWorkspace> ws;  // reused by fde_gmres / fde_bicgstab
};
struct fde_mg_s {
  std::shared_ptr<Hierarchy> h;
};
struct fde_precond_s {
  std::shared_ptr<Precond> pc;
};
struct fde_slab_s {
  std::unique_ptr<SlabOp> op;
};
struct fde_dist_comm_s {
  std::shared_ptr<SlabComm> c;
};
struct fde_dist_march_s {
  std::unique_ptr<DistMarch> m;
  DevBuf<double> tmp;
};
struct fde_march_s {
  Problem p;
  Grid g;
  fde_driver_config cfg;
  std::shared_ptr<StructuredOp> op;  // coefficients of t^{m-1} when time dependent
  std::shared_ptr<StructuredOp> next;  // time dependent: the step-m operator
  size_t next_m = 0;                   // step the next operator / preconditioner hold
  FieldScratch fields;
  std::shared_ptr<Precond> pc;
  std::unique_ptr<KrylovWorkspace> ws;
  DevBuf<double> u, b, src, x;
  std::vector<double> host_src;
  double scale = 0.0;  // 2 hx^alpha (problem.cpp:82)
  size_t m = 0;
  // pipelined host I/O (fde_march_prefetch_source / _solution_async)
  cudaStream_t cs = nullptr;            // copy stream
  cudaEvent_t ev_step = nullptr;        // u^m final on the compute stream
  // u and x swap between the same two allocations: one event per allocation,
  // recorded after the last D2H that reads it
  cudaEvent_t ev_d2h[2] = {};
  const double* d2h_buf[2] = {nullptr, nullptr};
  // prefetched sources: a ring of three device buffers, up to two in flight
  DevBuf<double> ring[3];
  cudaEvent_t ev_ready[3] = {};  // H2D into ring[i] done (copy stream)
  cudaEvent_t ev_free[3] = {};   // the rhs assembly that read ring[i] done (compute stream)
  int pending[2] = {-1, -1};     // FIFO of filled ring slots
  int npending = 0;
  int cur_src = -1;
  void ensure_io() {
    if (cs) return;
    FDE_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    FDE_CUDA(cudaEventCreateWithFlags(&ev_step, cudaEventDisableTiming));
    for (cudaEvent_t& e : ev_d2h) FDE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (int i = 0; i < 3; ++i) {
      FDE_CUDA(cudaEventCreateWithFlags(&ev_ready[i], cudaEventDisableTiming));
      FDE_CUDA(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming));
    }
  }
  ~fde_march_s() {
    if (cs) {
      cudaStreamSynchronize(cs);
      cudaStreamDestroy(cs);
      cudaEventDestroy(ev_step);
      for (cudaEvent_t e : ev_d2h) cudaEventDestroy(e);
      for (int i = 0; i < 3; ++i) {
        cudaEventDestroy(ev_ready[i]);
        cudaEventDestroy(ev_free[i]);
      }
    }
  }
};

namespace {

thread_local std::string g_error;

template <class F>
int guard(F&& f) {
  try {
    f();
    return FDE_OK;
  } catch (const InvalidArgument& e) {
    g_error = e.what();
    return FDE_EINVAL;
  } catch (const RuntimeError& e) {
    g_error = e.what();
    return FDE_ERUNTIME;
  } catch (const CudaError& e) {
    g_error = e.what();
    return FDE_ECUDA;
  } catch (const std::bad_alloc&) {
    g_error = "out of host memory";
    return FDE_ENOMEM;
  } catch (const std::exception& e) {
    g_error = e.what();
    return FDE_ERUNTIME;
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw InvalidArgument(what);
}

cudaStream_t stream_of(void* s) { return static_cast<cudaStream_t>(s); }

// fde_problem (C callbacks or preset) -> Problem
Problem to_problem(const fde_problem* c) {
  need(c != nullptr, "null problem");
  Problem p;
  if (c->preset >= 101 && c->preset <= 103) {  // the reference's manufactured examples
    p = make_example_problem(c->preset - 100, c->alpha, c->beta, c->ax, c->bx, c->ay, c->by);
    need(c->time_dependent_coeffs == (p.time_dependent_coeffs ? 1 : 0),
         "example problems fix time_dependent_coeffs (example 2 only)");
  } else if (c->preset) {
    need(!c->time_dependent_coeffs, "BASELINE presets have time-independent coefficients");
    p = make_preset(c->preset, c->seed, c->source_kind, 0, 0.0);
  } else {
    need(c->d_plus && c->d_minus && c->e_plus && c->e_minus, "problem is missing a coefficient field");
    void* ctx = c->ctx;
    auto wrap3 = [ctx](fde_field_fn f) {
      return std::function<double(double, double, double)>(
          [f, ctx](double x, double y, double t) { return f(x, y, t, ctx); });
    };
    p.d_plus = wrap3(c->d_plus);
    p.d_minus = wrap3(c->d_minus);
    p.e_plus = wrap3(c->e_plus);
    p.e_minus = wrap3(c->e_minus);
    if (c->source) p.source = wrap3(c->source);
    if (c->initial) {
      fde_initial_fn f = c->initial;
      p.initial = [f, ctx](double x, double y) { return f(x, y, ctx); };
    }
  }
  p.alpha = c->alpha;
  p.beta = c->beta;
  p.ax = c->ax;
  p.bx = c->bx;
  p.ay = c->ay;
  p.by = c->by;
  p.t_final = c->t_final;
  p.pq = c->pq;
  if (!c->preset) p.time_dependent_coeffs = c->time_dependent_coeffs != 0;
  need(p.pq == 0 || p.pq == 1, "pq must be 0 ((1,0)) or 1 ((1,-1))");
  return p;
}

void fill_result(const KrylovResult& r, fde_krylov_result* out) {
  if (!out) return;
  out->total_iterations = r.total_iterations;
  out->converged = r.converged ? 1 : 0;
  out->history_length = r.residual_history.size();
  size_t nh = r.residual_history.size();
  if (!out->history) nh = 0;
  if (nh > out->history_capacity) nh = out->history_capacity;
  for (size_t k = 0; k < nh; ++k) out->history[k] = r.residual_history[k];
  out->n_history = nh;
}

std::shared_ptr<Precond> make_pc(int kind, const Problem& p, const Grid& g, size_t m,
                                 const std::shared_ptr<StructuredOp>& op, double omega,
                                 size_t cycles, int coarse, size_t sweeps) {
  switch (kind) {  // make_preconditioner, precond.cpp:135-157
    case PC_NONE:
      return std::make_shared<Precond>(PC_NONE, nullptr, op->size(), 1);
    case PC_P2:
      return std::make_shared<Precond>(PC_P2, build_p2_hierarchy(*op, omega), op->size(), cycles);
    case PC_MGM:
      return std::make_shared<Precond>(
          PC_MGM, build_geometric_hierarchy(p, g, m, omega, coarse, sweeps), op->size(), cycles);
    case PC_P2_EXACT:
      return std::make_shared<Precond>(
          std::make_shared<BandedLu>(build_p2_csr(*op), op->n1()), op->size());
    case PC_MGM_GALERKIN: {  // precond.cpp:150-155
      const auto plan = plan_level_dims(op->n1(), op->n2(), anisotropy_ratio(*op, p.alpha, p.beta),
                                        p.alpha, p.beta);
      return std::make_shared<Precond>(
          PC_MGM_GALERKIN, build_galerkin_csr_hierarchy(*op, plan, omega, coarse, sweeps),
          op->size(), cycles);
    }
  }
  throw InvalidArgument("unknown preconditioner kind");
}

KrylovWorkspace& workspace_for(std::unique_ptr<KrylovWorkspace>& ws, size_t n, size_t restart) {
  const size_t need_rst = restart < 5 ? 5 : restart;
  if (!ws || ws->n() != n || ws->restart() < need_rst)
    ws = std::make_unique<KrylovWorkspace>(n, need_rst);
  return *ws;
}

}  // namespace

extern "C" {

const char* fde_last_error(void) { return g_error.c_str(); }
int fde_abi_version(void) { return FDE_B200_ABI_VERSION; }
unsigned long long fde_kernel_launches(void) { return g_kernel_launches.load(); }
int fde_fp64_peak(double* tflops, void* stream) {
  return guard([&] {
    need(tflops != nullptr, "null argument");
    *tflops = fp64_peak_tflops(stream_of(stream));
  });
}

int fde_wsgd_weights(double gamma, size_t K, int pq, double* g, double* w) {
  return guard([&] {
    need(g && w, "null output");
    const auto gg = binom_coeffs(gamma, K);
    const auto ww = wsgd_weights(gamma, K, pq);
    std::memcpy(g, gg.data(), gg.size() * sizeof(double));
    std::memcpy(w, ww.data(), ww.size() * sizeof(double));
  });
}

int fde_op_create(size_t n1, size_t n2, double inv_r, double s_over_r, const double* col_x,
                  const double* row_x, const double* col_y, const double* row_y,
                  const double* dp, const double* dm, const double* ep, const double* em,
                  fde_op* out) {
  return guard([&] {
    need(out && col_x && row_x && col_y && row_y && dp && dm && ep && em, "null argument");
    const size_t n = n1 * n2;
    auto h = std::make_unique<fde_op_s>();
    h->op = std::make_shared<StructuredOp>(
        n1, n2, inv_r, s_over_r, ToeplitzDev({col_x, col_x + n1}, {row_x, row_x + n1}),
        ToeplitzDev({col_y, col_y + n2}, {row_y, row_y + n2}), std::vector<double>(dp, dp + n),
        std::vector<double>(dm, dm + n), std::vector<double>(ep, ep + n),
        std::vector<double>(em, em + n));
    *out = h.release();
  });
}

int fde_op_create_fractional(size_t n1, size_t n2, double inv_r, double s_over_r,
                             double alpha, double beta, int pq, const double* dp,
                             const double* dm, const double* ep, const double* em,
                             fde_op* out) {
  return guard([&] {
    need(out && dp && dm && ep && em, "null argument");
    const size_t n = n1 * n2;
    auto h = std::make_unique<fde_op_s>();
    h->op = std::make_shared<StructuredOp>(
        n1, n2, inv_r, s_over_r, ToeplitzDev::fractional(alpha, n1, pq),
        ToeplitzDev::fractional(beta, n2, pq), std::vector<double>(dp, dp + n),
        std::vector<double>(dm, dm + n), std::vector<double>(ep, ep + n),
        std::vector<double>(em, em + n));
    *out = h.release();
  });
}

int fde_op_size(fde_op op, size_t* n) {
  return guard([&] {
    need(op && n, "null argument");
    *n = op->op->size();
  });
}
int fde_op_apply(fde_op op, const double* x, double* y, void* stream) {
  return guard([&] {
    need(op && x && y, "null argument");
    need(x != y, "apply cannot run in place");
    op->op->apply(x, y, stream_of(stream));
  });
}
int fde_op_apply_rhs(fde_op op, const double* x, double* y, void* stream) {
  return guard([&] {
    need(op && x && y, "null argument");
    need(x != y, "apply_rhs cannot run in place");
    op->op->apply_rhs(x, y, stream_of(stream));
  });
}
int fde_op_diagonal(fde_op op, double* d) {
  return guard([&] {
    need(op && d, "null argument");
    const auto& v = op->op->diagonal();
    std::memcpy(d, v.data(), v.size() * sizeof(double));
  });
}
int fde_op_scale(fde_op op, double s) {
  return guard([&] {
    need(op != nullptr, "null argument");
    op->op->scale(s);
  });
}
int fde_op_destroy(fde_op op) {
  return guard([&] { delete op; });
}

int fde_problem_preset(int cfg, unsigned long long seed, int source_kind, size_t steps,
                       double tau, fde_problem* out, size_t* n_out, size_t* steps_out) {
  return guard([&] {
    need(out != nullptr, "null output");
    const PresetInfo in = preset_info(cfg);
    const size_t st = steps ? steps : in.steps;
    std::memset(out, 0, sizeof *out);
    out->alpha = in.alpha;
    out->beta = in.beta;
    out->ax = 0.0;
    out->bx = 1.0;
    out->ay = 0.0;
    out->by = 1.0;
    out->t_final = (tau > 0 ? tau : in.tau) * static_cast<double>(st);
    out->pq = in.pq;
    out->preset = cfg;
    out->source_kind = source_kind >= 0 ? source_kind : in.source_kind;
    out->seed = seed;
    if (n_out) *n_out = in.n;
    if (steps_out) *steps_out = st;
  });
}

int fde_problem_example(int which, double alpha, double beta, double ax, double bx, double ay,
                        double by, fde_problem* out) {
  return guard([&] {
    need(out != nullptr, "null output");
    const Problem p = make_example_problem(which, alpha, beta, ax, bx, ay, by);  // validates
    std::memset(out, 0, sizeof *out);
    out->alpha = alpha;
    out->beta = beta;
    out->ax = ax;
    out->bx = bx;
    out->ay = ay;
    out->by = by;
    out->t_final = p.t_final;
    out->time_dependent_coeffs = p.time_dependent_coeffs ? 1 : 0;
    out->preset = 100 + which;
  });
}

int fde_problem_example_default(int which, double alpha, double beta, fde_problem* out) {
  const double len = which == 1 ? 2.0 : 1.0;
  return fde_problem_example(which, alpha, beta, 0.0, len, 0.0, len, out);
}

int fde_error_inf(const fde_problem* p, size_t n1, size_t n2, size_t steps, double t,
                  const double* u, double* err) {
  return guard([&] {
    need(u != nullptr && err != nullptr, "null argument");
    const Problem pr = to_problem(p);
    const Grid g(pr, n1, n2, steps);
    *err = error_inf(std::vector<double>(u, u + g.size()), pr, g, t);
  });
}

int fde_grid(const fde_problem* p, size_t n1, size_t n2, size_t steps, double* out) {
  return guard([&] {
    need(out != nullptr, "null output");
    const Grid g(to_problem(p), n1, n2, steps);
    out[0] = g.hx;
    out[1] = g.hy;
    out[2] = g.dt;
    out[3] = g.inv_r;
    out[4] = g.s_over_r;
  });
}

int fde_assemble_step_operator(const fde_problem* p, size_t n1, size_t n2, size_t steps,
                               size_t m, fde_op* out) {
  return guard([&] {
    need(out != nullptr, "null output");
    const Problem pr = to_problem(p);
    const Grid g(pr, n1, n2, steps);
    auto h = std::make_unique<fde_op_s>();
    h->op = assemble_step_operator(pr, g, m);
    *out = h.release();
  });
}

int fde_sample_initial(const fde_problem* p, size_t n1, size_t n2, size_t steps, double* u) {
  return guard([&] {
    need(u != nullptr, "null output");
    const Problem pr = to_problem(p);
    const Grid g(pr, n1, n2, steps);
    const auto v = sample_initial(pr, g);
    std::memcpy(u, v.data(), v.size() * sizeof(double));
  });
}

int fde_sample_source(const fde_problem* p, size_t n1, size_t n2, size_t steps, size_t m,
                      double* v) {
  return guard([&] {
    need(v != nullptr, "null output");
    need(m >= 1, "step index starts at 1");
    const Problem pr = to_problem(p);
    const Grid g(pr, n1, n2, steps);
    sample_source(pr, g, m, v);
  });
}

int fde_plan_level_dims(size_t n1, size_t n2, double ratio0, double alpha, double beta,
                        size_t* dims, size_t max_levels, size_t* n_levels) {
  return guard([&] {
    need(dims && n_levels, "null output");
    const auto d = plan_level_dims(n1, n2, ratio0, alpha, beta);
    *n_levels = d.size();
    for (size_t l = 0; l < d.size() && l < max_levels; ++l) {
      dims[2 * l] = d[l].first;
      dims[2 * l + 1] = d[l].second;
    }
  });
}

int fde_anisotropy_ratio(fde_op op, double alpha, double beta, double* ratio) {
  return guard([&] {
    need(op && ratio, "null argument");
    *ratio = anisotropy_ratio(*op->op, alpha, beta);
  });
}

int fde_transfer(size_t n1, size_t n2, int coarsen_x, int coarsen_y, int op, const double* in,
                 double* out, void* stream) {
  return guard([&] {
    need(in && out, "null argument");
    const Xfer t = make_xfer((int)n1, (int)n2, coarsen_x != 0, coarsen_y != 0);
    if (op == 0) xfer_prolong(t, in, out, stream_of(stream));
    else if (op == 1) xfer_restrict(t, in, out, 0.5, stream_of(stream));
    else if (op == 2) xfer_restrict(t, in, out, 1.0, stream_of(stream));
    else throw InvalidArgument("transfer op must be 0, 1 or 2");
  });
}

int fde_mg_build_geometric(const fde_problem* p, size_t n1, size_t n2, size_t steps, size_t m,
                           double omega, int coarse, size_t coarse_sweeps, fde_mg* out) {
  return guard([&] {
    need(out != nullptr, "null output");
    const Problem pr = to_problem(p);
    const Grid g(pr, n1, n2, steps);
    auto h = std::make_unique<fde_mg_s>();
    h->h = build_geometric_hierarchy(pr, g, m, omega, coarse, coarse_sweeps);
    *out = h.release();
  });
}

int fde_mg_create(const fde_op* levels, size_t n_levels, double omega, int coarse,
                  size_t coarse_sweeps, fde_mg* out) {
  return guard([&] {
    need(out && levels && n_levels > 0, "null argument");
    std::vector<LevelOp> lv;
    std::vector<std::pair<size_t, size_t>> dims;
    for (size_t l = 0; l < n_levels; ++l) {
      need(levels[l] != nullptr, "null level operator");
      LevelOp o;
      o.sop = levels[l]->op;
      dims.emplace_back(o.sop->n1(), o.sop->n2());
      lv.push_back(o);
    }
    auto h = std::make_unique<fde_mg_s>();
    h->h = std::make_shared<Hierarchy>(std::move(lv), dims, MODE_GEOMETRIC, omega, coarse,
                                       coarse_sweeps);
    *out = h.release();
  });
}

int fde_mg_build_p2(fde_op fine, double omega, fde_mg* out) {
  return guard([&] {
    need(fine && out, "null argument");
    auto h = std::make_unique<fde_mg_s>();
    h->h = build_p2_hierarchy(*fine->op, omega);
    *out = h.release();
  });
}

int fde_mg_depth(fde_mg h, size_t* depth) {
  return guard([&] {
    need(h && depth, "null argument");
    *depth = h->h->depth();
  });
}
int fde_mg_level_dims(fde_mg h, size_t level, size_t* n1, size_t* n2) {
  return guard([&] {
    need(h && n1 && n2, "null argument");
    need(level < h->h->depth(), "level out of range");
    *n1 = h->h->dims(level).first;
    *n2 = h->h->dims(level).second;
  });
}
int fde_mg_vcycle(fde_mg h, const double* b, double* x, int zero_guess, void* stream) {
  return guard([&] {
    need(h && b && x, "null argument");
    h->h->vcycle(b, x, zero_guess != 0, stream_of(stream));
  });
}
int fde_mg_destroy(fde_mg h) {
  return guard([&] { delete h; });
}

int fde_precond_create(int kind, const fde_problem* p, size_t n1, size_t n2, size_t steps,
                       size_t m, fde_op op, double omega, size_t cycles, int coarse,
                       size_t coarse_sweeps, fde_precond* out) {
  return guard([&] {
    need(out && op, "null argument");
    auto h = std::make_unique<fde_precond_s>();
    if (kind == PC_MGM || kind == PC_MGM_GALERKIN) {
      need(p != nullptr, "this preconditioner needs the problem");
      const Problem pr = to_problem(p);
      const Grid g(pr, n1, n2, steps);
      h->pc = make_pc(kind, pr, g, m, op->op, omega, cycles, coarse, coarse_sweeps);
    } else {
      h->pc = make_pc(kind, Problem{}, Grid{}, m, op->op, omega, cycles, coarse, coarse_sweeps);
    }
    *out = h.release();
  });
}
int fde_precond_apply(fde_precond pc, const double* r, double* z, void* stream) {
  return guard([&] {
    need(pc && r && z, "null argument");
    pc->pc->apply(r, z, stream_of(stream));
  });
}
int fde_precond_destroy(fde_precond pc) {
  return guard([&] { delete pc; });
}

int fde_gmres(fde_op a, fde_precond m, const fde_solver_config* cfg, const double* b,
              double* x, fde_krylov_result* res, void* stream) {
  return guard([&] {
    need(a && cfg && b && x, "null argument");
    need(b != x, "the solution must not alias the right-hand side (x is zeroed first)");
    SolverConfig c{cfg->tol, cfg->restart, cfg->max_outer};
    need(c.restart > 0 && c.tol > 0.0, "invalid solver configuration");
    KrylovWorkspace& ws = workspace_for(a->ws, a->op->size(), c.restart);
    fill_result(ws.gmres(*a->op, m ? m->pc.get() : nullptr, c, b, x, stream_of(stream)), res);
  });
}

int fde_bicgstab(fde_op a, fde_precond m, const fde_solver_config* cfg, const double* b,
                 double* x, fde_krylov_result* res, void* stream) {
  return guard([&] {
    need(a && cfg && b && x, "null argument");
    need(b != x, "the solution must not alias the right-hand side (x is zeroed first)");
    SolverConfig c{cfg->tol, cfg->restart, cfg->max_outer};
    need(c.tol > 0.0, "invalid solver configuration");
    KrylovWorkspace& ws = workspace_for(a->ws, a->op->size(), c.restart);
    fill_result(ws.bicgstab(*a->op, m ? m->pc.get() : nullptr, c, b, x, stream_of(stream)),
                res);
  });
}

void fde_driver_config_default(fde_driver_config* c) {
  if (!c) return;
  c->precond = PC_NONE;  // driver.hpp:12-21
  c->tol = 1e-7;
  c->restart = 20;
  c->max_outer = 100;
  c->omega = 0.9;
  c->cycles = 1;
  c->coarse = COARSE_SWEEPS;
  c->coarse_sweeps = 3;
  c->solver = 0;
}

int fde_march_create(const fde_problem* p, size_t n1, size_t n2, size_t steps,
                     const fde_driver_config* cfg, fde_march* out) {
  return guard([&] {
    need(out && cfg, "null argument");
    need(cfg->solver == 0 || cfg->solver == 1, "solver must be 0 (gmres) or 1 (bicgstab)");
    auto h = std::make_unique<fde_march_s>();
    h->p = to_problem(p);
    h->g = Grid(h->p, n1, n2, steps);
    h->cfg = *cfg;
    const size_t n = h->g.size();
    // driver.cpp:22-27: u0, operator and preconditioner (time-independent coefficients)
    const std::vector<double> u0 = sample_initial(h->p, h->g);
    if (h->p.time_dependent_coeffs) {
      // driver.cpp:23-27,37-41: op holds t^0; the step-1 operator and
      // preconditioner are built up front and refreshed in place per step
      h->op = assemble_step_operator(h->p, h->g, 0);
      h->next = assemble_step_operator(h->p, h->g, 1);
      h->next_m = 1;
      h->pc = make_pc(cfg->precond, h->p, h->g, 1, h->next, cfg->omega, cfg->cycles,
                      cfg->coarse, cfg->coarse_sweeps);
    } else {
      h->op = assemble_step_operator(h->p, h->g, 1);
      h->pc = make_pc(cfg->precond, h->p, h->g, 1, h->op, cfg->omega, cfg->cycles, cfg->coarse,
                      cfg->coarse_sweeps);
    }
    h->ws = std::make_unique<KrylovWorkspace>(n, cfg->restart < 5 ? 5 : cfg->restart);
    h->u.upload(u0.data(), n);
    h->b.alloc(n);
    h->src.alloc(n);
    h->x.alloc(n);
    h->scale = 2.0 * std::pow(h->g.hx, h->p.alpha);
    *out = h.release();
  });
}

int fde_march_step(fde_march h, const double* source, int source_mode, void* stream,
                   size_t* iterations, double* residual) {
  return guard([&] {
    need(h != nullptr, "null handle");
    NvtxRange trace("fde:time-step");
    cudaStream_t s = stream_of(stream);
    const size_t n = h->g.size();
    const size_t m = h->m + 1;
    const double* src = h->src.get();
    if (h->p.time_dependent_coeffs && h->next_m != m) {
      // driver.cpp:37-41: re-assemble the step-m operator and preconditioner
      refresh_step_operator(*h->next, h->p, h->g, m, h->fields, s);
      const int kind = h->pc->kind();
      if (kind == PC_MGM) {
        Hierarchy* hh = h->pc->mutable_hierarchy();
        if (!refresh_geometric_hierarchy(*hh, h->p, h->g, m, h->fields, s))
          h->pc = make_pc(kind, h->p, h->g, m, h->next, h->cfg.omega, h->cfg.cycles,
                          h->cfg.coarse, h->cfg.coarse_sweeps);  // the level plan moved
      } else if (kind == PC_P2 || kind == PC_P2_EXACT || kind == PC_MGM_GALERKIN) {
        h->next->sync_host(s);  // build_p2 / to_csr read the operator's fields
        h->pc = make_pc(kind, h->p, h->g, m, h->next, h->cfg.omega, h->cfg.cycles,
                        h->cfg.coarse, h->cfg.coarse_sweeps);
      }
      h->next_m = m;
    }
    if (source_mode == 0) {
      if (h->p.example.which) {
        example_source_device(h->p, h->g, m, h->src.get(), s);
      } else if (h->p.preset) {
        // same counter hash on the device: uniforms bit-identical, Gaussians
        // within an ulp or two of the host's log/cos (Appendix A of the survey)
        generate_source_device(h->p, h->g, m, h->src.get(), s);
      } else {
        h->host_src.resize(n);
        sample_source(h->p, h->g, m, h->host_src.data());
        FDE_CUDA(cudaMemcpyAsync(h->src.get(), h->host_src.data(), n * sizeof(double),
                                 cudaMemcpyHostToDevice, s));
      }
    } else if (source_mode == 1) {
      need(source != nullptr, "null source");
      FDE_CUDA(cudaMemcpyAsync(h->src.get(), source, n * sizeof(double), cudaMemcpyHostToDevice, s));
    } else if (source_mode == 2) {
      need(source != nullptr, "null source");
      src = source;
    } else if (source_mode == 3) {
      need(h->npending > 0, "no prefetched source (fde_march_prefetch_source)");
      const int b = h->pending[0];
      h->pending[0] = h->pending[1];
      --h->npending;
      FDE_CUDA(cudaStreamWaitEvent(s, h->ev_ready[b], 0));
      src = h->ring[b].get();
      h->cur_src = b;
    } else {
      throw InvalidArgument("source_mode must be 0, 1, 2 or 3");
    }
    // the solve overwrites h->x: a solution copy that still reads THAT
    // allocation must finish first (u and x alternate between two allocations,
    // each with its own event, recorded after the last copy that reads it).
    // The copy of u^{m-1} reads h->u, which this step only reads: no wait, so
    // the D2H of one step overlaps the next step's solve.
    if (h->cs)
      for (int i = 0; i < 2; ++i)
        if (h->d2h_buf[i] == h->x.get()) FDE_CUDA(cudaStreamWaitEvent(s, h->ev_d2h[i], 0));
    // assemble_rhs (problem.cpp:73-89): b = apply_rhs(u) + 2 hx^alpha v, fused
    EpiArgs e;
    e.src = src;
    e.src_scale = h->scale;
    h->op->run(h->u.get(), h->b.get(), -1.0, EPI_RHS, e, s);
    if (source_mode == 3) FDE_CUDA(cudaEventRecord(h->ev_free[h->cur_src], s));
    SolverConfig c{h->cfg.tol, h->cfg.restart, h->cfg.max_outer};
    const Precond* pc = h->pc->kind() == PC_NONE ? nullptr : h->pc.get();
    const StructuredOp& a = h->p.time_dependent_coeffs ? *h->next : *h->op;
    const KrylovResult r = h->cfg.solver == 1
                               ? h->ws->bicgstab(a, pc, c, h->b.get(), h->x.get(), s)
                               : h->ws->gmres(a, pc, c, h->b.get(), h->x.get(), s);
    std::swap(h->u, h->x);
    if (h->p.time_dependent_coeffs) std::swap(h->op, h->next);  // driver.cpp:51
    h->ensure_io();
    FDE_CUDA(cudaEventRecord(h->ev_step, s));  // u^m final; orders the copy stream
    h->m = m;
    if (iterations) *iterations = r.total_iterations;
    if (residual) *residual = r.residual_history.back();
  });
}

int fde_march_steps_taken(fde_march h, size_t* m) {
  return guard([&] {
    need(h && m, "null argument");
    *m = h->m;
  });
}

int fde_march_solution(fde_march h, double* u, int to_host, void* stream) {
  return guard([&] {
    need(h && u, "null argument");
    cudaStream_t s = stream_of(stream);
    FDE_CUDA(cudaMemcpyAsync(u, h->u.get(), h->g.size() * sizeof(double),
                             to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    if (to_host) FDE_CUDA(cudaStreamSynchronize(s));
  });
}

int fde_march_prefetch_source(fde_march h, const double* host_source) {
  return guard([&] {
    need(h && host_source, "null argument");
    need(h->npending < 2, "two prefetched sources are already pending");
    h->ensure_io();
    const size_t n = h->g.size();
    int b = 0;  // a ring slot that is neither pending nor the last one consumed
    while (b == h->cur_src || (h->npending > 0 && h->pending[0] == b) ||
           (h->npending > 1 && h->pending[1] == b))
      ++b;
    if (h->ring[b].size() != n) h->ring[b].alloc(n);
    // the slot last fed an earlier step's rhs assembly: order after it
    FDE_CUDA(cudaStreamWaitEvent(h->cs, h->ev_free[b], 0));
    FDE_CUDA(cudaMemcpyAsync(h->ring[b].get(), host_source, n * sizeof(double),
                             cudaMemcpyHostToDevice, h->cs));
    FDE_CUDA(cudaEventRecord(h->ev_ready[b], h->cs));
    h->pending[h->npending++] = b;
  });
}

int fde_march_solution_async(fde_march h, double* host_u) {
  return guard([&] {
    need(h && host_u, "null argument");
    h->ensure_io();
    FDE_CUDA(cudaStreamWaitEvent(h->cs, h->ev_step, 0));  // u^m written by the last step
    FDE_CUDA(cudaMemcpyAsync(host_u, h->u.get(), h->g.size() * sizeof(double),
                             cudaMemcpyDeviceToHost, h->cs));
    // slot of this allocation (only two exist: slot 1 is the other one's or free)
    const int slot = (h->d2h_buf[0] == h->u.get() || h->d2h_buf[0] == nullptr) ? 0 : 1;
    FDE_CUDA(cudaEventRecord(h->ev_d2h[slot], h->cs));
    h->d2h_buf[slot] = h->u.get();
  });
}

int fde_march_wait(fde_march h) {
  return guard([&] {
    need(h != nullptr, "null handle");
    if (h->cs) FDE_CUDA(cudaStreamSynchronize(h->cs));
  });
}

int fde_march_solution_ptr(fde_march h, const double** u_dev) {
  return guard([&] {
    need(h && u_dev, "null argument");
    *u_dev = h->u.get();
  });
}

int fde_march_destroy(fde_march h) {
  return guard([&] { delete h; });
}

int fde_time_march(const fde_problem* p, size_t n1, size_t n2, size_t steps,
                   const fde_driver_config* cfg, double* solution, size_t* step_iterations,
                   double* step_residuals, double* wall_seconds) {
  fde_march h = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  int rc = fde_march_create(p, n1, n2, steps, cfg, &h);
  if (rc != FDE_OK) return rc;
  for (size_t m = 0; m < steps && rc == FDE_OK; ++m) {
    size_t it = 0;
    double res = 0.0;
    rc = fde_march_step(h, nullptr, 0, nullptr, &it, &res);
    if (step_iterations) step_iterations[m] = it;
    if (step_residuals) step_residuals[m] = res;
  }
  if (rc == FDE_OK && solution) rc = fde_march_solution(h, solution, 1, nullptr);
  const int rc2 = fde_march_destroy(h);
  if (wall_seconds)
    *wall_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return rc != FDE_OK ? rc : rc2;
}

int fde_slab_create(const fde_problem* p, size_t nf1, size_t nf2, size_t d1, size_t d2,
                    size_t steps, size_t m, size_t r0, size_t r1, size_t c0, size_t c1,
                    fde_slab* out) {
  return guard([&] {
    need(out != nullptr, "null output");
    auto h = std::make_unique<fde_slab_s>();
    h->op = std::make_unique<SlabOp>(to_problem(p), nf1, nf2, d1, d2, steps, m, r0, r1, c0, c1);
    *out = h.release();
  });
}
int fde_slab_ypass(fde_slab h, const double* xT, double* QT, double sign, void* stream) {
  return guard([&] {
    need(h && xT && QT, "null argument");
    h->op->ypass(xT, QT, sign, stream_of(stream));
  });
}
int fde_slab_xpass(fde_slab h, const double* x, const double* Q, double* out, double sign,
                   int epi, const double* b, const double* dinv, double omega, const double* src,
                   double src_scale, void* stream) {
  return guard([&] {
    need(h && x && Q && out, "null argument");
    need(epi >= EPI_STORE && epi <= EPI_JACOBI, "unknown epilogue");
    need(epi != EPI_RHS || src, "rhs epilogue needs src");
    need((epi != EPI_RESID && epi != EPI_JACOBI) || b, "epilogue needs b");
    need(epi != EPI_JACOBI || dinv, "jacobi epilogue needs dinv");
    EpiArgs e;
    e.b = b;
    e.dinv = dinv;
    e.omega = omega;
    e.src = src;
    e.src_scale = src_scale;
    h->op->xpass(x, Q, out, sign, epi, e, stream_of(stream));
  });
}
int fde_slab_diagonal(fde_slab h, double* d) {
  return guard([&] {
    need(h && d, "null argument");
    const auto& v = h->op->diagonal();
    std::memcpy(d, v.data(), v.size() * sizeof(double));
  });
}
int fde_slab_destroy(fde_slab h) {
  return guard([&] { delete h; });
}
int fde_transpose(const double* in, double* out, size_t rows, size_t cols, void* stream) {
  return guard([&] {
    need(in && out && in != out, "transpose needs distinct buffers");
    if (rows && cols) launch_transpose(in, out, (int)cols, (int)rows, stream_of(stream));
  });
}
int fde_transfer_rows(size_t n1, size_t n2, int coarsen_x, int coarsen_y, int op, int add,
                      const double* in, size_t in_lo, double* out, size_t out_lo,
                      size_t out_rows, void* stream) {
  return guard([&] {
    need(in && out, "null argument");
    const Xfer t = make_xfer((int)n1, (int)n2, coarsen_x != 0, coarsen_y != 0);
    if (op == 0) {
      need(out_lo + out_rows <= n2, "fine row window out of range");
      xfer_prolong_rows(t, in, (int)in_lo, out, (int)out_lo, (int)out_rows, add != 0,
                        stream_of(stream));
    } else if (op == 1 || op == 2) {
      need(out_lo + out_rows <= (size_t)t.k2, "coarse row window out of range");
      xfer_restrict_rows(t, in, (int)in_lo, out, (int)out_lo, (int)out_rows, op == 1 ? 0.5 : 1.0,
                         stream_of(stream));
    } else {
      throw InvalidArgument("transfer op must be 0, 1 or 2");
    }
  });
}
int fde_vec(int op, size_t n, double a, const double* x, const double* y, double* out,
            void* stream) {
  return guard([&] {
    need(x && out, "null argument");
    cudaStream_t s = stream_of(stream);
    switch (op) {
      case 0: need(y != nullptr, "null y"); vec_diag_scale(n, a, x, y, out, s); break;
      case 1: vec_axpy(n, a, x, out, s); break;
      case 2: need(y != nullptr, "null y"); vec_jacobi_update(n, a, x, y, out, s); break;
      case 3: vec_copy_scale(n, a, x, out, s); break;
      default: throw InvalidArgument("unknown vector op");
    }
  });
}
int fde_block_permute(const double* in, double* out, size_t nc, size_t d2,
                      const long long* offsets_host, int nranks, int dir, void* stream) {
  return guard([&] {
    need(in && out && offsets_host && nranks > 0 && nranks <= 64, "bad block permute arguments");
    need(offsets_host[0] == 0 && (size_t)offsets_host[nranks] == d2, "offsets must span [0, d2]");
    long long off[65];
    for (int r = 0; r <= nranks; ++r) off[r] = offsets_host[r];
    block_permute(in, out, nc, d2, off, nranks, dir, stream_of(stream));
  });
}
int fde_axpy_dev(size_t n, const double* a_dev, double sgn, const double* x, double* out,
                 void* stream) {
  return guard([&] {
    need(a_dev && x && out, "null argument");
    vec_axpy_dev(n, a_dev, sgn, x, out, stream_of(stream));
  });
}
int fde_dot(size_t n, const double* x, const double* y, double* out_dev, int sqrt_out,
            void* stream) {
  return guard([&] {
    need(x && y && out_dev, "null argument");
    static thread_local std::unique_ptr<Reducer> red;
    if (!red) red = std::make_unique<Reducer>();
    red->dot(n, x, y, out_dev, stream_of(stream), sqrt_out != 0);
  });
}


/* ------------------------------------------------ multi-GPU step (dist.cuh) */
int fde_dist_unique_id(unsigned char* id128) {
  return guard([&] {
    need(id128 != nullptr, "null id");
    nccl_unique_id(id128);
  });
}
int fde_dist_comm_create(const unsigned char* id128, int rank, int world, fde_dist_comm* out) {
  return guard([&] {
    need(id128 && out, "null argument");
    auto h = std::make_unique<fde_dist_comm_s>();
    h->c = make_nccl_comm(id128, rank, world);
    *out = h.release();
  });
}
int fde_dist_comm_destroy(fde_dist_comm c) {
  delete c;
  return FDE_OK;
}
static SolverConfig solver_cfg_of(const fde_driver_config* cfg) {
  SolverConfig sc;
  sc.tol = cfg->tol;
  sc.restart = cfg->restart;
  sc.max_outer = cfg->max_outer;
  return sc;
}
int fde_dist_march_create(fde_dist_comm c, const fde_problem* p, size_t n1, size_t n2,
                          size_t steps, const fde_driver_config* cfg, size_t agglomerate,
                          fde_dist_march* out) {
  return guard([&] {
    need(c && cfg && out, "null argument");
    need(cfg->solver == 0, "the y-slab march runs GMRES");
    need(cfg->precond == PC_NONE || cfg->precond == PC_MGM, "the y-slab march offers none / mgm");
    need(cfg->cycles == 1 || cfg->precond == PC_NONE, "the y-slab V-cycle runs one cycle");
    auto h = std::make_unique<fde_dist_march_s>();
    h->m = std::make_unique<DistMarch>(c->c, to_problem(p), n1, n2, steps, solver_cfg_of(cfg),
                                       cfg->omega, cfg->coarse, cfg->coarse_sweeps, agglomerate,
                                       cfg->precond == PC_MGM);
    *out = h.release();
  });
}
int fde_dist_march_rows(fde_dist_march h, size_t* r0, size_t* r1) {
  return guard([&] {
    need(h && r0 && r1, "null argument");
    *r0 = h->m->r0();
    *r1 = h->m->r1();
  });
}
int fde_dist_march_step(fde_dist_march h, const double* source_local, void* stream,
                        size_t* iterations, double* residual) {
  return guard([&] {
    need(h != nullptr, "null march");
    const DistReport r = h->m->step(source_local, stream_of(stream));
    if (iterations) *iterations = r.iterations;
    if (residual) *residual = r.final_rel;
  });
}
int fde_dist_march_solution(fde_dist_march h, double* u_local, int to_host, void* stream) {
  return guard([&] {
    need(h && u_local, "null argument");
    cudaStream_t s = stream_of(stream);
    FDE_CUDA(cudaMemcpyAsync(u_local, h->m->solution(), h->m->local_size() * sizeof(double),
                             to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
    if (to_host) FDE_CUDA(cudaStreamSynchronize(s));
  });
}
int fde_dist_march_solution_ptr(fde_dist_march h, const double** u_dev) {
  return guard([&] {
    need(h && u_dev, "null argument");
    *u_dev = h->m->solution();
  });
}
int fde_dist_march_apply(fde_dist_march h, const double* x_local, double* y_local, void* stream) {
  return guard([&] {
    need(h && x_local && y_local && x_local != y_local, "apply needs distinct buffers");
    h->m->level().run(x_local, y_local, 1.0, EPI_STORE, EpiArgs{}, stream_of(stream));
  });
}
int fde_dist_march_vcycle(fde_dist_march h, const double* b_local, double* x_local, void* stream) {
  return guard([&] {
    need(h && b_local && x_local && b_local != x_local, "V-cycle needs distinct buffers");
    need(h->m->hierarchy() != nullptr, "the march was created without a preconditioner");
    h->m->hierarchy()->vcycle(b_local, x_local, stream_of(stream));
  });
}
int fde_dist_march_collectives(fde_dist_march h, unsigned long long* n) {
  return guard([&] {
    need(h && n, "null argument");
    *n = h->m->comm().collectives();
  });
}
int fde_dist_split_rows(size_t n, int nranks, size_t* offsets) {
  return guard([&] {
    need(offsets && nranks > 0, "bad arguments");
    const auto o = split_ranges(n, nranks);
    for (int r = 0; r <= nranks; ++r) offsets[r] = o[r];
  });
}
int fde_dist_induced_rows(const size_t* fine_offsets, int nranks, size_t d2, int coarsen_y,
                          size_t* coarse_offsets) {
  return guard([&] {
    need(fine_offsets && coarse_offsets && nranks > 0, "bad arguments");
    const std::vector<size_t> f(fine_offsets, fine_offsets + nranks + 1);
    const auto o = induced_coarse_rows(f, d2, coarsen_y != 0);
    for (int r = 0; r <= nranks; ++r) coarse_offsets[r] = o[r];
  });
}
int fde_dist_march_destroy(fde_dist_march h) {
  delete h;
  return FDE_OK;
}

int fde_vdist_run(const fde_problem* p, size_t n1, size_t n2, size_t steps,
                  const fde_driver_config* cfg, int nranks, size_t agglomerate, int what,
                  size_t nrun, const double* in_full, double* out_full, size_t* iterations,
                  double* residuals, unsigned long long* collectives) {
  return guard([&] {
    need(cfg && out_full, "null argument");
    need(what >= 0 && what <= 2, "what must be 0 (march), 1 (apply) or 2 (V-cycle)");
    need(what == 0 || in_full, "apply / V-cycle need an input vector");
    need(cfg->solver == 0 && (cfg->precond == PC_NONE || cfg->precond == PC_MGM),
         "the y-slab march runs GMRES with none / mgm");
    need(what != 2 || cfg->precond == PC_MGM, "V-cycle needs precond mgm");
    const Problem prob = to_problem(p);
    auto comms = make_virtual_comms(nranks);
    const int dev = current_device();
    cudaStream_t s = nullptr;
    FDE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    std::vector<std::string> errs(nranks);
    std::vector<int> codes(nranks, 0);
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r)
      th.emplace_back([&, r] {
        try {
          FDE_CUDA(cudaSetDevice(dev));
          DistMarch m(comms[r], prob, n1, n2, steps, solver_cfg_of(cfg), cfg->omega, cfg->coarse,
                      cfg->coarse_sweeps, agglomerate, cfg->precond == PC_MGM);
          const size_t nl = m.local_size(), off = m.r0() * n1;
          DevBuf<double> a(nl + 1), b(nl + 1);
          const double* res = nullptr;
          if (what == 0) {
            for (size_t k = 0; k < nrun; ++k) {
              const DistReport rep = m.step(nullptr, s);
              if (r == 0 && iterations) iterations[k] = rep.iterations;
              if (r == 0 && residuals) residuals[k] = rep.final_rel;
            }
            res = m.solution();
          } else {
            FDE_CUDA(cudaMemcpyAsync(a.get(), in_full + off, nl * sizeof(double),
                                     cudaMemcpyHostToDevice, s));
            if (what == 1) m.level().run(a.get(), b.get(), 1.0, EPI_STORE, EpiArgs{}, s);
            else m.hierarchy()->vcycle(a.get(), b.get(), s);
            res = b.get();
          }
          FDE_CUDA(cudaMemcpyAsync(out_full + off, res, nl * sizeof(double),
                                   cudaMemcpyDeviceToHost, s));
          FDE_CUDA(cudaStreamSynchronize(s));
          if (r == 0 && collectives) *collectives = m.comm().collectives();
        } catch (const InvalidArgument& e) {
          errs[r] = e.what();
          codes[r] = 1;
          abort_virtual(*comms[r]);
        } catch (const std::exception& e) {
          errs[r] = e.what();
          codes[r] = 2;
          abort_virtual(*comms[r]);
        }
      });
    for (auto& t : th) t.join();
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    for (int r = 0; r < nranks; ++r)
      if (codes[r] == 1 && errs[r] != "a virtual rank failed") throw InvalidArgument(errs[r]);
    for (int r = 0; r < nranks; ++r)
      if (codes[r]) throw RuntimeError("virtual rank " + std::to_string(r) + ": " + errs[r]);
  });
}

}  // extern "C"
