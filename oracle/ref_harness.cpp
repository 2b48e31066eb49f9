// Harness around the UNMODIFIED reference sources (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libfde_ref.so).
//
// TEST INFRASTRUCTURE ONLY: this file is the checker's adapter to the real
// reference.  Only tests/, __graft_entry__.smoke() and bench.py's cpu-baseline
// / --impl reference legs may load the library it builds.
//
// It builds the five BASELINE configurations as fde::FdeProblem objects
// (counter-hash seeded sources, custom coefficient
// lambdas, t_final = tau * steps) and exposes flat extern "C" entry points
// for ctypes.  Nothing here re-implements reference arithmetic except where
// the reference has no code at all:
//   * WSGD (p,q) = (1,-1) weights (cfg3; absent from the reference,
//     proj/include/fde/weights.hpp:7-9) -- restated in wsgd_weights_pq below
//     and fed to the reference's public ToeplitzBlock(col,row) constructor
//     (proj/include/fde/structured.hpp:22);
//   * the per-step loop that records every u^m (driver.cpp:34-52 restated over
//     the reference's own assemble_rhs / make_preconditioner / gmres), used
//     for golden trajectories.  ref_time_march calls fde::time_march itself.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fde/driver.hpp"
#include "fde/krylov.hpp"
#include "fde/multigrid.hpp"
#include "fde/precond.hpp"
#include "fde/problem.hpp"
#include "fde/structured.hpp"
#include "fde/weights.hpp"

namespace {

thread_local std::string g_err;

// ---- synthetic inputs ------------------------------
inline std::uint64_t mix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline std::uint64_t src_key(std::uint64_t seed, std::uint64_t m, std::uint64_t j,
                             std::uint64_t i) {
  return seed ^ (m << 42) ^ (j << 21) ^ i;
}
inline double u01(std::uint64_t key) {
  return static_cast<double>(mix64(key) >> 11) * 0x1.0p-53;
}
inline double gauss(std::uint64_t key) {
  const double a = u01(key), b = u01(key ^ (1ull << 63));
  return std::sqrt(-2.0 * std::log(1.0 - a)) * std::cos(2.0 * M_PI * b);
}

}  // namespace

extern "C" {

// Mirrors the layout of fde_spec in paper_1706_06844_b200 tests (ctypes).
struct ref_spec {
  int cfg;            // 1..5 (BASELINE configs), or 0 = cfg1 fields with pq/alpha overrides
  int n1, n2;         // grid (0 = config default)
  int steps;          // time steps (0 = config default)
  int precond;        // 0 none, 1 p2, 2 mgm
  int restart;        // GMRES restart
  int max_outer;
  int cycles;         // V-cycles per preconditioner apply
  int coarse;         // 0 lu, 1 sweeps, 2 none
  int coarse_sweeps;
  int pq;             // 0 = (1,0), 1 = (1,-1)
  int source_kind;    // 0 = U[0,1), 1 = 1e-2 N(0,1), 2 = zero
  double tol;
  double omega;
  double alpha, beta; // 0 = config default
  double tau;         // 0 = config default
  unsigned long long seed;
};

const char* ref_last_error() { return g_err.c_str(); }

}  // extern "C"

namespace {

struct Cfg {
  int n;
  double alpha, beta, tau;
  int steps;
  int pq;
  int source_kind;
};

Cfg defaults(int cfg) {
  switch (cfg) {
    case 0:
    case 1: return {63, 1.8, 1.6, 1.0 / 64, 64, 0, 0};
    case 2: return {255, 1.5, 1.7, 1.0 / 256, 32, 0, 0};
    case 3: return {1023, 1.1, 1.9, 1.0 / 128, 16, 1, 1};
    case 4: return {2047, 1.6, 1.4, 1.0 / 64, 8, 0, 0};
    case 5: return {2047, 1.7, 1.3, 1.0 / 64, 1, 0, 0};
  }
  throw std::invalid_argument("unknown config id");
}

struct Setup {
  fde::FdeProblem p;
  fde::Grid g;
  int pq = 0;
};

Setup make_setup(const ref_spec& s) {
  Cfg c = defaults(s.cfg);
  const int n1 = s.n1 > 0 ? s.n1 : c.n;
  const int n2 = s.n2 > 0 ? s.n2 : c.n;
  const int steps = s.steps > 0 ? s.steps : c.steps;
  const double tau = s.tau > 0 ? s.tau : c.tau;
  fde::FdeProblem p;
  p.name = "cfg" + std::to_string(s.cfg);
  p.alpha = s.alpha > 0 ? s.alpha : c.alpha;
  p.beta = s.beta > 0 ? s.beta : c.beta;
  p.ax = 0.0; p.bx = 1.0; p.ay = 0.0; p.by = 1.0;
  p.t_final = tau * static_cast<double>(steps);
  p.time_dependent_coeffs = false;
  switch (s.cfg) {
    case 0:
    case 1: {
      auto one = [](double, double, double) { return 1.0; };
      p.d_plus = one; p.d_minus = one; p.e_plus = one; p.e_minus = one;
      break;
    }
    case 2:
    case 4:
      p.d_plus = [](double x, double y, double) { return 1.0 + x + y; };
      p.d_minus = [](double x, double y, double) { return 2.0 - x + y; };
      p.e_plus = [](double x, double y, double) { return 1.0 + x * y; };
      p.e_minus = [](double x, double y, double) { return 1.0 + (1.0 - x) * (1.0 - y); };
      break;
    case 3:
      p.d_plus = [](double x, double, double) {
        const double s = std::sin(M_PI * x);
        return 1.0 + s * s;
      };
      p.d_minus = [](double, double y, double) {
        const double c = std::cos(M_PI * y);
        return 1.0 + c * c;
      };
      p.e_plus = [](double x, double y, double) { return 2.0 + x - y; };
      p.e_minus = [](double x, double y, double) { return 2.0 - x + y; };
      break;
    case 5: {
      // reference coefficient preset 1 (problem.cpp:196-209) on [0,1]^2
      fde::FdeProblem e = fde::make_example_on(1, p.alpha, p.beta, 0.0, 1.0, 0.0, 1.0);
      p.d_plus = e.d_plus; p.d_minus = e.d_minus; p.e_plus = e.e_plus; p.e_minus = e.e_minus;
      break;
    }
    default: throw std::invalid_argument("unknown config id");
  }
  p.initial = [](double x, double y) {
    return x * x * (1.0 - x) * (1.0 - x) * y * y * (1.0 - y) * (1.0 - y);
  };
  const int skind = s.source_kind >= 0 ? s.source_kind : c.source_kind;
  fde::Grid g(p, static_cast<std::size_t>(n1), static_cast<std::size_t>(n2),
              static_cast<std::size_t>(steps));
  const double hx = g.hx, hy = g.hy, dt = g.dt;
  const std::uint64_t seed = s.seed;
  p.source = [hx, hy, dt, seed, skind](double x, double y, double t) {
    if (skind == 2) return 0.0;
    const long i = std::lround(x / hx) - 1, j = std::lround(y / hy) - 1;
    const long m = std::lround(t / dt + 0.5);
    const std::uint64_t key = src_key(seed, static_cast<std::uint64_t>(m),
                                      static_cast<std::uint64_t>(j),
                                      static_cast<std::uint64_t>(i));
    return skind == 1 ? 1e-2 * gauss(key) : u01(key);
  };
  Setup out{p, g, s.pq >= 0 ? s.pq : c.pq};
  return out;
}

// ---- (p,q) = (1,-1) weights: NOT in the reference (restated; unpinned) ----
// WSGD: w_k = l1 g_k + l2 g_{k-(p-q)}, l1 = (gamma-2q)/(2(p-q)),
// l2 = (2p-gamma)/(2(p-q)); (1,0) reproduces weights.cpp:42-47.
std::vector<double> wsgd_weights_pq(double gamma, std::size_t K, int pq) {
  if (pq == 0) return fde::wsgd_weights(gamma, K).w;
  const std::vector<double> g = fde::binom_coeffs(gamma, K);
  const double l1 = (gamma + 2.0) / 4.0, l2 = (2.0 - gamma) / 4.0;
  std::vector<double> w(K + 1);
  for (std::size_t k = 0; k <= K; ++k) w[k] = l1 * g[k] + (k >= 2 ? l2 * g[k - 2] : 0.0);
  return w;
}

fde::ToeplitzBlock block_pq(double gamma, std::size_t n, int pq) {
  if (pq == 0) return fde::ToeplitzBlock::fractional(gamma, n);
  // same layout as structured.cpp:47-55, different weight table
  const std::vector<double> w = wsgd_weights_pq(gamma, n < 2 ? 2 : n, pq);
  std::vector<double> col(n), row(n, 0.0);
  for (std::size_t i = 0; i < n; ++i) col[i] = -w[i + 1];
  row[0] = -w[1];
  if (n > 1) row[1] = -w[0];
  return fde::ToeplitzBlock(std::move(col), std::move(row));
}

// assemble_step_operator (problem.cpp:50-71) with the (p,q) block choice.
fde::StructuredFdeOperator step_op(const fde::FdeProblem& p, const fde::Grid& g,
                                   std::size_t m, int pq) {
  if (pq == 0) return fde::assemble_step_operator(p, g, m);
  const double t = static_cast<double>(m) * g.dt;
  const std::size_t n = g.size();
  std::vector<double> dp(n), dm(n), ep(n), em(n);
  for (std::size_t j = 0; j < g.n2; ++j)
    for (std::size_t i = 0; i < g.n1; ++i) {
      const std::size_t q = i + j * g.n1;
      dp[q] = p.d_plus(g.x(i), g.y(j), t);
      dm[q] = p.d_minus(g.x(i), g.y(j), t);
      ep[q] = p.e_plus(g.x(i), g.y(j), t);
      em[q] = p.e_minus(g.x(i), g.y(j), t);
    }
  return fde::StructuredFdeOperator(g.n1, g.n2, g.inv_r, g.s_over_r,
                                    block_pq(p.alpha, g.n1, pq), block_pq(p.beta, g.n2, pq),
                                    std::move(dp), std::move(dm), std::move(ep),
                                    std::move(em));
}

// build_geometric_hierarchy (multigrid.cpp:407-441) with the (p,q) block choice.
fde::mg::MgHierarchy geometric(const fde::FdeProblem& p, const fde::Grid& g,
                               std::size_t m, int pq, double omega,
                               fde::mg::CoarseSolve coarse, std::size_t sweeps) {
  if (pq == 0) return fde::mg::build_geometric_hierarchy(p, g, m, omega, coarse, sweeps);
  auto fine = std::make_shared<fde::StructuredFdeOperator>(step_op(p, g, m, pq));
  const auto dims = fde::mg::plan_level_dims(
      g.n1, g.n2, fde::mg::anisotropy_ratio(*fine, p.alpha, p.beta), p.alpha, p.beta);
  std::vector<fde::mg::MgLevel> levels;
  for (std::size_t l = 0; l < dims.size(); ++l) {
    fde::mg::MgLevel lev;
    if (l == 0) {
      lev.op = fine;
    } else {
      const fde::Grid lg(p, dims[l].first, dims[l].second, g.steps);
      auto op = std::make_shared<fde::StructuredFdeOperator>(step_op(p, lg, m, pq));
      op->scale(std::pow(g.hx / lg.hx, p.alpha));
      lev.op = op;
    }
    lev.n1 = dims[l].first;
    lev.n2 = dims[l].second;
    levels.push_back(std::move(lev));
  }
  for (std::size_t l = 0; l + 1 < levels.size(); ++l)
    levels[l].transfer = fde::mg::GridTransfer(dims[l].first, dims[l].second,
                                               dims[l + 1].first < dims[l].first,
                                               dims[l + 1].second < dims[l].second);
  return fde::mg::MgHierarchy(std::move(levels), fde::mg::CoarseningMode::geometric,
                              omega, coarse, sweeps);
}

fde::mg::CoarseSolve coarse_of(int c) {
  return c == 0 ? fde::mg::CoarseSolve::lu
                : (c == 1 ? fde::mg::CoarseSolve::sweeps : fde::mg::CoarseSolve::none);
}

class HierPrecond final : public fde::Precond {
 public:
  HierPrecond(fde::mg::MgHierarchy h, std::size_t n, std::size_t cycles)
      : h_(std::move(h)), n_(n), cycles_(cycles) {}
  void apply(const double* r, double* z) const override {
    std::fill_n(z, n_, 0.0);  // precond.cpp:22-26
    for (std::size_t c = 0; c < cycles_; ++c) h_.vcycle(r, z);
  }

 private:
  fde::mg::MgHierarchy h_;
  std::size_t n_, cycles_;
};

std::unique_ptr<fde::Precond> make_pc(const ref_spec& s, const Setup& st,
                                      const fde::StructuredFdeOperator& op) {
  if (s.precond == 2)
    return std::make_unique<HierPrecond>(
        geometric(st.p, st.g, 1, st.pq, s.omega, coarse_of(s.coarse),
                  static_cast<std::size_t>(s.coarse_sweeps)),
        st.g.size(), static_cast<std::size_t>(s.cycles));
  if (s.precond == 1)
    return fde::make_preconditioner(fde::PrecondKind::p2, st.p, st.g, 1, op, s.omega,
                                    static_cast<std::size_t>(s.cycles));
  return nullptr;
}

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

}  // namespace

extern "C" {

int ref_wsgd_weights(double gamma, int K, int pq, double* g, double* w) {
  return guarded([&] {
    const std::vector<double> gg = fde::binom_coeffs(gamma, static_cast<std::size_t>(K));
    const std::vector<double> ww = wsgd_weights_pq(gamma, static_cast<std::size_t>(K), pq);
    std::memcpy(g, gg.data(), gg.size() * sizeof(double));
    std::memcpy(w, ww.data(), ww.size() * sizeof(double));
  });
}

int ref_toeplitz_apply_both(double gamma, int n, int pq, const double* x, double* y,
                            double* yt) {
  return guarded([&] { block_pq(gamma, static_cast<std::size_t>(n), pq).apply_both(x, y, yt); });
}

int ref_toeplitz_apply_colrow(int n, const double* col, const double* row, const double* x,
                              double* y, double* yt) {
  return guarded([&] {
    fde::ToeplitzBlock t(std::vector<double>(col, col + n), std::vector<double>(row, row + n));
    t.apply_both(x, y, yt);
  });
}

int ref_grid(const ref_spec* s, double* out /* hx hy dt inv_r s_over_r */) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    out[0] = st.g.hx; out[1] = st.g.hy; out[2] = st.g.dt;
    out[3] = st.g.inv_r; out[4] = st.g.s_over_r;
  });
}

int ref_coefficients(const ref_spec* s, double* dp, double* dm, double* ep, double* em) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    std::copy(op.dp().begin(), op.dp().end(), dp);
    std::copy(op.dm().begin(), op.dm().end(), dm);
    std::copy(op.ep().begin(), op.ep().end(), ep);
    std::copy(op.em().begin(), op.em().end(), em);
  });
}

int ref_op_apply(const ref_spec* s, int sign, const double* x, double* y) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    if (sign >= 0) op.apply(x, y); else op.apply_rhs(x, y);
  });
}

int ref_op_diagonal(const ref_spec* s, double* d) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    std::copy(op.diagonal().begin(), op.diagonal().end(), d);
  });
}

int ref_dense(const ref_spec* s, double* a /* N*N column-major */) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const Eigen::MatrixXd m = fde::dense_assemble(step_op(st.p, st.g, 1, st.pq));
    std::memcpy(a, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
  });
}

// Level plan; returns the number of levels (dims as n1,n2 pairs), <0 on error.
int ref_plan(const ref_spec* s, int* dims, int max_levels, double* ratio0) {
  int nl = -1;
  const int rc = guarded([&] {
    const Setup st = make_setup(*s);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    const double r = fde::mg::anisotropy_ratio(op, st.p.alpha, st.p.beta);
    if (ratio0) *ratio0 = r;
    const auto d = fde::mg::plan_level_dims(st.g.n1, st.g.n2, r, st.p.alpha, st.p.beta);
    nl = static_cast<int>(d.size());
    for (int l = 0; l < nl && l < max_levels; ++l) {
      dims[2 * l] = static_cast<int>(d[static_cast<std::size_t>(l)].first);
      dims[2 * l + 1] = static_cast<int>(d[static_cast<std::size_t>(l)].second);
    }
  });
  return rc ? -1 : nl;
}

int ref_plan_raw(int n1, int n2, double ratio0, double alpha, double beta, int* dims,
                 int max_levels) {
  int nl = -1;
  const int rc = guarded([&] {
    const auto d = fde::mg::plan_level_dims(static_cast<std::size_t>(n1),
                                            static_cast<std::size_t>(n2), ratio0, alpha, beta);
    nl = static_cast<int>(d.size());
    for (int l = 0; l < nl && l < max_levels; ++l) {
      dims[2 * l] = static_cast<int>(d[static_cast<std::size_t>(l)].first);
      dims[2 * l + 1] = static_cast<int>(d[static_cast<std::size_t>(l)].second);
    }
  });
  return rc ? -1 : nl;
}

// Grid transfers (multigrid.cpp:160-227): op 0 prolong, 1 restrict_full, 2 restrict_transpose.
int ref_transfer(int n1, int n2, int cx, int cy, int op, const double* in, double* out) {
  return guarded([&] {
    fde::mg::GridTransfer t(static_cast<std::size_t>(n1), static_cast<std::size_t>(n2),
                            cx != 0, cy != 0);
    if (op == 0) t.prolong(in, out);
    else if (op == 1) t.restrict_full(in, out);
    else t.restrict_transpose(in, out);
  });
}

// One V-cycle x <- vcycle(b, x) of the step-operator hierarchy (mgm) or the
// banded P2 Galerkin hierarchy (p2).
int ref_vcycle(const ref_spec* s, const double* b, double* x) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    if (s->precond == 1) {
      const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
      fde::mg::MgHierarchy h = fde::mg::build_galerkin_hierarchy(
          fde::build_p2(op).matrix, st.g.n1, st.g.n2, s->omega, fde::mg::CoarseSolve::none);
      h.vcycle(b, x);
      return;
    }
    const fde::mg::MgHierarchy h = geometric(st.p, st.g, 1, st.pq, s->omega,
                                             coarse_of(s->coarse),
                                             static_cast<std::size_t>(s->coarse_sweeps));
    h.vcycle(b, x);
  });
}

int ref_precond_apply(const ref_spec* s, const double* r, double* z) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    auto pc = make_pc(*s, st, op);
    if (pc) pc->apply(r, z); else std::memcpy(z, r, sizeof(double) * st.g.size());
  });
}

int ref_initial(const ref_spec* s, double* u) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const std::vector<double> v = fde::sample_initial(st.p, st.g);
    std::copy(v.begin(), v.end(), u);
  });
}

// Raw source samples v(x_i, y_j, t^{m-1/2}) (problem.cpp:81-87 call pattern).
int ref_source(const ref_spec* s, int m, double* v) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const double t_half = (static_cast<double>(m) - 0.5) * st.g.dt;
    for (std::size_t j = 0; j < st.g.n2; ++j)
      for (std::size_t i = 0; i < st.g.n1; ++i)
        v[i + j * st.g.n1] = st.p.source(st.g.x(i), st.g.y(j), t_half);
  });
}

int ref_rhs(const ref_spec* s, int m, const double* u_prev, double* b) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    const std::vector<double> u(u_prev, u_prev + st.g.size());
    const std::vector<double> v =
        fde::assemble_rhs(st.p, st.g, static_cast<std::size_t>(m), u, op);
    std::copy(v.begin(), v.end(), b);
  });
}

// One GMRES solve (krylov.cpp:34-166) with zero initial guess.
int ref_gmres(const ref_spec* s, const double* b, double* x, int* iterations, int* converged,
              double* history, int max_history, int* n_history) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    auto pc = make_pc(*s, st, op);
    fde::SolverConfig c;
    c.tol = s->tol;
    c.restart = static_cast<std::size_t>(s->restart);
    c.max_outer = static_cast<std::size_t>(s->max_outer);
    c.preconditioner = pc.get();
    const fde::KrylovResult r =
        fde::gmres(op, c, std::vector<double>(b, b + st.g.size()));
    std::copy(r.solution.begin(), r.solution.end(), x);
    *iterations = static_cast<int>(r.total_iterations);
    *converged = r.converged ? 1 : 0;
    const int nh = static_cast<int>(r.residual_history.size());
    *n_history = nh;
    for (int k = 0; k < nh && k < max_history; ++k) history[k] = r.residual_history[k];
  });
}

// Per-step time march (driver.cpp:34-52 over reference assemble_rhs/gmres),
// recording every u^m when u_steps != NULL.
int ref_march_timed(const ref_spec* s, double* u_out, int* its, double* res, double* u_steps,
                    double* wall, double* step_seconds);

int ref_march(const ref_spec* s, double* u_out, int* its, double* res, double* u_steps,
              double* wall) {
  return ref_march_timed(s, u_out, its, res, u_steps, wall, nullptr);
}

// Same loop; step_seconds[m-1] = wall time of step m alone (rhs + gmres).
int ref_march_timed(const ref_spec* s, double* u_out, int* its, double* res, double* u_steps,
                    double* wall, double* step_seconds) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<double> u = fde::sample_initial(st.p, st.g);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    auto pc = make_pc(*s, st, op);
    fde::SolverConfig c;
    c.tol = s->tol;
    c.restart = static_cast<std::size_t>(s->restart);
    c.max_outer = static_cast<std::size_t>(s->max_outer);
    c.preconditioner = pc.get();
    const std::size_t n = st.g.size();
    for (std::size_t m = 1; m <= st.g.steps; ++m) {
      const auto ts = std::chrono::steady_clock::now();
      const std::vector<double> b = fde::assemble_rhs(st.p, st.g, m, u, op);
      fde::KrylovResult r = fde::gmres(op, c, b);
      if (step_seconds)
        step_seconds[m - 1] =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count();
      its[m - 1] = static_cast<int>(r.total_iterations);
      res[m - 1] = r.residual_history.back();
      u = std::move(r.solution);
      if (u_steps) std::copy(u.begin(), u.end(), u_steps + (m - 1) * n);
    }
    std::copy(u.begin(), u.end(), u_out);
    if (wall)
      *wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// The reference's own fde::time_march (driver.cpp:10-69), (1,0) weights only.
int ref_time_march(const ref_spec* s, double* u_out, int* its, double* res, double* wall) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    if (st.pq != 0) throw std::invalid_argument("time_march supports (p,q)=(1,0) only");
    fde::DriverConfig c;
    c.precond = s->precond == 2 ? fde::PrecondKind::mgm
                                : (s->precond == 1 ? fde::PrecondKind::p2 : fde::PrecondKind::none);
    c.tol = s->tol;
    c.restart = static_cast<std::size_t>(s->restart);
    c.max_outer = static_cast<std::size_t>(s->max_outer);
    c.omega = s->omega;
    c.cycles = static_cast<std::size_t>(s->cycles);
    c.coarse = coarse_of(s->coarse);
    c.coarse_sweeps = static_cast<std::size_t>(s->coarse_sweeps);
    const fde::SolveReport r = fde::time_march(st.p, st.g, c);
    std::copy(r.solution.begin(), r.solution.end(), u_out);
    for (std::size_t m = 0; m < r.step_iterations.size(); ++m) {
      its[m] = static_cast<int>(r.step_iterations[m]);
      res[m] = r.step_residuals[m];
    }
    *wall = r.wall_seconds;
  });
}

// Timing helpers for the CPU baseline (single thread, the reference's native mode).
int ref_time_apply(const ref_spec* s, int reps, double* seconds_each) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const fde::StructuredFdeOperator op = step_op(st.p, st.g, 1, st.pq);
    std::vector<double> x(st.g.size()), y(st.g.size());
    for (std::size_t k = 0; k < x.size(); ++k) x[k] = 2.0 * u01(k) - 1.0;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      op.apply(x.data(), y.data());
      seconds_each[r] =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

int ref_time_vcycle(const ref_spec* s, int reps, double* seconds_each) {
  return guarded([&] {
    const Setup st = make_setup(*s);
    const fde::mg::MgHierarchy h = geometric(st.p, st.g, 1, st.pq, s->omega,
                                             coarse_of(s->coarse),
                                             static_cast<std::size_t>(s->coarse_sweeps));
    std::vector<double> b(st.g.size()), x(st.g.size());
    for (std::size_t k = 0; k < b.size(); ++k) b[k] = 2.0 * u01(k) - 1.0;
    for (int r = 0; r < reps; ++r) {
      std::fill(x.begin(), x.end(), 0.0);
      const auto t0 = std::chrono::steady_clock::now();
      h.vcycle(b.data(), x.data());
      seconds_each[r] =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
  });
}

}  // extern "C"
