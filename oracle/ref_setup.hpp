// Problem setup shared by the oracle harnesses (TEST INFRASTRUCTURE ONLY):
// the BASELINE configurations as fde::FdeProblem objects over the UNMODIFIED
// reference headers, the (p,q) = (1,-1) blocks the
// reference lacks, and the reference-built V-cycle preconditioner.  Included
// by ref_harness.cpp (libfde_ref.so) and adapter.cpp (libfde_adapter.so).
#pragma once

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

// Mirrors the layout of fde_spec in paper_1706_06844_b200 tests (ctypes).
// Mirrors the layout of fde_spec in paper_1706_06844_b200 tests (ctypes).
struct ref_spec {
  int cfg;            // 1..5 (BASELINE configs), or 0 = cfg1 fields with pq/alpha overrides
  int n1, n2;         // grid (0 = config default)
  int steps;          // time steps (0 = config default)
  int precond;        // 0 none, 1 p2, 2 mgm, 3 p2-exact, 4 mgm-galerkin
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

namespace refh {

// ---- synthetic inputs ------------------------------
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

struct Cfg {
  int n;
  double alpha, beta, tau;
  int steps;
  int pq;
  int source_kind;
};

inline Cfg defaults(int cfg) {
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

// The reference's manufactured examples (cfg 101..103 -> make_example(k),
// problem.cpp:257-260; defaults of builtin_examples, problem.cpp:262-265;
// the table command's Grid(p, n, n, n), cli.cpp:172).
inline Setup make_example_setup(const ref_spec& s) {
  const int which = s.cfg - 100;
  const double al = s.alpha > 0 ? s.alpha : 1.8;
  const double be = s.beta > 0 ? s.beta : (which == 1 ? 1.6 : 1.9);
  fde::FdeProblem p = fde::make_example(which, al, be);
  const int n1 = s.n1 > 0 ? s.n1 : 32, n2 = s.n2 > 0 ? s.n2 : n1;
  const int steps = s.steps > 0 ? s.steps : n1;
  fde::Grid g(p, static_cast<std::size_t>(n1), static_cast<std::size_t>(n2),
              static_cast<std::size_t>(steps));
  return Setup{p, g, 0};
}

inline Setup make_setup(const ref_spec& s) {
  if (s.cfg > 100) return make_example_setup(s);
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
inline std::vector<double> wsgd_weights_pq(double gamma, std::size_t K, int pq) {
  if (pq == 0) return fde::wsgd_weights(gamma, K).w;
  const std::vector<double> g = fde::binom_coeffs(gamma, K);
  const double l1 = (gamma + 2.0) / 4.0, l2 = (2.0 - gamma) / 4.0;
  std::vector<double> w(K + 1);
  for (std::size_t k = 0; k <= K; ++k) w[k] = l1 * g[k] + (k >= 2 ? l2 * g[k - 2] : 0.0);
  return w;
}

inline fde::ToeplitzBlock block_pq(double gamma, std::size_t n, int pq) {
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
inline fde::StructuredFdeOperator step_op(const fde::FdeProblem& p, const fde::Grid& g,
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
inline fde::mg::MgHierarchy geometric(const fde::FdeProblem& p, const fde::Grid& g,
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

inline fde::mg::CoarseSolve coarse_of(int c) {
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

inline std::unique_ptr<fde::Precond> make_pc(const ref_spec& s, const Setup& st,
                                      const fde::StructuredFdeOperator& op) {
  if (s.precond == 2)
    return std::make_unique<HierPrecond>(
        geometric(st.p, st.g, 1, st.pq, s.omega, coarse_of(s.coarse),
                  static_cast<std::size_t>(s.coarse_sweeps)),
        st.g.size(), static_cast<std::size_t>(s.cycles));
  if (s.precond == 1)
    return fde::make_preconditioner(fde::PrecondKind::p2, st.p, st.g, 1, op, s.omega,
                                    static_cast<std::size_t>(s.cycles));
  if (s.precond == 3)
    return fde::make_preconditioner(fde::PrecondKind::p2_exact, st.p, st.g, 1, op, s.omega,
                                    static_cast<std::size_t>(s.cycles));
  if (s.precond == 4)
    return fde::make_preconditioner(fde::PrecondKind::mgm_galerkin, st.p, st.g, 1, op, s.omega,
                                    static_cast<std::size_t>(s.cycles), coarse_of(s.coarse),
                                    static_cast<std::size_t>(s.coarse_sweeps));
  return nullptr;
}

}  // namespace refh
