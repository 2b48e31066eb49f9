#include <algorithm>
#include <cmath>

#include "problem.cuh"

namespace fde_b200 {

Grid::Grid(const Problem& p, size_t n1_, size_t n2_, size_t steps_) {
  if (n1_ == 0 || n2_ == 0 || steps_ == 0)
    throw InvalidArgument("grid needs n1, n2, steps >= 1");
  if (!(p.bx > p.ax) || !(p.by > p.ay) || !(p.t_final > 0.0))
    throw InvalidArgument("degenerate domain");
  n1 = n1_;
  n2 = n2_;
  steps = steps_;
  ax = p.ax;
  bx = p.bx;
  ay = p.ay;
  by = p.by;
  t_final = p.t_final;
  hx = (bx - ax) / static_cast<double>(n1 + 1);
  hy = (by - ay) / static_cast<double>(n2 + 1);
  dt = t_final / static_cast<double>(steps);
  r = dt / (2.0 * std::pow(hx, p.alpha));
  s = dt / (2.0 * std::pow(hy, p.beta));
  inv_r = 1.0 / r;
  s_over_r = s / r;
}

std::shared_ptr<StructuredOp> assemble_step_operator(const Problem& p, const Grid& g,
                                                     size_t m) {
  if (!p.d_plus || !p.d_minus || !p.e_plus || !p.e_minus)
    throw InvalidArgument("problem is missing a coefficient field");
  const double t = static_cast<double>(m) * g.dt;
  const size_t n = g.size();
  std::vector<double> dp(n), dm(n), ep(n), em(n);
  for (size_t j = 0; j < g.n2; ++j) {
    const double y = g.y(j);
    for (size_t i = 0; i < g.n1; ++i) {
      const double x = g.x(i);
      const size_t q = i + j * g.n1;
      dp[q] = p.d_plus(x, y, t);
      dm[q] = p.d_minus(x, y, t);
      ep[q] = p.e_plus(x, y, t);
      em[q] = p.e_minus(x, y, t);
    }
  }
  return std::make_shared<StructuredOp>(g.n1, g.n2, g.inv_r, g.s_over_r,
                                        ToeplitzDev::fractional(p.alpha, g.n1, p.pq),
                                        ToeplitzDev::fractional(p.beta, g.n2, p.pq),
                                        std::move(dp), std::move(dm), std::move(ep),
                                        std::move(em));
}

std::vector<double> sample_initial(const Problem& p, const Grid& g) {
  if (!p.initial) throw InvalidArgument("problem has no initial data");
  std::vector<double> u(g.size());
  for (size_t j = 0; j < g.n2; ++j)
    for (size_t i = 0; i < g.n1; ++i) u[i + j * g.n1] = p.initial(g.x(i), g.y(j));
  return u;
}

namespace {

double preset_value(int kind, uint64_t key) {
  if (kind == 2) return 0.0;
  if (kind == 1) {
    const double a = hash_u01(key), b = hash_u01(key ^ (1ull << 63));
    return 1e-2 * (std::sqrt(-2.0 * std::log(1.0 - a)) * std::cos(2.0 * M_PI * b));
  }
  return hash_u01(key);
}

__global__ void k_source(uint64_t seed, uint64_t m, int n1, int n2, int kind, double* v) {
  pdl_enter();
  const size_t n = (size_t)n1 * n2;
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    const uint64_t i = p % n1, j = p / n1;
    const uint64_t key = source_key(seed, m, j, i);
    double val;
    if (kind == 2) {
      val = 0.0;
    } else if (kind == 1) {
      const double a = hash_u01(key), b = hash_u01(key ^ (1ull << 63));
      val = 1e-2 * (sqrt(-2.0 * log(1.0 - a)) * cos(2.0 * M_PI * b));
    } else {
      val = hash_u01(key);
    }
    v[p] = val;
  }
}

}  // namespace

void sample_source(const Problem& p, const Grid& g, size_t m, double* v) {
  if (p.preset) {  // identical to evaluating the harness's source(x, y, t) lambda
    for (size_t j = 0; j < g.n2; ++j)
      for (size_t i = 0; i < g.n1; ++i)
        v[i + j * g.n1] = preset_value(p.source_kind, source_key(p.seed, m, j, i));
    return;
  }
  if (!p.source) throw InvalidArgument("problem has no source");
  const double t_half = (static_cast<double>(m) - 0.5) * g.dt;
  for (size_t j = 0; j < g.n2; ++j)
    for (size_t i = 0; i < g.n1; ++i) v[i + j * g.n1] = p.source(g.x(i), g.y(j), t_half);
}

void generate_source_device(const Problem& p, const Grid& g, size_t m, double* v,
                            cudaStream_t s) {
  if (!p.preset) throw InvalidArgument("device source generation needs a BASELINE preset");
  const size_t n = g.size();
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_k(k_source, blocks, 256, 0, s, p.seed, m, (int)g.n1, (int)g.n2, p.source_kind, v);
  FDE_LAUNCH_CHECK();
}

std::shared_ptr<Hierarchy> build_geometric_hierarchy(const Problem& p, const Grid& g, size_t m,
                                                     double omega, int coarse,
                                                     size_t coarse_sweeps) {
  auto fine = assemble_step_operator(p, g, m);
  const auto dims =
      plan_level_dims(g.n1, g.n2, anisotropy_ratio(*fine, p.alpha, p.beta), p.alpha, p.beta);
  std::vector<LevelOp> levels;
  for (size_t l = 0; l < dims.size(); ++l) {
    LevelOp lev;
    if (l == 0) {
      lev.sop = fine;
    } else {
      const Grid lg(p, dims[l].first, dims[l].second, g.steps);
      lev.sop = assemble_step_operator(p, lg, m);
      // rediscretised levels carry their own hx^alpha; rescale onto the fine level
      lev.sop->scale(std::pow(g.hx / lg.hx, p.alpha));
    }
    levels.push_back(std::move(lev));
  }
  return std::make_shared<Hierarchy>(std::move(levels), dims, MODE_GEOMETRIC, omega, coarse,
                                     coarse_sweeps);
}

namespace {

// 1D prolongation weights of fine index f from coarse indices (GridTransfer:
// coarse c at fine 2c+1-par, stencil [1/2, 1, 1/2]; identity if not coarsened).
int prolong_weights(int f, int k, int par, bool coarsened, int* c, double* w) {
  if (!coarsened) {
    c[0] = f;
    w[0] = 1.0;
    return 1;
  }
  const int t = f - 1 + par;
  int cnt = 0;
  if ((t & 1) == 0) {
    const int j = t >> 1;
    if (j >= 0 && j < k) { c[cnt] = j; w[cnt++] = 1.0; }
  } else {
    const int jl = (t - 1) >> 1;
    if (jl >= 0 && jl < k) { c[cnt] = jl; w[cnt++] = 0.5; }
    if (jl + 1 >= 0 && jl + 1 < k) { c[cnt] = jl + 1; w[cnt++] = 0.5; }
  }
  return cnt;
}

// A_c = P^T A P on 9-point stencil planes (sparse.cpp:131-136 for CSR).
std::vector<double> galerkin(const std::vector<double>& a, const Xfer& t) {
  const size_t nf = (size_t)t.n1 * t.n2, nc = (size_t)t.k1 * t.k2;
  std::vector<double> ac(9 * nc, 0.0);
  for (int b1 = 0; b1 < t.k2; ++b1)
    for (int a1 = 0; a1 < t.k1; ++a1) {
      const size_t c1 = (size_t)a1 + (size_t)b1 * t.k1;
      const int fa = t.cx ? 2 * a1 + 1 - t.par1 : a1;
      const int fb = t.cy ? 2 * b1 + 1 - t.par2 : b1;
      const int rx = t.cx ? 1 : 0, ry = t.cy ? 1 : 0;
      for (int dj = -ry; dj <= ry; ++dj)
        for (int di = -rx; di <= rx; ++di) {
          const int i1 = fa + di, j1 = fb + dj;
          if (i1 < 0 || j1 < 0 || i1 >= t.n1 || j1 >= t.n2) continue;
          const double p1 = (di == 0 ? 1.0 : 0.5) * (dj == 0 ? 1.0 : 0.5);
          const size_t f1 = (size_t)i1 + (size_t)j1 * t.n1;
          for (int ej = -1; ej <= 1; ++ej)
            for (int ei = -1; ei <= 1; ++ei) {
              const double av = a[(size_t)((ej + 1) * 3 + ei + 1) * nf + f1];
              if (av == 0.0) continue;
              const int i2 = i1 + ei, j2 = j1 + ej;
              int ca[2], cb[2];
              double wa[2], wb[2];
              const int na = prolong_weights(i2, t.k1, t.par1, t.cx, ca, wa);
              const int nb = prolong_weights(j2, t.k2, t.par2, t.cy, cb, wb);
              for (int qb = 0; qb < nb; ++qb)
                for (int qa = 0; qa < na; ++qa) {
                  const int oa = ca[qa] - a1, ob = cb[qb] - b1;
                  if (oa < -1 || oa > 1 || ob < -1 || ob > 1)
                    throw RuntimeError("galerkin operator left the 9-point pattern");
                  ac[(size_t)((ob + 1) * 3 + oa + 1) * nc + c1] += p1 * av * wa[qa] * wb[qb];
                }
            }
        }
    }
  return ac;
}

}  // namespace

std::shared_ptr<Hierarchy> build_p2_hierarchy(const StructuredOp& op, double omega) {
  const size_t n1 = op.n1(), n2 = op.n2(), n = n1 * n2;
  std::vector<double> a(9 * n, 0.0);
  for (size_t j = 0; j < n2; ++j)
    for (size_t i = 0; i < n1; ++i) {  // build_p2, precond.cpp:50-73
      const size_t p = i + j * n1;
      const double cx = op.dp()[p] + op.dm()[p];
      const double cy = op.s_over_r() * (op.ep()[p] + op.em()[p]);
      a[4 * n + p] = op.inv_r() + 2.0 * cx + 2.0 * cy;
      if (i > 0) a[3 * n + p] = -cx;
      if (i + 1 < n1) a[5 * n + p] = -cx;
      if (j > 0) a[1 * n + p] = -cy;
      if (j + 1 < n2) a[7 * n + p] = -cy;
    }
  const auto dims = level_dims(n1, n2);
  std::vector<LevelOp> levels;
  for (size_t l = 0; l < dims.size(); ++l) {
    if (l > 0) {
      const Xfer t = make_xfer((int)dims[l - 1].first, (int)dims[l - 1].second,
                               dims[l].first < dims[l - 1].first,
                               dims[l].second < dims[l - 1].second);
      a = galerkin(a, t);
    }
    LevelOp lev;
    lev.stencil = std::make_shared<StencilOp>(dims[l].first, dims[l].second, a);
    levels.push_back(std::move(lev));
  }
  return std::make_shared<Hierarchy>(std::move(levels), dims, MODE_GALERKIN, omega, COARSE_NONE,
                                     3);
}

Csr build_p2_csr(const StructuredOp& op) {
  const size_t n1 = op.n1(), n2 = op.n2(), n = n1 * n2;
  std::vector<Csr::Triplet> t;
  t.reserve(5 * n);
  for (size_t j = 0; j < n2; ++j)
    for (size_t i = 0; i < n1; ++i) {  // precond.cpp:50-73
      const uint32_t p = (uint32_t)(i + j * n1);
      const double cx = op.dp()[p] + op.dm()[p];
      const double cy = op.s_over_r() * (op.ep()[p] + op.em()[p]);
      t.push_back({p, p, op.inv_r() + 2.0 * cx + 2.0 * cy});
      if (i > 0) t.push_back({p, p - 1, -cx});
      if (i + 1 < n1) t.push_back({p, p + 1, -cx});
      if (j > 0) t.push_back({p, (uint32_t)(p - n1), -cy});
      if (j + 1 < n2) t.push_back({p, (uint32_t)(p + n1), -cy});
    }
  return Csr::from_triplets(n, n, std::move(t));
}

std::shared_ptr<Hierarchy> build_galerkin_csr_hierarchy(const StructuredOp& op,
                                                        std::vector<std::pair<size_t, size_t>> dims,
                                                        double omega, int coarse,
                                                        size_t coarse_sweeps) {
  if (op.n1() > 128 || op.n2() > 128)
    throw InvalidArgument("galerkin variant limited to 128 x 128 grids");  // precond.cpp:121-123
  if (dims.empty() || dims.front() != std::make_pair(op.n1(), op.n2()))
    throw InvalidArgument("plan does not start at the fine grid");
  Csr a = structured_to_csr(op);
  std::vector<LevelOp> levels;
  for (size_t l = 0; l < dims.size(); ++l) {
    if (l > 0)
      a = rap(prolong_matrix(make_xfer((int)dims[l - 1].first, (int)dims[l - 1].second,
                                       dims[l].first < dims[l - 1].first,
                                       dims[l].second < dims[l - 1].second)),
              a);
    LevelOp lev;
    lev.csr = std::make_shared<CsrOp>(a);
    levels.push_back(std::move(lev));
  }
  return std::make_shared<Hierarchy>(std::move(levels), dims, MODE_GALERKIN, omega, coarse,
                                     coarse_sweeps);
}

ExampleSpec make_example_spec(int which, double alpha, double beta, double ax, double bx,
                              double ay, double by) {
  if (which < 1 || which > 3) throw InvalidArgument("example index must be 1..3");
  if (!(alpha > 1.0 && alpha <= 2.0 && beta > 1.0 && beta <= 2.0))
    throw InvalidArgument("fractional orders must lie in (1, 2]");
  if (!(bx > ax) || !(by > ay)) throw InvalidArgument("degenerate domain");
  ExampleSpec s;
  s.which = which;
  s.alpha = alpha;
  s.beta = beta;
  s.ax = ax;
  s.bx = bx;
  s.ay = ay;
  s.by = by;
  s.amp = which == 1 ? 16.0 : 1.0;
  // quartic xi^2 (len - xi)^2 (example 1) / sextic xi^3 (len - xi)^3 profiles
  auto profile = [which](double len, EndPoly& q) {
    if (which == 1) {
      const double c[] = {0.0, 0.0, len * len, -2.0 * len, 1.0};
      q.n = 5;
      for (int p = 0; p < q.n; ++p) q.c[p] = c[p];
    } else {
      const double c[] = {0.0, 0.0, 0.0, len * len * len, -3.0 * len * len, 3.0 * len, -1.0};
      q.n = 7;
      for (int p = 0; p < q.n; ++p) q.c[p] = c[p];
    }
  };
  profile(bx - ax, s.px);
  profile(by - ay, s.py);
  auto factors = [](double gamma, EndPoly& q) {  // frac_deriv's per-term constants
    for (int p = 0; p < q.n; ++p) {
      q.keep[p] = false;
      if (q.c[p] == 0.0) continue;
      const double qq = static_cast<double>(p) + 1.0 - gamma;
      if (qq <= 0.0 && std::fabs(qq - std::nearbyint(qq)) < 1e-12) continue;
      q.keep[p] = true;
      q.f[p] = q.c[p] * std::tgamma(static_cast<double>(p) + 1.0) / std::tgamma(qq);
      q.e[p] = qq - 1.0;
    }
  };
  factors(alpha, s.px);
  factors(beta, s.py);
  if (which == 1) {
    s.ga = std::tgamma(3.0 - alpha);
    s.gb = std::tgamma(3.0 - beta);
  }
  return s;
}

Problem make_example_problem(int which, double alpha, double beta, double ax, double bx,
                             double ay, double by) {
  const ExampleSpec s = make_example_spec(which, alpha, beta, ax, bx, ay, by);
  Problem p;
  p.alpha = alpha;
  p.beta = beta;
  p.ax = ax;
  p.bx = bx;
  p.ay = ay;
  p.by = by;
  p.t_final = 1.0;
  p.time_dependent_coeffs = which == 2;
  p.example = s;
  p.d_plus = [s](double x, double y, double t) { return example_coeff(s, 0, x, y, t); };
  p.d_minus = [s](double x, double y, double t) { return example_coeff(s, 1, x, y, t); };
  p.e_plus = [s](double x, double y, double t) { return example_coeff(s, 2, x, y, t); };
  p.e_minus = [s](double x, double y, double t) { return example_coeff(s, 3, x, y, t); };
  p.source = [s](double x, double y, double t) { return example_source(s, x, y, t); };
  p.initial = [s](double x, double y) { return example_initial(s, x, y); };
  p.exact = [s](double x, double y, double t) { return example_exact(s, x, y, t); };
  return p;
}

Problem make_example_default(int which, double alpha, double beta) {
  const double len = which == 1 ? 2.0 : 1.0;
  return make_example_problem(which, alpha, beta, 0.0, len, 0.0, len);
}

double error_inf(const std::vector<double>& u, const Problem& p, const Grid& g, double t) {
  if (!p.exact) throw InvalidArgument("problem has no exact solution");
  if (u.size() != g.size()) throw InvalidArgument("size mismatch");
  double e = 0.0;
  for (size_t j = 0; j < g.n2; ++j)
    for (size_t i = 0; i < g.n1; ++i) {
      const double ref = p.exact(g.x(i), g.y(j), t);
      e = std::max(e, std::fabs(u[i + j * g.n1] - ref));
    }
  return e;
}

PresetInfo preset_info(int cfg) {
  switch (cfg) {
    case 1: return {63, 1.8, 1.6, 1.0 / 64, 64, 0, 0};
    case 2: return {255, 1.5, 1.7, 1.0 / 256, 32, 0, 0};
    case 3: return {1023, 1.1, 1.9, 1.0 / 128, 16, 1, 1};
    case 4: return {2047, 1.6, 1.4, 1.0 / 64, 8, 0, 0};
    case 5: return {2047, 1.7, 1.3, 1.0 / 64, 1, 0, 0};
  }
  throw InvalidArgument("unknown BASELINE config id (1..5)");
}

Problem make_preset(int cfg, uint64_t seed, int source_kind, size_t steps, double tau) {
  const PresetInfo in = preset_info(cfg);
  Problem p;
  p.alpha = in.alpha;
  p.beta = in.beta;
  p.ax = 0.0;
  p.bx = 1.0;
  p.ay = 0.0;
  p.by = 1.0;
  p.t_final = (tau > 0 ? tau : in.tau) * static_cast<double>(steps ? steps : in.steps);
  p.pq = in.pq;
  p.preset = cfg;
  p.seed = seed;
  p.source_kind = source_kind >= 0 ? source_kind : in.source_kind;
  switch (cfg) {
    case 1: {
      auto one = [](double, double, double) { return 1.0; };
      p.d_plus = one;
      p.d_minus = one;
      p.e_plus = one;
      p.e_minus = one;
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
    case 5: {  // reference coefficient preset 1 (problem.cpp:196-209) on [0,1]^2
      const double al = p.alpha, be = p.beta, ax = 0.0, bx = 1.0, ay = 0.0, by = 1.0;
      const double ga = std::tgamma(3.0 - al), gb = std::tgamma(3.0 - be);
      p.d_plus = [=](double x, double y, double) {
        return ga * std::pow(1.0 + x - ax, al) * (1.0 + y - ay) * (1.0 + y - ay);
      };
      p.d_minus = [=](double x, double y, double) {
        return ga * std::pow(1.0 + bx - x, al) * (1.0 + by - y) * (1.0 + by - y);
      };
      p.e_plus = [=](double x, double y, double) {
        return gb * (1.0 + x - ax) * (1.0 + x - ax) * std::pow(1.0 + y - ay, be);
      };
      p.e_minus = [=](double x, double y, double) {
        return gb * (1.0 + bx - x) * (1.0 + bx - x) * std::pow(1.0 + by - y, be);
      };
      break;
    }
  }
  p.initial = [](double x, double y) {
    return x * x * (1.0 - x) * (1.0 - x) * y * y * (1.0 - y) * (1.0 - y);
  };
  const int kind = p.source_kind;
  const uint64_t sd = seed;
  // source(x, y, t) in the reference's callback form (used only for custom grids)
  p.source = [kind, sd](double, double, double) -> double {
    (void)kind;
    (void)sd;
    throw InvalidArgument("preset sources are indexed; use sample_source");
  };
  return p;
}

}  // namespace fde_b200
