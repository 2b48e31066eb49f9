#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>

#include "mg.cuh"

namespace fde_b200 {

size_t coarse_size(size_t n) { return (n - n % 2) / 2; }

double q_gamma_pi(double gamma) {
  // symbols.cpp:14-33 at xi = pi: z = 1 - e^{i pi} written as
  // 2 sin(xi/2) (sin(xi/2) - i cos(xi/2)); f = -(1 - gamma/2 conj z) z^gamma.
  const double xi = M_PI;
  const double s = std::sin(0.5 * xi), c = std::cos(0.5 * xi);
  const std::complex<double> z{2.0 * s * s, -2.0 * s * c};
  const std::complex<double> factor = -(1.0 - 0.5 * gamma * std::conj(z));
  return 2.0 * (factor * std::pow(z, gamma)).real();
}

double anisotropy_ratio(const StructuredOp& op, double alpha, double beta) {
  const auto mean = [](const std::vector<double>& a, const std::vector<double>& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] + b[i];
    return s / static_cast<double>(a.size());
  };
  const double cx = mean(op.dp(), op.dm()) * q_gamma_pi(alpha);
  const double cy = op.s_over_r() * mean(op.ep(), op.em()) * q_gamma_pi(beta);
  return cy / cx;
}

std::vector<std::pair<size_t, size_t>> plan_level_dims(size_t n1, size_t n2, double ratio0,
                                                       double alpha, double beta) {
  std::vector<std::pair<size_t, size_t>> dims{{n1, n2}};
  while (dims.back().first > 8 || dims.back().second > 8) {
    const auto [d1, d2] = dims.back();
    const double ratio = ratio0 * std::pow(double(n1 + 1) / double(d1 + 1), alpha) /
                         std::pow(double(n2 + 1) / double(d2 + 1), beta);
    bool cx = true, cy = true;
    if (ratio > 5.0) cx = false;
    else if (ratio < 1.0 / 5.0) cy = false;
    if (!cx && d2 <= 8) cx = true;
    if (!cy && d1 <= 8) cy = true;
    const size_t k1 = cx ? coarse_size(d1) : d1;
    const size_t k2 = cy ? coarse_size(d2) : d2;
    if ((cx && k1 == 0) || (cy && k2 == 0)) break;
    dims.emplace_back(k1, k2);
  }
  return dims;
}

std::vector<std::pair<size_t, size_t>> level_dims(size_t n1, size_t n2) {
  std::vector<std::pair<size_t, size_t>> dims{{n1, n2}};
  while (dims.back().first > 8 || dims.back().second > 8) {
    const size_t k1 = coarse_size(dims.back().first);
    const size_t k2 = coarse_size(dims.back().second);
    if (k1 == 0 || k2 == 0) break;
    dims.emplace_back(k1, k2);
  }
  return dims;
}

namespace {

// Dense row-major... column-major n x n matrix of a level (dense_assemble,
// structured.cpp:194-216, or the stencil planes).
std::vector<double> dense_of(const LevelOp& op, size_t n1, size_t n2) {
  const size_t n = n1 * n2;
  if (n > 4096) throw InvalidArgument("operator too large to densify");
  std::vector<double> m(n * n, 0.0);
  auto at = [&](size_t r, size_t c) -> double& { return m[r + c * n]; };
  if (op.sop) {
    const StructuredOp& o = *op.sop;
    for (size_t j = 0; j < n2; ++j)
      for (size_t i = 0; i < n1; ++i) {
        const size_t p = i + j * n1;
        at(p, p) += o.inv_r();
        for (size_t ii = 0; ii < n1; ++ii)
          at(p, ii + j * n1) +=
              o.dp()[p] * o.block_x().entry(i, ii) + o.dm()[p] * o.block_x().entry(ii, i);
        for (size_t jj = 0; jj < n2; ++jj)
          at(p, i + jj * n1) += o.s_over_r() * (o.ep()[p] * o.block_y().entry(j, jj) +
                                                o.em()[p] * o.block_y().entry(jj, j));
      }
  } else if (op.csr) {
    const Csr& c = op.csr->matrix();
    for (size_t r = 0; r < n; ++r)
      for (uint32_t k = c.ptr[r]; k < c.ptr[r + 1]; ++k) at(r, c.idx[k]) = c.val[k];
  } else {
    const std::vector<double>& c = op.stencil->coef();
    for (size_t j = 0; j < n2; ++j)
      for (size_t i = 0; i < n1; ++i) {
        const size_t p = i + j * n1;
        for (int dj = -1; dj <= 1; ++dj)
          for (int di = -1; di <= 1; ++di) {
            const long ii = (long)i + di, jj = (long)j + dj;
            if (ii < 0 || jj < 0 || ii >= (long)n1 || jj >= (long)n2) continue;
            at(p, (size_t)ii + (size_t)jj * n1) += c[(size_t)((dj + 1) * 3 + di + 1) * n + p];
          }
      }
  }
  return m;
}

// Row-pivoted LU in place (column-major), PA = LU; perm[i] = source row.
void lu_factor(std::vector<double>& a, size_t n, std::vector<int>& perm) {
  perm.resize(n);
  for (size_t i = 0; i < n; ++i) perm[i] = (int)i;
  auto A = [&](size_t i, size_t j) -> double& { return a[i + j * n]; };
  for (size_t k = 0; k < n; ++k) {
    size_t p = k;
    double best = std::fabs(A(k, k));
    for (size_t i = k + 1; i < n; ++i)
      if (std::fabs(A(i, k)) > best) {
        best = std::fabs(A(i, k));
        p = i;
      }
    if (p != k) {
      for (size_t j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
      std::swap(perm[k], perm[p]);
    }
    const double piv = A(k, k);
    if (piv == 0.0) throw RuntimeError("singular coarsest-level matrix");
    for (size_t i = k + 1; i < n; ++i) {
      const double l = A(i, k) / piv;
      A(i, k) = l;
      if (l == 0.0) continue;
      for (size_t j = k + 1; j < n; ++j) A(i, j) -= l * A(k, j);
    }
  }
}

__global__ void k_jacobi_update(size_t n, double omega, const double* __restrict__ dinv,
                                const double* __restrict__ r, double* __restrict__ x) {
  pdl_enter();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    x[i] += omega * dinv[i] * r[i];
}

}  // namespace

Hierarchy::Hierarchy(std::vector<LevelOp> levels, std::vector<std::pair<size_t, size_t>> dims,
                     int mode, double omega, int coarse, size_t coarse_sweeps)
    : levels_(std::move(levels)), dims_(std::move(dims)), mode_(mode), omega_(omega),
      coarse_(coarse), coarse_sweeps_(coarse_sweeps) {
  if (levels_.empty()) throw InvalidArgument("empty hierarchy");
  // bit 0: fold zero-guess smoothing into the residual pass, bit 1: fold the
  // prolongation correction into the post-smoothing pass (both bit-identical)
  if (const char* e = std::getenv("FDE_MG_FUSE")) fuse_ = std::atoi(e);
  if (levels_.size() != dims_.size()) throw InvalidArgument("level dims mismatch");
  if (!(omega_ > 0.0)) throw InvalidArgument("omega must be positive");
  if (coarse_ == COARSE_SWEEPS && coarse_sweeps_ == 0)
    throw InvalidArgument("coarse_sweeps must be positive");
  if (coarse_ < COARSE_LU || coarse_ > COARSE_NONE) throw InvalidArgument("unknown coarse solve");
  const size_t L = levels_.size();
  dinv_.resize(L);
  r_.resize(L);
  bc_.resize(L);
  xc_.resize(L);
  for (size_t l = 0; l < L; ++l) {
    const auto& d = levels_[l].diagonal();
    if (d.size() != dims_[l].first * dims_[l].second)
      throw InvalidArgument("level operator size does not match its dims");
    std::vector<double> inv(d.size());
    for (size_t i = 0; i < d.size(); ++i) {
      if (!(d[i] > 0.0)) throw InvalidArgument("operator diagonal must be strictly positive");
      inv[i] = 1.0 / d[i];
    }
    dinv_[l].upload(inv.data(), inv.size());
    if (levels_[l].sop) levels_[l].sop->freeze();  // 1/diag, inv_r, s/r are baked in from here on
    r_[l].alloc(d.size());
    if (l > 0) {
      bc_[l].alloc(d.size());
      xc_[l].alloc(d.size());
    }
  }
  for (size_t l = 0; l + 1 < L; ++l)
    xfer_.push_back(make_xfer((int)dims_[l].first, (int)dims_[l].second,
                              dims_[l + 1].first < dims_[l].first,
                              dims_[l + 1].second < dims_[l].second));
  for (size_t l = 0; l + 1 < L; ++l)
    if ((size_t)xfer_[l].k1 != dims_[l + 1].first || (size_t)xfer_[l].k2 != dims_[l + 1].second)
      throw InvalidArgument("level plan is not a coarsening chain");
  if (coarse_ == COARSE_LU) {
    const auto [c1, c2] = dims_.back();
    const size_t n = c1 * c2;
    std::vector<double> a = dense_of(levels_.back(), c1, c2);
    std::vector<int> perm;
    lu_factor(a, n, perm);
    lu_.upload(a.data(), a.size());
    perm_.upload(perm.data(), perm.size());
  }
  plan_tail();
}

// The tail starts at the first level from which every level is structured,
// small (kTailMaxN unknowns, kTailMaxLine per line) and fits the shared-memory
// budget with its iterate, right-hand side and diagonal tables, and the
// coarsest solve is sweeps or none.  Level 0 joins only for zero-guess cycles.
void Hierarchy::plan_tail() {
  tail_ = 0;
  if (const char* e = std::getenv("FDE_MG_TAIL"))
    if (e[0] == '0') return;
  if (coarse_ == COARSE_LU) return;
  size_t max_n = kTailMaxN;
  if (const char* e = std::getenv("FDE_MG_TAIL_N")) max_n = std::min<size_t>(std::atol(e), max_n);
  const size_t L = levels_.size();
  size_t start = L, need = 0;
  while (start > 0) {
    const size_t l = start - 1;
    const auto [n1, n2] = dims_[l];
    const size_t n = n1 * n2;
    // this level's x, b and tables; two scratch vectors of the first level's size
    const size_t with = need + 2 * n + (2 * n1 - 1) + (2 * n2 - 1);
    if (!levels_[l].sop || n > max_n || n1 > (size_t)kTailMaxLine ||
        n2 > (size_t)kTailMaxLine || L - l > (size_t)kTailMaxLevels ||
        with + 2 * n > (size_t)kTailSmemMax)
      break;
    need = with;
    start = l;
  }
  if (start >= L) return;
  if (start + 1 == L && coarse_ == COARSE_NONE) return;  // nothing to run
  TailDesc& d = tail_desc_;
  d = TailDesc{};
  d.nl = (int)(L - start);
  d.coarse = coarse_;
  d.sweeps = (int)coarse_sweeps_;
  d.omega = omega_;
  d.rsc = mode_ == MODE_GALERKIN ? 1.0 : 0.5;
  int off = 0;
  auto take = [&](size_t n) {
    const int o = off;
    off += (int)((n + 1) & ~size_t(1));  // 16-byte aligned vectors
    return o;
  };
  const size_t n0 = dims_[start].first * dims_[start].second;
  d.s0 = take(n0);
  d.s1 = take(n0);
  for (size_t l = start; l < L; ++l) {
    const StructuredOp& o = *levels_[l].sop;
    TailLevel& t = d.lv[l - start];
    t.n1 = (int)dims_[l].first;
    t.n2 = (int)dims_[l].second;
    t.inv_r = o.inv_r();
    t.sr = o.s_over_r();
    const LineBlockDev bx = o.block_x().dev(), by = o.block_y().dev();
    t.colx = bx.col;
    t.rowx = bx.row;
    t.coly = by.col;
    t.rowy = by.row;
    t.dp = o.dp_dev();
    t.dm = o.dm_dev();
    t.epT = o.epT_dev();
    t.emT = o.emT_dev();
    t.dinv = dinv_[l].get();
    t.xo = take((size_t)t.n1 * t.n2);
    t.bo = take((size_t)t.n1 * t.n2);
    t.tabx = take(2 * (size_t)t.n1 - 1);
    t.taby = take(2 * (size_t)t.n2 - 1);
    if (l + 1 < L) t.t = xfer_[l];
  }
  d.smem = off;
  if (off > kTailSmemMax) return;
  tail_ = start == 0 ? L : start;  // L marks "level 0" (0 means no tail)
}

void Hierarchy::refactor_coarse(cudaStream_t s) {
  if (coarse_ != COARSE_LU) return;
  const auto [c1, c2] = dims_.back();
  if (levels_.back().sop) levels_.back().sop->sync_host(s);
  std::vector<double> a = dense_of(levels_.back(), c1, c2);
  std::vector<int> perm;
  lu_factor(a, c1 * c2, perm);
  FDE_CUDA(cudaStreamSynchronize(s));
  lu_.upload(a.data(), a.size());  // same sizes: buffers keep their addresses
  perm_.upload(perm.data(), perm.size());
}

void Hierarchy::vcycle(const double* b, double* x, bool zero_guess, cudaStream_t s) const {
  NvtxRange trace("fde:vcycle");
  cycle(0, b, x, zero_guess, s);
}

// Does level l, entered with a zero guess, start with x = omega dinv b as a
// separate pass (so the restriction producing b can write it instead)?
bool Hierarchy::zero_guess_is_diag_scale(size_t l) const {
  const LevelOp& lev = levels_[l];
  const bool mapped = lev.sop && lev.sop->maps_input();
  if (l + 1 == levels_.size())
    return coarse_ == COARSE_SWEEPS && !(mapped && (fuse_ & 1) && coarse_sweeps_ > 1);
  return !(mapped && (fuse_ & 1));
}

void Hierarchy::cycle(size_t l, const double* b, double* x, bool zero, cudaStream_t s,
                      bool prescaled) const {
  if (tail_ && zero && l == (tail_ == levels_.size() ? 0 : tail_)) {
    TailDesc d = tail_desc_;
    d.b = b;
    d.x = x;
    d.prescaled = prescaled ? 1 : 0;
    launch_vcycle_tail(d, s);
    return;
  }
  const LevelOp& lev = levels_[l];
  const size_t n = lev.size();
  const double* dinv = dinv_[l].get();
  EpiArgs jac;
  jac.b = b;
  jac.dinv = dinv;
  jac.omega = omega_;
  // damped-Jacobi sweep x += omega dinv (b - A x), multigrid.cpp:358-360,380-382
  auto sweep = [&]() {
    if (lev.sop) {
      lev.run(x, x, EPI_JACOBI, jac, s);  // fused, in place (whole lines staged)
    } else {
      lev.run(x, r_[l].get(), EPI_RESID, jac, s);
      int blocks = (int)((n + 255) / 256);
      if (blocks > 148 * 8) blocks = 148 * 8;
      launch_k(k_jacobi_update, blocks, 256, 0, s, n, omega_, dinv, r_[l].get(), x);
      FDE_LAUNCH_CHECK();
    }
  };
  // zero-guess smoothing x = omega dinv b (multigrid.cpp:355-356) and the
  // correction x + P xc (multigrid.cpp:377-378) ride on the next operator
  // application's column transpose where the level has one (fine levels)
  const bool mapped = lev.sop && lev.sop->maps_input();
  InMap zin{};
  zin.kind = 1;
  zin.a = b;
  zin.d = dinv;
  zin.w = omega_;
  zin.ld = (int)dims_[l].first;
  if (l + 1 == levels_.size()) {  // multigrid.cpp:322-350
    if (coarse_ == COARSE_LU) {
      lu_solve((int)n, lu_.get(), perm_.get(), b, x, s);
    } else if (coarse_ == COARSE_SWEEPS) {
      size_t k = 1;
      if (!zero) {
        sweep();
      } else if (mapped && (fuse_ & 1) && coarse_sweeps_ > 1) {
        lev.sop->run_mapped(zin, x, x, 1.0, EPI_JACOBI, jac, s);  // first two sweeps
        k = 2;
      } else if (!prescaled) {
        vec_diag_scale(n, omega_, dinv, b, x, s);
      }
      for (; k < coarse_sweeps_; ++k) sweep();
    }
    return;
  }
  EpiArgs res;
  res.b = b;
  if (zero && mapped && (fuse_ & 1)) {
    lev.sop->run_mapped(zin, x, r_[l].get(), 1.0, EPI_RESID, res, s);  // x, r = b - A x
  } else {
    if (zero) {
      if (!prescaled) vec_diag_scale(n, omega_, dinv, b, x, s);
    } else {
      sweep();
    }
    lev.run(x, r_[l].get(), EPI_RESID, res, s);  // r = b - A x
  }
  const double rsc = mode_ == MODE_GALERKIN ? 1.0 : 0.5;
  const bool fuse_smooth = zero_guess_is_diag_scale(l + 1);
  if (fuse_smooth)
    xfer_restrict_smooth(xfer_[l], r_[l].get(), bc_[l + 1].get(), rsc, dinv_[l + 1].get(), omega_,
                         xc_[l + 1].get(), s);
  else
    xfer_restrict(xfer_[l], r_[l].get(), bc_[l + 1].get(), rsc, s);
  if (l + 2 == levels_.size() && coarse_ == COARSE_NONE) xc_[l + 1].zero(s);
  cycle(l + 1, bc_[l + 1].get(), xc_[l + 1].get(), true, s, fuse_smooth);
  if (mapped && (fuse_ & 2)) {
    InMap pin{};
    pin.kind = 2;
    pin.a = x;
    pin.t = xfer_[l];
    pin.c = xc_[l + 1].get();
    pin.ld = (int)dims_[l].first;
    lev.sop->run_mapped(pin, x, x, 1.0, EPI_JACOBI, jac, s);  // x += P xc, post-smooth
  } else {
    xfer_prolong_add(xfer_[l], xc_[l + 1].get(), x, s);  // x += P xc
    sweep();                                              // post-smooth
  }
}

}  // namespace fde_b200
