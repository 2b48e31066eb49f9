#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <utility>

#include "krylov.cuh"

namespace fde_b200 {
namespace {

__global__ void k_copy_scale(size_t n, double a, const double* __restrict__ x,
                             double* __restrict__ y) {
  pdl_enter();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = x[i] * a;
}
void copy_scale(size_t n, double a, const double* x, double* y, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_k(k_copy_scale, blocks, 256, 0, s, n, a, x, y);
  FDE_LAUNCH_CHECK();
}

// Small scalar transfers between device scratch and the pinned host staging
// (UVA-mapped): one tiny kernel instead of a DMA copy, so the solver's
// per-iteration round trip never queues behind bulk host copies running on
// other streams (the march's pipelined source / solution transfers).
__global__ void k_copy_small(double* __restrict__ dst, const double* __restrict__ src, int n) {
  pdl_enter();
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
void copy_small(double* dst, const double* src, size_t n, cudaStream_t s) {
  launch_k(k_copy_small, 1, 128, 0, s, dst, src, (int)n);
  FDE_LAUNCH_CHECK();
}

// device-to-device vector copy on the SMs (a DMA copy would queue behind the
// march's bulk host transfers on the copy engines)
__global__ void k_copy(size_t n, const double* __restrict__ x, double* __restrict__ y) {
  pdl_enter();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}
void copy_vec(size_t n, const double* x, double* y, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  launch_k(k_copy, blocks ? blocks : 1, 256, 0, s, n, x, y);
  FDE_LAUNCH_CHECK();
}

// back_substitute (krylov.cpp:19-30)
std::vector<double> back_substitute(const std::vector<double>& h, size_t ld,
                                    const std::vector<double>& g, size_t k) {
  std::vector<double> y(k, 0.0);
  for (size_t i = k; i-- > 0;) {
    double v = g[i];
    for (size_t j = i + 1; j < k; ++j) v -= h[j * ld + i] * y[j];
    y[i] = h[i * ld + i] != 0.0 ? v / h[i * ld + i] : 0.0;
  }
  return y;
}

}  // namespace

Precond::Precond(int kind, std::shared_ptr<Hierarchy> h, size_t n, size_t cycles)
    : kind_(kind), h_(std::move(h)), n_(n), cycles_(cycles) {
  if (kind_ != PC_NONE && !h_) throw InvalidArgument("preconditioner needs a hierarchy");
  if (kind_ != PC_NONE && cycles_ == 0) throw InvalidArgument("cycles must be >= 1");
  if (const char* e = std::getenv("FDE_NO_GRAPH")) use_graphs_ = e[0] != '1';
}

Precond::Precond(std::shared_ptr<BandedLu> lu, size_t n)
    : kind_(PC_P2_EXACT), lu_(std::move(lu)), n_(n), cycles_(1) {
  if (!lu_ || lu_->size() != n_) throw InvalidArgument("p2-exact needs its factorisation");
}

Precond::~Precond() {
  for (Entry& e : graphs_) cudaGraphExecDestroy(e.exec);
  if (cap_) cudaStreamDestroy(cap_);
}

void Precond::record(const double* r, double* z, cudaStream_t s) const {
  // z = 0; cycles x vcycle(r, z): the first cycle is the zero-guess path
  // (the reference scans z, multigrid.cpp:387-392).  With one cycle the
  // zero fill is dead work: every path of the zero-guess cycle writes z.
  if (cycles_ > 1 || h_->coarse() == COARSE_NONE)
    FDE_CUDA(cudaMemsetAsync(z, 0, n_ * sizeof(double), s));
  for (size_t c = 0; c < cycles_; ++c) h_->vcycle(r, z, c == 0, s);
}

void Precond::apply(const double* r, double* z, cudaStream_t s) const {
  if (kind_ == PC_NONE) {
    copy_vec(n_, r, z, s);
    return;
  }
  if (kind_ == PC_P2_EXACT) {
    lu_->solve(r, z, s);
    return;
  }
  if (!use_graphs_) {
    record(r, z, s);
    return;
  }
  for (const Entry& e : graphs_)
    if (e.r == r && e.z == z) {
      FDE_CUDA(cudaGraphLaunch(e.exec, s));
      g_kernel_launches.fetch_add(e.kernels, std::memory_order_relaxed);
      return;
    }
  if (graphs_.size() >= 8) {  // bounded cache (callers normally reuse a few buffers)
    for (Entry& e : graphs_) cudaGraphExecDestroy(e.exec);
    graphs_.clear();
  }
  if (!cap_) FDE_CUDA(cudaStreamCreateWithFlags(&cap_, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  const unsigned long long before = g_kernel_launches.load();
  FDE_CUDA(cudaStreamBeginCapture(cap_, cudaStreamCaptureModeRelaxed));
  try {
    record(r, z, cap_);
  } catch (...) {
    cudaStreamEndCapture(cap_, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  FDE_CUDA(cudaStreamEndCapture(cap_, &g));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t err = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  FDE_CUDA(err);
  // captured launches were counted while recording; replays count again
  graphs_.push_back(Entry{r, z, exec, g_kernel_launches.load() - before});
  FDE_CUDA(cudaGraphLaunch(exec, s));
}

KrylovWorkspace::KrylovWorkspace(size_t n, size_t restart) : n_(n), rst_(restart) {
  if (restart == 0) throw InvalidArgument("invalid solver configuration");
  v_.resize(rst_ + 1);
  std::vector<const double*> ptrs(rst_ + 1);
  for (size_t k = 0; k <= rst_; ++k) {
    v_[k].alloc(n);
    ptrs[k] = v_[k].get();
  }
  for (DevBuf<double>* b : {&t_, &r_, &z_, &w_, &w2_, &trial_}) b->alloc(n);
  dsc_.alloc(4 * (rst_ + 2) + 16);
  dcoef_.alloc(rst_ + 1);
  dptr_.upload(ptrs.data(), ptrs.size());
  FDE_CUDA(cudaMallocHost(&hsc_, sizeof(double) * (4 * (rst_ + 2) + 16 + rst_ + 1)));
  hstride_ = rst_ + 4;
  FDE_CUDA(cudaMallocHost(&hstep_, sizeof(double) * 2 * hstride_));
  for (cudaEvent_t& e : ev_step_) FDE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (const char* e = std::getenv("FDE_GMRES_SPECULATE")) speculate_ = e[0] != '0';
}

KrylovWorkspace::~KrylovWorkspace() {
  for (cudaEvent_t e : ev_step_)
    if (e) cudaEventDestroy(e);
  if (hstep_) cudaFreeHost(hstep_);
  if (hsc_) cudaFreeHost(hsc_);
}

void KrylovWorkspace::precondition(const Precond* m, const double* r, double* z,
                                   cudaStream_t s) {
  if (m) m->apply(r, z, s);
  else copy_vec(n_, r, z, s);
}

void KrylovWorkspace::fetch(size_t count, cudaStream_t s) {
  copy_small(hsc_, dsc_.get(), count, s);
  FDE_CUDA(cudaStreamSynchronize(s));
}

double KrylovWorkspace::nrm2_host(const double* v, cudaStream_t s) {
  red_.dot(n_, v, v, dsc_.get(), s, true);
  fetch(1, s);
  return hsc_[0];
}

double KrylovWorkspace::dot_host(const double* x, const double* y, cudaStream_t s) {
  red_.dot(n_, x, y, dsc_.get(), s, false);
  fetch(1, s);
  return hsc_[0];
}

double KrylovWorkspace::true_rel(const StructuredOp& a, const Precond* m, const double* b,
                                 const double* x, double norm_b, cudaStream_t s) {
  EpiArgs e;
  e.b = b;
  a.run(x, r_.get(), 1.0, EPI_RESID, e, s);  // r = b - A x (krylov.cpp:60-61)
  precondition(m, r_.get(), z_.get(), s);
  return nrm2_host(z_.get(), s) / norm_b;
}

KrylovResult KrylovWorkspace::gmres(const StructuredOp& a, const Precond* m,
                                    const SolverConfig& cfg, const double* b, double* x_out,
                                    cudaStream_t s) {
  NvtxRange trace("fde:gmres");
  const size_t n = n_;
  if (a.size() != n) throw InvalidArgument("rhs size mismatch");
  if (cfg.restart == 0 || !(cfg.tol > 0.0)) throw InvalidArgument("invalid solver configuration");
  if (cfg.restart > rst_) throw InvalidArgument("restart exceeds the workspace");
  const size_t rst = cfg.restart, ld = rst + 1;
  KrylovResult res;
  double* x = x_out;
  double* trial = trial_.get();
  FDE_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));

  precondition(m, b, z_.get(), s);
  const double norm_b = nrm2_host(z_.get(), s);
  if (norm_b == 0.0) {
    res.converged = true;
    res.residual_history.push_back(0.0);
    return res;
  }
  std::vector<double> h(ld * rst, 0.0), g(ld, 0.0), cs(rst, 0.0), sn(rst, 0.0), y;
  double* const dh = dsc_.get();              // h column slots [0, rst]
  double* const dnorm0 = dsc_.get() + ld;     // ||w|| before MGS
  double* const dnrmw = dsc_.get() + ld + 1;  // ||w|| after MGS
  double* const dreo = dsc_.get() + ld + 2;   // re-orthogonalisation coefficients
  auto lincomb_into = [&](const double* x0, double* out, const std::vector<double>& coef) {
    std::copy(coef.begin(), coef.end(), hsc_ + 4 * (rst_ + 2) + 16);
    copy_small(dcoef_.get(), hsc_ + 4 * (rst_ + 2) + 16, coef.size(), s);
    vec_lincomb(n, x0, dptr_.get(), dcoef_.get(), (int)coef.size(), out, s);
    FDE_CUDA(cudaStreamSynchronize(s));  // the pinned staging slot is reused
  };

  // z_ holds M^-1 (b - A x) for solution version zver (norm zbeta).  The
  // reference recomputes it at outer 0 (x = 0: exactly M^-1 b) and after an
  // accepted verification (same x): identical bits, so those applies and
  // V-cycles are reused instead of recomputed; counts and history unchanged.
  unsigned long xver = 0, zver = 0;  // x = 0 and z_ = M^-1 b now
  double zbeta = norm_b;
  auto residual_z = [&]() -> double {
    if (zver == xver) return zbeta;
    EpiArgs e;
    e.b = b;
    a.run(x, r_.get(), 1.0, EPI_RESID, e, s);  // r = b - A x (krylov.cpp:60-61,71-72)
    precondition(m, r_.get(), z_.get(), s);
    zbeta = nrm2_host(z_.get(), s);
    zver = xver;
    return zbeta;
  };

  for (size_t outer = 0; outer < cfg.max_outer && !res.converged; ++outer) {
    const double beta = residual_z();
    const double rel0 = beta / norm_b;
    if (outer == 0) res.residual_history.push_back(rel0);
    if (rel0 <= cfg.tol) {
      res.converged = true;
      break;
    }
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    copy_scale(n, 1.0 / beta, z_.get(), v_[0].get(), s);  // scal(1/beta); v[0] = z

    size_t spanned = 0;
    bool cycle_done = false;
    // Device work of Arnoldi step i: w = M^-1 A v_i, the Gram-Schmidt
    // projections, and the staging of the Hessenberg column for the host.
    // Steps alternate two w buffers and two pinned staging slots so the next
    // step can be enqueued before the host has read this one.
    bool enq[2] = {false, false}, chained[2] = {false, false};
    auto wbuf = [&](size_t i) { return (i & 1) ? w2_.get() : w_.get(); };
    auto enqueue = [&](size_t i) {
      NvtxRange step_trace("fde:arnoldi-step");
      double* w = wbuf(i);
      a.apply(v_[i].get(), t_.get(), s);
      precondition(m, t_.get(), w, s);
      // modified Gram-Schmidt (krylov.cpp:92-97): one cooperative launch with
      // w resident in shared memory (and v_{i+1} = w / ||w|| formed on the
      // way out), else each subtraction fused with the next projection: i + 2
      // passes over w instead of 2 (i + 1) + 2
      const bool ch = red_.mgs_chain(n, w, dptr_.get(), (int)i, dh, dnorm0, dnrmw,
                                     v_[i + 1].get(), s);
      if (!ch) {
        red_.norm_dot(n, w, v_[0].get(), dnorm0, dh, s);
        for (size_t k = 0; k <= i; ++k)
          red_.mgs(n, w, v_[k].get(), dh + k, k < i ? v_[k + 1].get() : w,
                   k < i ? dh + k + 1 : dnrmw, k == i, s);
      }
      copy_small(hstep_ + (i & 1) * hstride_, dsc_.get(), ld + 2, s);
      FDE_CUDA(cudaEventRecord(ev_step_[i & 1], s));
      enq[i & 1] = true;
      chained[i & 1] = ch;
    };
    double est_prev = rel0;
    for (size_t i = 0; i < rst && !cycle_done; ++i) {
      if (!enq[i & 1]) enqueue(i);
      // Speculate step i + 1 while the host waits for step i: it only needs
      // v_{i+1}, which the chained Gram-Schmidt forms on the device.  Worth it
      // while step i cannot converge (estimates fall by well under 20x per
      // step here); a step i that converges, breaks down or needs a second
      // Gram-Schmidt pass discards it.  Arithmetic is unchanged either way.
      if (speculate_ && chained[i & 1] && i + 1 < rst && est_prev > 20.0 * cfg.tol)
        enqueue(i + 1);
      FDE_CUDA(cudaEventSynchronize(ev_step_[i & 1]));
      const double* hs = hstep_ + (i & 1) * hstride_;
      enq[i & 1] = false;
      for (size_t k = 0; k <= i; ++k) h[i * ld + k] = hs[k];
      const double norm0 = hs[ld];
      double hip = hs[ld + 1];
      bool reorth = false;
      double* const w = wbuf(i);
      if (hip < 1e-8 * norm0) {  // second pass (krylov.cpp:98-104)
        reorth = true;
        enq[(i + 1) & 1] = false;  // a speculated step used the first-pass v_{i+1}
        red_.dot(n, v_[0].get(), w, dreo, s);
        for (size_t k = 0; k <= i; ++k)
          red_.mgs(n, w, v_[k].get(), dreo + k, k < i ? v_[k + 1].get() : w,
                   k < i ? dreo + k + 1 : dnrmw, k == i, s);
        fetch(ld + 2 + i + 1, s);
        for (size_t k = 0; k <= i; ++k) h[i * ld + k] += hsc_[ld + 2 + k];
        hip = hsc_[ld + 1];
      }
      const bool happy = hip <= 1e-14 * (norm0 > 0.0 ? norm0 : 1.0);

      for (size_t k = 0; k + 1 <= i; ++k) {  // apply previous rotations
        const double tmp = cs[k] * h[i * ld + k] + sn[k] * h[i * ld + k + 1];
        h[i * ld + k + 1] = -sn[k] * h[i * ld + k] + cs[k] * h[i * ld + k + 1];
        h[i * ld + k] = tmp;
      }
      const double denom = std::hypot(h[i * ld + i], hip);
      cs[i] = denom > 0.0 ? h[i * ld + i] / denom : 1.0;
      sn[i] = denom > 0.0 ? hip / denom : 0.0;
      h[i * ld + i] = denom;
      g[i + 1] = -sn[i] * g[i];
      g[i] = cs[i] * g[i];

      ++res.total_iterations;
      spanned = i + 1;
      const double est = std::fabs(g[i + 1]) / norm_b;
      est_prev = est;
      res.residual_history.push_back(est);
      // (the chained Gram-Schmidt already formed v_{i+1} unless a second pass ran)
      if (!happy && (!chained[i & 1] || reorth)) copy_scale(n, 1.0 / hip, w, v_[i + 1].get(), s);

      if (est <= cfg.tol || happy) {  // verify the estimate (krylov.cpp:132-149)
        y = back_substitute(h, ld, g, spanned);
        lincomb_into(x, trial, y);
        std::swap(x, trial);
        ++xver;
        if (residual_z() / norm_b <= cfg.tol) {  // true_rel (krylov.cpp:59-64)
          res.converged = true;
          cycle_done = true;
        } else if (happy) {
          cycle_done = true;
        } else {
          std::swap(x, trial);  // estimate lied: keep iterating
          ++xver;
        }
      }
    }
    // a step speculated past the end of the cycle is dropped (its outputs
    // are rewritten before any use)
    if (!res.converged && !cycle_done) {
      y = back_substitute(h, ld, g, spanned);
      lincomb_into(x, x, y);
      ++xver;
    }
  }
  const double final_rel = residual_z() / norm_b;
  if (final_rel <= cfg.tol) res.converged = true;
  if (res.residual_history.empty()) res.residual_history.push_back(final_rel);
  else res.residual_history.back() = final_rel;
  if (x != x_out)
    copy_vec(n, x, x_out, s);
  return res;
}

KrylovResult KrylovWorkspace::bicgstab(const StructuredOp& a, const Precond* m,
                                       const SolverConfig& cfg, const double* b, double* x,
                                       cudaStream_t s) {
  NvtxRange trace("fde:bicgstab");
  const size_t n = n_;
  if (a.size() != n) throw InvalidArgument("rhs size mismatch");
  if (cfg.restart == 0 || cfg.max_outer == 0 || !(cfg.tol > 0.0))
    throw InvalidArgument("invalid solver configuration");
  // BiCGSTAB vectors reuse the Arnoldi basis storage
  if (rst_ < 5) throw InvalidArgument("bicgstab needs a workspace with restart >= 5");
  double *r = v_[0].get(), *rh = v_[1].get(), *p = v_[2].get(), *v = v_[3].get(),
         *sv = v_[4].get(), *tv = v_[5 % (rst_ + 1)].get();
  double *tmp = t_.get(), *tmp2 = r_.get();
  const size_t max_it = cfg.restart * cfg.max_outer;
  KrylovResult res;
  FDE_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  precondition(m, b, r, s);  // r = M^-1 (b - A 0)
  const double norm_b = nrm2_host(r, s);
  if (norm_b == 0.0) {
    res.converged = true;
    res.residual_history.push_back(0.0);
    return res;
  }
  copy_vec(n, r, rh, s);
  res.residual_history.push_back(1.0);
  auto true_res = [&](const double* xv, double* out) {  // out = M^-1 (b - A xv)
    EpiArgs e;
    e.b = b;
    a.run(xv, tmp2, 1.0, EPI_RESID, e, s);
    precondition(m, tmp2, out, s);
    return nrm2_host(out, s) / norm_b;
  };
  // Fused iteration: every reduction lands in the device scalar block sc,
  // alpha / omega / beta are formed there, and the host reads the block twice
  // per iteration (after the half step and after the full step) for the
  // breakdown and convergence tests -- the same tests, in the same order, as
  // the restatement in oracle/fde_oracle.c.
  double* const sc = dsc_.get();
  int rho_cur = BICG_RHO_A;
  red_.dot(n, rh, r, sc + rho_cur, s, false);
  fetch(BICG_SLOTS, s);
  double rho_host = hsc_[rho_cur];
  for (size_t it = 0; it < max_it; ++it) {
    if (rho_host == 0.0) break;
    const int rho_old = rho_cur ^ 1;  // the previous iteration's <rh, r>
    if (it == 0) {
      copy_vec(n, r, p, s);
    } else {
      red_.bicg_p(n, r, v, p, sc, rho_cur, rho_old, s);
    }
    a.apply(p, tmp, s);
    precondition(m, tmp, v, s);
    red_.dot(n, rh, v, sc + BICG_RV, s, false);
    red_.bicg_s(n, r, v, sv, sc, rho_cur, s);  // alpha, s = r - alpha v, ||s||
    fetch(BICG_SLOTS, s);                      // host read 1 of 2
    if (hsc_[BICG_RV] == 0.0) break;
    const double alpha = hsc_[BICG_ALPHA];
    ++res.total_iterations;
    const double srel = hsc_[BICG_NS] / norm_b;
    if (srel <= cfg.tol) {  // half step: verify x + alpha p
      double* trial = trial_.get();
      copy_vec(n, x, trial, s);
      vec_axpy(n, alpha, p, trial, s);
      const double trel = true_res(trial, tv);
      if (trel <= cfg.tol) {
        copy_vec(n, trial, x, s);
        res.residual_history.push_back(trel);
        res.converged = true;
        break;
      }
    }
    a.apply(sv, tmp, s);
    precondition(m, tmp, tv, s);
    red_.bicg_tt(n, tv, sv, sc, s);
    // omega, x += alpha p + omega s, r = s - omega t, ||r||, next <rh, r>
    red_.bicg_xr(n, p, sv, tv, rh, x, r, sc, rho_old, s);
    fetch(BICG_SLOTS, s);  // host read 2 of 2
    rho_cur = rho_old;
    rho_host = hsc_[rho_cur];
    const double omg = hsc_[BICG_OMEGA];
    const double rel = hsc_[BICG_NR] / norm_b;
    res.residual_history.push_back(rel);
    if (rel <= cfg.tol) {
      if (true_res(x, tmp) <= cfg.tol) {
        res.converged = true;
        break;
      }
    }
    if (omg == 0.0) break;
  }
  const double final_rel = true_res(x, tmp);
  if (final_rel <= cfg.tol) res.converged = true;
  res.residual_history.back() = final_rel;
  return res;
}

}  // namespace fde_b200
