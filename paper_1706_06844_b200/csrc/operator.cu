// Host setup of the device-resident operator: WSGD weights, circulant
// spectra, twiddle tables, coefficient fields (reference structured.cpp,
// weights.cpp).  Setup arithmetic runs once per level in long double so the
// device tables are correctly rounded.
#include <cmath>
#include <complex>
#include <map>
#include <cstdlib>
#include <mutex>

#include "operator.cuh"

namespace fde_b200 {

std::vector<double> binom_coeffs(double gamma, size_t K) {
  if (!(gamma > 1.0) || !(gamma <= 2.0))
    throw InvalidArgument("weights: gamma must lie in (1, 2]");
  std::vector<double> g(K + 1);
  g[0] = 1.0;
  for (size_t k = 1; k <= K; ++k) g[k] = g[k - 1] * (1.0 - (gamma + 1.0) / double(k));
  return g;
}

std::vector<double> wsgd_weights(double gamma, size_t K, int pq) {
  if (K < 2) throw InvalidArgument("weights: K must be >= 2");
  const std::vector<double> g = binom_coeffs(gamma, K);
  std::vector<double> w(K + 1);
  if (pq == 0) {
    const double cg = 0.5 * gamma, cg1 = 0.5 * (2.0 - gamma);
    w[0] = cg;
    for (size_t k = 1; k <= K; ++k) w[k] = cg * g[k] + cg1 * g[k - 1];
  } else if (pq == 1) {
    const double l1 = (gamma + 2.0) / 4.0, l2 = (2.0 - gamma) / 4.0;
    for (size_t k = 0; k <= K; ++k) w[k] = l1 * g[k] + (k >= 2 ? l2 * g[k - 2] : 0.0);
  } else {
    throw InvalidArgument("weights: (p,q) selector must be 0 for (1,0) or 1 for (1,-1)");
  }
  return w;
}

size_t next_pow2(size_t n) {
  size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

namespace {

using cld = std::complex<long double>;
constexpr long double kPiL = 3.141592653589793238462643383279502884L;

// exp(-2 pi i k / n), correctly rounded to double via long double.
double2 unit_root(size_t k, size_t n) {
  const long double a = 2.0L * kPiL * (long double)k / (long double)n;
  return make_double2((double)cosl(a), (double)-sinl(a));
}

// In-place forward DFT of power-of-two length in long double (setup only).
void fft_ld(std::vector<cld>& a) {
  const size_t n = a.size();
  if (n <= 1) return;
  for (size_t i = 1, j = 0; i < n; ++i) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    for (size_t k = 0; k < len / 2; ++k) {
      const long double ang = -2.0L * kPiL * (long double)k / (long double)len;
      const cld w(cosl(ang), sinl(ang));
      for (size_t i = 0; i < n; i += len) {
        const cld u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
    }
  }
}

struct TwiddleTables {
  DevBuf<double2> twM;
};

const TwiddleTables& twiddles(int logM) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<TwiddleTables>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = cache[logM];
  if (!slot) {
    const size_t M = size_t(1) << logM;
    // compact per-stage layout: exp(-2 pi i j / Q), j < Q / 2, at Q / 2 + j for
    // every power of two Q <= M.  A stage with NS butterflies per group and
    // radix R reads the NS contiguous entries from NS R / 2, so the twiddles a
    // line kernel touches cover a few KB of L1 lines instead of strided
    // sectors all over a 16 M-byte table.
    std::vector<double2> tm(M, make_double2(1.0, 0.0));
    for (size_t Q = 2; Q <= M; Q <<= 1)
      for (size_t j = 0; j < Q / 2; ++j) tm[Q / 2 + j] = unit_root(j, Q);
    auto t = std::make_unique<TwiddleTables>();
    t->twM.upload(tm.data(), M);
    slot = std::move(t);
  }
  return *slot;
}

}  // namespace

ToeplitzDev::ToeplitzDev(std::vector<double> first_col, std::vector<double> first_row)
    : n_(first_col.size()), col_(std::move(first_col)), row_(std::move(first_row)) {
  if (n_ == 0 || row_.size() != n_)
    throw InvalidArgument("toeplitz column and row sizes must match");
  if (col_[0] != row_[0]) throw InvalidArgument("toeplitz corner entry mismatch");
  L_ = next_pow2(2 * n_ - 1);
  dcol_ = std::make_shared<DevBuf<double>>();
  drow_ = std::make_shared<DevBuf<double>>();
  dcol_->upload(col_.data(), n_);
  drow_->upload(row_.data(), n_);
  if (n_ <= size_t(kDirectMax)) {
    logM_ = 0;
    return;
  }
  const size_t M = L_ / 2;
  logM_ = 0;
  while ((size_t(1) << logM_) < M) ++logM_;
  if (logM_ > 13) throw InvalidArgument("line length beyond the supported FFT sizes (n <= 8191)");
  // circulant column (structured.cpp:21-30), spectrum scaled by 1/(2L)
  std::vector<cld> c(L_, cld(0.0L, 0.0L));
  for (size_t i = 0; i < n_; ++i) c[i] = (long double)col_[i];
  for (size_t j = 1; j < n_; ++j) c[L_ - j] = (long double)row_[j];
  fft_ld(c);
  // Per-k constants of the fused unpack -> multiply -> repack step
  // (line_conv.cu): with S~ = S / (2L), a = S~[k], b = conj(S~[M-k]),
  // W = exp(-2 pi i k / L) = cw + i sw:
  //   a_k = 2 (a + b + sw (a - b)),  b_k = 2 i cw (a - b).
  // Compact layout: a_k at index k (k < M); b_c at M + c for c <= M / 2 only,
  // because b_{M-k} = -conj(b_k) (cw flips sign, a and conj(b) swap).
  std::vector<double2> ab(M + M / 2 + 2, make_double2(0.0, 0.0));
  const long double sc = 1.0L / (2.0L * (long double)L_);
  for (size_t k = 0; k < M; ++k) {
    const cld a = c[k] * sc, b = std::conj(c[M - k] * sc);
    const long double ang = 2.0L * kPiL * (long double)k / (long double)L_;
    const long double cw = cosl(ang), sw = -sinl(ang);
    const cld ak = 2.0L * (a + b + sw * (a - b));
    const cld bk = 2.0L * cld(0.0L, cw) * (a - b);
    ab[k] = make_double2((double)ak.real(), (double)ak.imag());
    if (k <= M / 2) ab[M + k] = make_double2((double)bk.real(), (double)bk.imag());
  }
  spec_ = std::make_shared<DevBuf<double2>>();
  spec_->upload(ab.data(), ab.size());
}

ToeplitzDev ToeplitzDev::fractional(double gamma, size_t n, int pq) {
  if (n == 0) throw InvalidArgument("empty toeplitz block");
  const std::vector<double> w = wsgd_weights(gamma, n < 2 ? 2 : n, pq);
  std::vector<double> col(n), row(n, 0.0);
  for (size_t i = 0; i < n; ++i) col[i] = -w[i + 1];
  row[0] = -w[1];
  if (n > 1) row[1] = -w[0];
  return ToeplitzDev(std::move(col), std::move(row));
}

LineBlockDev ToeplitzDev::dev() const {
  LineBlockDev d{};
  d.n = (int)n_;
  d.logM = logM_;
  d.col = dcol_->get();
  d.row = drow_->get();
  if (logM_) {
    const TwiddleTables& t = twiddles(logM_);
    d.ab = spec_->get();
    d.twM = t.twM.get();
  }
  return d;
}

StructuredOp::StructuredOp(size_t n1, size_t n2, double inv_r, double s_over_r,
                           ToeplitzDev ax, ToeplitzDev ay, std::vector<double> dp,
                           std::vector<double> dm, std::vector<double> ep,
                           std::vector<double> em)
    : n1_(n1), n2_(n2), inv_r_(inv_r), s_over_r_(s_over_r), inv_r0_(inv_r),
      s_over_r0_(s_over_r), ax_(std::move(ax)),
      ay_(std::move(ay)), dp_(std::move(dp)), dm_(std::move(dm)), ep_(std::move(ep)),
      em_(std::move(em)) {
  const size_t n = n1_ * n2_;
  if (n == 0) throw InvalidArgument("empty operator");
  if (ax_.size() != n1_ || ay_.size() != n2_)
    throw InvalidArgument("toeplitz block size mismatch");
  if (dp_.size() != n || dm_.size() != n || ep_.size() != n || em_.size() != n)
    throw InvalidArgument("coefficient field size mismatch");
  if (!(inv_r_ > 0.0)) throw InvalidArgument("1/r must be positive");
  if (!(s_over_r_ > 0.0)) throw InvalidArgument("s/r must be positive");
  for (size_t p = 0; p < n; ++p)
    if (dp_[p] < 0.0 || dm_[p] < 0.0 || ep_[p] < 0.0 || em_[p] < 0.0)
      throw InvalidArgument("negative diffusion coefficient sample");
  const double ax0 = ax_.first_col()[0];
  const double ay0 = ay_.first_col()[0];
  diag_.resize(n);
  for (size_t p = 0; p < n; ++p)
    diag_[p] = inv_r_ + (dp_[p] + dm_[p]) * ax0 + s_over_r_ * (ep_[p] + em_[p]) * ay0;
  upload();
  d_q_.alloc(n);
  d_xT_.alloc(n);
  if (const char* e = std::getenv("FDE_NO_TRANSPOSE")) transpose_columns_ = e[0] != '1';
}

void StructuredOp::upload() {
  const size_t n = n1_ * n2_;
  d_dp_.upload(dp_.data(), n);
  d_dm_.upload(dm_.data(), n);
  d_diag_.upload(diag_.data(), n);
  std::vector<double> t(n);  // ep/em transposed for the column pass
  for (size_t j = 0; j < n2_; ++j)
    for (size_t i = 0; i < n1_; ++i) t[i * n2_ + j] = ep_[i + j * n1_];
  d_epT_.upload(t.data(), n);
  for (size_t j = 0; j < n2_; ++j)
    for (size_t i = 0; i < n1_; ++i) t[i * n2_ + j] = em_[i + j * n1_];
  d_emT_.upload(t.data(), n);
}

void StructuredOp::scale(double s) {
  if (frozen_)
    throw InvalidArgument("scale(): the operator is a level of a multigrid hierarchy "
                          "(scale it before building the hierarchy)");
  scales_.push_back(s);
  inv_r_ *= s;
  s_over_r_ *= s;
  for (double& v : dp_) v *= s;
  for (double& v : dm_) v *= s;
  for (double& v : diag_) v *= s;
  const size_t n = n1_ * n2_;
  d_dp_.upload(dp_.data(), n);
  d_dm_.upload(dm_.data(), n);
  d_diag_.upload(diag_.data(), n);
}

namespace {

struct Scales {
  int n;
  double v[8];
};

// Explicitly rounded operations: the same sequence as the host construction
// (no FMA contraction), so refreshed diagonals equal a fresh host build.
__global__ void k_refresh(size_t n, double inv_r0, double sr0, double ax0, double ay0,
                          Scales sc, const double* __restrict__ dp, const double* __restrict__ dm,
                          const double* __restrict__ ep, const double* __restrict__ em,
                          double* __restrict__ odp, double* __restrict__ odm,
                          double* __restrict__ diag, double* __restrict__ dinv, int* flag) {
  pdl_enter();
  int bad = 0;
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    double a = dp[p], b = dm[p];
    const double e = ep[p], f = em[p];
    if (a < 0.0 || b < 0.0 || e < 0.0 || f < 0.0) bad |= 1;
    // inv_r + (dp + dm) ax0 + s/r (ep + em) ay0   (structured.cpp:119-122)
    double d = __dadd_rn(inv_r0, __dmul_rn(__dadd_rn(a, b), ax0));
    d = __dadd_rn(d, __dmul_rn(__dmul_rn(sr0, __dadd_rn(e, f)), ay0));
    for (int k = 0; k < sc.n; ++k) {  // scale(s): dp, dm, diag *= s
      a = __dmul_rn(a, sc.v[k]);
      b = __dmul_rn(b, sc.v[k]);
      d = __dmul_rn(d, sc.v[k]);
    }
    odp[p] = a;
    odm[p] = b;
    diag[p] = d;
    if (dinv) {
      if (!(d > 0.0)) bad |= 2;
      dinv[p] = __ddiv_rn(1.0, d);
    }
  }
  if (bad) atomicOr(flag, bad);
}

}  // namespace

void StructuredOp::refresh(const double* dp, const double* dm, const double* ep,
                           const double* em, double* dinv, int* flag, cudaStream_t s) {
  const size_t n = n1_ * n2_;
  Scales sc{};
  if (scales_.size() > 8) throw InvalidArgument("too many scale() factors to refresh");
  sc.n = (int)scales_.size();
  for (int k = 0; k < sc.n; ++k) sc.v[k] = scales_[k];
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(k_refresh, (int)blocks, 256, 0, s, n, inv_r0_, s_over_r0_, ax_.first_col()[0],
                                        ay_.first_col()[0], sc, dp, dm, ep, em, d_dp_.get(),
                                        d_dm_.get(), d_diag_.get(), dinv, flag);
  FDE_LAUNCH_CHECK();
  launch_transpose(ep, d_epT_.get(), (int)n1_, (int)n2_, s);  // column-pass layout
  launch_transpose(em, d_emT_.get(), (int)n1_, (int)n2_, s);
  host_stale_ = true;
}

void StructuredOp::sync_host(cudaStream_t s) {
  if (!host_stale_) return;
  const size_t n = n1_ * n2_;
  std::vector<double> t(n);
  FDE_CUDA(cudaMemcpyAsync(dp_.data(), d_dp_.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
  FDE_CUDA(cudaMemcpyAsync(dm_.data(), d_dm_.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
  FDE_CUDA(cudaMemcpyAsync(diag_.data(), d_diag_.get(), n * sizeof(double),
                           cudaMemcpyDeviceToHost, s));
  FDE_CUDA(cudaMemcpyAsync(t.data(), d_epT_.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
  FDE_CUDA(cudaStreamSynchronize(s));
  for (size_t j = 0; j < n2_; ++j)
    for (size_t i = 0; i < n1_; ++i) ep_[i + j * n1_] = t[i * n2_ + j];
  FDE_CUDA(cudaMemcpyAsync(t.data(), d_emT_.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
  FDE_CUDA(cudaStreamSynchronize(s));
  for (size_t j = 0; j < n2_; ++j)
    for (size_t i = 0; i < n1_; ++i) em_[i + j * n1_] = t[i * n2_ + j];
  host_stale_ = false;
}

// FFT-path column passes read a transposed copy of the input from this many
// columns up (fewer columns: strided gathers, one transpose launch saved)
// L2 residency of the transposed-input and Q scratch (tmem.cuh): evict_last
// stores, discard after the single read
#ifndef FDE_L2_SCRATCH
#define FDE_L2_SCRATCH 1
#endif
// Row pass waits for the column pass only in its first epilogue (line_conv.cu)
#ifndef FDE_LATE_WAIT
#define FDE_LATE_WAIT 1
#endif
#ifndef FDE_XT_MIN
#define FDE_XT_MIN 512  // measured: 128 or 256 (-0.4 to -1 %), 1024 (-0.3 %) slower
#endif
bool StructuredOp::maps_input() const {
  // (the paired kernels, logM >= 10, bulk-copy contiguous lines: always transposed)
  const int lm = ay_.dev().logM;
  return lm && (lm >= 10 || (n1_ >= FDE_XT_MIN && transpose_columns_));
}

void StructuredOp::run(const double* x, double* out, double sign, int epi, const EpiArgs& e,
                       cudaStream_t s) const {
  run_impl(nullptr, x, out, sign, epi, e, s);
}

void StructuredOp::run_mapped(const InMap& in, double* x, double* out, double sign, int epi,
                              const EpiArgs& e, cudaStream_t s) const {
  if (!maps_input()) throw InvalidArgument("operator input map needs the transposed column pass");
  run_impl(&in, x, out, sign, epi, e, s);
}

void StructuredOp::run_impl(const InMap* in, const double* x, double* out, double sign, int epi,
                            const EpiArgs& e, cudaStream_t s) const {
  NvtxRange trace("fde:apply");
  YPass yp{};
  yp.blk = ay_.dev();
  yp.n1 = (int)n1_;
  yp.n2 = (int)n2_;
  yp.x = x;
  // FFT-path columns read a transposed copy (coalesced) instead of stride-n1 gathers
  if (in) {
    launch_transpose_mapped(*in, const_cast<double*>(x), d_xT_.get(), (int)n1_, (int)n2_, s);
    yp.x = d_xT_.get();
    yp.xT = 1;
    yp.scratch_x = FDE_L2_SCRATCH;
  } else if (maps_input()) {
    launch_transpose(x, d_xT_.get(), (int)n1_, (int)n2_, s);
    yp.x = d_xT_.get();
    yp.xT = 1;
    yp.scratch_x = FDE_L2_SCRATCH;
  }
  yp.keep_q = FDE_L2_SCRATCH;
  yp.epT = d_epT_.get();
  yp.emT = d_emT_.get();
  yp.c = sign * s_over_r_;
  yp.q = d_q_.get();
#ifdef FDE_EXP_QTX
  if (yp.xT) {  // column pass writes Q transposed in place of its input, then one transpose
    yp.q = d_xT_.get();
    yp.qT = 1;
    launch_line_pass(yp, s);
    launch_transpose(d_xT_.get(), d_q_.get(), (int)n2_, (int)n1_, s);
  } else {
    launch_line_pass(yp, s);
  }
#else
  const bool y_saturates = launch_line_pass(yp, s);
#endif
  XPass xp{};
  xp.blk = ax_.dev();
  xp.n1 = (int)n1_;
  xp.n2 = (int)n2_;
  xp.x = x;
  xp.dp = d_dp_.get();
  xp.dm = d_dm_.get();
  xp.q = d_q_.get();
  xp.scratch_q = FDE_L2_SCRATCH;
  xp.inv_r = inv_r_;
  xp.sign = sign;
  xp.epi = epi;
  xp.out = out;
  xp.b = e.b;
  xp.dinv = e.dinv;
  xp.omega = e.omega;
  xp.src = e.src;
  xp.src_scale = e.src_scale;
#ifndef FDE_EXP_QTX
  xp.late_wait = FDE_LATE_WAIT && y_saturates;
#endif
  launch_line_pass(xp, s);
}

}  // namespace fde_b200
