#include <cmath>

#include "slab.cuh"

namespace fde_b200 {

SlabOp::SlabOp(const Problem& p, size_t nf1, size_t nf2, size_t d1, size_t d2, size_t steps,
               size_t m, size_t r0, size_t r1, size_t c0, size_t c1)
    : n1_(d1), n2_(d2), r0_(r0), r1_(r1), c0_(c0), c1_(c1),
      ax_(ToeplitzDev::fractional(p.alpha, d1, p.pq)),
      ay_(ToeplitzDev::fractional(p.beta, d2, p.pq)) {
  if (r0 > r1 || r1 > d2 || c0 > c1 || c1 > d1) throw InvalidArgument("slab range out of the grid");
  if (!p.d_plus || !p.d_minus || !p.e_plus || !p.e_minus)
    throw InvalidArgument("problem is missing a coefficient field");
  const Grid g(p, d1, d2, steps);
  double scale = 1.0;
  if (d1 != nf1 || d2 != nf2) {
    const Grid gf(p, nf1, nf2, steps);
    scale = std::pow(gf.hx / g.hx, p.alpha);
  }
  // StructuredOp::scale (structured.cpp:154-162) applied to the slab's pieces
  inv_r_ = g.inv_r;
  s_over_r_ = g.s_over_r;
  if (scale != 1.0) {
    inv_r_ *= scale;
    s_over_r_ *= scale;
  }
  const double t = static_cast<double>(m) * g.dt;
  const size_t nr = r1 - r0, nc = c1 - c0;
  std::vector<double> dp(nr * d1), dm(nr * d1), epT(nc * d2), emT(nc * d2);
  diag_.resize(nr * d1);
  const double ax0 = ax_.first_col()[0], ay0 = ay_.first_col()[0];
  for (size_t j = r0; j < r1; ++j)
    for (size_t i = 0; i < d1; ++i) {
      const double x = g.x(i), y = g.y(j);
      double a = p.d_plus(x, y, t), b = p.d_minus(x, y, t);
      const double e1 = p.e_plus(x, y, t), e2 = p.e_minus(x, y, t);
      if (a < 0.0 || b < 0.0 || e1 < 0.0 || e2 < 0.0)
        throw InvalidArgument("negative diffusion coefficient sample");
      // the unscaled operator's diagonal, then scaled like StructuredOp
      double dg = g.inv_r + (a + b) * ax0 + g.s_over_r * (e1 + e2) * ay0;
      if (scale != 1.0) {
        a *= scale;
        b *= scale;
        dg *= scale;
      }
      const size_t q = (j - r0) * d1 + i;
      dp[q] = a;
      dm[q] = b;
      diag_[q] = dg;
    }
  for (size_t i = c0; i < c1; ++i)
    for (size_t j = 0; j < d2; ++j) {
      const double x = g.x(i), y = g.y(j);
      epT[(i - c0) * d2 + j] = p.e_plus(x, y, t);
      emT[(i - c0) * d2 + j] = p.e_minus(x, y, t);
    }
  d_dp_.upload(dp.data(), dp.size());
  d_dm_.upload(dm.data(), dm.size());
  d_epT_.upload(epT.data(), epT.size());
  d_emT_.upload(emT.data(), emT.size());
}

void SlabOp::ypass(const double* xT, double* QT, double sign, cudaStream_t s) const {
  if (c1_ == c0_) return;
  YPass yp{};
  yp.blk = ay_.dev();
  yp.n1 = (int)(c1_ - c0_);  // lines = local columns
  yp.n2 = (int)n2_;
  yp.x = xT;
  yp.xT = 1;
  yp.epT = d_epT_.get();
  yp.emT = d_emT_.get();
  yp.c = sign * s_over_r_;
  yp.q = QT;
  yp.qT = 1;
  launch_line_pass(yp, s);
}

void SlabOp::xpass(const double* x, const double* Q, double* out, double sign, int epi,
                   const EpiArgs& e, cudaStream_t s) const {
  if (r1_ == r0_) return;
  XPass xp{};
  xp.blk = ax_.dev();
  xp.n1 = (int)n1_;
  xp.n2 = (int)(r1_ - r0_);  // lines = local rows
  xp.x = x;
  xp.dp = d_dp_.get();
  xp.dm = d_dm_.get();
  xp.q = Q;
  xp.inv_r = inv_r_;
  xp.sign = sign;
  xp.epi = epi;
  xp.out = out;
  xp.b = e.b;
  xp.dinv = e.dinv;
  xp.omega = e.omega;
  xp.src = e.src;
  xp.src_scale = e.src_scale;
  launch_line_pass(xp, s);
}

}  // namespace fde_b200
