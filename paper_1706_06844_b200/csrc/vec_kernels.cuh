// Vector, reduction and grid-transfer kernels for the multigrid and Krylov
// layers (reference: proj/src/kernels.cpp, multigrid.cpp:17-71,160-227,
// krylov.cpp).  Scalars produced by reductions stay in device memory; the
// Krylov host loop reads them back in one small copy per iteration.
#pragma once
#include "devbuf.cuh"
#include "transfer.cuh"

namespace fde_b200 {

// x = (a * d) .* b                         (zero-guess smoothing, multigrid.cpp:355-356)
void vec_diag_scale(size_t n, double a, const double* d, const double* b, double* x,
                    cudaStream_t s);
// y += a * x                               (kernels::axpy, fma like the AVX2 backend)
void vec_axpy(size_t n, double a, const double* x, double* y, cudaStream_t s);
// y += sgn * (*a_dev) * x
void vec_axpy_dev(size_t n, const double* a_dev, double sgn, const double* x, double* y,
                  cudaStream_t s);
// y = x * (1 / *a_dev)                     (v_{i+1} = w / ||w||, krylov.cpp:127-130)
void vec_scale_inv_dev(size_t n, const double* a_dev, const double* x, double* y,
                       cudaStream_t s);
// x *= a
void vec_scal(size_t n, double a, double* x, cudaStream_t s);
// out += a * d .* r   (Jacobi update, multigrid.cpp:380-382)
void vec_jacobi_update(size_t n, double a, const double* d, const double* r, double* out,
                       cudaStream_t s);
// y = x * a
void vec_copy_scale(size_t n, double a, const double* x, double* y, cudaStream_t s);
// out = x - y
void vec_sub(size_t n, const double* x, const double* y, double* out, cudaStream_t s);
// out = x0 + sum_k c[k] * v[k]   accumulated in k order (krylov.cpp:136-137,153-155)
void vec_lincomb(size_t n, const double* x0, const double* const* v_dev, const double* c_dev,
                 int k, double* out, cudaStream_t s);

// Device scalar slots of the fused BiCGSTAB iteration (krylov.cu): reductions
// land here, the quotients alpha, omega, beta are formed on the device, and
// the host reads the block back twice per iteration for its control flow.
enum BicgSlot : int {
  BICG_RHO_A = 0,  // <rh, r>, alternating with BICG_RHO_B between iterations
  BICG_RHO_B = 1,
  BICG_RV = 2,     // <rh, v>
  BICG_ALPHA = 3,
  BICG_NS = 4,     // ||s||
  BICG_TT = 5,     // <t, t>
  BICG_TS = 6,     // <t, s>
  BICG_OMEGA = 7,
  BICG_NR = 8,     // ||r||
  BICG_SLOTS = 9
};

// Deterministic two-level dot product: per-block partials + last-block sum in
// fixed order.  Writes <x,y> to *out_dev (and sqrt to *out_dev if sqrt_out).
class Reducer {
 public:
  Reducer();
  void dot(size_t n, const double* x, const double* y, double* out_dev, cudaStream_t s,
           bool sqrt_out = false);
  // *norm_out = ||w||, *dot_out = <v, w> in one pass (first MGS projection)
  void norm_dot(size_t n, const double* w, const double* v, double* norm_out, double* dot_out,
                cudaStream_t s);
  // Fused BiCGSTAB passes on the device scalar block sc[BICG_SLOTS]:
  //   bicg_s : alpha = sc[rho_slot] / sc[RV]; s = r - alpha v; sc[NS] = ||s||
  //   bicg_tt: sc[TT] = <t,t>, sc[TS] = <t,s>
  //   bicg_xr: omega = TS/TT; x += alpha p + omega s; r = s - omega t;
  //            sc[NR] = ||r||, sc[rho_out] = <rh, r>
  //   bicg_p : p = r + beta (p - omega v), beta = (rho_new/rho_old)(alpha/omega)
  void bicg_s(size_t n, const double* r, const double* v, double* sv, double* sc, int rho_slot,
              cudaStream_t s);
  void bicg_tt(size_t n, const double* t, const double* sv, double* sc, cudaStream_t s);
  void bicg_xr(size_t n, const double* p, const double* sv, const double* t, const double* rh,
               double* x, double* r, double* sc, int rho_out, cudaStream_t s);
  void bicg_p(size_t n, const double* r, const double* v, double* p, const double* sc,
              int rho_new, int rho_old, cudaStream_t s);
  // w -= (*hk) v_k, then *out = <v_next, w> (sqrt when sqrt_out; v_next may be w)
  void mgs(size_t n, double* w, const double* vk, const double* hk, const double* vnext,
           double* out, bool sqrt_out, cudaStream_t s);
  // The whole Gram-Schmidt of GMRES iteration `last` (krylov.cpp:92-97,
  // 127-130) in one cooperative launch: *dnorm0 = ||w||, dh[k] = <w_k, v_k>
  // with w_{k+1} = w_k - dh[k] v_k for k <= last, *dnrmw = ||w_{last+1}||, and
  // vout = w_{last+1} / *dnrmw -- or, when *dnrmw < 1e-8 *dnorm0 (a second
  // pass follows), w_{last+1} written back to w.  False (nothing launched)
  // when w does not fit the SMs' shared memory or cooperative launch is off.
  bool mgs_chain(size_t n, double* w, const double* const* v_dev, int last, double* dh,
                 double* dnorm0, double* dnrmw, double* vout, cudaStream_t s);

 private:
  DevBuf<double> partials_;
  DevBuf<unsigned int> counter_;
  DevBuf<unsigned long long> chain_flags_;  // flag-carrying partial sums of the chain's reductions
};

Xfer make_xfer(int n1, int n2, bool cx, bool cy);
// coarse = scale-weighted transpose of prolongation (restrict_full: 0.5,
// restrict_transpose: 1.0), same operation order as restrict_rows/cols.
// restriction fused with the coarse level's zero-guess smoothing xc = omega dinv_c bc
void xfer_restrict_smooth(const Xfer& t, const double* fine, double* coarse, double scale,
                          const double* dinv_c, double omega, double* xc, cudaStream_t s);
void xfer_restrict(const Xfer& t, const double* fine, double* coarse, double scale,
                   cudaStream_t s);
// fine += P coarse (prolong then axpy 1.0, multigrid.cpp:377-378)
void xfer_prolong_add(const Xfer& t, const double* coarse, double* fine, cudaStream_t s);
// fine = P coarse
void xfer_prolong(const Xfer& t, const double* coarse, double* fine, cudaStream_t s);
// Row-window variants for y-slabs: the fine buffer holds global fine rows
// starting at f_lo, the coarse buffer global coarse rows starting at c_lo.
// restrict writes coarse rows [c_lo, c_lo + c_rows); prolong writes fine
// rows [f_lo, f_lo + f_rows) (add: +=).  Needed neighbour rows must be present.
void xfer_restrict_rows(const Xfer& t, const double* fine, int f_lo, double* coarse, int c_lo,
                        int c_rows, double scale, cudaStream_t s);
void xfer_prolong_rows(const Xfer& t, const double* coarse, int c_lo, double* fine, int f_lo,
                       int f_rows, bool add, cudaStream_t s);

// All-to-all chunk layout <-> [nc][d2] (see fde_block_permute); off[0..P].
void block_permute(const double* in, double* out, size_t nc, size_t d2, const long long* off,
                   int nranks, int dir, cudaStream_t s);

// x = U^-1 L^-1 P b on one CTA (coarsest CoarseSolve::lu, multigrid.cpp:324-328).
void lu_solve(int n, const double* lu, const int* perm, const double* b, double* x,
              cudaStream_t s);

// Measured DFMA throughput of the current device in TFLOP/s (best of three
// timed launches of a pure FP64 FMA kernel): the roofline denominator of the
// FP64-issue-bound line kernels, taken in the run that reports the fraction.
double fp64_peak_tflops(cudaStream_t s);

}  // namespace fde_b200
