#include <cstdlib>
#include "vec_kernels.cuh"
#include "tmem.cuh"

namespace fde_b200 {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 8;

inline int blocks_for(size_t n) {
  const size_t b = (n + kThreads - 1) / kThreads;
  return (int)(b < (size_t)kMaxBlocks ? (b ? b : 1) : kMaxBlocks);
}

#define GRID_STRIDE(i, n) \
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (n); i += (size_t)gridDim.x * blockDim.x)

__global__ void k_diag_scale(size_t n, double a, const double* __restrict__ d,
                             const double* __restrict__ b, double* __restrict__ x) {
  pdl_enter();
  GRID_STRIDE(i, n) x[i] = a * d[i] * b[i];
}
__global__ void k_axpy(size_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  pdl_enter();
  GRID_STRIDE(i, n) y[i] = fma(a, x[i], y[i]);
}
__global__ void k_axpy_dev(size_t n, const double* __restrict__ a, double sgn,
                           const double* __restrict__ x, double* __restrict__ y) {
  pdl_enter();
  const double av = sgn * *a;
  GRID_STRIDE(i, n) y[i] = fma(av, x[i], y[i]);
}
__global__ void k_scale_inv_dev(size_t n, const double* __restrict__ a, const double* x,
                                double* y) {
  pdl_enter();
  const double inv = 1.0 / *a;
  GRID_STRIDE(i, n) y[i] = x[i] * inv;
}
__global__ void k_jacobi_upd(size_t n, double a, const double* __restrict__ d,
                             const double* __restrict__ r, double* __restrict__ x) {
  pdl_enter();
  GRID_STRIDE(i, n) x[i] += a * d[i] * r[i];
}
__global__ void k_copy_scale2(size_t n, double a, const double* __restrict__ x,
                              double* __restrict__ y) {
  pdl_enter();
  GRID_STRIDE(i, n) y[i] = x[i] * a;
}
__global__ void k_scal(size_t n, double a, double* x) {
  pdl_enter();
  GRID_STRIDE(i, n) x[i] *= a;
}
__global__ void k_sub(size_t n, const double* __restrict__ x, const double* __restrict__ y,
                      double* out) {
  pdl_enter();
  GRID_STRIDE(i, n) out[i] = x[i] - y[i];
}
__global__ void k_lincomb(size_t n, const double* x0, const double* const* __restrict__ v,
                          const double* __restrict__ c, int k, double* out) {
  pdl_enter();
  GRID_STRIDE(i, n) {
    double acc = x0[i];
    for (int q = 0; q < k; ++q) acc = fma(c[q], v[q][i], acc);
    out[i] = acc;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__global__ void k_dot(size_t n, const double* __restrict__ x, const double* __restrict__ y,
                      double* __restrict__ partials, unsigned int* counter, double* out,
                      int sqrt_out) {
  pdl_enter();
  __shared__ double ws[kThreads / 32];
  __shared__ bool last;
  double acc = 0.0;
  GRID_STRIDE(i, n) acc = fma(x[i], y[i], acc);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kThreads / 32 ? ws[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) {
      partials[blockIdx.x] = v;
      __threadfence();
      last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  // last block: fixed-order sum of the partials (deterministic)
  __threadfence();
  double v = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += ((volatile double*)partials)[b];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) t += ws[w];
    *out = sqrt_out ? sqrt(t) : t;
    *counter = 0u;
  }
}

// Last-block finalisation shared by the fused reductions: block partial v of
// reduction r lands in partials[r * kMaxBlocks + block]; the last block to
// arrive sums each reduction's partials in block order (deterministic).
template <int NR>
__device__ __forceinline__ void reduce_finish(double (&v)[NR], double* partials,
                                              unsigned int* counter, double* const (&out)[NR],
                                              const int (&sqrt_out)[NR]) {
  __shared__ double ws[NR][kThreads / 32];
  __shared__ bool last;
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const double t = warp_sum(v[r]);
    if ((threadIdx.x & 31) == 0) ws[r][threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      double t = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) t += ws[r][w];
      partials[r * kMaxBlocks + blockIdx.x] = t;
    }
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    double t = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
      t += ((volatile double*)partials)[r * kMaxBlocks + b];
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) ws[r][threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      double t = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) t += ws[r][w];
      *out[r] = sqrt_out[r] ? sqrt(t) : t;
    }
    *counter = 0u;
  }
}

// L2 eviction-priority hints for the Gram-Schmidt chain: w (read and written
// every pass) and v_{k+1} (projected now, subtracted in the next pass) are
// kept (evict_last); v_k has its last use of the pass (evict_first).  With
// w and v_{k+1} L2-resident a pass streams one basis vector from HBM.
__device__ __forceinline__ uint64_t policy_keep() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_stream() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

__device__ __forceinline__ double2 ld2_hint(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

// out0 = ||w|| (sqrt of <w,w>), out1 = <v, w> in one pass over w (MGS start).
__global__ void k_norm_dot(size_t n, const double* __restrict__ w, const double* __restrict__ v,
                           double* partials, unsigned int* counter, double* out0, double* out1) {
  pdl_enter();
  double acc[2] = {0.0, 0.0};
  const uint64_t keep = policy_keep();
  GRID_STRIDE(i, n) {
    const double wi = ld_hint(w + i, keep);
    acc[0] = fma(wi, wi, acc[0]);
    acc[1] = fma(ld_hint(v + i, keep), wi, acc[1]);
  }
  double* const outs[2] = {out0, out1};
  const int sq[2] = {1, 0};
  reduce_finish<2>(acc, partials, counter, outs, sq);
}

// One modified Gram-Schmidt step fused with the next projection:
//   w -= (*hk) v_k;  *out = <v_next, w>   (v_next == w: *out = ||w||)
__global__ void k_mgs(size_t n, double* __restrict__ w, const double* __restrict__ vk,
                      const double* __restrict__ hk, const double* vnext, double* partials,
                      unsigned int* counter, double* out, int sqrt_out) {
  pdl_enter();
  const double h = -*hk;
  double acc[1] = {0.0};
  const bool last = vnext == w;
  const uint64_t keep = policy_keep(), stream = policy_stream();
  GRID_STRIDE(i, n) {
    const double wi = fma(h, ld_hint(vk + i, stream), ld_hint(w + i, keep));  // axpy(-h, v_k, w)
    st_hint(w + i, wi, keep);
    acc[0] = fma(last ? wi : ld_hint(vnext + i, keep), wi, acc[0]);
  }
  double* const outs[1] = {out};
  const int sq[1] = {sqrt_out};
  reduce_finish<1>(acc, partials, counter, outs, sq);
}

// ---- fused BiCGSTAB updates (scalars stay on the device) --------------------
// sc[] slots: see BicgSlot (vec_kernels.cuh).  Quotients are formed on the
// device from finished reductions, in the oracle's order of operations.
// s = r - alpha v with alpha = rho / <rh, v>;  *ns = ||s||
__global__ void k_bicg_s(size_t n, const double* __restrict__ r, const double* __restrict__ v,
                         double* __restrict__ sv, double* sc, int rho_slot, double* partials,
                         unsigned int* counter) {
  pdl_enter();
  const double alpha = sc[rho_slot] / sc[BICG_RV];
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) {
    const double si = r[i] - alpha * v[i];
    sv[i] = si;
    acc[0] = fma(si, si, acc[0]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[BICG_ALPHA] = alpha;
  double* const outs[1] = {sc + BICG_NS};
  const int sq[1] = {1};
  reduce_finish<1>(acc, partials, counter, outs, sq);
}
// tt = <t, t>, ts = <t, s> in one pass over t
__global__ void k_bicg_tt(size_t n, const double* __restrict__ t, const double* __restrict__ sv,
                          double* sc, double* partials, unsigned int* counter) {
  pdl_enter();
  double acc[2] = {0.0, 0.0};
  GRID_STRIDE(i, n) {
    const double ti = t[i];
    acc[0] = fma(ti, ti, acc[0]);
    acc[1] = fma(ti, sv[i], acc[1]);
  }
  double* const outs[2] = {sc + BICG_TT, sc + BICG_TS};
  const int sq[2] = {0, 0};
  reduce_finish<2>(acc, partials, counter, outs, sq);
}
// omega = ts / tt (0 when tt == 0);  x += alpha p + omega s;  r = s - omega t;
// *nr = ||r||, sc[rho_out] = <rh, r> (the next iteration's rho)
__global__ void k_bicg_xr(size_t n, const double* __restrict__ p, const double* __restrict__ sv,
                          const double* __restrict__ t, const double* __restrict__ rh,
                          double* __restrict__ x, double* __restrict__ r, double* sc, int rho_out,
                          double* partials, unsigned int* counter) {
  pdl_enter();
  const double alpha = sc[BICG_ALPHA];
  const double tt = sc[BICG_TT];
  const double omg = tt > 0.0 ? sc[BICG_TS] / tt : 0.0;
  double acc[2] = {0.0, 0.0};
  GRID_STRIDE(i, n) {
    const double si = sv[i];
    x[i] += alpha * p[i] + omg * si;
    const double ri = si - omg * t[i];
    r[i] = ri;
    acc[0] = fma(ri, ri, acc[0]);
    acc[1] = fma(rh[i], ri, acc[1]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[BICG_OMEGA] = omg;
  double* const outs[2] = {sc + BICG_NR, sc + rho_out};
  const int sq[2] = {1, 0};
  reduce_finish<2>(acc, partials, counter, outs, sq);
}
// p = r + beta (p - omega v), beta = (rho_new / rho_old) (alpha / omega)
__global__ void k_bicg_p(size_t n, const double* __restrict__ r, const double* __restrict__ v,
                         double* __restrict__ p, const double* sc, int rho_new, int rho_old) {
  pdl_enter();
  const double omg = sc[BICG_OMEGA];
  const double beta = (sc[rho_new] / sc[rho_old]) * (sc[BICG_ALPHA] / omg);
  GRID_STRIDE(i, n) p[i] = r[i] + beta * (p[i] - omg * v[i]);
}

// ---- grid transfers ---------------------------------------------------------
// restrict_rows (multigrid.cpp:46-58): v = f[fc]; v += .5 f[fc-1]; v += .5 f[fc+1]; scale*v
__device__ __forceinline__ double rrow(const double* f, int n, int fc, double sc) {
  double v = f[fc];
  if (fc > 0) v += 0.5 * f[fc - 1];
  if (fc + 1 < n) v += 0.5 * f[fc + 1];
  return sc * v;
}

// Row windows let the same kernels run on a y-slab: the fine buffer holds
// global fine rows [f_lo, f_lo + rows), the coarse buffer global coarse rows
// [c_lo, c_lo + rows).  Full-grid calls use f_lo = c_lo = 0.
// xs != nullptr: also x_c = (omega dinv_c) bc, the next level's zero-guess
// smoothing (multigrid.cpp:355-356), in the same pass
__global__ void k_restrict(Xfer t, const double* __restrict__ f, int f_lo,
                           double* __restrict__ c, int c_lo, int c_rows, double sc,
                           double* __restrict__ xs = nullptr,
                           const double* __restrict__ dinv = nullptr, double omega = 0.0) {
  pdl_enter();
  const size_t nc = (size_t)t.k1 * c_rows;
  GRID_STRIDE(q, nc) {
    const int a = (int)(q % t.k1), bb = (int)(q / t.k1) + c_lo;  // global coarse row
    auto frow = [&](int r) { return f + (size_t)(r - f_lo) * t.n1; };
    double out;
    if (!t.cx) {  // restrict_cols only (multigrid.cpp:60-71)
      const int fb = 2 * bb + 1 - t.par2;
      double v = frow(fb)[a];
      if (fb > 0) v += 0.5 * frow(fb - 1)[a];
      if (fb + 1 < t.n2) v += 0.5 * frow(fb + 1)[a];
      out = v * sc;
    } else if (!t.cy) {  // restrict_rows only
      out = rrow(frow(bb), t.n1, 2 * a + 1 - t.par1, sc);
    } else {  // rows then columns of the row-restricted temporary
      const int fa = 2 * a + 1 - t.par1, fb = 2 * bb + 1 - t.par2;
      double v = rrow(frow(fb), t.n1, fa, sc);
      if (fb > 0) v += 0.5 * rrow(frow(fb - 1), t.n1, fa, sc);
      if (fb + 1 < t.n2) v += 0.5 * rrow(frow(fb + 1), t.n1, fa, sc);
      out = v * sc;
    }
    c[q] = out;
    if (xs) xs[q] = omega * dinv[q] * out;  // vec_diag_scale's (a d) b
  }
}

template <bool ADD>
__global__ void k_prolong(Xfer t, const double* __restrict__ c, int c_lo,
                          double* __restrict__ f, int f_lo, int f_rows) {
  pdl_enter();
  const size_t nf = (size_t)t.n1 * f_rows;
  GRID_STRIDE(q, nf) {
    const int i = (int)(q % t.n1), j = (int)(q / t.n1) + f_lo;  // global fine row
    const double v = prolong_point(t, c, c_lo, i, j);
    if (ADD) f[q] += v;
    else f[q] = v;
  }
}

// ---- the whole modified Gram-Schmidt of one GMRES iteration, one launch ----
// Cooperative grid of one 1024-thread CTA per SM; CTA b keeps its slice of w
// in shared memory for the whole chain, so a projection pass streams only the
// basis vectors (v_{k+1} from HBM, v_k again from L2) instead of reading and
// writing w every pass.  Same per-element arithmetic as k_norm_dot / k_mgs /
// k_copy_scale; the grid-wide sums combine per-CTA partials in CTA order
// (deterministic, identical in every CTA).
constexpr int kChainThreads = 1024;

// Grid-wide sums of (a, b) without atomics: every CTA publishes its two
// partial sums as four 8-byte words {32 bits of the double, 32-bit epoch}
// (an aligned 8-byte access is single-copy atomic, so a word carries its own
// "valid" flag and no fence or counter is needed -- the data IS the flag),
// and thread k of every CTA polls CTA k's words until they carry this epoch:
// one L2 round trip per reduction instead of three (arrive, poll, read the
// partials).  Slots are double-buffered by epoch parity: a CTA can run at
// most one reduction ahead of the slowest reader.  Every warp then adds the
// gathered partials in CTA order (lane-strided, shuffle tree) exactly as
// the counter version did: identical bits, identical in every CTA.
constexpr int kChainMaxGrid = 160;  // CTAs (one per SM); 2.5 KB of gather slots
struct ChainShared {
  double red[2][kChainThreads / 32];
  double gath[2][kChainMaxGrid];
};
// TWO = false: only a is summed (b's words are neither written nor polled)
template <bool TWO>
__device__ __forceinline__ double2 chain_grid_sum(double a, double b, ChainShared& sh,
                                                  unsigned long long* ll, unsigned& phase) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grid = (int)gridDim.x;
  a = warp_sum(a);
  if (TWO) b = warp_sum(b);
  if (lane == 0) {
    sh.red[0][warp] = a;
    if (TWO) sh.red[1][warp] = b;
  }
  __syncthreads();
  ++phase;
  if (grid == 1) {  // a single CTA: the warp partials are the whole sum, nothing leaves the SM
    double ta = warp_sum(sh.red[0][lane]), tb = TWO ? warp_sum(sh.red[1][lane]) : 0.0;
    ta = __shfl_sync(0xffffffffu, ta, 0);
    if (TWO) tb = __shfl_sync(0xffffffffu, tb, 0);
    __syncthreads();  // sh.red is rewritten by the next reduction
    return make_double2(ta, tb);
  }
  unsigned long long* const slots = ll + (size_t)(phase & 1) * 4 * grid;
  if (warp == 0) {  // the 32 warp partials, shuffle tree (fixed order)
    double ta = warp_sum(sh.red[0][lane]), tb = TWO ? warp_sum(sh.red[1][lane]) : 0.0;
    ta = __shfl_sync(0xffffffffu, ta, 0);
    if (TWO) tb = __shfl_sync(0xffffffffu, tb, 0);
    if (lane < (TWO ? 4 : 2)) {
      const double val = lane < 2 ? ta : tb;
      const unsigned half = (lane & 1) ? (unsigned)__double2hiint(val) : (unsigned)__double2loint(val);
      const unsigned long long word = ((unsigned long long)phase << 32) | half;
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(slots + 4 * blockIdx.x + lane),
                   "l"(word)
                   : "memory");
    }
  }
  if ((int)threadIdx.x < grid) {
    const unsigned long long* const p = slots + 4 * threadIdx.x;
    unsigned long long w0, w1, w2 = 0, w3 = 0;
    for (;;) {
      asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(p) : "memory");
      if (TWO)
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w2), "=l"(w3) : "l"(p + 2) : "memory");
      if ((unsigned)(w0 >> 32) == phase && (unsigned)(w1 >> 32) == phase &&
          (!TWO || ((unsigned)(w2 >> 32) == phase && (unsigned)(w3 >> 32) == phase)))
        break;
      __nanosleep(40);  // (200 / 1000 ns measured: 8.5 / 8.7 us per projection against 8.2)
    }
    sh.gath[0][threadIdx.x] = __hiloint2double((int)(unsigned)w1, (int)(unsigned)w0);
    if (TWO) sh.gath[1][threadIdx.x] = __hiloint2double((int)(unsigned)w3, (int)(unsigned)w2);
  }
  __syncthreads();
  double ta = 0.0, tb = 0.0;
  for (int k = lane; k < grid; k += 32) {
    ta += sh.gath[0][k];
    if (TWO) tb += sh.gath[1][k];
  }
  ta = warp_sum(ta);
  if (TWO) tb = warp_sum(tb);
  return make_double2(__shfl_sync(0xffffffffu, ta, 0), TWO ? __shfl_sync(0xffffffffu, tb, 0) : 0.0);
}

__global__ void __launch_bounds__(kChainThreads, 1)
    k_mgs_chain(size_t n, size_t chunk, double* __restrict__ w, const double* const* __restrict__ v,
                int last, double* dh, double* dnorm0, double* dnrmw, double* __restrict__ vout,
                unsigned long long* flags) {
  extern __shared__ __align__(16) double ws[];  // this CTA's slice of w
  __shared__ ChainShared sh;
  const size_t lo = blockIdx.x * chunk;
  const int cnt = lo < n ? (int)((n - lo < chunk) ? n - lo : chunk) : 0;
  const uint64_t keep = policy_keep(), stream = policy_stream();
  unsigned phase = 0;
  double2 sums;
  auto grid_sum = [&](double a, double b) { sums = chain_grid_sum<true>(a, b, sh, flags, phase); };
  auto grid_sum1 = [&](double a) { sums = chain_grid_sum<false>(a, 0.0, sh, flags, phase); };

  // pairs of elements (16-byte loads; the slice start is even), plus the odd
  // last element of the last slice
  double2* const ws2 = reinterpret_cast<double2*>(ws);
  const int pairs = cnt >> 1, tail = (cnt & 1) ? cnt - 1 : -1;
  // ||w|| and <w, v_0> while w moves into shared memory (k_norm_dot)
  {
    const double* v0 = v[0] + lo;
    const double* wg = w + lo;
    double a0 = 0.0, a1 = 0.0;
#pragma unroll 4
    for (int e = threadIdx.x; e < pairs; e += kChainThreads) {
      const double2 wi = ld2_hint(wg + 2 * e, stream), vi = ld2_hint(v0 + 2 * e, keep);
      ws2[e] = wi;
      a0 = fma(wi.x, wi.x, a0);
      a1 = fma(vi.x, wi.x, a1);
      a0 = fma(wi.y, wi.y, a0);
      a1 = fma(vi.y, wi.y, a1);
    }
    if (threadIdx.x == 0 && tail >= 0) {
      const double wi = wg[tail];
      ws[tail] = wi;
      a0 = fma(wi, wi, a0);
      a1 = fma(v0[tail], wi, a1);
    }
    grid_sum(a0, a1);
  }
  const double norm0 = sqrt(sums.x);
  double h = sums.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *dnorm0 = norm0;
    dh[0] = h;
  }
  double hip = 0.0;
  // w -= h_k v_k fused with <v_{k+1}, w> (k_mgs); the last pass forms ||w||
  for (int k = 0; k <= last; ++k) {
    const double* vk = v[k] + lo;
    const double* vn = k < last ? v[k + 1] + lo : nullptr;
    const double nh = -h;
    double acc = 0.0;
    if (vn) {
#pragma unroll 4
      for (int e = threadIdx.x; e < pairs; e += kChainThreads) {
        const double2 a = ld2_hint(vk + 2 * e, stream), b = ld2_hint(vn + 2 * e, keep);
        double2 wi = ws2[e];
        wi.x = fma(nh, a.x, wi.x);
        wi.y = fma(nh, a.y, wi.y);
        ws2[e] = wi;
        acc = fma(b.x, wi.x, acc);
        acc = fma(b.y, wi.y, acc);
      }
    } else {
#pragma unroll 4
      for (int e = threadIdx.x; e < pairs; e += kChainThreads) {
        const double2 a = ld2_hint(vk + 2 * e, stream);
        double2 wi = ws2[e];
        wi.x = fma(nh, a.x, wi.x);
        wi.y = fma(nh, a.y, wi.y);
        ws2[e] = wi;
        acc = fma(wi.x, wi.x, acc);
        acc = fma(wi.y, wi.y, acc);
      }
    }
    if (threadIdx.x == 0 && tail >= 0) {
      const double wi = fma(nh, vk[tail], ws[tail]);
      ws[tail] = wi;
      acc = fma(vn ? vn[tail] : wi, wi, acc);
    }
    grid_sum1(acc);
    if (k < last) {
      h = sums.x;
      if (blockIdx.x == 0 && threadIdx.x == 0) dh[k + 1] = h;
    } else {
      hip = sqrt(sums.x);
      if (blockIdx.x == 0 && threadIdx.x == 0) *dnrmw = hip;
    }
  }
  // v_{i+1} = w (1 / ||w||) (copy_scale, krylov.cpp:127-130); a second
  // Gram-Schmidt pass (hip < 1e-8 norm0, krylov.cpp:98-104) needs w itself
  if (hip < 1e-8 * norm0) {
    for (int e = threadIdx.x; e < cnt; e += kChainThreads) w[lo + e] = ws[e];
  } else {
    const double a = 1.0 / hip;
    double2* const out2 = reinterpret_cast<double2*>(vout + lo);
    for (int e = threadIdx.x; e < pairs; e += kChainThreads) {
      const double2 wi = ws2[e];
      out2[e] = make_double2(wi.x * a, wi.y * a);
    }
    if (threadIdx.x == 0 && tail >= 0) vout[lo + tail] = ws[tail] * a;
  }
}

// The same chain with w in TENSOR MEMORY and the current basis vector in shared
// memory.  A pass of k_mgs_chain brings two slices per SM through L2 (v_{k+1}
// from HBM, v_k again from L2) and measured 11 us with the grid barrier taken
// out -- the L2 -> SM path, not HBM, bounds it.  Here the slice of v_{k+1} a
// pass streams for its dot product is left in shared memory and is the v_k of
// the next pass's subtraction, so a pass reads ONE vector slice through L2;
// the CTA's slice of w (226 KB at n = 2047, the whole shared memory before)
// lives in the SM's 256 KB of tensor memory instead: thread t of warp q owns
// lane 32 (q % 4) + t % 32, columns 64 (q / 4) .. + 63, i.e. 16 double2 = the
// pairs t + 1024 c (c < 16) of the slice.  Same per-element arithmetic, same
// element -> thread map, same partial-sum order as k_mgs_chain: identical bits.
constexpr int kChainSlots = 16;  // double2 per thread in tensor memory
#ifndef FDE_CHAIN_ASYNC
#define FDE_CHAIN_ASYNC 1  // v_{k+1} by per-thread asynchronous copies into its shared-memory slots
// (measured: each 16-byte cp.async.cg fetches its whole 32-byte sector, so a pass moves 68 MB L2 -> SM
// for a 33.5 MB vector; .ca halves that and runs 10.2 us per projection against 8.5; one 512-byte bulk
// copy per warp and slot with an mbarrier per slot group also halves it and runs 8.9 -- the pass is no
// longer bound by that path, the per-thread .cg copies stay)
#endif
#ifndef FDE_CHAIN_LOADS
#define FDE_CHAIN_LOADS 4  // 16-byte loads of v_{k+1} in flight per thread; 8 / 16 spill at 64 registers: 10.3 -> 13.1 / 14.5 us per pass
#endif
// (an L2 bulk prefetch of the next pass's slice measured +1.3 us per pass in
// isolation and nothing in the step: left out)
__global__ void __launch_bounds__(kChainThreads, 1)
    k_mgs_chain_tmem(size_t n, size_t chunk, double* __restrict__ w,
                     const double* const* __restrict__ v, int last, double* dh, double* dnorm0,
                     double* dnrmw, double* __restrict__ vout,
                     unsigned long long* flags) {
  extern __shared__ __align__(16) double vs[];  // this CTA's slice of the pass's basis vector
  __shared__ ChainShared sh;
  __shared__ uint32_t s_tbase;
  __shared__ double w_tail;  // the odd last element of the last slice
  const size_t lo = blockIdx.x * chunk;
  const int cnt = lo < n ? (int)((n - lo < chunk) ? n - lo : chunk) : 0;
  const uint64_t keep = policy_keep(), stream = policy_stream();
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&s_tbase);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = s_tbase;
  const uint32_t tw = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
  unsigned phase = 0;
  double2 sums;
  auto grid_sum = [&](double a, double b) { sums = chain_grid_sum<true>(a, b, sh, flags, phase); };
  auto grid_sum1 = [&](double a) { sums = chain_grid_sum<false>(a, 0.0, sh, flags, phase); };
  double2* const vs2 = reinterpret_cast<double2*>(vs);
  const int pairs = cnt >> 1, tail = (cnt & 1) ? cnt - 1 : -1;
  // ||w|| and <w, v_0>: w moves into tensor memory, v_0 into shared memory
  {
    const double* v0 = v[0] + lo;
    const double* wg = w + lo;
    double a0 = 0.0, a1 = 0.0;
#if FDE_CHAIN_ASYNC
    // v_0 straight into its shared-memory slots (no registers), w through
    // registers into tensor memory; <w, v_0> in a second walk, slot order
#pragma unroll
    for (int g = 0; g < kChainSlots; g += 4) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e = threadIdx.x + (g + c) * kChainThreads;
        if (e < pairs) cp_async16_hint(vs2 + e, v0 + 2 * e, keep);
      }
      cp_async_commit();
    }
#pragma unroll 1  // (unrolled, the loads of every round are hoisted and spill)
    for (int g = 0; g < kChainSlots && g * kChainThreads < pairs; g += 4) {  // (live slot groups only)
      double2 wv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e = threadIdx.x + (g + c) * kChainThreads;
        wv[c] = e < pairs ? ld2_hint(wg + 2 * e, stream) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // (zero beyond the slice: adds +0.0)
        a0 = fma(wv[c].x, wv[c].x, a0);
        a0 = fma(wv[c].y, wv[c].y, a0);
      }
      tmem_st4(tw + 4 * g, wv);
    }
    tmem_wait_st();
#pragma unroll
    for (int g = 0; g < kChainSlots; g += 4) {
      cp_async_wait_group_le(3 - g / 4);
      if (g * kChainThreads >= pairs) continue;  // short slices: the slot group is empty in every thread
      double2 wv[4];
      tmem_ld4(tw + 4 * g, wv);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e = threadIdx.x + (g + c) * kChainThreads;
        if (e < pairs) {
          const double2 b = vs2[e];
          a1 = fma(b.x, wv[c].x, a1);
          a1 = fma(b.y, wv[c].y, a1);
        }
      }
    }
#else
#pragma unroll
    for (int g = 0; g < kChainSlots; g += 4) {
      double2 wv[4], vv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e = threadIdx.x + (g + c) * kChainThreads;
        wv[c] = e < pairs ? ld2_hint(wg + 2 * e, stream) : make_double2(0.0, 0.0);
        vv[c] = e < pairs ? ld2_hint(v0 + 2 * e, keep) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e = threadIdx.x + (g + c) * kChainThreads;
        if (e < pairs) {
          vs2[e] = vv[c];
          a0 = fma(wv[c].x, wv[c].x, a0);
          a1 = fma(vv[c].x, wv[c].x, a1);
          a0 = fma(wv[c].y, wv[c].y, a0);
          a1 = fma(vv[c].y, wv[c].y, a1);
        }
      }
      tmem_st4(tw + 4 * g, wv);
    }
#endif
    if (threadIdx.x == 0 && tail >= 0) {
      const double wi = wg[tail];
      w_tail = wi;
      a0 = fma(wi, wi, a0);
      a1 = fma(v0[tail], wi, a1);
    }
    tmem_wait_st();
    grid_sum(a0, a1);
  }
  const double norm0 = sqrt(sums.x);
  double h = sums.y;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *dnorm0 = norm0;
    dh[0] = h;
  }
  double hip = 0.0;
  // w -= h_k v_k (v_k from shared memory) fused with <v_{k+1}, w> (v_{k+1}
  // streamed once, left in shared memory for the next pass); the last pass
  // forms ||w||
  for (int k = 0; k <= last; ++k) {
    const double* vk = v[k] + lo;
    const double* vn = k < last ? v[k + 1] + lo : nullptr;
    const double nh = -h;
    double acc = 0.0;
#if FDE_CHAIN_ASYNC
    // Every pair of the slice belongs to one thread (shared-memory slot and
    // tensor-memory slot alike), so the thread that has subtracted h_k v_k[e]
    // can overwrite its slot with v_{k+1}[e] by an asynchronous copy: all 16
    // loads of a thread are in flight at once and hold no register.  The dot
    // product follows in a second walk (w once more from tensor memory), in
    // the same slot order as the fused walk: identical bits.
#pragma unroll
    for (int g = 0; g < kChainSlots; g += 4) {
      if (g * kChainThreads >= pairs) {  // empty slot group (uniform over the CTA)
        if (vn) cp_async_commit();       // keeps the group count the waits below assume
        continue;
      }
      double2 wv[4];
      tmem_ld4(tw + 4 * g, wv);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e = threadIdx.x + (g + c) * kChainThreads;
        if (e < pairs) {
          const double2 a = vs2[e];
          double2 wi = wv[c];
          wi.x = fma(nh, a.x, wi.x);
          wi.y = fma(nh, a.y, wi.y);
          wv[c] = wi;
          if (!vn) {
            acc = fma(wi.x, wi.x, acc);
            acc = fma(wi.y, wi.y, acc);
          }
        }
      }
      tmem_st4(tw + 4 * g, wv);  // (depends on every vs2[e] read of the group)
      if (vn) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int e = threadIdx.x + (g + c) * kChainThreads;
          if (e < pairs) cp_async16_hint(vs2 + e, vn + 2 * e, keep);
        }
        cp_async_commit();
      }
    }
    if (vn) {
      tmem_wait_st();
#pragma unroll
      for (int g = 0; g < kChainSlots; g += 4) {
        cp_async_wait_group_le(3 - g / 4);
        if (g * kChainThreads >= pairs) continue;
        double2 wv[4];
        tmem_ld4(tw + 4 * g, wv);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int e = threadIdx.x + (g + c) * kChainThreads;
          if (e < pairs) {
            const double2 b = vs2[e];
            acc = fma(b.x, wv[c].x, acc);
            acc = fma(b.y, wv[c].y, acc);
          }
        }
      }
    }
#else
#pragma unroll
    for (int g8 = 0; g8 < kChainSlots; g8 += FDE_CHAIN_LOADS) {
      // FDE_CHAIN_LOADS slices of v_{k+1} in flight per thread, then tensor
      // memory in groups of 4 slots
      double2 nv[FDE_CHAIN_LOADS];
      if (vn) {
#pragma unroll
        for (int c = 0; c < FDE_CHAIN_LOADS; ++c) {
          const int e = threadIdx.x + (g8 + c) * kChainThreads;
          nv[c] = e < pairs ? ld2_hint(vn + 2 * e, keep) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int g = g8; g < g8 + FDE_CHAIN_LOADS; g += 4) {
        double2 wv[4];
        tmem_ld4(tw + 4 * g, wv);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int e = threadIdx.x + (g + c) * kChainThreads;
          if (e < pairs) {
            const double2 a = vs2[e];
            double2 wi = wv[c];
            wi.x = fma(nh, a.x, wi.x);
            wi.y = fma(nh, a.y, wi.y);
            wv[c] = wi;
            if (vn) {
              acc = fma(nv[g - g8 + c].x, wi.x, acc);
              acc = fma(nv[g - g8 + c].y, wi.y, acc);
              vs2[e] = nv[g - g8 + c];
            } else {
              acc = fma(wi.x, wi.x, acc);
              acc = fma(wi.y, wi.y, acc);
            }
          }
        }
        tmem_st4(tw + 4 * g, wv);
      }
    }
#endif
    if (threadIdx.x == 0 && tail >= 0) {
      const double wi = fma(nh, vk[tail], w_tail);
      w_tail = wi;
      acc = fma(vn ? vn[tail] : wi, wi, acc);
    }
    tmem_wait_st();
    grid_sum1(acc);
    if (k < last) {
      h = sums.x;
      if (blockIdx.x == 0 && threadIdx.x == 0) dh[k + 1] = h;
    } else {
      hip = sqrt(sums.x);
      if (blockIdx.x == 0 && threadIdx.x == 0) *dnrmw = hip;
    }
  }
  // v_{i+1} = w (1 / ||w||) (copy_scale, krylov.cpp:127-130); a second
  // Gram-Schmidt pass (hip < 1e-8 norm0, krylov.cpp:98-104) needs w itself
  const bool keep_w = hip < 1e-8 * norm0;
  const double a = keep_w ? 1.0 : 1.0 / hip;
  double2* const out2 = reinterpret_cast<double2*>((keep_w ? w : vout) + lo);
#pragma unroll
  for (int g = 0; g < kChainSlots; g += 4) {
    if (g * kChainThreads >= pairs) continue;
    double2 wv[4];
    tmem_ld4(tw + 4 * g, wv);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int e = threadIdx.x + (g + c) * kChainThreads;
      if (e < pairs) out2[e] = keep_w ? wv[c] : make_double2(wv[c].x * a, wv[c].y * a);
    }
  }
  if (threadIdx.x == 0 && tail >= 0) (keep_w ? w : vout)[lo + tail] = keep_w ? w_tail : w_tail * a;
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tbase);
}


#ifndef FDE_CHAIN_TMEM
#define FDE_CHAIN_TMEM 1  // w in tensor memory, one basis-vector slice per pass through L2
#endif
// slices from this many doubles per SM up run the tensor-memory chain; below,
// the allocation and the fixed 16-slot walk cost more than the second L2
// stream (cfg1 894 -> 808, cfg2 650 -> 611 steps/s with it)
#ifndef FDE_CHAIN_MIN_SLICE
#define FDE_CHAIN_MIN_SLICE 4096  // doubles per CTA below which the chain runs on fewer CTAs than SMs (0: always one per SM)
#endif
#ifndef FDE_CHAIN_TMEM_MIN
#define FDE_CHAIN_TMEM_MIN 4096
#endif

struct RankOffsets {
  long long o[65];
  int n;
};
__global__ void k_block_permute(const double* __restrict__ in, double* __restrict__ out,
                                size_t nc, size_t d2, RankOffsets ro, int dir) {
  pdl_enter();
  const size_t total = nc * d2;
  GRID_STRIDE(q, total) {
    const size_t c = q / d2, j = q % d2;
    int s = 0;
    while (s + 1 < ro.n && (long long)j >= ro.o[s + 1]) ++s;
    const size_t rows = (size_t)(ro.o[s + 1] - ro.o[s]);
    const size_t src = nc * (size_t)ro.o[s] + c * rows + (j - (size_t)ro.o[s]);
    if (dir == 0) out[q] = in[src];
    else out[src] = in[q];
  }
}

// Single-CTA forward/back substitution with a row-pivoted LU (column-major).
__global__ void k_lu_solve(int n, const double* __restrict__ lu, const int* __restrict__ perm,
                           const double* __restrict__ b, double* __restrict__ x) {
  pdl_enter();
  extern __shared__ double y[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = b[perm[i]];
  __syncthreads();
  for (int j = 0; j < n; ++j) {  // L (unit diagonal): y_i -= l_ij y_j
    const double yj = y[j];
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) y[i] -= lu[i + (size_t)j * n] * yj;
    __syncthreads();
  }
  for (int j = n - 1; j >= 0; --j) {  // U
    if (threadIdx.x == 0) y[j] = y[j] / lu[j + (size_t)j * n];
    __syncthreads();
    const double yj = y[j];
    for (int i = threadIdx.x; i < j; i += blockDim.x) y[i] -= lu[i + (size_t)j * n] * yj;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = y[i];
}

}  // namespace

void vec_diag_scale(size_t n, double a, const double* d, const double* b, double* x,
                    cudaStream_t s) {
  launch_k(k_diag_scale, blocks_for(n), kThreads, 0, s, n, a, d, b, x);
  FDE_LAUNCH_CHECK();
}
void vec_axpy(size_t n, double a, const double* x, double* y, cudaStream_t s) {
  launch_k(k_axpy, blocks_for(n), kThreads, 0, s, n, a, x, y);
  FDE_LAUNCH_CHECK();
}
void vec_axpy_dev(size_t n, const double* a, double sgn, const double* x, double* y,
                  cudaStream_t s) {
  launch_k(k_axpy_dev, blocks_for(n), kThreads, 0, s, n, a, sgn, x, y);
  FDE_LAUNCH_CHECK();
}
void vec_scale_inv_dev(size_t n, const double* a, const double* x, double* y, cudaStream_t s) {
  launch_k(k_scale_inv_dev, blocks_for(n), kThreads, 0, s, n, a, x, y);
  FDE_LAUNCH_CHECK();
}
void vec_scal(size_t n, double a, double* x, cudaStream_t s) {
  launch_k(k_scal, blocks_for(n), kThreads, 0, s, n, a, x);
  FDE_LAUNCH_CHECK();
}
void vec_jacobi_update(size_t n, double a, const double* d, const double* r, double* out,
                       cudaStream_t s) {
  launch_k(k_jacobi_upd, blocks_for(n), kThreads, 0, s, n, a, d, r, out);
  FDE_LAUNCH_CHECK();
}
void vec_copy_scale(size_t n, double a, const double* x, double* y, cudaStream_t s) {
  launch_k(k_copy_scale2, blocks_for(n), kThreads, 0, s, n, a, x, y);
  FDE_LAUNCH_CHECK();
}
void vec_sub(size_t n, const double* x, const double* y, double* out, cudaStream_t s) {
  launch_k(k_sub, blocks_for(n), kThreads, 0, s, n, x, y, out);
  FDE_LAUNCH_CHECK();
}
void vec_lincomb(size_t n, const double* x0, const double* const* v, const double* c, int k,
                 double* out, cudaStream_t s) {
  launch_k(k_lincomb, blocks_for(n), kThreads, 0, s, n, x0, v, c, k, out);
  FDE_LAUNCH_CHECK();
}

Reducer::Reducer() : partials_(2 * kMaxBlocks), counter_(1) {
  FDE_CUDA(cudaMemset(counter_.get(), 0, sizeof(unsigned int)));
}
void Reducer::dot(size_t n, const double* x, const double* y, double* out, cudaStream_t s,
                  bool sqrt_out) {
  launch_k(k_dot, blocks_for(n), kThreads, 0, s, n, x, y, partials_.get(), counter_.get(), out,
                                           sqrt_out ? 1 : 0);
  FDE_LAUNCH_CHECK();
}

void Reducer::bicg_s(size_t n, const double* r, const double* v, double* sv, double* sc,
                     int rho_slot, cudaStream_t s) {
  launch_k(k_bicg_s, blocks_for(n), kThreads, 0, s, n, r, v, sv, sc, rho_slot, partials_.get(),
           counter_.get());
  FDE_LAUNCH_CHECK();
}
void Reducer::bicg_tt(size_t n, const double* t, const double* sv, double* sc, cudaStream_t s) {
  launch_k(k_bicg_tt, blocks_for(n), kThreads, 0, s, n, t, sv, sc, partials_.get(),
           counter_.get());
  FDE_LAUNCH_CHECK();
}
void Reducer::bicg_xr(size_t n, const double* p, const double* sv, const double* t,
                      const double* rh, double* x, double* r, double* sc, int rho_out,
                      cudaStream_t s) {
  launch_k(k_bicg_xr, blocks_for(n), kThreads, 0, s, n, p, sv, t, rh, x, r, sc, rho_out,
           partials_.get(), counter_.get());
  FDE_LAUNCH_CHECK();
}
void Reducer::bicg_p(size_t n, const double* r, const double* v, double* p, const double* sc,
                     int rho_new, int rho_old, cudaStream_t s) {
  launch_k(k_bicg_p, blocks_for(n), kThreads, 0, s, n, r, v, p, sc, rho_new, rho_old);
  FDE_LAUNCH_CHECK();
}

void Reducer::norm_dot(size_t n, const double* w, const double* v, double* norm_out,
                       double* dot_out, cudaStream_t s) {
  launch_k(k_norm_dot, blocks_for(n), kThreads, 0, s, n, w, v, partials_.get(), counter_.get(),
                                                norm_out, dot_out);
  FDE_LAUNCH_CHECK();
}
bool Reducer::mgs_chain(size_t n, double* w, const double* const* v_dev, int last, double* dh,
                        double* dnorm0, double* dnrmw, double* vout, cudaStream_t s) {
  struct Setup {
    int grid;
    size_t max_smem;
  };
  static DeviceCache<Setup> setup;  // per device: cooperative grid, opt-in shared memory
  const Setup& su = setup.get([](int dev) {
    Setup r{0, 0};
    int sms = 0, coop = 0, optin = 0;
    FDE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FDE_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    FDE_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (const char* e = std::getenv("FDE_MGS_CHAIN"))
      if (e[0] == '0') coop = 0;
    if (coop) {
      size_t room = (size_t)optin;
      for (auto kern : {k_mgs_chain, k_mgs_chain_tmem}) {
        cudaFuncAttributes fa{};
        FDE_CUDA(cudaFuncGetAttributes(&fa, kern));
        if ((size_t)optin - fa.sharedSizeBytes < room) room = (size_t)optin - fa.sharedSizeBytes;
      }
      r.max_smem = room;
      for (auto kern : {k_mgs_chain, k_mgs_chain_tmem})
        FDE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)r.max_smem));
      r.grid = sms;
    }
    return r;
  });
  const size_t max_smem = su.max_smem;
  if (su.grid == 0 || su.grid > kChainMaxGrid) return false;
  // short vectors: one CTA per FDE_CHAIN_MIN_SLICE doubles instead of one per
  // SM (cfg1's 3969 unknowns: a single CTA, whose reductions never leave it)
  int grid = su.grid;
#if FDE_CHAIN_MIN_SLICE > 0
  {
    const size_t want = (n + FDE_CHAIN_MIN_SLICE - 1) / FDE_CHAIN_MIN_SLICE;
    if (want < (size_t)grid) grid = want < 1 ? 1 : (int)want;
  }
#endif
  const size_t chunk = ((n + grid - 1) / grid + 1) & ~size_t(1);
  if (chunk * sizeof(double) > max_smem) return false;
  const bool in_tmem = FDE_CHAIN_TMEM && chunk >= FDE_CHAIN_TMEM_MIN &&
                       chunk <= 2 * (size_t)kChainSlots * kChainThreads;
  if (chain_flags_.size() == 0) {
    chain_flags_.alloc(8 * (size_t)su.grid);  // 2 epoch parities x 4 flag words per CTA
  }
  // epochs restart at 1 in every launch: clear the flag words
  FDE_CUDA(cudaMemsetAsync(chain_flags_.get(), 0, 8 * (size_t)grid * sizeof(unsigned long long), s));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kChainThreads);
  cfg.dynamicSmemBytes = chunk * sizeof(double);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, in_tmem ? k_mgs_chain_tmem : k_mgs_chain, n, chunk, w, v_dev,
                                last, dh, dnorm0, dnrmw,
                                vout, chain_flags_.get()),
             "kernel launch");
  FDE_LAUNCH_CHECK();
  return true;
}

void Reducer::mgs(size_t n, double* w, const double* vk, const double* hk, const double* vnext,
                  double* out, bool sqrt_out, cudaStream_t s) {
  launch_k(k_mgs, blocks_for(n), kThreads, 0, s, n, w, vk, hk, vnext, partials_.get(),
                                           counter_.get(), out, sqrt_out ? 1 : 0);
  FDE_LAUNCH_CHECK();
}

Xfer make_xfer(int n1, int n2, bool cx, bool cy) {
  Xfer t{};
  t.n1 = n1;
  t.n2 = n2;
  t.k1 = cx ? (n1 - n1 % 2) / 2 : n1;
  t.k2 = cy ? (n2 - n2 % 2) / 2 : n2;
  t.par1 = (n1 + 1) % 2;
  t.par2 = (n2 + 1) % 2;
  t.cx = cx;
  t.cy = cy;
  if (t.k1 == 0 || t.k2 == 0 || (!cx && !cy)) throw InvalidArgument("grid too small to coarsen");
  return t;
}
void xfer_restrict_rows(const Xfer& t, const double* fine, int f_lo, double* coarse, int c_lo,
                        int c_rows, double scale, cudaStream_t s) {
  const size_t nc = (size_t)t.k1 * c_rows;
  if (!nc) return;
  launch_k(k_restrict, blocks_for(nc), kThreads, 0, s, t, fine, f_lo, coarse, c_lo, c_rows, scale,
           (double*)nullptr, (const double*)nullptr, 0.0);
  FDE_LAUNCH_CHECK();
}
void xfer_prolong_rows(const Xfer& t, const double* coarse, int c_lo, double* fine, int f_lo,
                       int f_rows, bool add, cudaStream_t s) {
  const size_t nf = (size_t)t.n1 * f_rows;
  if (!nf) return;
  if (add) launch_k(k_prolong<true>, blocks_for(nf), kThreads, 0, s, t, coarse, c_lo, fine, f_lo, f_rows);
  else launch_k(k_prolong<false>, blocks_for(nf), kThreads, 0, s, t, coarse, c_lo, fine, f_lo, f_rows);
  FDE_LAUNCH_CHECK();
}
void xfer_restrict(const Xfer& t, const double* fine, double* coarse, double scale,
                   cudaStream_t s) {
  xfer_restrict_rows(t, fine, 0, coarse, 0, t.k2, scale, s);
}
void xfer_restrict_smooth(const Xfer& t, const double* fine, double* coarse, double scale,
                          const double* dinv_c, double omega, double* xc, cudaStream_t s) {
  const size_t nc = (size_t)t.k1 * t.k2;
  if (!nc) return;
  launch_k(k_restrict, blocks_for(nc), kThreads, 0, s, t, fine, 0, coarse, 0, t.k2, scale, xc, dinv_c,
                                                 omega);
  FDE_LAUNCH_CHECK();
}
void xfer_prolong_add(const Xfer& t, const double* coarse, double* fine, cudaStream_t s) {
  xfer_prolong_rows(t, coarse, 0, fine, 0, t.n2, true, s);
}
void xfer_prolong(const Xfer& t, const double* coarse, double* fine, cudaStream_t s) {
  xfer_prolong_rows(t, coarse, 0, fine, 0, t.n2, false, s);
}
void block_permute(const double* in, double* out, size_t nc, size_t d2, const long long* off,
                   int nranks, int dir, cudaStream_t s) {
  RankOffsets ro{};
  for (int r = 0; r <= nranks; ++r) ro.o[r] = off[r];
  ro.n = nranks;
  const size_t total = nc * d2;
  if (!total) return;
  launch_k(k_block_permute, blocks_for(total), kThreads, 0, s, in, out, nc, d2, ro, dir);
  FDE_LAUNCH_CHECK();
}
void lu_solve(int n, const double* lu, const int* perm, const double* b, double* x,
              cudaStream_t s) {
  launch_k(k_lu_solve, 1, 256, (size_t)n * sizeof(double), s, n, lu, perm, b, x);
  FDE_LAUNCH_CHECK();
}

// ---- FP64 roofline denominator, measured where the bench runs ---------------
// Eight independent DFMA chains per thread (inline PTX: the compiler keeps
// every one), 8 CTAs of 256 threads per SM: saturates the FP64 pipe.
namespace {
__global__ void __launch_bounds__(256) k_dfma_probe(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

double fp64_peak_tflops(cudaStream_t s) {
  int dev = current_device(), sms = 0;
  FDE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int blocks = sms * 8, threads = 256, iters = 2048;
  DevBuf<double> out((size_t)blocks * threads);
  cudaEvent_t e0, e1;
  FDE_CUDA(cudaEventCreate(&e0));
  FDE_CUDA(cudaEventCreate(&e1));
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {  // first repetition warms up
    FDE_CUDA(cudaEventRecord(e0, s));
    k_dfma_probe<<<blocks, threads, 0, s>>>(out.get(), iters, 0.999999, 1e-7);
    FDE_LAUNCH_CHECK();
    FDE_CUDA(cudaEventRecord(e1, s));
    FDE_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FDE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    const double tf = 2.0 * 8 * 16 * (double)iters * blocks * threads / (ms * 1e9);
    if (rep > 0 && tf > best) best = tf;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

}  // namespace fde_b200
