// Kernels for the batched Toeplitz line convolutions (see line_conv.cuh).
//
// Per line (length n <= M, L = 2M): three complex length-M transforms --
// one forward of the packed real input, two inverses of the packed T x and
// T^T x spectra -- as Stockham radix-16 stages (16 points per thread in
// registers, plus one radix-2/4/8 stage when log2 M is not a multiple of 4).
// Shared memory is only the inter-stage exchange buffer, SoA re/im doubles
// with an XOR swizzle that makes every stage's 8-byte accesses bank-conflict
// free (half-warp phases).  Stage twiddles cost one table load per butterfly;
// the other powers come from a depth-4 product tree (the FP64 pipe has the
// headroom, the L1/shared-memory pipe does not).
#include <type_traits>

#include "line_conv.cuh"
#include "tmem.cuh"

namespace fde_b200 {
namespace {

// XOR swizzle of the exchange buffers; conflict free for every stage's
// 8-byte accesses (half-warp phases) when SH = log2(points per thread).
template <int SH>
__device__ __forceinline__ int swz(int p) { return p ^ ((p >> SH) & 15); }

// spectral constants a_k, b_k of one k: a single 256-bit read-only load
__device__ __forceinline__ void ld_ab(const double4* p, double2& a, double2& b) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
      : "l"(p));
}

// ---- small DFTs on registers; INV = false uses exp(-2 pi i / R) -----------
template <bool INV>
__device__ __forceinline__ double2 rot90(double2 a) {  // * (-i) forward, * (+i) inverse
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
// a * exp(-+ 2 pi i e / 16) for a compile-time exponent e (0..15)
template <bool INV, int E>
__device__ __forceinline__ double2 tw16(double2 a) {
  constexpr int e = E & 15;
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  constexpr double h = 0.70710678118654752440;
  if constexpr (e == 0) return a;
  else if constexpr (e == 4) return rot90<INV>(a);
  else if constexpr (e == 8) return make_double2(-a.x, -a.y);
  else if constexpr (e == 12) return rot90<!INV>(a);
  else {
    // cos and sin of 2 pi e / 16
    constexpr double cr = e == 1 ? c1 : e == 2 ? h : e == 3 ? s1 : e == 5 ? -s1 : e == 6 ? -h
                        : e == 7 ? -c1 : e == 9 ? -c1 : e == 10 ? -h : e == 11 ? -s1
                        : e == 13 ? s1 : e == 14 ? h : c1;
    constexpr double sn = e == 1 ? s1 : e == 2 ? h : e == 3 ? c1 : e == 5 ? c1 : e == 6 ? h
                        : e == 7 ? s1 : e == 9 ? -s1 : e == 10 ? -h : e == 11 ? -c1
                        : e == 13 ? -c1 : e == 14 ? -h : -s1;
    constexpr double ci = INV ? sn : -sn;  // forward root exp(-i theta)
    return make_double2(a.x * cr - a.y * ci, a.x * ci + a.y * cr);
  }
}

// in place DFT4 of (a0, a1, a2, a3)
template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 b0 = cadd(a0, a2), b2 = csub(a0, a2);
  const double2 b1 = cadd(a1, a3), b3 = rot90<INV>(csub(a1, a3));
  a0 = cadd(b0, b1);
  a2 = csub(b0, b1);
  a1 = cadd(b2, b3);
  a3 = csub(b2, b3);
}

template <int R, bool INV, bool HALF>
struct Dft;
template <bool INV, bool HALF>
struct Dft<2, INV, HALF> {
  __device__ __forceinline__ static void run(double2 (&u)[2]) {
    const double2 t = u[0];
    u[0] = cadd(t, u[1]);
    u[1] = csub(t, u[1]);
  }
};
template <bool INV, bool HALF>
struct Dft<4, INV, HALF> {
  __device__ __forceinline__ static void run(double2 (&u)[4]) {
    dft4<INV>(u[0], u[1], u[2], u[3]);
  }
};
template <bool INV, bool HALF>
struct Dft<8, INV, HALF> {
  __device__ __forceinline__ static void run(double2 (&u)[8]) {
    // radix-2 DIF split, twiddle W8^k, two DFT4s (HALF: inputs 4..7 are zero)
    double2 a[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (HALF) {
        a[k] = u[k];
        a[k + 4] = u[k];
      } else {
        a[k] = cadd(u[k], u[k + 4]);
        a[k + 4] = csub(u[k], u[k + 4]);
      }
    }
    a[5] = tw16<INV, 2>(a[5]);
    a[6] = tw16<INV, 4>(a[6]);
    a[7] = tw16<INV, 6>(a[7]);
    dft4<INV>(a[0], a[1], a[2], a[3]);  // X[0], X[2], X[4], X[6]
    dft4<INV>(a[4], a[5], a[6], a[7]);  // X[1], X[3], X[5], X[7]
    u[0] = a[0]; u[2] = a[1]; u[4] = a[2]; u[6] = a[3];
    u[1] = a[4]; u[3] = a[5]; u[5] = a[6]; u[7] = a[7];
  }
};
// DFT16 = DFT4 (over n2) -> twiddle W16^(n1 k1) -> DFT4 (over n1).
// HALF: inputs 8..15 are zero (zero-padded forward input, first stage).
template <bool INV, bool HALF>
struct Dft<16, INV, HALF> {
  __device__ __forceinline__ static void run(double2 (&u)[16]) {
    double2 a[4][4];  // a[n1][k1]
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
      if (HALF) {  // u[n1 + 8] = u[n1 + 12] = 0
        const double2 x0 = u[n1], x1 = u[n1 + 4];
        a[n1][0] = cadd(x0, x1);
        a[n1][2] = csub(x0, x1);
        const double2 r = rot90<INV>(x1);
        a[n1][1] = cadd(x0, r);
        a[n1][3] = csub(x0, r);
      } else {
        a[n1][0] = u[n1];
        a[n1][1] = u[n1 + 4];
        a[n1][2] = u[n1 + 8];
        a[n1][3] = u[n1 + 12];
        dft4<INV>(a[n1][0], a[n1][1], a[n1][2], a[n1][3]);
      }
    }
    a[1][1] = tw16<INV, 1>(a[1][1]);
    a[1][2] = tw16<INV, 2>(a[1][2]);
    a[1][3] = tw16<INV, 3>(a[1][3]);
    a[2][1] = tw16<INV, 2>(a[2][1]);
    a[2][2] = tw16<INV, 4>(a[2][2]);
    a[2][3] = tw16<INV, 6>(a[2][3]);
    a[3][1] = tw16<INV, 3>(a[3][1]);
    a[3][2] = tw16<INV, 6>(a[3][2]);
    a[3][3] = tw16<INV, 9>(a[3][3]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      dft4<INV>(a[0][k1], a[1][k1], a[2][k1], a[3][k1]);
      u[k1] = a[0][k1];
      u[k1 + 4] = a[1][k1];
      u[k1 + 8] = a[2][k1];
      u[k1 + 12] = a[3][k1];
    }
  }
};

// Output-pruned DFTs: only outputs 0 .. R/2 - 1 (the last inverse stage, whose
// upper half lands on positions >= M/2 that the zero-padded lines discard).
template <bool INV>
__device__ __forceinline__ void dft4_lo(double2& a0, double2& a1, double2 a2, double2 a3) {
  const double2 b0 = cadd(a0, a2), b2 = csub(a0, a2);
  const double2 b1 = cadd(a1, a3), b3 = rot90<INV>(csub(a1, a3));
  a0 = cadd(b0, b1);
  a1 = cadd(b2, b3);
}
template <int R, bool INV>
struct DftLo;
template <bool INV>
struct DftLo<8, INV> {
  __device__ __forceinline__ static void run(double2 (&u)[8]) {
    double2 a[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[k] = cadd(u[k], u[k + 4]);
      a[k + 4] = csub(u[k], u[k + 4]);
    }
    a[5] = tw16<INV, 2>(a[5]);
    a[6] = tw16<INV, 4>(a[6]);
    a[7] = tw16<INV, 6>(a[7]);
    dft4_lo<INV>(a[0], a[1], a[2], a[3]);  // X[0], X[2]
    dft4_lo<INV>(a[4], a[5], a[6], a[7]);  // X[1], X[3]
    u[0] = a[0]; u[2] = a[1];
    u[1] = a[4]; u[3] = a[5];
  }
};
template <bool INV>
struct DftLo<16, INV> {
  __device__ __forceinline__ static void run(double2 (&u)[16]) {
    double2 a[4][4];  // a[n1][k1]
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
      a[n1][0] = u[n1];
      a[n1][1] = u[n1 + 4];
      a[n1][2] = u[n1 + 8];
      a[n1][3] = u[n1 + 12];
      dft4<INV>(a[n1][0], a[n1][1], a[n1][2], a[n1][3]);
    }
    a[1][1] = tw16<INV, 1>(a[1][1]);
    a[1][2] = tw16<INV, 2>(a[1][2]);
    a[1][3] = tw16<INV, 3>(a[1][3]);
    a[2][1] = tw16<INV, 2>(a[2][1]);
    a[2][2] = tw16<INV, 4>(a[2][2]);
    a[2][3] = tw16<INV, 6>(a[2][3]);
    a[3][1] = tw16<INV, 3>(a[3][1]);
    a[3][2] = tw16<INV, 6>(a[3][2]);
    a[3][3] = tw16<INV, 9>(a[3][3]);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      dft4_lo<INV>(a[0][k1], a[1][k1], a[2][k1], a[3][k1]);
      u[k1] = a[0][k1];
      u[k1 + 4] = a[1][k1];
    }
  }
};

template <int R>
struct Log2;
template <> struct Log2<2> { static constexpr int v = 1; };
template <> struct Log2<4> { static constexpr int v = 2; };
template <> struct Log2<8> { static constexpr int v = 3; };
template <> struct Log2<16> { static constexpr int v = 4; };

// w^r for r = 1..R-1 from w^1 by a shallow product tree (depth <= 4).
template <int R>
__device__ __forceinline__ void powers(double2 w1, double2 (&w)[R]) {
  w[1] = w1;
  if constexpr (R > 2) {
    w[2] = cmul(w1, w1);
    w[3] = cmul(w[2], w1);
  }
  if constexpr (R > 4) {
    w[4] = cmul(w[2], w[2]);
    w[5] = cmul(w[4], w1);
    w[6] = cmul(w[4], w[2]);
    w[7] = cmul(w[4], w[3]);
  }
  if constexpr (R > 8) {
    w[8] = cmul(w[4], w[4]);
#pragma unroll
    for (int r = 9; r < 16; ++r) w[r] = cmul(w[8], w[r - 8]);
  }
}

// Stage twiddle base W_{NS R}^(j mod NS) for butterfly q (index into exp(-2 pi i k/M)).
template <int LOGM, int P, int NSL, int R>
__device__ __forceinline__ void load_tw(double2 (&pre)[P], int tl, const double2* twM) {
  constexpr int M = 1 << LOGM, T = M / P, NS = 1 << NSL, B = P / R;
  constexpr int TWSH = LOGM - NSL - Log2<R>::v;
  if constexpr (NS > 1) {
#pragma unroll
    for (int q = 0; q < B; ++q) pre[q] = twM[((tl + q * T) & (NS - 1)) << TWSH];  // plain: stays after the barrier
  }
}

template <int LOGM, int P, int NSL>
struct NextRadix {  // radix of the stage that starts at NSL
  static constexpr int REM = LOGM - NSL;
  static constexpr int v = REM >= Log2<P>::v ? P : (1 << REM);
};

// One Stockham stage on v[s] = a[tl + s*T] (P slots per thread).  Radix R,
// NS = 2^NSL.  Non-final stages exchange through shared memory; the final
// stage leaves results in the same slots.
template <int LOGM, int P, bool INV, int NSL, int R, bool LAST, bool HALF>
__device__ __forceinline__ void stage(double2 (&v)[P], double* re, double* im, int tl,
                                      const double2* twM, double2 (&pre)[P]) {
  constexpr int M = 1 << LOGM, T = M / P, NS = 1 << NSL, B = P / R, SH = Log2<P>::v;
  (void)M;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    double2 u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[q + r * B];
    if (NS > 1) {  // this stage's W^(jm), loaded before the previous exchange
      double2 w1 = pre[q];
      if (INV) w1.y = -w1.y;
      double2 w[R];
      powers<R>(w1, w);
#pragma unroll
      for (int r = 1; r < R; ++r) u[r] = cmul(u[r], w[r]);
    }
    Dft<R, INV, HALF>::run(u);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q + r * B] = u[r];
  }
  if constexpr (!LAST) {
    load_tw<LOGM, P, NSL + Log2<R>::v, NextRadix<LOGM, P, NSL + Log2<R>::v>::v>(pre, tl, twM);
    __syncthreads();  // everyone finished reading the previous contents
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int j = tl + q * T;
      const int base = ((j >> NSL) << (NSL + Log2<R>::v)) + (j & (NS - 1));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int p = swz<SH>(base + r * NS);
        re[p] = v[q + r * B].x;
        im[p] = v[q + r * B].y;
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const int p = swz<SH>(tl + s * T);
      v[s] = make_double2(re[p], im[p]);
    }
  }
}

// Full length-M transform: radix-P stages, then one smaller radix stage.
template <int LOGM, int P, bool INV, int NSL, bool HALF>
struct Fft {
  __device__ __forceinline__ static void run(double2 (&v)[P], double* re, double* im, int tl,
                                             const double2* twM, double2 (&pre)[P]) {
    constexpr int REM = LOGM - NSL, LP = Log2<P>::v;
    if constexpr (REM >= LP) {
      stage<LOGM, P, INV, NSL, P, REM == LP, HALF>(v, re, im, tl, twM, pre);
      if constexpr (REM > LP) Fft<LOGM, P, INV, NSL + LP, false>::run(v, re, im, tl, twM, pre);
    } else if constexpr (REM == 3) {
      stage<LOGM, P, INV, NSL, 8, true, false>(v, re, im, tl, twM, pre);
    } else if constexpr (REM == 2) {
      stage<LOGM, P, INV, NSL, 4, true, false>(v, re, im, tl, twM, pre);
    } else if constexpr (REM == 1) {
      stage<LOGM, P, INV, NSL, 2, true, false>(v, re, im, tl, twM, pre);
    }
  }
};

#ifndef FDE_PTS
#define FDE_PTS 16
#endif
// points per thread by FFT size: short lines take fewer points per thread,
// so more threads share a line and the serial butterfly chain shrinks
#ifndef FDE_PTS_SMALL
#define FDE_PTS_SMALL 4  // M <= 256
#endif
#ifndef FDE_PTS_9
#define FDE_PTS_9 8
#endif
#ifndef FDE_PTS_10
#define FDE_PTS_10 8
#endif
#ifndef FDE_L2_PREFETCH
#define FDE_L2_PREFETCH 0  // measured: cfg4 +0.3 % steps/s without
#endif
#ifndef FDE_MINB_BIG
#define FDE_MINB_BIG 2
#endif
#ifndef FDE_MINB_P8
#define FDE_MINB_P8 2
#endif

template <int LOGM>
struct FftShape {
  static constexpr int P =
      LOGM <= 8 ? FDE_PTS_SMALL : (LOGM == 9 ? FDE_PTS_9 : (LOGM == 10 ? FDE_PTS_10 : FDE_PTS));
  static constexpr int M = 1 << LOGM;
  static constexpr int T = M / P;                      // threads per line
  static constexpr int LPB = T >= 128 ? 1 : 128 / T;   // lines per CTA
  static constexpr int THREADS = T * LPB;
  static constexpr int BUF = M + (T < 16 ? T : 0);     // per-buffer stride (doubles)
  static constexpr size_t SMEM = size_t(LPB) * 2 * BUF * sizeof(double);
  static constexpr int MINB = THREADS >= 256 ? (P == 8 && THREADS == 256 ? FDE_MINB_P8 : 1)
                                             : (LOGM == 9 ? 2 : (LOGM >= 10 ? FDE_MINB_BIG : 3));
};

// One CTA convolves LPB lines of length n <= M with T_b and T_b^T.
template <int LOGM, class Pol>
__global__ void __launch_bounds__(FftShape<LOGM>::THREADS, FftShape<LOGM>::MINB)
    fft_line_kernel(const Pol p) {
  pdl_enter();
  using S = FftShape<LOGM>;
  constexpr int M = S::M, T = S::T, BUF = S::BUF, P = S::P, H = P / 2, SH = Log2<P>::v;
  extern __shared__ double smem[];
  // lines per CTA is a launch-time choice (<= S::LPB): small levels use more CTAs
  const int ls = threadIdx.x / T, tl = threadIdx.x - ls * T;
  const int line = blockIdx.x * (int)(blockDim.x / T) + ls;
  const bool active = line < p.nlines();
  const int n = p.blk.n;
  double* const ra = smem + (size_t)ls * 2 * BUF;
  double* const ia = ra + BUF;

  // 0) warm L2 with the epilogue operands of this line (consumed ~3 FFTs later)
#if FDE_L2_PREFETCH
  if (active)
    for (int c = tl; c * 16 < n; c += T) p.prefetch(line, c);
#endif

  // 1) z_m = x_2m + i x_2m+1, m = tl + s*T; zero padded (n <= M: s < P/2 only)
  double2 v[P];
#pragma unroll
  for (int s = 0; s < H; ++s) {
    const int i0 = 2 * (tl + s * T);
    v[s].x = (active && i0 < n) ? p.load(line, i0) : 0.0;
    v[s].y = (active && i0 + 1 < n) ? p.load(line, i0 + 1) : 0.0;
    v[s + H] = make_double2(0.0, 0.0);
  }

  // 2) forward FFT_M -> Z[tl + s*T] in registers; publish for the partner reads
  double2 pre[P];
#ifndef FDE_EXP_NOFFT
  Fft<LOGM, P, false, 0, true>::run(v, ra, ia, tl, p.blk.twM, pre);
#endif
  __syncthreads();
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int q = swz<SH>(tl + s * T);
    ra[q] = v[s].x;
    ia[q] = v[s].y;
  }
  __syncthreads();

  // 3) spectral step.  Unpacking the real spectrum X[k], X[M-k] from Z,
  //    multiplying by S / conj(S) and repacking both real outputs for the
  //    half-length inverses collapses (per k) to
  //      Qy[k] = a_k Z[k] + b_k conj(Z[M-k]),  Qt[k] = conj(a_k) Z[k] - conj(b_k) conj(Z[M-k])
  //    with a_k, b_k precomputed per block (operator.cu): 8 products per k.
  //    Qy stays in v, Qt in qt (the compiler may keep part of it in
  //    L1-backed local memory: shared memory stays one buffer per line).
  double2 qt[P];
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int k = tl + s * T;
    const int qm = swz<SH>((M - k) & (M - 1));
    const double zr = v[s].x, zi = v[s].y;
    const double mr = ra[qm], mi = ia[qm];
    double2 ca, cb;  // a_k, b_k
    ld_ab(p.blk.ab + k, ca, cb);
    const double t1 = ca.x * zr, t2 = ca.y * zi, t3 = ca.x * zi, t4 = ca.y * zr;
    const double u1 = cb.x * mr, u2 = cb.y * mi, u3 = cb.y * mr, u4 = cb.x * mi;
    v[s] = make_double2((t1 - t2) + (u1 + u2), (t3 + t4) + (u3 - u4));
    qt[s] = make_double2((t1 + t2) + (u2 - u1), (t3 - t4) + (u3 + u4));
  }

  // 4) unnormalised inverse FFT_M of each packed spectrum -> q = T x (re: even
  //    positions, im: odd); only m < M/2 (s < P/2) carries outputs since n <= M.
#ifndef FDE_EXP_NOFFT
  Fft<LOGM, P, true, 0, false>::run(v, ra, ia, tl, p.blk.twM, pre);
#endif
  double2 ty[H];
#pragma unroll
  for (int s = 0; s < H; ++s) ty[s] = v[s];
#pragma unroll
  for (int s = 0; s < P; ++s) v[s] = qt[s];
#ifndef FDE_EXP_NOFFT
  Fft<LOGM, P, true, 0, false>::run(v, ra, ia, tl, p.blk.twM, pre);
#endif

  // 5) epilogue at the positions the inputs came from: fetch a group of
  //    operands, then finish it (one memory latency per group)
  if (!active) return;
  constexpr int G = H < 4 ? H : 4;
#pragma unroll
  for (int g = 0; g < H; g += G) {
    typename Pol::Ops o[2 * G];
#pragma unroll
    for (int s = g; s < g + G; ++s) {
      const int i0 = 2 * (tl + s * T);
#ifdef FDE_EXP_NOEPI
      o[2 * (s - g)] = typename Pol::Ops{};
      o[2 * (s - g) + 1] = typename Pol::Ops{};
#else
      if (i0 < n) o[2 * (s - g)] = p.fetch(line, i0);
      if (i0 + 1 < n) o[2 * (s - g) + 1] = p.fetch(line, i0 + 1);
#endif
    }
#pragma unroll
    for (int s = g; s < g + G; ++s) {
      const int i0 = 2 * (tl + s * T);
      if (i0 < n) p.finish(line, i0, ty[s].x, v[s].x, o[2 * (s - g)]);
      if (i0 + 1 < n) p.finish(line, i0 + 1, ty[s].y, v[s].y, o[2 * (s - g) + 1]);
    }
  }
}

// ---------------------------------------------------------------------------
// Paired-spectrum line kernel (M = 2^LOGM with LOGM % log2(P) != 0).
//
// The forward transform runs its radix-P stages first and the short radix
// R0 = 2^(LOGM mod log2 P) stage last; the two inverses run R0 first.  The
// last forward stage hands thread tl the butterflies {j, NS0 - j} (thread 0:
// the self-paired 0 and NS0/2), so every Z[k] and its spectral partner
// Z[M - k] sit in the same thread's registers, and the first inverse stage
// (radix R0, stride NS0) reads exactly those slots: no shared-memory round
// trip between the forward transform, the spectral step and the inverses.
// The packed spectra Qy, Qt and the first inverse's output are parked in
// tensor memory (tmem.cuh), so registers hold one 16-point set per thread and
// three CTAs share an SM.  Exchange buffers alternate (one barrier per
// exchange).
#ifndef FDE_PAIRED_DBUF
#define FDE_PAIRED_DBUF 0
#endif
template <int LOGM, int P>
struct PairedShape {
  static constexpr int M = 1 << LOGM, T = M / P, LP = Log2<P>::v;
  // log2 M a multiple of log2 P (M = 4096): the last radix-P stage splits
  // into a radix-P/2 stage and the paired radix-2 stage (16 16 8 | 2)
  static constexpr bool SPLIT = LOGM % LP == 0;
  static constexpr int REM = SPLIT ? 1 : LOGM % LP;  // log2 R0
  static constexpr int R0 = 1 << REM;
  // radix of the stage at NSL, forward (the split stage ends where R0 begins)
  // and inverse (the split stage follows the paired stage)
  template <int NSL>
  static constexpr int fwd_radix() { return SPLIT && LOGM - NSL == LP ? P / 2 : P; }
  template <int NSL>
  static constexpr int inv_radix() { return SPLIT && NSL == REM ? P / 2 : P; }
  static constexpr int B0 = P / R0;      // butterflies per thread in the R0 stage
  static constexpr int NS0 = M / R0;     // = B0 * T
  static constexpr int LPC = T >= 128 ? 1 : 128 / T;  // lines per CTA (lockstep)
  static constexpr int THREADS = T * LPC;
  static constexpr int BUF = M;          // doubles per re / im plane
  // alternating exchange buffers need an even exchange count per transform
  // (both inverses start on buffer 0 with no barrier in between)
  static constexpr int NBUF = (FDE_PAIRED_DBUF && (LOGM / LP) % 2 == 0) ? 2 : 1;
  // per line: exchange buffer(s) + the next line's input (BUF doubles)
  static constexpr size_t LINE_DOUBLES = (size_t(NBUF) * 2 + 1) * BUF;
  static constexpr size_t SMEM = LPC * LINE_DOUBLES * sizeof(double);
  static constexpr int TCOLS = 8 * P;    // Qy (4P words) + Qt (4P words) per thread
  // TMEM has 128 lanes: a CTA of several 128-thread warpgroups (one long
  // line, M = 8192) gives each warpgroup its own TCOLS-column range
  static constexpr int WG = THREADS / 128;
  static constexpr int TCOLS_CTA = TCOLS * WG;
  static_assert(REM != 0 && LOGM >= 2 * LP, "paired kernel needs a short stage");
  static constexpr int KX = LP;                 // radix-P -> radix-P exchanges
  static constexpr int KPF = 0;                 // into the paired forward stage
  static constexpr int KPI = P == 16 ? 3 : 2;   // out of the paired inverse stage
  static_assert(T % 32 == 0 && THREADS % 128 == 0 && (LPC == 1 || THREADS == 128),
                "whole warpgroups, one lane quadrant per warp");
  static_assert(TCOLS_CTA <= 512 && (TCOLS_CTA & (TCOLS_CTA - 1)) == 0, "TMEM allocation");
};

#ifndef FDE_L2_PREFETCH_PAIRED
#define FDE_L2_PREFETCH_PAIRED 0  // measured: cfg4 74.7 -> 75.5 steps/s without (cp.async staging covers dp/dm)
#endif
#ifndef FDE_EPI_AHEAD
#define FDE_EPI_AHEAD 1  // measured: cfg4 75.8 -> 75.9 steps/s
#endif
#ifndef FDE_X_TMEM_JACOBI
#define FDE_X_TMEM_JACOBI 0  // the Jacobi instance spills with the stash: measured +0.4 % steps/s without
#endif
#ifndef FDE_X_TMEM
#define FDE_X_TMEM 1  // measured: n=2047 apply 166.8 -> 165.6 us (L2 flushed), cfg4 +0.1 %
#endif
#ifndef FDE_P8_Y10
#define FDE_P8_Y10 0  // column passes at M = 1024 with 8 points/thread (one line per CTA): measured no change
#endif
#ifndef FDE_TMEM_LD64
#define FDE_TMEM_LD64 1  // one 32x32b.x64 load + wait per spectrum (measured +0.1 %)
#endif
#ifndef FDE_PAIRED12
#define FDE_PAIRED12 1
#endif
#ifndef FDE_PAIRED13
#define FDE_PAIRED13 1
#endif
#ifndef FDE_PAIRED_MINB
#define FDE_PAIRED_MINB 4  // CTAs per SM at M = 2048 (128 registers)
#endif
#ifndef FDE_PAIRED_MINB10
#define FDE_PAIRED_MINB10 5
#endif

// butterfly handled in slot q of the paired R0 stage
template <int B, int T>
__device__ __forceinline__ int paired_bfly(int tl, int q) {
  constexpr int NS = B * T;
  if (tl == 0) return q * T;
  return q < B / 2 ? tl + q * T : NS - tl - (q - B / 2) * T;
}

// twiddle + DFT of this thread's B = P / R butterflies (slots q + r * B)
template <int LOGM, int P, bool INV, int NSL, int R, bool PAIRED, bool HALF, bool LOWOUT = false>
__device__ __forceinline__ void pstage_compute(double2 (&v)[P], int tl, const double2 (&w1s)[P]) {
#ifdef FDE_EXP_NOFFT
  return;
#endif
  constexpr int B = P / R, NS = 1 << NSL;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    double2 u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[q + r * B];
    if constexpr (NS > 1) {
      double2 w1 = w1s[q];
      if (INV) w1.y = -w1.y;
      double2 w[R];
      powers<R>(w1, w);
#pragma unroll
      for (int r = 1; r < R; ++r) u[r] = cmul(u[r], w[r]);
    }
    if constexpr (LOWOUT) {
      DftLo<R, INV>::run(u);
#pragma unroll
      for (int r = 0; r < R / 2; ++r) v[q + r * B] = u[r];
    } else {
      Dft<R, INV, HALF>::run(u);
#pragma unroll
      for (int r = 0; r < R; ++r) v[q + r * B] = u[r];
    }
  }
}

template <int LOGM, int P, int NSL, int R, bool PAIRED>
__device__ __forceinline__ void pstage_twiddles(double2 (&w1s)[P], int tl, const double2* twM) {
  constexpr int T = (1 << LOGM) / P, B = P / R, NS = 1 << NSL;
  constexpr int TWSH = LOGM - NSL - Log2<R>::v;
  if constexpr (NS > 1) {
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int j = PAIRED ? paired_bfly<B, T>(tl, q) : tl + q * T;
      w1s[q] = twM[(j & (NS - 1)) << TWSH];
    }
  }
}

// Stockham write of a finished stage (NSL, R) to plane (re, im)
// Exchange-buffer swizzle p ^ ((p >> K) & 15) (K = 0: none).  Each exchange
// picks the K that makes both its write and its read pattern free of 8-byte
// bank conflicts (the paired stage's (j, NS - j) accesses need their own).
template <int K>
__device__ __forceinline__ int swzk(int p) {
  if constexpr (K == 0) return p;
  else return p ^ ((p >> K) & 15);
}

template <int LOGM, int P, int NSL, int R, bool PAIRED, int K>
__device__ __forceinline__ void pstage_write(const double2 (&v)[P], double* re, double* im,
                                             int tl) {
#ifdef FDE_EXP_NOXCHG
  return;
#endif
  constexpr int T = (1 << LOGM) / P, B = P / R, NS = 1 << NSL;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int j = PAIRED ? paired_bfly<B, T>(tl, q) : tl + q * T;
    const int base = ((j >> NSL) << (NSL + Log2<R>::v)) + (j & (NS - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = swzk<K>(base + r * NS);
      re[p] = v[q + r * B].x;
      im[p] = v[q + r * B].y;
    }
  }
}

// inputs of stage (R, PAIRED): butterfly j reads j + r * M / R
template <int LOGM, int P, int R, bool PAIRED, int K>
__device__ __forceinline__ void pstage_read(double2 (&v)[P], const double* re, const double* im,
                                            int tl) {
#ifdef FDE_EXP_NOXCHG
  return;
#endif
  constexpr int M = 1 << LOGM, T = M / P, B = P / R;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int j = PAIRED ? paired_bfly<B, T>(tl, q) : tl + q * T;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = swzk<K>(j + r * (M / R));
      v[q + r * B] = make_double2(re[p], im[p]);
    }
  }
}

#ifndef FDE_PRUNE_LAST
#define FDE_PRUNE_LAST 1
#endif
// Forward transform, radix-P stages from NSL, ending with the paired R0 stage.
// On entry the stage at NSL has its inputs in v; the exchange buffer toggles.
template <int LOGM, int P, int NSL, bool HALF>
struct PFwd {
  __device__ __forceinline__ static void run(double2 (&v)[P], double* buf, int& cur, int tl,
                                             const double2* twM, double2 (&w1s)[P]) {
    using S = PairedShape<LOGM, P>;
    constexpr int R = S::template fwd_radix<NSL>();  // P, or P/2 for the split stage
    static_assert(LOGM - NSL >= Log2<R>::v, "");
    pstage_compute<LOGM, P, false, NSL, R, false, HALF>(v, tl, w1s);
    double* re = buf + cur * 2 * S::BUF;
    if constexpr (S::NBUF == 1) __syncthreads();
    constexpr int NX = NSL + Log2<R>::v;
    constexpr bool LASTP = (LOGM - NX) == S::REM;  // next stage is the paired R0 stage
    constexpr int K = LASTP ? S::KPF : S::KX;
    pstage_write<LOGM, P, NSL, R, false, K>(v, re, re + S::BUF, tl);
    if constexpr (LASTP) {
      pstage_twiddles<LOGM, P, NX, S::R0, true>(w1s, tl, twM);
      __syncthreads();
      pstage_read<LOGM, P, S::R0, true, K>(v, re, re + S::BUF, tl);
      cur ^= S::NBUF - 1;
      pstage_compute<LOGM, P, false, NX, S::R0, true, false>(v, tl, w1s);
    } else {
      constexpr int RN = S::template fwd_radix<NX>();
      pstage_twiddles<LOGM, P, NX, RN, false>(w1s, tl, twM);
      __syncthreads();
      pstage_read<LOGM, P, RN, false, K>(v, re, re + S::BUF, tl);
      cur ^= S::NBUF - 1;
      PFwd<LOGM, P, NX, false>::run(v, buf, cur, tl, twM, w1s);
    }
  }
};

// Inverse stages from NSL (radix P, or P/2 for the split stage right after
// the paired one; inputs in v); the last stays in registers.
// hook(): called once the last stage's inputs are in registers (the exchange
// buffer is then free for the epilogue operands, see fft_line_kernel_paired)
template <int LOGM, int P, int NSL>
struct PInvTail {
  template <class Hook>
  __device__ __forceinline__ static void run(double2 (&v)[P], double* buf, int& cur, int tl,
                                             const double2* twM, double2 (&w1s)[P],
                                             const Hook& hook) {
    using S = PairedShape<LOGM, P>;
    constexpr int R = S::template inv_radix<NSL>();
    constexpr int NX = NSL + Log2<R>::v;
    static_assert(NX <= LOGM, "");
    // last stage (radix P): slots q + r B with r >= P/2 hold positions >= M/2 (unused)
    pstage_compute<LOGM, P, true, NSL, R, false, false, (NX >= LOGM) && FDE_PRUNE_LAST>(v, tl,
                                                                                        w1s);
    if constexpr (NX < LOGM) {
      constexpr int RN = S::template inv_radix<NX>();
      double* re = buf + cur * 2 * S::BUF;
      if constexpr (S::NBUF == 1) __syncthreads();
      pstage_write<LOGM, P, NSL, R, false, S::KX>(v, re, re + S::BUF, tl);
      pstage_twiddles<LOGM, P, NX, RN, false>(w1s, tl, twM);
      __syncthreads();
      pstage_read<LOGM, P, RN, false, S::KX>(v, re, re + S::BUF, tl);
      cur ^= S::NBUF - 1;
      if constexpr (NX + Log2<RN>::v >= LOGM) hook();  // the next stage is the last
      PInvTail<LOGM, P, NX>::run(v, buf, cur, tl, twM, w1s, hook);
    }
  }
};

// Full inverse: paired R0 stage (NS = 1) on the spectral slots, then the tail.
template <int LOGM, int P, class Hook>
__device__ __forceinline__ void pinverse(double2 (&v)[P], double* buf, int& cur, int tl,
                                         const double2* twM, double2 (&w1s)[P],
                                         const Hook& hook) {
  using S = PairedShape<LOGM, P>;
  constexpr int RN = S::template inv_radix<S::REM>();
  pstage_compute<LOGM, P, true, 0, S::R0, true, false>(v, tl, w1s);
  double* re = buf + cur * 2 * S::BUF;
  if constexpr (S::NBUF == 1) __syncthreads();
  pstage_write<LOGM, P, 0, S::R0, true, S::KPI>(v, re, re + S::BUF, tl);
  pstage_twiddles<LOGM, P, S::REM, RN, false>(w1s, tl, twM);
  __syncthreads();
  pstage_read<LOGM, P, RN, false, S::KPI>(v, re, re + S::BUF, tl);
  cur ^= S::NBUF - 1;
  if constexpr (S::REM + Log2<RN>::v >= LOGM) hook();  // the tail is one stage
  PInvTail<LOGM, P, S::REM>::run(v, buf, cur, tl, twM, w1s, hook);
}

// spectral partner slot of slot s = q + r * B0 (tl != 0 / tl == 0)
template <int B, int R>
constexpr int partner_slot(int s, bool t0) {
  const int q = s % B, r = s / B;
  if (!t0) return (q + B / 2) % B + (R - 1 - r) * B;
  const int q2 = (B - q) % B;
  const int r2 = q == 0 ? (R - r) % R : R - 1 - r;
  return q2 + r2 * B;
}

// Per-line I/O views for the paired kernel: pointers are offset to the
// thread's first position 2*tl once, so every slot's accesses use
// compile-time displacements d = pos - 2*tl (no per-access 64-bit index math).
template <class Pol, int EPI>
struct LineIO;

// YPass: EPI carries the layout flags, bit 0 = xT (x transposed), bit 1 = qT
template <int EPI>
struct LineIO<YPass, EPI> {
  static constexpr bool XT = EPI & 1, QT = (EPI >> 1) & 1;
  const double* x;
  const double* ep;
  const double* em;
  double* q;
  int n1;
  double c;
  struct Ops {
    double ep, em;
  };
  __device__ __forceinline__ LineIO(const YPass& p, int line, int pos0) {
    const size_t n1s = p.n1, n2 = p.n2;
    n1 = p.n1;
    x = XT ? p.x + line * n2 + pos0 : p.x + line + pos0 * n1s;
    ep = p.epT + line * n2 + pos0;
    em = p.emT + line * n2 + pos0;
    q = QT ? p.q + line * n2 + pos0 : p.q + line + pos0 * n1s;
    c = p.c;
  }
  __device__ __forceinline__ double load(int d) const {
    return XT ? x[d] : x[(size_t)d * n1];
  }
  __device__ __forceinline__ const double* xaddr(int d) const {
    return XT ? x + d : x + (size_t)d * n1;
  }
  // the two operand streams staged through shared memory, and the rest
  __device__ __forceinline__ const double* staged(int k, int d) const { return (k ? em : ep) + d; }
  static constexpr bool kKeepX = false;  // the epilogue does not read x
  __device__ __forceinline__ Ops fetch_rest(int, double s0, double s1, double) const {
    return Ops{s0, s1};
  }
  struct Glob {};  // no operands beyond the two staged streams
  __device__ __forceinline__ Glob fetch_glob(int) const { return Glob{}; }
  __device__ __forceinline__ Ops combine(const Glob&, double s0, double s1, double) const {
    return Ops{s0, s1};
  }
  __device__ __forceinline__ Ops fetch(int d) const { return Ops{ep[d], em[d]}; }
  __device__ __forceinline__ void finish(int d, double ty, double tt, const Ops& o) const {
    const double v = c * (o.ep * ty + o.em * tt);
    if (QT) q[d] = v;
    else q[(size_t)d * n1] = v;
  }
};

template <int EPI>
struct LineIO<XPass, EPI> {
  const double* x;
  const double* dp;
  const double* dm;
  const double* q;
  const double* e1;  // src (RHS) or b (RESID / JACOBI)
  const double* e2;  // dinv (JACOBI)
  double* out;
  double inv_r, sign, s2;  // s2: src_scale (RHS) or omega (JACOBI)
  struct Ops {
    double x, dp, dm, q, e1, e2;
  };
  __device__ __forceinline__ LineIO(const XPass& p, int line, int pos0) {
    const size_t o = (size_t)line * p.n1 + pos0;
    x = p.x + o;
    dp = p.dp + o;
    dm = p.dm + o;
    q = p.q ? p.q + o : nullptr;
    e1 = EPI == EPI_RHS ? p.src + o : (EPI == EPI_STORE ? nullptr : p.b + o);
    e2 = EPI == EPI_JACOBI ? p.dinv + o : nullptr;
    out = p.out + o;
    inv_r = p.inv_r;
    sign = p.sign;
    s2 = EPI == EPI_RHS ? p.src_scale : p.omega;
  }
  __device__ __forceinline__ double load(int d) const { return x[d]; }
  __device__ __forceinline__ const double* xaddr(int d) const { return x + d; }
  __device__ __forceinline__ const double* staged(int k, int d) const { return (k ? dm : dp) + d; }
  // the line's own input stays in shared memory for the epilogue (xv)
  static constexpr bool kKeepX = true;
  // global operands (Q, rhs/b, dinv) of one position, fetched ahead of use
  struct Glob {
    double q, e1, e2;
  };
  __device__ __forceinline__ Glob fetch_glob(int d) const {
    Glob g;
    g.q = q ? q[d] : 0.0;
    g.e1 = EPI == EPI_STORE ? 0.0 : e1[d];
    g.e2 = EPI == EPI_JACOBI ? e2[d] : 0.0;
    return g;
  }
  __device__ __forceinline__ Ops combine(const Glob& g, double s0, double s1, double xv) const {
    return Ops{xv, s0, s1, g.q, g.e1, g.e2};
  }
  __device__ __forceinline__ Ops fetch_rest(int d, double s0, double s1, double xv) const {
    Ops o;
    o.x = xv;
    o.dp = s0;
    o.dm = s1;
    o.q = q ? q[d] : 0.0;
    o.e1 = EPI == EPI_STORE ? 0.0 : e1[d];
    o.e2 = EPI == EPI_JACOBI ? e2[d] : 0.0;
    return o;
  }
  __device__ __forceinline__ Ops fetch(int d) const {
    Ops o;
    o.x = x[d];
    o.dp = dp[d];
    o.dm = dm[d];
    o.q = q ? q[d] : 0.0;
    o.e1 = EPI == EPI_STORE ? 0.0 : e1[d];
    o.e2 = EPI == EPI_JACOBI ? e2[d] : 0.0;
    return o;
  }
  __device__ __forceinline__ void finish(int d, double ty, double tt, const Ops& o) const {
    // structured.cpp:128,134-135,146: y = inv_r x; y += s dp t; y += s dm tt; y += Q
    double y = inv_r * o.x;
    y += sign * o.dp * ty;
    y += sign * o.dm * tt;
    if (q) y += o.q;
    if constexpr (EPI == EPI_RHS) out[d] = y + s2 * o.e1;
    else if constexpr (EPI == EPI_RESID) out[d] = o.e1 - y;
    else if constexpr (EPI == EPI_JACOBI) out[d] = o.x + s2 * o.e2 * (o.e1 - y);
    else out[d] = y;
  }
};

// points per thread of the paired kernel: 16 at M = 2048; at M = 1024 either
// 8 (one line per 128-thread CTA) or 16 (two lines per CTA, 64 threads each)
#ifndef FDE_P16_M1024
#define FDE_P16_M1024 1  // measured: 5-6 % faster 1023-point passes than 8 points/thread
#endif
#ifndef FDE_PAIRED9
#define FDE_PAIRED9 0  // M = 512, 16 points/thread, 4 lines per CTA: measured slower (V-cycle +3 %)
#endif
#ifndef FDE_PAIRED8
#define FDE_PAIRED8 0  // M = 256, 8 points/thread, 4 lines per CTA: measured slower (V-cycle +5 %)
#endif
template <int LOGM>
constexpr int paired_pts_for(bool ypass) {
  return LOGM == 8 || (LOGM == 10 && (!FDE_P16_M1024 || (ypass && FDE_P8_Y10))) ? 8 : 16;
}
template <int LOGM, class Pol>
constexpr int paired_pts() { return paired_pts_for<LOGM>(std::is_same<Pol, YPass>::value); }
template <int LOGM, class Pol>
constexpr int paired_minb() {  // CTAs per SM; per 128 threads for larger CTAs
  constexpr int th = PairedShape<LOGM, paired_pts<LOGM, Pol>()>::THREADS;
  constexpr int b = paired_pts<LOGM, Pol>() == 16 ? FDE_PAIRED_MINB : FDE_PAIRED_MINB10;
  return b * 128 / th > 0 ? b * 128 / th : 1;
}

template <int LOGM, class Pol, int EPI>
__global__ void __launch_bounds__(PairedShape<LOGM, paired_pts<LOGM, Pol>()>::THREADS,
                                  paired_minb<LOGM, Pol>())
    fft_line_kernel_paired(const Pol p) {
  pdl_enter();
  constexpr int P = paired_pts<LOGM, Pol>();
  using S = PairedShape<LOGM, P>;
  using IO = LineIO<Pol, EPI>;
  constexpr int T = S::T, H = P / 2, R0 = S::R0, B0 = S::B0, NS0 = S::NS0;
  extern __shared__ __align__(16) double smem_all[];
  // S::LPC lines per CTA in lockstep: thread tl of line slot ls
  const int ls = threadIdx.x / T, tl = threadIdx.x - ls * T, warp = threadIdx.x >> 5;
  double* const smem = smem_all + ls * S::LINE_DOUBLES;  // this line's buffers
  double* const xbuf = smem + S::NBUF * 2 * S::BUF;  // next line's input (own slots only)
  // the TMEM base address lands in the first exchange-buffer word (read into a
  // register before any exchange): no static shared memory, so four CTAs fit
  // a 196 KB carveout and the rest of the SM's L1 caches the spectral tables
  uint32_t* const s_tbase = reinterpret_cast<uint32_t*>(smem_all);
  const int n = p.blk.n, nl = p.nlines();
  constexpr int LPC = S::LPC;
  // line of this slot in the CTA's group starting at `base` (clamped: a slot
  // past the last line recomputes it and stores nothing)
  auto line_of = [&](int base) { return base + ls < nl ? base + ls : nl - 1; };

  // Persistent CTA: lines blockIdx.x, + gridDim.x, ...  Each thread copies the
  // next line's input slots (its own positions) into xbuf while the current
  // line is transformed, so only the first line waits for HBM.
  auto prefetch_x = [&](int line) {
#ifdef FDE_EXP_NOX
    return;
#endif
    const IO io(p, line, 2 * tl);
#pragma unroll
    for (int s = 0; s < H; ++s) {
      const int i0 = 2 * (tl + s * T), d = 2 * s * T;
      cp_async8(xbuf + i0, io.xaddr(i0 < n ? d : 0), i0 < n ? 8 : 0);
      cp_async8(xbuf + i0 + 1, io.xaddr(i0 + 1 < n ? d + 1 : 0), i0 + 1 < n ? 8 : 0);
    }
    cp_async_commit();
  };
#ifdef FDE_EXP_STAGGER
  {
    const int slot = blockIdx.x / 148;
    for (int k = 0; k < slot; ++k) __nanosleep(FDE_EXP_STAGGER);
  }
#endif
  if (warp == 0) tmem_alloc<S::TCOLS_CTA>(s_tbase);
  if (blockIdx.x * LPC < nl) prefetch_x(line_of(blockIdx.x * LPC));
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *s_tbase;  // the first exchange write follows a barrier
  if constexpr (S::NBUF != 1) __syncthreads();
  // this warp's lane quadrant, and its warpgroup's column range
  const uint32_t tq = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * S::TCOLS);
  const uint32_t tqy = tq, tqt = tq + 4 * P;                    // Qy, Qt column ranges
  constexpr bool kStashX = IO::kKeepX && FDE_X_TMEM && (FDE_X_TMEM_JACOBI || EPI != EPI_JACOBI);
  const uint32_t tqx = tqy + 4 * H;  // stashed row input (Qy columns past T x's)
  const double* const ep0 = smem;            // staged epilogue operands (exchange buffer)
  const double* const ep1 = smem + S::BUF;

#pragma unroll 1
  for (int base = blockIdx.x * LPC; base < nl; base += gridDim.x * LPC) {
    const int line = line_of(base);
    const bool live = base + ls < nl;  // uniform per line slot
    const int next = base + gridDim.x * LPC;
    const IO io(p, line, 2 * tl);
#if FDE_L2_PREFETCH_PAIRED
    // compile-time trip count (16 T >= M >= n): no loop-carried predicate to spill
#pragma unroll
    for (int i = 0; i < (S::M + 16 * T - 1) / (16 * T); ++i)
      if ((tl + i * T) * 16 < n) p.prefetch(line, tl + i * T);
#endif
    // 1) z_m = x_2m + i x_2m+1, m = tl + s*T, from this thread's xbuf slots
    //    (zero filled beyond n); then start the next line's copy
    cp_async_wait_all();
    double2 v[P];
#pragma unroll
    for (int s = 0; s < H; ++s) {
      const double2 t = *reinterpret_cast<const double2*>(xbuf + 2 * (tl + s * T));
      v[s] = t;
      v[s + H] = make_double2(0.0, 0.0);
    }
    if (!IO::kKeepX && next < nl) prefetch_x(line_of(next));

    // 2) forward transform; ends with this thread's paired slots in v
    double2 w1s[P];
    int cur = 0;
    PFwd<LOGM, P, 0, true>::run(v, smem, cur, tl, p.blk.twM, w1s);

    // 3) spectral step (see fft_line_kernel): partners are in registers;
    //    results go to tensor memory in groups of 4 slots
    {
      const bool t0 = tl == 0;
      const double4* abv = p.blk.ab;
#pragma unroll
      for (int g = 0; g < P; g += 4) {
        double2 qy[4], qt[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int s = g + c, q = s % B0, r = s / B0;
          const int k = paired_bfly<B0, T>(tl, q) + r * NS0;
          const double2 z = v[s];
          const double2 zm0 = v[partner_slot<B0, R0>(s, true)];
          const double2 zm1 = v[partner_slot<B0, R0>(s, false)];
          const double mr = t0 ? zm0.x : zm1.x, mi = t0 ? zm0.y : zm1.y;
#ifdef FDE_EXP_NOAB
          const double2 ca = make_double2(1.0 + k, 0.5), cb = make_double2(0.25, 0.125 * k);
#else
          double2 ca, cb;
          ld_ab(abv + k, ca, cb);
#endif
          const double t1 = ca.x * z.x, t2 = ca.y * z.y, t3 = ca.x * z.y, t4 = ca.y * z.x;
          const double u1 = cb.x * mr, u2 = cb.y * mi, u3 = cb.y * mr, u4 = cb.x * mi;
          qy[c] = make_double2((t1 - t2) + (u1 + u2), (t3 + t4) + (u3 - u4));
          qt[c] = make_double2((t1 + t2) + (u2 - u1), (t3 - t4) + (u3 + u4));
        }
        tmem_st4(tqy + 4 * g, qy);
        tmem_st4(tqt + 4 * g, qt);
      }
    }
    tmem_wait_st();

    // 4) inverse of Qy -> T x (packed; its H output slots are parked in the Qy
    //    columns), then 5) inverse of Qt -> T^T x.  One copy of the inverse
    //    code (instruction-cache footprint); both start on exchange buffer 0.
    //    Once the second inverse's last stage has its inputs in registers, the
    //    exchange buffer receives two epilogue operand streams (cp.async),
    //    overlapped with that stage's butterflies.
    const int n_inv = 2 + (n < 0);  // opaque trip count: ptxas keeps the loop rolled
#pragma unroll 1
    for (int it = 0; it < n_inv; ++it) {
      const uint32_t src = it ? tqt : tqy;
      if constexpr (P == 16 && FDE_TMEM_LD64) {
        tmem_ld16(src, v);  // the whole spectrum in one load and one wait
      } else {
#pragma unroll
        for (int g = 0; g < P; g += 4) {
          double2 t[4];
          tmem_ld4(src + 4 * g, t);
#pragma unroll
          for (int c = 0; c < 4; ++c) v[g + c] = t[c];
        }
      }
      if constexpr (kStashX) {
        // row pass: the line's own input moves from xbuf to the Qy columns
        // the first inverse no longer needs (H slots from column 4H), so the
        // next line's copy overlaps both inverses instead of waiting for the
        // epilogue (each thread touches only its own xbuf slots)
        if (it == 0) {
#pragma unroll
          for (int g = 0; g < H; g += 4) {
            double2 t[4];
#pragma unroll
            for (int c = 0; c < 4; ++c)
              t[c] = *reinterpret_cast<const double2*>(xbuf + 2 * (tl + (g + c) * T));
            tmem_st4(tqx + 4 * g, t);
          }
          if (next < nl) prefetch_x(line_of(next));
        }
      }
      cur = 0;
      auto stage_epilogue = [&]() {
        if (it == 0) return;
#ifdef FDE_EXP_NOEPI
        return;
#endif
        __syncthreads();  // every thread has read its last-stage inputs
#pragma unroll
        for (int s = 0; s < H; ++s) {
          const int i0 = 2 * (tl + s * T), d = 2 * s * T;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ok = i0 + e < n;
            cp_async8(smem + i0 + e, io.staged(0, ok ? d + e : 0), ok ? 8 : 0);
            cp_async8(smem + S::BUF + i0 + e, io.staged(1, ok ? d + e : 0), ok ? 8 : 0);
          }
        }
        cp_async_commit();
      };
      pinverse<LOGM, P>(v, smem, cur, tl, p.blk.twM, w1s, stage_epilogue);
      if (it == 0) {
#pragma unroll
        for (int g = 0; g < H; g += 4) {
          double2 t[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) t[c] = v[g + c];
          tmem_st4(tqy + 4 * g, t);
        }
        tmem_wait_st();
      }
    }

    // 6) epilogue in groups of 4 slots (8 positions); own staged slots only.
    //    Every operand of a group is fetched before any of its stores, with
    //    out-of-range positions clamped to the thread's first position
    //    (2 tl < n) and only the stores predicated: the global loads of a
    //    group are all in flight together (a tail group fetched element by
    //    element behind its own stores serialised one L2 latency per load).
#if FDE_EPI_AHEAD
    // group 0's global operands are in flight while the staged streams land
    typename IO::Glob gn[8];
    auto fetch_group = [&](int g) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i0 = 2 * (tl + (g + c) * T), d = 2 * (g + c) * T;
        gn[2 * c] = io.fetch_glob(i0 < n ? d : 0);
        gn[2 * c + 1] = io.fetch_glob(i0 + 1 < n ? d + 1 : 0);
      }
    };
    fetch_group(0);
#endif
    cp_async_wait_all();
#pragma unroll
    for (int g = 0; g < H; g += 4) {
      double2 ty[4], tx[4];
      tmem_ld4(tqy + 4 * g, ty);
      if constexpr (kStashX) tmem_ld4(tqx + 4 * g, tx);
      typename IO::Ops o[8];
#if FDE_EPI_AHEAD
      // later groups fetch at their top (fetching group g + 4 before group g
      // is used spills ~230 B in the Jacobi instance: measured 2 % slower)
      if (g > 0) fetch_group(g);
      typename IO::Glob gc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) gc[c] = gn[c];
#endif
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i0 = 2 * (tl + (g + c) * T);
        [[maybe_unused]] const int d = 2 * (g + c) * T;
        const double2 a = *reinterpret_cast<const double2*>(ep0 + i0);
        const double2 b = *reinterpret_cast<const double2*>(ep1 + i0);
        const double2 xv = kStashX       ? tx[c]
                           : IO::kKeepX ? *reinterpret_cast<const double2*>(xbuf + i0)
                                        : make_double2(0.0, 0.0);
#ifdef FDE_EXP_NOEPI
        o[2 * c] = typename IO::Ops{a.x, b.x};
        o[2 * c + 1] = typename IO::Ops{a.y, b.y};
#elif FDE_EPI_AHEAD
        o[2 * c] = io.combine(gc[2 * c], a.x, b.x, xv.x);
        o[2 * c + 1] = io.combine(gc[2 * c + 1], a.y, b.y, xv.y);
#else
        o[2 * c] = io.fetch_rest(i0 < n ? d : 0, a.x, b.x, xv.x);
        o[2 * c + 1] = io.fetch_rest(i0 + 1 < n ? d + 1 : 0, a.y, b.y, xv.y);
#endif
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i0 = 2 * (tl + (g + c) * T), d = 2 * (g + c) * T;
        if (live && i0 < n) io.finish(d, ty[c].x, v[g + c].x, o[2 * c]);
        if (live && i0 + 1 < n) io.finish(d + 1, ty[c].y, v[g + c].y, o[2 * c + 1]);
      }
    }
    // row pass without the stash: the next line's input lands once this
    // line's epilogue is done
    if (IO::kKeepX && !kStashX && next < nl) prefetch_x(line_of(next));
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<S::TCOLS_CTA>(tbase);
}

// Warp-per-line direct Toeplitz product for short lines (n <= kDirectMax):
// up to four outputs per lane, x broadcast by shuffles, the block's first
// column / row staged in shared memory.  Exact sums, no FFT latency chain --
// this is what the coarse multigrid levels run.
template <class P>
__global__ void __launch_bounds__(256) direct_line_kernel(const P p) {
  pdl_enter();
  constexpr int E = kDirectMax / 32;
  __shared__ double s_col[kDirectMax], s_row[kDirectMax];
  const int n = p.blk.n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    s_col[i] = p.blk.col[i];
    s_row[i] = p.blk.row[i];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = blockIdx.x * 8 + warp;
  if (line >= p.nlines()) return;
  double xv[E], ty[E], tt[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane + 32 * e;
    xv[e] = i < n ? p.load(line, i) : 0.0;
    ty[e] = 0.0;
    tt[e] = 0.0;
  }
#pragma unroll
  for (int kb = 0; kb < E; ++kb) {
    if (32 * kb >= n) break;
    const int kend = n - 32 * kb < 32 ? n - 32 * kb : 32;
    for (int kk = 0; kk < kend; ++kk) {
      const int k = 32 * kb + kk;
      const double xk = __shfl_sync(0xffffffffu, xv[kb], kk);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = lane + 32 * e;
        if (i < n) {
          ty[e] = fma(i >= k ? s_col[i - k] : s_row[k - i], xk, ty[e]);  // T(i,k)
          tt[e] = fma(k >= i ? s_col[k - i] : s_row[i - k], xk, tt[e]);  // T(k,i)
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane + 32 * e;
    if (i < n) p.finish(line, i, ty[e], tt[e], p.fetch(line, i));
  }
}

// 32 x 32 tiles, 32 x 8 threads; padded shared tile (8-byte banks).
__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ in,
                                                        double* __restrict__ out, int n1, int n2) {
  pdl_enter();
  __shared__ double tile[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int i = i0 + tx, j = j0 + ty + k;
    if (i < n1 && j < n2) tile[ty + k][tx] = in[(size_t)j * n1 + i];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int j = j0 + tx, i = i0 + ty + k;
    if (i < n1 && j < n2) out[(size_t)i * n2 + j] = tile[tx][ty + k];
  }
}

// Same tiling with the input map applied on the way in; the mapped values are
// also stored row-major when xout is set (read and written by the same thread).
template <int K>
__global__ void __launch_bounds__(256) transpose_map_kernel(const InMap m, double* xout,
                                                            double* __restrict__ out, int n1,
                                                            int n2) {
  pdl_enter();
  __shared__ double tile[32][33];
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int i = i0 + tx, j = j0 + ty + k;
    if (i < n1 && j < n2) {
      const double v = m.at<K>(i, j);
      tile[ty + k][tx] = v;
      if (xout) xout[(size_t)j * n1 + i] = v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int j = j0 + tx, i = i0 + ty + k;
    if (i < n1 && j < n2) out[(size_t)i * n2 + j] = tile[tx][ty + k];
  }
}

template <class P>
int lines_of(const P& p) {
  return std::is_same<P, YPass>::value ? p.n1 : p.n2;
}

template <int LOGM, class P>
void launch_fft(const P& p, cudaStream_t s) {
  using S = FftShape<LOGM>;
  static bool configured = false;  // per template instance
  if (!configured) {
    FDE_CUDA(cudaFuncSetAttribute(fft_line_kernel<LOGM, P>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    configured = true;
  }
  // spread small levels over the SMs: fewer lines per CTA until the grid
  // covers two waves (CTAs stay a whole number of warps)
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    FDE_CUDA(cudaGetDevice(&dev));
    FDE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int lines = lines_of(p);
  int lpb = S::LPB;
  const int min_lpb = S::T >= 32 ? 1 : 32 / S::T;
  while (lpb > min_lpb && (lines + lpb - 1) / lpb < 2 * sms) lpb /= 2;
  const int grid = (lines + lpb - 1) / lpb;
  const size_t smem = size_t(lpb) * 2 * S::BUF * sizeof(double);
  launch_k(fft_line_kernel<LOGM, P>, grid, S::T * lpb, smem, s, p);
  FDE_LAUNCH_CHECK();
}

#ifndef FDE_PAIRED
#define FDE_PAIRED 1
#endif

// Shared-memory carveout (percent of the 228 KB maximum): 85 % selects the
// 196 KB configuration, which still holds four CTAs (4 x 49,152 B + 1 KB
// reserved each) and leaves 60 KB of L1 for the spectral constants and
// twiddles (measured 165 -> 160 us per n = 2047 apply against the maximum).
#ifndef FDE_PAIRED_CARVEOUT
#define FDE_PAIRED_CARVEOUT 85
#endif
template <int LOGM, class P, int EPI>
void launch_paired_epi(const P& p, cudaStream_t s) {
  constexpr int PP = paired_pts<LOGM, P>();
  using S = PairedShape<LOGM, PP>;
  static bool configured = false;
  if (!configured) {
    FDE_CUDA(cudaFuncSetAttribute(fft_line_kernel_paired<LOGM, P, EPI>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    // resident CTAs are register-bound; give shared memory the whole carveout
    FDE_CUDA(cudaFuncSetAttribute(fft_line_kernel_paired<LOGM, P, EPI>,
                                  cudaFuncAttributePreferredSharedMemoryCarveout,
                                  FDE_PAIRED_CARVEOUT));
    configured = true;
  }
  static int max_ctas = 0;  // resident CTAs on the device (persistent grid)
  if (!max_ctas) {
    // registers, shared memory and tensor-memory columns per SM, whichever
    // binds (the occupancy API does not see the TMEM allocation)
    int dev = 0, sms = 0, smem_sm = 0, smem_rsv = 0, regs_sm = 0;
    FDE_CUDA(cudaGetDevice(&dev));
    FDE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FDE_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    FDE_CUDA(cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev));
    FDE_CUDA(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev));
    cudaFuncAttributes fa{};
    FDE_CUDA(cudaFuncGetAttributes(&fa, fft_line_kernel_paired<LOGM, P, EPI>));
    const int regs_cta = ((fa.numRegs * 32 + 255) / 256 * 256) * (S::THREADS / 32);
    int per_sm = regs_sm / regs_cta;
    const int by_smem = smem_sm / (int)(S::SMEM + fa.sharedSizeBytes + smem_rsv);
    const int by_tmem = 512 / S::TCOLS_CTA;
    per_sm = per_sm < by_smem ? per_sm : by_smem;
    per_sm = per_sm < by_tmem ? per_sm : by_tmem;
    max_ctas = sms * (per_sm > 0 ? per_sm : 1);
  }
  const int groups = (lines_of(p) + S::LPC - 1) / S::LPC;
  launch_k(fft_line_kernel_paired<LOGM, P, EPI>, groups < max_ctas ? groups : max_ctas, S::THREADS,
                                         S::SMEM, s, p);
  FDE_LAUNCH_CHECK();
}

template <int LOGM, class P>
void launch_paired(const P& p, cudaStream_t s) {
  if constexpr (std::is_same<P, YPass>::value) {
    switch ((p.xT ? 1 : 0) | (p.qT ? 2 : 0)) {
      case 1: return launch_paired_epi<LOGM, P, 1>(p, s);
      case 2: return launch_paired_epi<LOGM, P, 2>(p, s);
      case 3: return launch_paired_epi<LOGM, P, 3>(p, s);
      default: return launch_paired_epi<LOGM, P, 0>(p, s);
    }
  } else {
    switch (p.epi) {
      case EPI_RHS: return launch_paired_epi<LOGM, P, EPI_RHS>(p, s);
      case EPI_RESID: return launch_paired_epi<LOGM, P, EPI_RESID>(p, s);
      case EPI_JACOBI: return launch_paired_epi<LOGM, P, EPI_JACOBI>(p, s);
      default: return launch_paired_epi<LOGM, P, EPI_STORE>(p, s);
    }
  }
}

template <class P>
void launch_any(const P& p, cudaStream_t s) {
  const int lines = lines_of(p);
  if (lines <= 0) return;
  switch (p.blk.logM) {
    case 0:
      launch_k(direct_line_kernel<P>, (lines + 7) / 8, 256, 0, s, p);
      FDE_LAUNCH_CHECK();
      return;
    case 6: return launch_fft<6>(p, s);
    case 7: return launch_fft<7>(p, s);
    case 8: return FDE_PAIRED8 ? launch_paired<8>(p, s) : launch_fft<8>(p, s);
    case 9: return FDE_PAIRED9 ? launch_paired<9>(p, s) : launch_fft<9>(p, s);
    case 10: return FDE_PAIRED ? launch_paired<10>(p, s) : launch_fft<10>(p, s);
    case 11: return FDE_PAIRED ? launch_paired<11>(p, s) : launch_fft<11>(p, s);
    case 12: return FDE_PAIRED12 ? launch_paired<12>(p, s) : launch_fft<12>(p, s);
    case 13:  // n <= 8191 (cfg5's largest grid): one 512-thread line per SM
      return FDE_PAIRED13 ? launch_paired<13>(p, s) : launch_fft<13>(p, s);
    default: throw InvalidArgument("line length beyond the supported FFT sizes");
  }
}

}  // namespace

void launch_line_pass(const YPass& p, cudaStream_t s) { launch_any(p, s); }
void launch_transpose(const double* in, double* out, int n1, int n2, cudaStream_t s) {
  const dim3 grid((n1 + 31) / 32, (n2 + 31) / 32);
  launch_k(transpose_kernel, grid, 256, 0, s, in, out, n1, n2);
  FDE_LAUNCH_CHECK();
}
void launch_transpose_mapped(const InMap& m, double* xout, double* out, int n1, int n2,
                             cudaStream_t s) {
  const dim3 grid((n1 + 31) / 32, (n2 + 31) / 32);
  switch (m.kind) {
    case 0: launch_k(transpose_map_kernel<0>, grid, 256, 0, s, m, xout, out, n1, n2); break;
    case 1: launch_k(transpose_map_kernel<1>, grid, 256, 0, s, m, xout, out, n1, n2); break;
    case 2: launch_k(transpose_map_kernel<2>, grid, 256, 0, s, m, xout, out, n1, n2); break;
    default: throw InvalidArgument("unknown operator input map");
  }
  FDE_LAUNCH_CHECK();
}
void launch_line_pass(const XPass& p, cudaStream_t s) { launch_any(p, s); }

}  // namespace fde_b200
