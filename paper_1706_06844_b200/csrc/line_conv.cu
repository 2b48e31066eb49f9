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
#include <initializer_list>
#include <type_traits>

#include "line_conv.cuh"
#include "tmem.cuh"

namespace fde_b200 {
namespace {

// XOR swizzle of the exchange buffers; conflict free for every stage's
// 8-byte accesses (half-warp phases) when SH = log2(points per thread).
template <int SH>
__device__ __forceinline__ int swz(int p) { return p ^ ((p >> SH) & 15); }

// Programmatic-launch protocol of a column pass / row pass pair.  Nothing a
// row pass does before its epilogue depends on the column pass (it transforms
// x, the column pass writes Q), so a row pass launched right behind its column
// pass (XPass::late_wait) waits for it only before its first epilogue: its
// first lines run in the slots the column pass's early finishers leave (2047
// lines on 592 slots: the last round is half empty), and on small levels the
// two grids run side by side.  What it reads before that wait (x, coefficient
// streams, through L2) was written by kernels BEFORE the column pass; the
// column pass therefore lets its dependents launch only after its own wait,
// i.e. once everything before it is complete and flushed.  Returns whether
// the caller still owes the wait.  (Doing the kernel's memory-free setup --
// mbarriers, tensor-memory allocation -- before the wait measured slower:
// 88.2 -> 83.0 steps/s.)
__device__ __forceinline__ bool pass_enter(const YPass&) {
  pdl_wait();
  pdl_launch_dependents();
  return false;
}
__device__ __forceinline__ bool pass_enter(const XPass& p) {
  pdl_launch_dependents();
  if (p.late_wait) return true;
  pdl_wait();
  return false;
}
// Spectral constants of one k from the compact table (operator.cu): a_k at
// index k (k < M), b_c at M + c for c <= M/2; b_k = b_k (k <= M/2) or
// -conj(b_{M-k}).  48 KB per block at M = 2048: together with the stage
// twiddles it stays resident in the L1 the line kernels leave (64 KB).
template <int M>
__device__ __forceinline__ void ld_ab(const double2* ab, int k, double2& a, double2& b) {
#ifdef FDE_EXP_NOSPEC
  a = make_double2(1.0 + k, 0.5);  // timing experiment: no constant loads (wrong results)
  b = make_double2(0.25, 2.0 - k);
  return;
#endif
#ifdef FDE_EXP_ABSMALL
  k &= 255;  // timing experiment: an always-L1-resident slice of the table (wrong results)
#endif
  asm("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(a.x), "=d"(a.y) : "l"(ab + k));
  const bool flip = k > M / 2;
  const double2* pb = ab + M + (flip ? M - k : k);
  double br, bi;
  asm("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(br), "=d"(bi) : "l"(pb));
  b = make_double2(flip ? -br : br, bi);
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
  (void)M;
  if constexpr (NS > 1) {  // compact table: exp(-2 pi i j / (NS R)) at NS R / 2 + j
#pragma unroll
    for (int q = 0; q < B; ++q) pre[q] = twM[NS * R / 2 + ((tl + q * T) & (NS - 1))];  // plain: stays after the barrier
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
// resident CTAs the plain FFT kernels are compiled for: 4 (128 registers)
// lets a 511- / 255-line level sit in one wave (V-cycle cfg4 627.5 -> 622.6 us)
#ifndef FDE_MINB_9
#define FDE_MINB_9 4
#endif
#ifndef FDE_MINB_SMALL
#define FDE_MINB_SMALL 4
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
                                             : (LOGM == 9 ? FDE_MINB_9 : (LOGM >= 10 ? FDE_MINB_BIG : FDE_MINB_SMALL));
};

// One CTA convolves LPB lines of length n <= M with T_b and T_b^T.
template <int LOGM, class Pol>
__global__ void __launch_bounds__(FftShape<LOGM>::THREADS, FftShape<LOGM>::MINB)
    fft_line_kernel(const Pol p) {
  const bool late_wait = pass_enter(p);
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
    v[s].x = (active && i0 < n) ? p.load(line, i0) : 0.0;  // (row pass: through L2, see pass_enter)
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
    ld_ab<M>(p.blk.ab, k, ca, cb);
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
  if (late_wait) pdl_wait();
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
#ifndef FDE_BAR_IMM
#define FDE_BAR_IMM 0
#endif
#ifndef FDE_CTA_THREADS
#define FDE_CTA_THREADS 128  // measured: 128-thread CTAs 140 us per n = 2047 apply, 256: 171, 512: 177
#endif
// Barrier over one line group of NT threads inside the 512-thread CTA of the
// paired kernel (named barrier 1 + group index; barrier 0 is the whole CTA).
template <int NT>
__device__ __forceinline__ void group_bar() {
#ifdef FDE_EXP_NOBAR
  return;  // timing experiment (wrong results)
#endif
  if constexpr (NT >= FDE_CTA_THREADS) {
    __syncthreads();
  } else {
#if FDE_BAR_IMM
    // immediate barrier ids (a register id costs an R2UR per barrier)
    switch ((int)threadIdx.x / NT) {
      case 0: asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); break;
      case 1: asm volatile("bar.sync 2, %0;" ::"n"(NT) : "memory"); break;
      case 2: asm volatile("bar.sync 3, %0;" ::"n"(NT) : "memory"); break;
      default: asm volatile("bar.sync 4, %0;" ::"n"(NT) : "memory"); break;
    }
#else
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)threadIdx.x / NT), "n"(NT) : "memory");
#endif
  }
}

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
  static constexpr int BUF = M;          // doubles per landing plane (input line / coefficient line)
  static constexpr int SLOTS = M + (M >> 3);  // padded 16-byte exchange slots (pslot, K >= 3)
  // alternating exchange buffers need an even exchange count per transform
  // (both inverses start on buffer 0 with no barrier in between)
  // per line: the exchange buffer (it also stages the line's input and the
  // epilogue coefficient streams); after the lines a control block with two
  // mbarriers per line slot and the TMEM base address
  // per line: the padded exchange slots; their first 2 BUF doubles double as
  // the two coefficient planes of the epilogue
  static constexpr size_t LINE_DOUBLES = size_t(2) * SLOTS;
  // One CTA of 512 threads per SM holds NG independent line groups (each the
  // THREADS threads of LPC lockstep lines, synchronised by its own named
  // barrier): 4 x 32 KB of exchange buffers plus one small control block fit
  // the 132 KB shared-memory configuration, which leaves ~90 KB of L1
  // (measured, tools/l1_probe.cu) -- separate 128-thread CTAs would each pay
  // the control block and land in the 164 KB configuration (~56 KB of L1).
  static constexpr int CTA_THREADS = FDE_CTA_THREADS > THREADS ? FDE_CTA_THREADS : THREADS;
  static constexpr size_t CTRL_BYTES = 128;
  static constexpr int TCOLS = 8 * P;    // Qy (4P words) + Qt (4P words) per thread
  // TMEM has 128 lanes: a CTA of several 128-thread warpgroups (one long
  // line, M = 8192) gives each warpgroup its own TCOLS-column range
  static constexpr int WG = THREADS / 128;
  static constexpr int NG = CTA_THREADS / THREADS;  // line groups per CTA
  static constexpr int TCOLS_CTA = TCOLS * WG * NG;
  static constexpr size_t SMEM = size_t(NG) * LPC * LINE_DOUBLES * sizeof(double) + CTRL_BYTES;
  static_assert(REM != 0 && LOGM >= 2 * LP, "paired kernel needs a short stage");
  static_assert(T % 32 == 0 && THREADS % 128 == 0 && (LPC == 1 || THREADS == 128),
                "whole warpgroups, one lane quadrant per warp");
  static_assert(TCOLS_CTA <= 512 && (TCOLS_CTA & (TCOLS_CTA - 1)) == 0, "TMEM allocation");
};

#ifndef FDE_P8_Y10
#define FDE_P8_Y10 0  // every column pass at M = 1024 with 8 points/thread (one line per CTA): cfg4 +0.5 %, but the n = 1023 apply 42 -> 48 us (1023 CTAs: two waves)
#endif
#ifndef FDE_P8_Y10_WAVE
#define FDE_P8_Y10_WAVE 1  // ... only when its lines fit one wave of resident CTAs (cfg4's 511-column levels): V-cycle 621.0 -> 616.4 us
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
#ifdef FDE_EXP_NOTW
  return;  // timing experiment (wrong results)
#endif
  if constexpr (NS > 1) {  // compact table: exp(-2 pi i j / (NS R)) at NS R / 2 + j
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int j = PAIRED ? paired_bfly<B, T>(tl, q) : tl + q * T;
      w1s[q] = twM[NS * R / 2 + (j & (NS - 1))];
    }
  }
}

// Exchange buffer of the paired kernel: one 16-byte slot per complex value,
// padded: slot(p) = p + (p >> K).  Each exchange picks K from its write
// pattern (write_pad) so that every 128-bit access of a quarter warp hits
// eight distinct 16-byte bank groups, on the write and on the read side
// (tools/bank_sim.py enumerates all of them).  Every butterfly's R accesses
// are base + compile-time offsets: slot(p0 + r S) - slot(p0) does not depend
// on the thread (checked by the same tool), so an exchange costs one address
// per butterfly and no index arithmetic per access -- the XOR swizzle this
// replaces spent ~2.5 integer instructions per access, a fifth of all issued
// instructions.
template <int K>
__host__ __device__ constexpr int pslot(int p) { return K ? p + (p >> K) : p; }
template <int NSL, int R>
constexpr int write_pad() {
  return NSL >= 3 ? 0 : (Log2<R>::v > 3 ? Log2<R>::v : 3);
}

// Stockham write of a finished stage (NSL, R)
template <int LOGM, int P, int NSL, int R, bool PAIRED, int K>
__device__ __forceinline__ void pstage_write(const double2 (&v)[P], double2* buf, int tl) {
#ifdef FDE_EXP_NOXCHG
  return;
#endif
  constexpr int T = (1 << LOGM) / P, B = P / R, NS = 1 << NSL;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int j = PAIRED ? paired_bfly<B, T>(tl, q) : tl + q * T;
    const int base = ((j >> NSL) << (NSL + Log2<R>::v)) + (j & (NS - 1));
    double2* const b = buf + pslot<K>(base);
#pragma unroll
    for (int r = 0; r < R; ++r) b[pslot<K>(r * NS)] = v[q + r * B];
  }
}

// inputs of stage (R, PAIRED): butterfly j reads j + r * M / R
template <int LOGM, int P, int R, bool PAIRED, int K>
__device__ __forceinline__ void pstage_read(double2 (&v)[P], const double2* buf, int tl) {
#ifdef FDE_EXP_NOXCHG
  return;
#endif
  constexpr int M = 1 << LOGM, T = M / P, B = P / R;
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int j = PAIRED ? paired_bfly<B, T>(tl, q) : tl + q * T;
    const double2* const b = buf + pslot<K>(j);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q + r * B] = b[pslot<K>(r * (M / R))];
  }
}

#ifndef FDE_PRUNE_LAST
#define FDE_PRUNE_LAST 1
#endif
// Forward transform, radix-P stages from NSL, ending with the paired R0 stage.
// On entry the stage at NSL has its inputs in v.  One exchange buffer: a
// barrier before the writes (everyone has read the previous contents) and one
// before the reads.
template <int LOGM, int P, int NSL, bool HALF>
struct PFwd {
  // pre(): called once the paired stage's inputs are in registers (the
  // spectral step follows that stage's butterflies)
  template <class Pre>
  __device__ __forceinline__ static void run(double2 (&v)[P], double2* buf, int tl,
                                             const double2* twM, double2 (&w1s)[P],
                                             const Pre& pre) {
    using S = PairedShape<LOGM, P>;
    constexpr int R = S::template fwd_radix<NSL>();  // P, or P/2 for the split stage
    static_assert(LOGM - NSL >= Log2<R>::v, "");
    pstage_compute<LOGM, P, false, NSL, R, false, HALF>(v, tl, w1s);
    group_bar<S::THREADS>();
    constexpr int NX = NSL + Log2<R>::v;
    constexpr bool LASTP = (LOGM - NX) == S::REM;  // next stage is the paired R0 stage
    constexpr int K = write_pad<NSL, R>();
    pstage_write<LOGM, P, NSL, R, false, K>(v, buf, tl);
    if constexpr (LASTP) {
      pstage_twiddles<LOGM, P, NX, S::R0, true>(w1s, tl, twM);
      group_bar<S::THREADS>();
      pstage_read<LOGM, P, S::R0, true, K>(v, buf, tl);
      pre();
      pstage_compute<LOGM, P, false, NX, S::R0, true, false>(v, tl, w1s);
    } else {
      constexpr int RN = S::template fwd_radix<NX>();
      pstage_twiddles<LOGM, P, NX, RN, false>(w1s, tl, twM);
      group_bar<S::THREADS>();
      pstage_read<LOGM, P, RN, false, K>(v, buf, tl);
      PFwd<LOGM, P, NX, false>::run(v, buf, tl, twM, w1s, pre);
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
  __device__ __forceinline__ static void run(double2 (&v)[P], double2* buf, int tl,
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
      constexpr int K = write_pad<NSL, R>();
      group_bar<S::THREADS>();
      pstage_write<LOGM, P, NSL, R, false, K>(v, buf, tl);
      pstage_twiddles<LOGM, P, NX, RN, false>(w1s, tl, twM);
      group_bar<S::THREADS>();
      pstage_read<LOGM, P, RN, false, K>(v, buf, tl);
      if constexpr (NX + Log2<RN>::v >= LOGM) hook();  // the next stage is the last
      PInvTail<LOGM, P, NX>::run(v, buf, tl, twM, w1s, hook);
    }
  }
};

// Full inverse: paired R0 stage (NS = 1) on the spectral slots, then the tail.
template <int LOGM, int P, class Hook>
__device__ __forceinline__ void pinverse(double2 (&v)[P], double2* buf, int tl,
                                         const double2* twM, double2 (&w1s)[P],
                                         const Hook& hook) {
  using S = PairedShape<LOGM, P>;
  constexpr int RN = S::template inv_radix<S::REM>();
  constexpr int K = write_pad<0, S::R0>();
  pstage_compute<LOGM, P, true, 0, S::R0, true, false>(v, tl, w1s);
  group_bar<S::THREADS>();
  pstage_write<LOGM, P, 0, S::R0, true, K>(v, buf, tl);
  pstage_twiddles<LOGM, P, S::REM, RN, false>(w1s, tl, twM);
  group_bar<S::THREADS>();
  pstage_read<LOGM, P, RN, false, K>(v, buf, tl);
  if constexpr (S::REM + Log2<RN>::v >= LOGM) hook();  // the tail is one stage
  PInvTail<LOGM, P, S::REM>::run(v, buf, tl, twM, w1s, hook);
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

// ---------------------------------------------------------------------------
// Line I/O of the paired kernel.
//
// Every stream of a pass (input line, coefficient lines, Q, b, dinv, output)
// has the same line offset line * n, and the host checks that all base
// addresses agree modulo 16 bytes, so one parity sx = (par + line * n) & 1
// says whether a line starts 8 bytes past a 16-byte boundary.  Such a line is
// processed as the VIRTUAL line (0, x_0, ..., x_{n-1}) of length nv = n + 1:
// a Toeplitz product is shift invariant, so output element e sits at virtual
// position e + sx, and every 16-byte pair (2m, 2m+1) of virtual positions is
// aligned in all streams -- bulk copies, 128-bit loads and 128-bit stores
// apply to odd lines too (n + 1 <= M is checked by the host).
// Pointers below address virtual position 0 (= element -sx).
#ifndef FDE_EPI_G_Y
#define FDE_EPI_G_Y 4  // 8 (every em pair of the line in flight at once): measured no change
#endif
#ifndef FDE_L2_STREAM
#define FDE_L2_STREAM 1  // evict_first hints on the coefficient streams
#endif
template <bool STREAM = false>
__device__ __forceinline__ double2 ld_pair(const double* v0, int pv, int sx, int nv) {
#ifdef FDE_EXP_NOEPILD
  return make_double2(1.0 + pv, 2.0 - sx);  // timing experiment: no epilogue operand loads
#endif
  const double* a = v0 + pv;
  if (pv >= sx && pv + 1 < nv) {
    if constexpr (STREAM && FDE_L2_STREAM) return ldcg_stream(reinterpret_cast<const double2*>(a));
    else return __ldcg(reinterpret_cast<const double2*>(a));
  }
  double2 r = make_double2(0.0, 0.0);  // edge pairs: element by element
  if (pv >= sx && pv < nv) r.x = __ldcg(a);
  if (pv + 1 < nv) r.y = __ldcg(a + 1);
  return r;
}
__device__ __forceinline__ void st_pair(double* v0, int pv, int sx, int nv, bool live, double2 r) {
#ifdef FDE_EXP_NOEPIST
  if (r.x != 1.2345) return;  // timing experiment: (practically) no stores
#endif
  double* a = v0 + pv;
  if (!live) return;
  if (pv >= sx && pv + 1 < nv) {
    *reinterpret_cast<double2*>(a) = r;
  } else {
    if (pv >= sx && pv < nv) a[0] = r.x;
    if (pv + 1 < nv) a[1] = r.y;
  }
}

template <class Pol, int EPI>
struct LineIO;

// YPass: EPI bit 1 = qT (Q written transposed, i.e. contiguous along the line).
// Stream 0 (ep) is staged through plane 0 of the exchange buffer, stream 1
// (em) is loaded in 16-byte pairs with the group's other global operands
// (plane 1 receives the next line's input meanwhile).
template <int EPI>
struct LineIO<YPass, EPI> {
  static constexpr bool QT = (EPI >> 1) & 1;
  static constexpr int G = FDE_EPI_G_Y;  // slots per epilogue group 
  const double* x;
  const double* ep;
  const double* em;
  double* q;
  size_t n1;
  double c;
  int sx, nv;
  uint64_t pol;  // L2 evict_last policy for the Q stores (0: plain stores)
  __device__ __forceinline__ LineIO(const YPass& p, int line, int sx_) {
    pol = p.keep_q ? l2_policy_evict_last() : 0;
    const ptrdiff_t o = (ptrdiff_t)line * p.n2 - sx_;
    sx = sx_;
    nv = p.n2 + sx_;
    n1 = (size_t)p.n1;
    x = p.x + o;
    ep = p.epT + o;
    em = p.emT + o;
    q = QT ? p.q + o : p.q + line - (ptrdiff_t)sx_ * p.n1;
    c = p.c;
  }
  __device__ __forceinline__ const double* input() const { return x; }
  __device__ __forceinline__ const double* staged(int k) const { return k ? em : ep; }
  struct Glob {
    double2 s1;
  };
  __device__ __forceinline__ Glob fetch_glob(int pv) const {
    return Glob{ld_pair<true>(em, pv, sx, nv)};
  }
  __device__ __forceinline__ void prefetch_rest(uint32_t) const {}
  __device__ __forceinline__ void finish(int pv, bool live, double2 ty, double2 tt, double2 s0,
                                         const Glob& g) const {
    const double2 s1 = g.s1;
    const double2 v = make_double2(c * (s0.x * ty.x + s1.x * tt.x), c * (s0.y * ty.y + s1.y * tt.y));
#ifdef FDE_EXP_NOEPIST
    if (v.x != 1.2345) return;
#endif
    if (QT) {
      st_pair(q, pv, sx, nv, live, v);
    } else if (live) {
      if (pol) {
        if (pv >= sx && pv < nv) st_l2_hint(q + (size_t)pv * n1, v.x, pol);
        if (pv + 1 < nv) st_l2_hint(q + (size_t)(pv + 1) * n1, v.y, pol);
      } else {
        if (pv >= sx && pv < nv) q[(size_t)pv * n1] = v.x;
        if (pv + 1 < nv) q[(size_t)(pv + 1) * n1] = v.y;
      }
    }
  }
};

// XPass: dp is staged through plane 0 of the exchange buffer; dm, the line's
// own input (again, for inv_r x), Q, b, dinv / src are loaded in 16-byte
// pairs, a group of slots at a time.
template <int EPI>
struct LineIO<XPass, EPI> {
  static constexpr int G = EPI == EPI_STORE ? 4 : 2;
  const double* x;
  const double* dp;
  const double* dm;
  const double* q;
  const double* e1;  // src (RHS) or b (RESID / JACOBI)
  const double* e2;  // dinv (JACOBI)
  double* out;
  double inv_r, sign, s2;  // s2: src_scale (RHS) or omega (JACOBI)
  int sx, nv;
  __device__ __forceinline__ LineIO(const XPass& p, int line, int sx_) {
    const ptrdiff_t o = (ptrdiff_t)line * p.n1 - sx_;
    sx = sx_;
    nv = p.n1 + sx_;
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
  __device__ __forceinline__ const double* input() const { return x; }
  __device__ __forceinline__ const double* staged(int k) const { return k ? dm : dp; }
  struct Glob {
    double2 s1, x, q, e1, e2;
  };
  __device__ __forceinline__ Glob fetch_glob(int pv) const {
    Glob g;
    g.s1 = ld_pair<true>(dm, pv, sx, nv);
    g.x = ld_pair<true>(x, pv, sx, nv);  // last read of x by this apply
    g.q = q ? ld_pair(q, pv, sx, nv) : make_double2(0.0, 0.0);
    g.e1 = EPI == EPI_STORE ? make_double2(0.0, 0.0) : ld_pair(e1, pv, sx, nv);
    g.e2 = EPI == EPI_JACOBI ? ld_pair(e2, pv, sx, nv) : make_double2(0.0, 0.0);
    return g;
  }
  // warm L2 with the line's directly loaded operands (Q was just written)
  __device__ __forceinline__ void prefetch_rest(uint32_t bytes) const {
    if constexpr (EPI != EPI_STORE) bulk_prefetch_l2(e1, bytes);
    if constexpr (EPI == EPI_JACOBI) bulk_prefetch_l2(e2, bytes);
  }
  __device__ __forceinline__ double one(double xv, double a, double b, double qv, double f1,
                                        double f2, double ty, double tt) const {
    // structured.cpp:128,134-135,146: y = inv_r x; y += s dp t; y += s dm tt; y += Q
    double y = inv_r * xv;
    y += sign * a * ty;
    y += sign * b * tt;
    if (q) y += qv;
    if constexpr (EPI == EPI_RHS) return y + s2 * f1;
    else if constexpr (EPI == EPI_RESID) return f1 - y;
    else if constexpr (EPI == EPI_JACOBI) return xv + s2 * f2 * (f1 - y);
    else return y;
  }
  __device__ __forceinline__ void finish(int pv, bool live, double2 ty, double2 tt, double2 s0,
                                         const Glob& g) const {
    const double2 s1 = g.s1;
    const double2 v = make_double2(one(g.x.x, s0.x, s1.x, g.q.x, g.e1.x, g.e2.x, ty.x, tt.x),
                                   one(g.x.y, s0.y, s1.y, g.q.y, g.e1.y, g.e2.y, ty.y, tt.y));
    st_pair(out, pv, sx, nv, live, v);
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
#ifndef FDE_SPEC_GROUP
#define FDE_SPEC_GROUP 4  // slots per tensor-memory store in the spectral step
#endif
#ifndef FDE_BULK_PF
#define FDE_BULK_PF 1  // L2 bulk prefetch of the line's operand streams at line start
#endif
template <int LOGM>
constexpr int paired_pts_for(bool ypass) {
  return LOGM == 8 || (LOGM == 10 && (!FDE_P16_M1024 || (ypass && FDE_P8_Y10))) ? 8 : 16;
}
// P8: the 8-point instance of a column pass at M = 1024, chosen at launch
template <int LOGM, class Pol, bool P8 = false>
constexpr int paired_pts() {
  return (P8 && LOGM == 10 && std::is_same<Pol, YPass>::value)
             ? 8
             : paired_pts_for<LOGM>(std::is_same<Pol, YPass>::value);
}

template <int LOGM, class Pol, int EPI, bool P8 = false>
#ifndef FDE_STAGGER_Y_NS
#define FDE_STAGGER_Y_NS 0
#endif
#ifndef FDE_PAIRED_CTAS
#define FDE_PAIRED_CTAS 4  // resident 128-thread CTAs per SM the register budget is cut for
#endif
__global__ void __launch_bounds__(PairedShape<LOGM, paired_pts<LOGM, Pol, P8>()>::CTA_THREADS,
                                  FDE_PAIRED_CTAS * 128 / PairedShape<LOGM, paired_pts<LOGM, Pol, P8>()>::CTA_THREADS)
    fft_line_kernel_paired(const Pol p) {
  const bool late_wait = pass_enter(p);
  constexpr int P = paired_pts<LOGM, Pol, P8>();
  using S = PairedShape<LOGM, P>;
  using IO = LineIO<Pol, EPI>;
  constexpr int T = S::T, H = P / 2, R0 = S::R0, B0 = S::B0, NS0 = S::NS0;
  extern __shared__ __align__(16) double smem_all[];
  // line group grp of the CTA; S::LPC lines per group in lockstep: thread tl
  // of line slot ls.  Groups are the kernel's "virtual CTAs": vb of nvb.
  const int grp = threadIdx.x / S::THREADS, tg = threadIdx.x - grp * S::THREADS;
  const int ls = tg / T, tl = tg - ls * T, warp = threadIdx.x >> 5;
  const int vb = grp * gridDim.x + blockIdx.x, nvb = gridDim.x * S::NG;  // balanced per SM
  // Shared memory per line: the exchange slots only.  During the last
  // inverse stage their first two planes of M doubles receive the first
  // epilogue coefficient stream (plane 0) and the NEXT line's input (plane 1)
  // by bulk copies that one thread issues (no LSU traffic, no registers).
  // Four CTAs stay within the 164 KB shared-memory configuration, which leaves
  // ~56 KB of L1 (tools/l1_probe.cu) for the stage twiddles and the stack;
  // with a third 16 KB plane per CTA (228 KB configuration, no L1 to speak of)
  // the n = 2047 apply measured 144 us against 134.
  double* const smem = smem_all + (grp * S::LPC + ls) * S::LINE_DOUBLES;
  double* const xin = smem + S::BUF;  // plane 1: where a line's input lands
  uint64_t* const bars =
      reinterpret_cast<uint64_t*>(smem_all + S::NG * S::LPC * S::LINE_DOUBLES);
  uint64_t* const bar_x = bars + 2 * (grp * S::LPC + ls);  // input line landed
  uint64_t* const bar_c = bar_x + 1;                       // coefficient stream landed
  uint32_t* const s_tbase = reinterpret_cast<uint32_t*>(bars + 2 * S::NG * S::LPC);
  const int n = p.blk.n, nl = p.nlines();
  constexpr int LPC = S::LPC;
  // line of this slot in the CTA's group starting at `base` (clamped: a slot
  // past the last line recomputes it and stores nothing)
  auto line_of = [&](int base) { return base + ls < nl ? base + ls : nl - 1; };
  auto sx_of = [&](int line) { return (p.par + line * n) & 1; };
  // 16-byte chunks of a line's virtual image; the input of the array's last
  // line must not be read past its end (its odd tail element is loaded by the
  // thread that owns it)
  auto chunks_of = [&](int line, bool exact) {
    const int nv = n + sx_of(line);
    return (uint32_t)((exact && line == nl - 1) ? nv / 2 : (nv + 1) / 2);
  };
  // Persistent groups: lines vb, + nvb, ...; thread 0 of a slot moves a
  // line's input into plane 1 with one bulk copy.
  auto issue_input = [&](int line) {
    const uint32_t bytes = chunks_of(line, true) * 16;
    const double* src = IO(p, line, sx_of(line)).input();
    mbar_expect_tx(bar_x, bytes);
    bulk_g2s(xin, src, bytes, bar_x);
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < 2 * S::NG * LPC; ++i) mbar_init(bars + i, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<S::TCOLS_CTA>(s_tbase);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = *s_tbase;
#if FDE_STAGGER_Y_NS
  // experiment: groups with one line fewer than the longest start late (4 / 8 us: no gain)
  if (std::is_same<Pol, YPass>::value) {
    const int per = nvb * LPC;
    if ((nl - vb * LPC + per - 1) / per < (nl + per - 1) / per) __nanosleep(FDE_STAGGER_Y_NS);
  }
#endif
  if (tl == 0 && vb * LPC < nl) issue_input(line_of(vb * LPC));
  // this warp's lane quadrant, and its warpgroup's column range
  const uint32_t tq = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * S::TCOLS);
  const uint32_t tqy = tq, tqt = tq + 4 * P;                    // Qy, Qt column ranges
  // both mbarriers complete once per line: their phase parity rides in bit 30
  // of the loop counter (one loop-carried register instead of two; a spilled
  // parity word cost an exposed local-memory load before every wait)
  int st = vb * LPC;
#pragma unroll 1
  for (; (st & 0x3fffffff) < nl; st = (st + nvb * LPC) ^ 0x40000000) {
    const int base = st & 0x3fffffff;
    const uint32_t phase = (uint32_t)st >> 30;
    const int line = line_of(base);
    const bool live = base + ls < nl;  // uniform per line slot
    const int next = base + nvb * LPC;
    const int sx = sx_of(line);
    const int nv = n + sx;
    // 1) z_m = x'_2m + i x'_2m+1, m = tl + s*T, from the bulk-copied virtual
    //    line (zero outside [sx, nv))
    mbar_wait(bar_x, phase);
    double2 v[P];
    {
      const IO io(p, line, sx);
      const bool tailfix = line == nl - 1 && (nv & 1);
#pragma unroll
      for (int s = 0; s < H; ++s) {
        const int pv = 2 * (tl + s * T);
        double2 t = *reinterpret_cast<const double2*>(xin + pv);
        if (tailfix && pv == nv - 1) t.x = __ldcg(io.input() + pv);
        v[s] = make_double2(pv >= sx && pv < nv ? t.x : 0.0, pv + 1 < nv ? t.y : 0.0);
        v[s + H] = make_double2(0.0, 0.0);
      }
#if FDE_BULK_PF
      if (tl == 0) {  // this line's operand streams and the next line's input -> L2
        const uint32_t bytes = chunks_of(line, false) * 16;
#if FDE_L2_STREAM
        bulk_prefetch_l2_stream(io.staged(0), bytes);
        bulk_prefetch_l2_stream(io.staged(1), bytes);
#else
        bulk_prefetch_l2(io.staged(0), bytes);
        bulk_prefetch_l2(io.staged(1), bytes);
#endif
        io.prefetch_rest(chunks_of(line, true) * 16);
        if (next < nl) {
          const int ln = line_of(next);
          bulk_prefetch_l2(IO(p, ln, sx_of(ln)).input(), chunks_of(ln, true) * 16);
        }
      }
#endif
    }

    // the transposed-input scratch was read for the last time by this line's
    // bulk copy: drop its L2 lines instead of writing them back
    if constexpr (std::is_same<Pol, YPass>::value) {
      if (p.scratch_x && live && line != nl - 1)
        l2_discard_range(p.x + (size_t)line * p.n2, n, tl, T);
    }

    // 2) forward transform; ends with this thread's paired slots in v
    double2 w1s[P];
    double2* const xbuf = reinterpret_cast<double2*>(smem);  // exchange slots
    PFwd<LOGM, P, 0, true>::run(v, xbuf, tl, p.blk.twM, w1s, [] {});
    // the previous line's Q (row pass): every thread of the group is past its
    // epilogue loads (the forward transform's barriers), so its lines can go
    if constexpr (std::is_same<Pol, XPass>::value) {
      const int pb = base - nvb * LPC;  // the group's previous lines
      if (p.scratch_q && p.q && pb >= vb * LPC && pb + ls < nl)
        l2_discard_range(p.q + (size_t)(pb + ls) * p.n1, n, tl, T);
    }

    // 3) spectral step (see fft_line_kernel): partners are in registers;
    //    results go to tensor memory in groups of 4 slots.  With
    //      P  = ar zr + bi mi,  Q  = br mr - ai zi,
    //      P' = ar zi + bi mr,  Q' = ai zr - br mi      (a = a_k, b = b_k, m = Z[M-k])
    //    Qy = (P + Q, P' + Q') and Qt = (P - Q, P' - Q'): 12 FP64 instructions per k.
    {
      const bool t0 = tl == 0;
      const double2* abv = p.blk.ab;
#pragma unroll
      for (int g = 0; g < P; g += FDE_SPEC_GROUP) {
        double2 qy[FDE_SPEC_GROUP], qt[FDE_SPEC_GROUP];
#pragma unroll
        for (int c = 0; c < FDE_SPEC_GROUP; ++c) {
          const int s = g + c, q = s % B0, r = s / B0;
          const int k = paired_bfly<B0, T>(tl, q) + r * NS0;
          const double2 z = v[s];
          const double2 zm0 = v[partner_slot<B0, R0>(s, true)];
          const double2 zm1 = v[partner_slot<B0, R0>(s, false)];
          const double mr = t0 ? zm0.x : zm1.x, mi = t0 ? zm0.y : zm1.y;
          double2 ca, cb;
          ld_ab<S::M>(abv, k, ca, cb);
          const double pr = ca.x * z.x + cb.y * mi, qr = cb.x * mr - ca.y * z.y;
          const double pi = ca.x * z.y + cb.y * mr, qi = ca.y * z.x - cb.x * mi;
          qy[c] = make_double2(pr + qr, pi + qi);
          qt[c] = make_double2(pr - qr, pi - qi);
        }
#if FDE_SPEC_GROUP == 4
        tmem_st4(tqy + 4 * g, qy);
        tmem_st4(tqt + 4 * g, qt);
#else
        tmem_st2(tqy + 4 * g, qy);
        tmem_st2(tqt + 4 * g, qt);
#endif
      }
    }
    tmem_wait_st();

    // 4) inverse of Qy -> T x (packed; its H output slots are parked in the Qy
    //    columns), then 5) inverse of Qt -> T^T x.  One copy of the inverse
    //    code (instruction-cache footprint).  Once the second inverse's last
    //    stage has its inputs in registers, the exchange buffer receives the
    //    two epilogue coefficient streams (bulk copies), overlapped with that
    //    stage's butterflies.
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
      auto stage_epilogue = [&]() {
        if (it == 0) return;
        group_bar<S::THREADS>();  // every thread has read its last-stage inputs
        if (tl == 0) {
          const uint32_t bytes = chunks_of(line, false) * 16;
          fence_proxy_async();
          mbar_expect_tx(bar_c, bytes);
#if FDE_L2_STREAM
          bulk_g2s_stream(smem, IO(p, line, sx).staged(0), bytes, bar_c);
#else
          bulk_g2s(smem, IO(p, line, sx).staged(0), bytes, bar_c);
#endif
          if (next < nl) issue_input(line_of(next));
        }
      };
      pinverse<LOGM, P>(v, xbuf, tl, p.blk.twM, w1s, stage_epilogue);
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

    // 6) epilogue in groups of IO::G slots (pairs of positions): every global
    //    operand of a group is in flight before any of its stores; the first
    //    group's are issued before the wait for the staged streams.
    {
      const IO io(p, line, sx);
      constexpr int G = IO::G < H ? IO::G : H;
      typename IO::Glob gl[G];
      auto fetch_group = [&](int g) {
#pragma unroll
        for (int c = 0; c < G; ++c) gl[c] = io.fetch_glob(2 * (tl + (g + c) * T));
      };
      if (late_wait) pdl_wait();  // Q (and everything older) is complete and visible
      fetch_group(0);
      mbar_wait(bar_c, phase);
#pragma unroll
      for (int g4 = 0; g4 < H; g4 += 4) {
        double2 ty[4];
        tmem_ld4(tqy + 4 * g4, ty);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int slot = g4 + c4;
          if (slot > 0 && slot % G == 0) fetch_group(slot);
          const int pv = 2 * (tl + slot * T);
          const double2 a = *reinterpret_cast<const double2*>(smem + pv);
          io.finish(pv, live, ty[c4], v[slot], a, gl[slot % G]);
        }
      }
    }
    // the exchange slots are rewritten by the next line's first exchange,
    // after the barrier that follows its input reads
  }
  tmem_fence_before();
  __syncthreads();
  if constexpr (std::is_same<Pol, XPass>::value) {
    const int pb = (st & 0x3fffffff) - nvb * LPC;  // the group's last lines
    if (p.scratch_q && p.q && pb >= vb * LPC && pb + ls < nl)
      l2_discard_range(p.q + (size_t)(pb + ls) * p.n1, n, tl, T);
  }
  if (warp == 0) tmem_dealloc<S::TCOLS_CTA>(tbase);
}

// Warp-per-line direct Toeplitz product for short lines (n <= kDirectMax):
// up to four outputs per lane, x broadcast by shuffles, the block's first
// column / row staged in shared memory.  Exact sums, no FFT latency chain --
// this is what the coarse multigrid levels run.
template <class P>
__global__ void __launch_bounds__(256) direct_line_kernel(const P p) {
  if (pass_enter(p)) pdl_wait();  // (short lines: no late wait)
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
  const uint64_t pol = l2_policy_evict_last();  // the transposed copy is read next, once
  const int i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int i = i0 + tx, j = j0 + ty + k;
    // the row pass reads x again: keep it in L2 over the column pass
    if (i < n1 && j < n2) tile[ty + k][tx] = ld_l2_hint(in + (size_t)j * n1 + i, pol);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int j = j0 + tx, i = i0 + ty + k;
    if (i < n1 && j < n2) st_l2_hint(out + (size_t)i * n2 + j, tile[tx][ty + k], pol);
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
  const uint64_t pol = l2_policy_evict_last();
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
    if (i < n1 && j < n2) st_l2_hint(out + (size_t)i * n2 + j, tile[tx][ty + k], pol);
  }
}

template <class P>
int lines_of(const P& p) {
  return std::is_same<P, YPass>::value ? p.n1 : p.n2;
}

template <int LOGM, class P>
bool launch_fft(const P& p, cudaStream_t s) {
  using S = FftShape<LOGM>;
  // per template instance and device: opt-in shared memory, SM count
  static DeviceCache<int> sm_count;
  const int sms = sm_count.get([](int dev) {
    FDE_CUDA(cudaFuncSetAttribute(fft_line_kernel<LOGM, P>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    int n = 0;
    FDE_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
  });
  // spread small levels over the SMs: fewer lines per CTA until the grid
  // covers two waves (CTAs stay a whole number of warps)
  const int lines = lines_of(p);
  int lpb = S::LPB;
  const int min_lpb = S::T >= 32 ? 1 : 32 / S::T;
  while (lpb > min_lpb && (lines + lpb - 1) / lpb < 2 * sms) lpb /= 2;
  const int grid = (lines + lpb - 1) / lpb;
  const size_t smem = size_t(lpb) * 2 * S::BUF * sizeof(double);
  launch_k(fft_line_kernel<LOGM, P>, grid, S::T * lpb, smem, s, p);
  FDE_LAUNCH_CHECK();
  return true;
}

#ifndef FDE_PAIRED
#define FDE_PAIRED 1
#endif

// Extra shared-memory carveout (percent) on top of what the resident CTAs
// need; 0 leaves the most L1.
#ifndef FDE_PAIRED_CARVEOUT_PAD
#define FDE_PAIRED_CARVEOUT_PAD 0
#endif
// Whether the paired kernel's aligned I/O applies: every line-contiguous
// stream's base address agrees modulo 16 bytes (then par = that parity in
// doubles), and the virtual line of an odd row still fits the zero-padded
// half (n + 1 <= M).  Otherwise the pass runs on fft_line_kernel.
inline int common_parity(std::initializer_list<const void*> ptrs) {
  int par = -1;
  for (const void* q : ptrs) {
    if (!q) continue;
    const uintptr_t a = reinterpret_cast<uintptr_t>(q);
    if (a & 7) return -1;
    const int b = (int)((a >> 3) & 1);
    if (par >= 0 && b != par) return -1;
    par = b;
  }
  return par;
}
inline int paired_parity(const XPass& p) {
  return common_parity({p.x, p.dp, p.dm, p.q, p.out, p.epi == EPI_RHS ? p.src : nullptr,
                        p.epi == EPI_RESID || p.epi == EPI_JACOBI ? p.b : nullptr,
                        p.epi == EPI_JACOBI ? p.dinv : nullptr});
}
inline int paired_parity(const YPass& p) {
  if (!p.xT) return -1;  // the bulk copy needs contiguous lines
  return common_parity({p.x, p.epT, p.emT, p.qT ? p.q : nullptr});
}

template <int LOGM, class P, int EPI, bool P8 = false>
bool launch_paired_epi(const P& p, cudaStream_t s) {
  constexpr int PP = paired_pts<LOGM, P, P8>();
  using S = PairedShape<LOGM, PP>;
  // resident CTAs on the device (persistent grid) and the shared-memory
  // carveout that just holds them: registers, tensor-memory columns and
  // shared memory per SM, whichever binds (the occupancy API does not see
  // the TMEM allocation).  What the carveout leaves of the SM's 256 KB is
  // L1: it keeps the spectral constants (64 KB per block at M = 2048) and
  // the twiddle tables resident across lines.
  static DeviceCache<int> resident;
  const int max_ctas = resident.get([](int dev) {
    int sms = 0, smem_sm = 0, smem_rsv = 0, regs_sm = 0;
    FDE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FDE_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    FDE_CUDA(cudaDeviceGetAttribute(&smem_rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev));
    FDE_CUDA(cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev));
    FDE_CUDA(cudaFuncSetAttribute(fft_line_kernel_paired<LOGM, P, EPI, P8>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    cudaFuncAttributes fa{};
    FDE_CUDA(cudaFuncGetAttributes(&fa, fft_line_kernel_paired<LOGM, P, EPI, P8>));
    const int regs_cta = ((fa.numRegs * 32 + 255) / 256 * 256) * (S::CTA_THREADS / 32);
    const int cta_smem = (int)(S::SMEM + fa.sharedSizeBytes) + smem_rsv;
    int per_sm = regs_sm / regs_cta;
    const int by_smem = smem_sm / cta_smem;
    const int by_tmem = 512 / S::TCOLS_CTA;
    per_sm = per_sm < by_smem ? per_sm : by_smem;
    per_sm = per_sm < by_tmem ? per_sm : by_tmem;
    if (per_sm < 1) per_sm = 1;
    int carve = (per_sm * cta_smem * 100 + smem_sm - 1) / smem_sm + FDE_PAIRED_CARVEOUT_PAD;
    if (carve > 100) carve = 100;
    FDE_CUDA(cudaFuncSetAttribute(fft_line_kernel_paired<LOGM, P, EPI, P8>,
                                  cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    return sms * per_sm;
  });
  const int groups = (lines_of(p) + S::LPC - 1) / S::LPC;
  const int ctas = (groups + S::NG - 1) / S::NG;
  launch_k(fft_line_kernel_paired<LOGM, P, EPI, P8>, ctas < max_ctas ? ctas : max_ctas,
           S::CTA_THREADS, S::SMEM, s, p);
  FDE_LAUNCH_CHECK();
  return true;
}

template <int LOGM, class P>
bool launch_paired(const P& p0, cudaStream_t s) {
  P p = p0;
  p.par = paired_parity(p);
  if (p.par < 0 || p.blk.n + 1 > (1 << LOGM)) return launch_fft<LOGM>(p0, s);
  if constexpr (std::is_same<P, YPass>::value) {
    if constexpr (LOGM == 10 && FDE_P8_Y10_WAVE && paired_pts<LOGM, P>() == 16) {
      // few enough columns for one wave of resident CTAs (4 per SM): one
      // line per CTA with 8 points per thread halves the serial chain
      static DeviceCache<int> wave;
      const int one_wave = wave.get([](int dev) {
        int sms = 0;
        FDE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        return FDE_PAIRED_CTAS * sms;
      });
      if (lines_of(p) <= one_wave) {
        if (p.qT) return launch_paired_epi<LOGM, P, 2, true>(p, s);
        return launch_paired_epi<LOGM, P, 0, true>(p, s);
      }
    }
    if (p.qT) return launch_paired_epi<LOGM, P, 2>(p, s);
    return launch_paired_epi<LOGM, P, 0>(p, s);
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
bool launch_any(const P& p, cudaStream_t s) {
  const int lines = lines_of(p);
  if (lines <= 0) return false;
  switch (p.blk.logM) {
    case 0:
      launch_k(direct_line_kernel<P>, (lines + 7) / 8, 256, 0, s, p);
      FDE_LAUNCH_CHECK();
      return true;
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

bool launch_line_pass(const YPass& p, cudaStream_t s) { return launch_any(p, s); }
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
bool launch_line_pass(const XPass& p, cudaStream_t s) { return launch_any(p, s); }

}  // namespace fde_b200
