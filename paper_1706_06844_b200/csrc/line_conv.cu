// Kernels for the batched Toeplitz line convolutions (see line_conv.cuh).
#include "line_conv.cuh"

#include <type_traits>

namespace fde_b200 {
namespace {

__device__ __forceinline__ int pad(int p) { return p + (p >> 5); }

// ---- small DFTs on registers; INV = false uses exp(-2 pi i / R) -----------
template <bool INV>
__device__ __forceinline__ double2 rot90(double2 a) {  // * (-i) forward, * (+i) inverse
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
template <bool INV>
__device__ __forceinline__ double2 rot45(double2 a) {  // * exp(-+ i pi/4)
  constexpr double h = 0.70710678118654752440;
  return INV ? make_double2((a.x - a.y) * h, (a.x + a.y) * h)
             : make_double2((a.x + a.y) * h, (a.y - a.x) * h);
}
template <bool INV>
__device__ __forceinline__ double2 rot135(double2 a) {  // * exp(-+ 3 i pi/4)
  constexpr double h = 0.70710678118654752440;
  return INV ? make_double2((-a.x - a.y) * h, (a.x - a.y) * h)
             : make_double2((a.y - a.x) * h, (-a.x - a.y) * h);
}

template <int R, bool INV>
struct Dft;
template <bool INV>
struct Dft<2, INV> {
  __device__ __forceinline__ static void run(double2 (&u)[2]) {
    const double2 a = u[0], b = u[1];
    u[0] = cadd(a, b);
    u[1] = csub(a, b);
  }
};
template <bool INV>
struct Dft<4, INV> {
  __device__ __forceinline__ static void run(double2 (&u)[4]) {
    const double2 a0 = cadd(u[0], u[2]), a2 = csub(u[0], u[2]);
    const double2 a1 = cadd(u[1], u[3]), a3 = rot90<INV>(csub(u[1], u[3]));
    u[0] = cadd(a0, a1);
    u[2] = csub(a0, a1);
    u[1] = cadd(a2, a3);
    u[3] = csub(a2, a3);
  }
};
template <bool INV>
struct Dft<8, INV> {
  __device__ __forceinline__ static void run(double2 (&u)[8]) {
    const double2 a0 = cadd(u[0], u[4]), a4 = csub(u[0], u[4]);
    const double2 a1 = cadd(u[1], u[5]), a5 = rot45<INV>(csub(u[1], u[5]));
    const double2 a2 = cadd(u[2], u[6]), a6 = rot90<INV>(csub(u[2], u[6]));
    const double2 a3 = cadd(u[3], u[7]), a7 = rot135<INV>(csub(u[3], u[7]));
    const double2 b0 = cadd(a0, a2), b2 = csub(a0, a2);
    const double2 b1 = cadd(a1, a3), b3 = rot90<INV>(csub(a1, a3));
    const double2 b4 = cadd(a4, a6), b6 = csub(a4, a6);
    const double2 b5 = cadd(a5, a7), b7 = rot90<INV>(csub(a5, a7));
    u[0] = cadd(b0, b1);
    u[4] = csub(b0, b1);
    u[2] = cadd(b2, b3);
    u[6] = csub(b2, b3);
    u[1] = cadd(b4, b5);
    u[5] = csub(b4, b5);
    u[3] = cadd(b6, b7);
    u[7] = csub(b6, b7);
  }
};

template <int R>
struct Log2;
template <> struct Log2<2> { static constexpr int v = 1; };
template <> struct Log2<4> { static constexpr int v = 2; };
template <> struct Log2<8> { static constexpr int v = 3; };

// One Stockham stage on NB simultaneous transforms held as v[b][s] =
// a_b[tl + s*T].  Stage s has radix R and NS = 2^NSL (product of previous
// radices).  The last stage (NS * R == M) leaves results in registers at the
// same slots; other stages exchange through shared memory.
template <int LOGM, bool INV, int NB, int NSL, int R, bool LAST>
__device__ __forceinline__ void stage(double2 (&v)[NB][8], double* const (&re)[NB],
                                      double* const (&im)[NB], int tl,
                                      const double2* twM) {
  constexpr int M = 1 << LOGM, T = M / 8, NS = 1 << NSL, B = 8 / R;
  constexpr int TWSH = LOGM - NSL - Log2<R>::v;  // twiddle index = r * jm << TWSH
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int j = tl + q * T;
    const int jm = j & (NS - 1);
    double2 w[R];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        w[r] = twM[(r * jm) << TWSH];  // plain load: not hoisted across barriers
        if (INV) w[r].y = -w[r].y;
      }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      double2 u[R];
#pragma unroll
      for (int r = 0; r < R; ++r) u[r] = v[b][q + r * B];
      if (NS > 1) {
#pragma unroll
        for (int r = 1; r < R; ++r) u[r] = cmul(u[r], w[r]);
      }
      Dft<R, INV>::run(u);
#pragma unroll
      for (int r = 0; r < R; ++r) v[b][q + r * B] = u[r];
    }
  }
  if (LAST) return;
  __syncthreads();  // everyone finished reading the previous stage's buffer
#pragma unroll
  for (int q = 0; q < B; ++q) {
    const int j = tl + q * T;
    const int base = ((j >> NSL) << (NSL + Log2<R>::v)) + (j & (NS - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = pad(base + r * NS);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        re[b][p] = v[b][q + r * B].x;
        im[b][p] = v[b][q + r * B].y;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int p = pad(tl + s * T);
#pragma unroll
    for (int b = 0; b < NB; ++b) v[b][s] = make_double2(re[b][p], im[b][p]);
  }
}

// Full length-M transform: radix-8 stages, then one radix-4/2 stage if needed.
template <int LOGM, bool INV, int NB, int NSL>
struct Fft {
  __device__ __forceinline__ static void run(double2 (&v)[NB][8], double* const (&re)[NB],
                                             double* const (&im)[NB], int tl,
                                             const double2* twM) {
    constexpr int REM = LOGM - NSL;
    if constexpr (REM >= 3) {
      stage<LOGM, INV, NB, NSL, 8, REM == 3>(v, re, im, tl, twM);
      if constexpr (REM > 3) Fft<LOGM, INV, NB, NSL + 3>::run(v, re, im, tl, twM);
    } else if constexpr (REM == 2) {
      stage<LOGM, INV, NB, NSL, 4, true>(v, re, im, tl, twM);
    } else if constexpr (REM == 1) {
      stage<LOGM, INV, NB, NSL, 2, true>(v, re, im, tl, twM);
    }
  }
};

template <int LOGM>
struct FftShape {
  static constexpr int M = 1 << LOGM;
  static constexpr int T = M / 8;                 // threads per line
  static constexpr int LPB = T >= 256 ? 1 : 256 / T;  // lines per CTA
  static constexpr int THREADS = T * LPB;
  static constexpr int MINB = THREADS >= 512 ? 1 : 2;  // <= 128 registers per thread
  static constexpr int MP = M + M / 32;           // padded buffer length (doubles)
  static constexpr size_t SMEM = size_t(LPB) * 4 * MP * sizeof(double);
};

// One CTA convolves LPB lines of length n <= M with T_b and T_b^T.
template <int LOGM, class P>
__global__ void __launch_bounds__(FftShape<LOGM>::THREADS, FftShape<LOGM>::MINB)
    fft_line_kernel(const P p) {
  using S = FftShape<LOGM>;
  constexpr int M = S::M, T = S::T, MP = S::MP;
  extern __shared__ double smem[];
  const int ls = threadIdx.x / T, tl = threadIdx.x - ls * T;
  const int line = blockIdx.x * S::LPB + ls;
  const bool active = line < p.nlines();
  const int n = p.blk.n;
  double* const base = smem + (size_t)ls * 4 * MP;
  double* const ra[1] = {base};
  double* const ia[1] = {base + MP};

  // 1) load the line: z_m = x_2m + i x_2m+1, m = tl + s*T; zero padding
  //    (n <= M so only s < 4 can be nonzero).
  double2 v[1][8];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int i0 = 2 * (tl + s * T);
    v[0][s].x = (active && i0 < n) ? p.load(line, i0) : 0.0;
    v[0][s].y = (active && i0 + 1 < n) ? p.load(line, i0 + 1) : 0.0;
    v[0][s + 4] = make_double2(0.0, 0.0);
  }

  // 2) forward FFT_M; result in smem (natural order)
  Fft<LOGM, false, 1, 0>::run(v, ra, ia, tl, p.blk.twM);
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int pp = pad(tl + s * T);
    ra[0][pp] = v[0][s].x;
    ia[0][pp] = v[0][s].y;
  }
  __syncthreads();

  // 3) unpack the real spectrum X[k], X[M-k]; multiply by S and conj(S);
  //    repack both real outputs for half-length inverse transforms.  The
  //    T x spectrum stays in registers (stage-0 layout), the T^T x one goes
  //    to the second buffer.
  double* const rb[1] = {base + 2 * MP};
  double* const ib[1] = {base + 3 * MP};
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int k = tl + s * T;
    const int km = (M - k) & (M - 1);
    const double2 zk = make_double2(ra[0][pad(k)], ia[0][pad(k)]);
    const double2 zm = make_double2(ra[0][pad(km)], ia[0][pad(km)]);
    const double2 wk = __ldg(&p.blk.twL[k]);
    const double2 pe = cadd(zk, conjg(zm));                    // 2 E[k]
    const double2 po = csub(zk, conjg(zm));                    // 2i O[k]
    const double2 iwpo = cmul(make_double2(-wk.y, wk.x), po);  // i W^k (2i O[k])
    const double2 x2k = csub(pe, iwpo);                        // 2 X[k]
    const double2 x2m = conjg(cadd(pe, iwpo));                 // 2 X[M-k]
    const double2 sk = __ldg(&p.blk.spec[k]);
    const double2 sm = __ldg(&p.blk.spec[M - k]);
    const double2 cw = conjg(wk);
    const double2 yk = cmul(x2k, sk), ym = cmul(x2m, sm);
    const double2 ay = cadd(yk, conjg(ym)), by = cmul(csub(yk, conjg(ym)), cw);
    v[0][s] = make_double2(ay.x - by.y, ay.y + by.x);  // A + i B
    const double2 tk = cmul(x2k, conjg(sk)), tm = cmul(x2m, conjg(sm));
    const double2 at = cadd(tk, conjg(tm)), bt = cmul(csub(tk, conjg(tm)), cw);
    rb[0][pad(k)] = at.x - bt.y;
    ib[0][pad(k)] = at.y + bt.x;
  }

  // 4) unnormalised inverse FFT_M of each packed spectrum -> q = T x (re: even
  //    positions, im: odd); only m < M/2 (s < 4) carries outputs since n <= M.
  Fft<LOGM, true, 1, 0>::run(v, ra, ia, tl, p.blk.twM);
  double2 ty[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) ty[s] = v[0][s];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int pp = pad(tl + s * T);
    v[0][s] = make_double2(rb[0][pp], ib[0][pp]);
  }
  Fft<LOGM, true, 1, 0>::run(v, rb, ib, tl, p.blk.twM);

  // 5) epilogue at the positions the inputs came from (x re-read hits L1/L2)
  if (!active) return;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int i0 = 2 * (tl + s * T);
    if (i0 < n) p.store(line, i0, ty[s].x, v[0][s].x, P::kNeedsX ? p.load(line, i0) : 0.0);
    if (i0 + 1 < n)
      p.store(line, i0 + 1, ty[s].y, v[0][s].y, P::kNeedsX ? p.load(line, i0 + 1) : 0.0);
  }
}

// Warp-per-line direct Toeplitz product for short lines (n <= 32).
template <class P>
__global__ void __launch_bounds__(256) direct_line_kernel(const P p) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = blockIdx.x * 8 + warp;
  if (line >= p.nlines()) return;
  const int n = p.blk.n;
  const double xv = lane < n ? p.load(line, lane) : 0.0;
  double ty = 0.0, tt = 0.0;
  const double* __restrict__ col = p.blk.col;
  const double* __restrict__ row = p.blk.row;
  for (int k = 0; k < n; ++k) {
    const double xk = __shfl_sync(0xffffffffu, xv, k);
    if (lane < n) {
      const double a = lane >= k ? __ldg(&col[lane - k]) : __ldg(&row[k - lane]);  // T(i,k)
      const double b = k >= lane ? __ldg(&col[k - lane]) : __ldg(&row[lane - k]);  // T(k,i)
      ty += a * xk;
      tt += b * xk;
    }
  }
  if (lane < n) p.store(line, lane, ty, tt, xv);
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
  const int lines = std::is_same<P, YPass>::value ? p.n1 : p.n2;
  const int grid = (lines + S::LPB - 1) / S::LPB;
  fft_line_kernel<LOGM, P><<<grid, S::THREADS, S::SMEM, s>>>(p);
  FDE_LAUNCH_CHECK();
}

template <class P>
void launch_any(const P& p, cudaStream_t s) {
  const int lines = std::is_same<P, YPass>::value ? p.n1 : p.n2;
  if (lines <= 0) return;
  switch (p.blk.logM) {
    case 0:
      direct_line_kernel<P><<<(lines + 7) / 8, 256, 0, s>>>(p);
      FDE_LAUNCH_CHECK();
      return;
    case 6: return launch_fft<6>(p, s);
    case 7: return launch_fft<7>(p, s);
    case 8: return launch_fft<8>(p, s);
    case 9: return launch_fft<9>(p, s);
    case 10: return launch_fft<10>(p, s);
    case 11: return launch_fft<11>(p, s);
    case 12: return launch_fft<12>(p, s);
    default: throw InvalidArgument("line length beyond the supported FFT sizes");
  }
}

}  // namespace

void launch_line_pass(const YPass& p, cudaStream_t s) { launch_any(p, s); }
void launch_line_pass(const XPass& p, cudaStream_t s) { launch_any(p, s); }

}  // namespace fde_b200
