// Batched Toeplitz line convolutions for the CN-WSGD operator apply.
//
// Restates StructuredFdeOperator::apply_impl (proj/src/structured.cpp:125-148)
// and ToeplitzBlock::apply_both (structured.cpp:74-89) the B200 way:
//
//  * Every grid line is one independent job: T x and T^T x of a lower
//    Hessenberg Toeplitz block via its length-L = next_pow2(2n-1) circulant
//    embedding.  The reference does 3 complex length-L FFTs per line; here a
//    real line costs 3 complex FFTs of length M = L/2 (real-input packing
//    z_m = x_2m + i x_2m+1 on the way in, the two real outputs T x and T^T x
//    unpacked the same way on the way out), and spectrum(T^T) = conj
//    spectrum(T) (c is real) so only one spectrum is stored, pre-scaled by
//    1/(2L) so the whole pipeline runs unnormalised transforms.
//  * FFTs are Stockham radix-16 stages (plus one radix-8/4/2 stage) with 16
//    points per thread held in registers (8 or 4 on short lines); shared
//    memory is only the exchange buffer between stages.  The two finest
//    line lengths (M >= 1024) run the paired-spectrum kernel: Z[k] and
//    Z[M-k] end in the same thread, the packed spectra are parked in tensor
//    memory (tcgen05.st/ld), lines and coefficient streams arrive by bulk
//    asynchronous copies, one persistent 128-thread CTA per line slot
//    (line_conv.cu).
//  * Two passes per apply: the y-pass (columns; of a transposed copy of x
//    from 512 columns up) runs first and writes Q = sign * s/r * (ep T_b x + em T_b^T x) using pre-transposed
//    ep/em; the x-pass (rows, contiguous) adds inv_r x + sign (dp T_a x +
//    dm T_a^T x) + Q and applies a fused epilogue (plain store, rhs source
//    add, residual b - Ax, damped-Jacobi update) -- all its streams coalesced.
//  * Lines with n <= kDirectMax (32) use a warp-per-line direct product
//    (coarse multigrid levels, semicoarsened n = 1 lines).
#pragma once
#include "common.cuh"
#include "transfer.cuh"

namespace fde_b200 {

constexpr int kDirectMax = 32;  // n <= this: direct Toeplitz product

// One Toeplitz block resident in HBM (built by ToeplitzDev, operator.cu).
struct LineBlockDev {
  int n;                 // line length
  int logM;              // FFT path: M = 2^logM = L/2; 0 -> direct path
  const double2* ab;     // spectral constants, compact: a_k at k (k < M), b_c at M + c (c <= M/2) (operator.cu)
  const double2* twM;    // stage twiddles, compact: exp(-2 pi i j / Q), j < Q/2, at Q/2 + j (Q = 2..M)
  const double* col;     // first column, n entries (direct path)
  const double* row;     // first row, n entries (direct path)
};

__device__ __forceinline__ void l2_prefetch(const double* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Operator input evaluated by the column-transpose pass, so a multigrid
// update folds into the next operator application instead of its own pass:
//   kind 0: a                       (plain)
//   kind 1: (w * d) * a              zero-guess smoothing x = omega dinv b (multigrid.cpp:355-356)
//   kind 2: a + (P c)                prolongation correction x + P xc (multigrid.cpp:377-378)
struct InMap {
  int kind;
  const double* a;
  const double* d;
  double w;
  Xfer t;
  const double* c;
  int ld;  // row length of a / d
  template <int K>
  __device__ __forceinline__ double at(int i, int j) const {
    const size_t p = (size_t)j * ld + i;
    if constexpr (K == 1) return w * d[p] * a[p];
    else if constexpr (K == 2) return a[p] + prolong_point(t, c, 0, i, j);
    else return a[p];
  }
};

enum Epilogue : int {
  EPI_STORE = 0,   // out = A x                       (LinOp::apply)
  EPI_RHS = 1,     // out = A~ x + src_scale * src     (assemble_rhs, problem.cpp:73-89)
  EPI_RESID = 2,   // out = b - A x                    (multigrid.cpp:363-364, krylov.cpp:71-72)
  EPI_JACOBI = 3,  // out = x + omega dinv (b - A x)   (multigrid.cpp:380-382)
};

// Column pass: line = x index i, position = y index j (stride n1).
// Epilogue protocol: fetch(line, pos) issues the plain loads of one output
// position, finish(...) computes and stores it; the kernel fetches a whole
// group of positions before finishing any, so one memory latency covers the
// group (plain loads: ptxas must not hoist them across the stage barriers).
struct YPass {
  static constexpr bool kNeedsX = false;
  struct Ops {
    double ep, em;
  };
  LineBlockDev blk;
  int n1, n2;
  const double* x;    // x transposed when xT is set: xT[i * n2 + j] = x[i + j * n1]
  int xT;
  const double* epT;  // ep transposed: epT[i * n2 + j] = ep[i + j * n1]
  const double* emT;
  double c;           // sign * s_over_r
  double* q;          // Q[i + j * n1], or Q transposed (Q[i * n2 + j]) when qT is set
  int qT;
  int par = 0;        // set by the launcher: common base-address parity (line_conv.cu)
  int scratch_x = 0;  // x is library scratch read once: its L2 lines are discarded after the read
  int keep_q = 0;     // Q is read once by the row pass that follows: stored evict_last
  __device__ __forceinline__ int nlines() const { return n1; }
  __device__ __forceinline__ double load(int line, int pos) const {
    return xT ? x[(size_t)line * n2 + pos] : x[(size_t)pos * n1 + line];
  }
  __device__ __forceinline__ Ops fetch(int line, int pos) const {
    const size_t t = (size_t)line * n2 + pos;
    return Ops{epT[t], emT[t]};
  }
  // warm L2 with this line's epilogue operands (one 128-byte line per call)
  __device__ __forceinline__ void prefetch(int line, int chunk) const {
    const size_t t = (size_t)line * n2 + (size_t)chunk * 16;
    if ((size_t)chunk * 16 < (size_t)n2) {
      l2_prefetch(epT + t);
      l2_prefetch(emT + t);
    }
  }
  __device__ __forceinline__ void finish(int line, int pos, double ty, double tt,
                                         const Ops& o) const {
    const double v = c * (o.ep * ty + o.em * tt);
#ifdef FDE_EXP_QT
    if (true) q[(size_t)line * n2 + pos] = v;
#else
    if (qT) q[(size_t)line * n2 + pos] = v;
#endif
    else q[(size_t)pos * n1 + line] = v;
  }
};

// Row pass: line = y index j, position = x index i (contiguous).  Every
// thread reads exactly the positions it writes, so the in-place Jacobi update
// (out == x) has no cross-thread hazard.
struct XPass {
  static constexpr bool kNeedsX = true;
  struct Ops {
    double x, dp, dm, q, e1, e2;
  };
  LineBlockDev blk;
  int n1, n2;
  const double* x;
  const double* dp;
  const double* dm;
  const double* q;     // y-pass result (nullptr: no y term)
  double inv_r, sign;
  int epi;
  double* out;
  const double* b;     // EPI_RESID / EPI_JACOBI
  const double* dinv;  // EPI_JACOBI
  double omega;
  const double* src;   // EPI_RHS
  double src_scale;
  int par = 0;         // set by the launcher: common base-address parity (line_conv.cu)
  int scratch_q = 0;   // q is library scratch read once: its L2 lines are discarded after the read
  // the launch right before this one was the column pass that writes q (it
  // releases its dependents only after its own wait, line_conv.cu pass_enter):
  // this pass waits for it in its first epilogue
  int late_wait = 0;
  __device__ __forceinline__ int nlines() const { return n2; }
  __device__ __forceinline__ double load(int line, int pos) const {
    // before a late wait: through L2 (this SM's L1 may hold the buffer's older contents)
    return late_wait ? __ldcg(x + (size_t)line * n1 + pos) : x[(size_t)line * n1 + pos];
  }
  __device__ __forceinline__ void prefetch(int line, int chunk) const {
    const size_t p = (size_t)line * n1 + (size_t)chunk * 16;
    if ((size_t)chunk * 16 < (size_t)n1) {
      l2_prefetch(dp + p);
      l2_prefetch(dm + p);
      if (q) l2_prefetch(q + p);
      if (epi == EPI_RHS) l2_prefetch(src + p);
      if (epi == EPI_RESID || epi == EPI_JACOBI) l2_prefetch(b + p);
      if (epi == EPI_JACOBI) l2_prefetch(dinv + p);
    }
  }
  __device__ __forceinline__ Ops fetch(int line, int pos) const {
    const size_t p = (size_t)line * n1 + pos;
    Ops o;
    o.x = x[p];
    o.dp = dp[p];
    o.dm = dm[p];
    o.q = q ? q[p] : 0.0;
    o.e1 = epi == EPI_RHS ? src[p] : (epi == EPI_STORE ? 0.0 : b[p]);
    o.e2 = epi == EPI_JACOBI ? dinv[p] : 0.0;
    return o;
  }
  __device__ __forceinline__ void finish(int line, int pos, double ty, double tt,
                                         const Ops& o) const {
    const size_t p = (size_t)line * n1 + pos;
    // structured.cpp:128,134-135,146: y = inv_r x; y += s dp t; y += s dm tt; y += Q
    double y = inv_r * o.x;
    y += sign * o.dp * ty;
    y += sign * o.dm * tt;
    if (q) y += o.q;
    switch (epi) {
      case EPI_RHS: out[p] = y + src_scale * o.e1; break;
      case EPI_RESID: out[p] = o.e1 - y; break;
      case EPI_JACOBI: out[p] = o.x + omega * o.e2 * (o.e1 - y); break;
      default: out[p] = y; break;
    }
  }
  // direct (short-line) kernel convenience
  __device__ __forceinline__ void store(int line, int pos, double ty, double tt, double) const {
    finish(line, pos, ty, tt, fetch(line, pos));
  }
};

// true: a kernel was launched (every column-pass kernel follows the protocol
// XPass::late_wait needs from the launch before it)
bool launch_line_pass(const YPass& p, cudaStream_t s);
// out[i * n2 + j] = in[i + j * n1] (tiled through shared memory)
void launch_transpose(const double* in, double* out, int n1, int n2, cudaStream_t s);
// out[i * n2 + j] = v(i, j) = m.at(i, j), and xout[i + j * n1] = v(i, j) when
// xout is set (it may alias m.a: each element is read and written by one thread)
void launch_transpose_mapped(const InMap& m, double* xout, double* out, int n1, int n2,
                             cudaStream_t s);
bool launch_line_pass(const XPass& p, cudaStream_t s);

}  // namespace fde_b200
