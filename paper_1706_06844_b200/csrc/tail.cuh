// Coarse tail of the V-cycle in one launch (reference: MgHierarchy::cycle,
// proj/src/multigrid.cpp:318-383, on the levels below ~1K unknowns).
//
// Below ~1K unknowns every level's operator application, transfer and
// smoothing step is a few microseconds of pure latency as its own kernel
// (cfg4 crosses ~16 such launches per V-cycle on its last three levels).  Here
// one CTA walks those levels with every level's iterate, right-hand side and
// Toeplitz diagonals resident in its shared memory: each phase (residual,
// restriction + zero-guess smoothing, coarsest sweeps, prolongation,
// post-smoothing) is separated from the next by a CTA barrier only.  The
// level operators stay diag x Toeplitz; their line products are direct sums
// (as the direct line kernel does for n <= 32).  Every other step follows
// the reference's arithmetic order, so the transfers are bit-identical to
// k_restrict / k_prolong; only the Toeplitz sums round differently from the
// FFT passes.
#pragma once
#include "transfer.cuh"

namespace fde_b200 {

constexpr int kTailMaxLevels = 12;
constexpr int kTailMaxN = 1024;       // unknowns of the tail's first level (measured best)
constexpr int kTailMaxLine = 512;     // line length per direction
constexpr int kTailSmemMax = 24576;   // shared-memory doubles (192 KB)

struct TailLevel {
  int n1, n2;
  double inv_r, sr;                   // inv_r, s_over_r
  const double *colx, *rowx;          // T_alpha first column / row (n1)
  const double *coly, *rowy;          // T_beta first column / row (n2)
  const double *dp, *dm, *epT, *emT;  // epT/emT: transposed (i * n2 + j)
  const double* dinv;
  int xo, bo;      // shared-memory offsets of the level's iterate and right-hand side
  int tabx, taby;  // offsets of the 2 n - 1 entry diagonal tables
  Xfer t;          // transfer to the next level
};

struct TailDesc {
  int nl;         // levels in the tail (>= 1); the last is the coarsest
  int coarse;     // COARSE_SWEEPS or COARSE_NONE
  int sweeps;     // coarsest sweeps
  int prescaled;  // x of the first level already holds omega dinv b
  int s0, s1;     // shared-memory offsets of two scratch vectors (first level's size)
  int smem;       // shared-memory doubles in use
  double omega, rsc;
  const double* b;  // first level: the caller's right-hand side
  double* x;        // first level: the caller's iterate (input if prescaled, output)
  TailLevel lv[kTailMaxLevels];
};

void launch_vcycle_tail(const TailDesc& d, cudaStream_t s);

}  // namespace fde_b200
