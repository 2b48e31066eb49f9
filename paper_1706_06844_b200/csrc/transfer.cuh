// GridTransfer geometry and the pointwise bilinear prolongation
// (multigrid.cpp:17-44,160-182), shared by the transfer kernels and the
// operator passes that fuse "x + P xc" into their loads.
#pragma once

namespace fde_b200 {

// Transfer between an n1 x n2 fine and a k1 x k2 coarse grid; cx/cy select
// the coarsened directions; coarse index j sits at fine 2j+1-par.
struct Xfer {
  int n1, n2, k1, k2, par1, par2, cx, cy;
};

// 1D prolongation in the reference's accumulation order: fine index i gets
// 1.0 * c[j] if it is the coarse point of j, else 0.5*c[left] then 0.5*c[right].
__host__ __device__ __forceinline__ double prow(const double* c, int k, int i, int par) {
  const int t = i - 1 + par;  // = 2j when i is the coarse point of j
  if ((t & 1) == 0) {
    const int j = t >> 1;
    return (j >= 0 && j < k) ? c[j] : 0.0;  // 0 + 1.0*c
  }
  const int jl = (t - 1) >> 1, jr = jl + 1;  // fine i = fc(jl)+1 = fc(jr)-1
  double v = 0.0;
  if (jl >= 0 && jl < k) v += 0.5 * c[jl];
  if (jr >= 0 && jr < k) v += 0.5 * c[jr];
  return v;
}

// (P c)(i, j): prolong_rows into an n1 x k2 temporary, then prolong_cols, the
// way GridTransfer::prolong composes them.  The coarse buffer holds global
// coarse rows from c_lo on (rows of width k1, or n1 when x is not coarsened).
__host__ __device__ __forceinline__ double prolong_point(const Xfer& t, const double* c, int c_lo,
                                                         int i, int j) {
  auto crow = [&](int r, int width) { return c + (size_t)(r - c_lo) * width; };
  if (!t.cx) {  // prolong_cols only: rows of width n1
    const int tt = j - 1 + t.par2;
    if ((tt & 1) == 0) {
      const int jc = tt >> 1;
      return (jc >= 0 && jc < t.k2) ? crow(jc, t.n1)[i] : 0.0;
    }
    const int jl = (tt - 1) >> 1, jr = jl + 1;
    double v = 0.0;
    if (jl >= 0 && jl < t.k2) v += 0.5 * crow(jl, t.n1)[i];
    if (jr >= 0 && jr < t.k2) v += 0.5 * crow(jr, t.n1)[i];
    return v;
  }
  if (!t.cy) return prow(crow(j, t.k1), t.k1, i, t.par1);  // prolong_rows only
  const int tt = j - 1 + t.par2;
  if ((tt & 1) == 0) {
    const int jc = tt >> 1;
    return (jc >= 0 && jc < t.k2) ? prow(crow(jc, t.k1), t.k1, i, t.par1) : 0.0;
  }
  const int jl = (tt - 1) >> 1, jr = jl + 1;
  double v = 0.0;
  if (jl >= 0 && jl < t.k2) v += 0.5 * prow(crow(jl, t.k1), t.k1, i, t.par1);
  if (jr >= 0 && jr < t.k2) v += 0.5 * prow(crow(jr, t.k1), t.k1, i, t.par1);
  return v;
}

}  // namespace fde_b200
