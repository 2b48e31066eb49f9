// Single-CTA coarse tail of the V-cycle (see tail.cuh).
#include "common.cuh"
#include "mg.cuh"
#include "tail.cuh"

namespace fde_b200 {
namespace {

constexpr int kTailThreads = 1024;

__device__ __forceinline__ void l2_prefetch_range(const double* p, int n, int gt, int nt) {
  for (int i = gt * 16; i < n; i += nt * 16)  // one 128-byte line per thread-step
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + i));
}

// sum_k D[i - k] v_k and sum_k D[k - i] v_k over one line (stride sv), with
// D[m + n - 1] = T(i, k) for m = i - k (ToeplitzBlock::entry); four partial
// sums each so the FMA chains overlap
__device__ __forceinline__ void line_sums(const double* D, int n, int i, const double* v, int sv,
                                          double& t, double& tt) {
  double a[4] = {0.0, 0.0, 0.0, 0.0}, b[4] = {0.0, 0.0, 0.0, 0.0};
  const double* dp = D + (n - 1) + i;  // D[i - k + n - 1] = dp[-k]
  const double* dm = D + (n - 1) - i;  // D[k - i + n - 1] = dm[k]
  int k = 0;
  for (; k + 4 <= n; k += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double vk = v[(k + u) * sv];
      a[u] = fma(dp[-(k + u)], vk, a[u]);
      b[u] = fma(dm[k + u], vk, b[u]);
    }
  }
  for (; k < n; ++k) {
    const double vk = v[k * sv];
    a[0] = fma(dp[-k], vk, a[0]);
    b[0] = fma(dm[k], vk, b[0]);
  }
  t = (a[0] + a[1]) + (a[2] + a[3]);
  tt = (b[0] + b[1]) + (b[2] + b[3]);
}

// (A x)_p in the line passes' order: Q = s/r (ep T_b x + em T_b^T x);
// y = inv_r x; y += dp T_a x; y += dm T_a^T x; y += Q (structured.cpp:125-152)
__device__ __forceinline__ double apply_at(const TailLevel& L, const double* tabs, const double* xs,
                                           int p) {
  const int n1 = L.n1, n2 = L.n2;
  const int i = p % n1, j = p / n1;
  double ty, tt, qy, qt;
  line_sums(tabs + L.tabx, n1, i, xs + j * n1, 1, ty, tt);
  line_sums(tabs + L.taby, n2, j, xs + i, n1, qy, qt);
  const size_t pt = (size_t)i * n2 + j;
  const double q = L.sr * (__ldg(L.epT + pt) * qy + __ldg(L.emT + pt) * qt);
  double y = L.inv_r * xs[p];
  y += __ldg(L.dp + p) * ty;
  y += __ldg(L.dm + p) * tt;
  y += q;
  return y;
}

// k_restrict's arithmetic (restrict_full / restrict_transpose, multigrid.cpp:
// 46-71,184-205) at coarse point q of the fine vector fs
__device__ __forceinline__ double restrict_at(const Xfer& t, const double* fs, double sc, int q) {
  const int a = q % t.k1, bb = q / t.k1;
  auto frow = [&](int r) { return fs + (size_t)r * t.n1; };
  auto rrow = [&](const double* f, int fc) {
    double v = f[fc];
    if (fc > 0) v += 0.5 * f[fc - 1];
    if (fc + 1 < t.n1) v += 0.5 * f[fc + 1];
    return sc * v;
  };
  if (!t.cx) {
    const int fb = 2 * bb + 1 - t.par2;
    double v = frow(fb)[a];
    if (fb > 0) v += 0.5 * frow(fb - 1)[a];
    if (fb + 1 < t.n2) v += 0.5 * frow(fb + 1)[a];
    return v * sc;
  }
  if (!t.cy) return rrow(frow(bb), 2 * a + 1 - t.par1);
  const int fa = 2 * a + 1 - t.par1, fb = 2 * bb + 1 - t.par2;
  double v = rrow(frow(fb), fa);
  if (fb > 0) v += 0.5 * rrow(frow(fb - 1), fa);
  if (fb + 1 < t.n2) v += 0.5 * rrow(frow(fb + 1), fa);
  return v * sc;
}

__global__ void __launch_bounds__(kTailThreads) k_vcycle_tail(const TailDesc d) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int last = d.nl - 1;
  const double w = d.omega;

  // Toeplitz diagonals of every tail level and an L2 prefetch of the
  // coefficient fields: constant data, so this overlaps the previous kernel
  for (int l = 0; l < d.nl; ++l) {
    const TailLevel& L = d.lv[l];
    for (int m = tid; m < 2 * L.n1 - 1; m += nt) {
      const int k = m - (L.n1 - 1);
      sm[L.tabx + m] = k >= 0 ? __ldg(L.colx + k) : __ldg(L.rowx - k);
    }
    for (int m = tid; m < 2 * L.n2 - 1; m += nt) {
      const int k = m - (L.n2 - 1);
      sm[L.taby + m] = k >= 0 ? __ldg(L.coly + k) : __ldg(L.rowy - k);
    }
    const int N = L.n1 * L.n2;
    l2_prefetch_range(L.dp, N, tid, nt);
    l2_prefetch_range(L.dm, N, tid, nt);
    l2_prefetch_range(L.epT, N, tid, nt);
    l2_prefetch_range(L.emT, N, tid, nt);
    l2_prefetch_range(L.dinv, N, tid, nt);
  }
  pdl_enter();

  // first level: b, and x = omega dinv b (zero-guess smoothing,
  // multigrid.cpp:355-356) unless the caller's x already holds it
  {
    const TailLevel& L = d.lv[0];
    for (int p = tid; p < L.n1 * L.n2; p += nt) {
      const double bv = __ldcg(d.b + p);
      sm[L.bo + p] = bv;
      sm[L.xo + p] = d.prescaled ? __ldcg(d.x + p) : w * __ldg(L.dinv + p) * bv;
    }
  }
  __syncthreads();

  // down: r = b - A x; b_c = R r, x_c = omega dinv_c b_c (multigrid.cpp:363-372)
  for (int l = 0; l < last; ++l) {
    const TailLevel& L = d.lv[l];
    double* r = sm + d.s0;
    for (int p = tid; p < L.n1 * L.n2; p += nt)
      r[p] = sm[L.bo + p] - apply_at(L, sm, sm + L.xo, p);
    __syncthreads();
    const TailLevel& C = d.lv[l + 1];
    const bool smooth = l + 1 < last || d.coarse == COARSE_SWEEPS;
    for (int q = tid; q < C.n1 * C.n2; q += nt) {
      const double bc = restrict_at(L.t, r, d.rsc, q);
      sm[C.bo + q] = bc;
      sm[C.xo + q] = smooth ? w * __ldg(C.dinv + q) * bc : 0.0;  // COARSE_NONE: x_c = 0
    }
    __syncthreads();
  }
  // coarsest: the remaining damped-Jacobi sweeps (multigrid.cpp:338-349)
  int cur = d.lv[last].xo;
  if (d.coarse == COARSE_SWEEPS) {
    const TailLevel& L = d.lv[last];
    int alt = d.s1;
    for (int k = 1; k < d.sweeps; ++k) {
      for (int p = tid; p < L.n1 * L.n2; p += nt) {
        const double xv = sm[cur + p];
        const double y = apply_at(L, sm, sm + cur, p);
        sm[alt + p] = xv + w * __ldg(L.dinv + p) * (sm[L.bo + p] - y);
      }
      __syncthreads();
      const int t = cur;
      cur = alt;
      alt = t;
    }
  }
  // up: w = x + P x_c, then x = w + omega dinv (b - A w) (multigrid.cpp:376-382)
  for (int l = last - 1; l >= 0; --l) {
    const TailLevel& L = d.lv[l];
    const int N = L.n1 * L.n2;
    double* wv = sm + d.s0;
    for (int q = tid; q < N; q += nt) {
      const int i = q % L.n1, j = q / L.n1;
      wv[q] = sm[L.xo + q] + prolong_point(L.t, sm + cur, 0, i, j);
    }
    __syncthreads();
    for (int p = tid; p < N; p += nt) {
      const double y = apply_at(L, sm, wv, p);
      sm[L.xo + p] = wv[p] + w * __ldg(L.dinv + p) * (sm[L.bo + p] - y);
    }
    __syncthreads();
    cur = L.xo;
  }
  const TailLevel& L0 = d.lv[0];
  for (int p = tid; p < L0.n1 * L0.n2; p += nt) d.x[p] = sm[cur + p];
}

}  // namespace

void launch_vcycle_tail(const TailDesc& d, cudaStream_t s) {
  static DeviceCache<bool> configured;  // per device
  configured.get([](int) {
    FDE_CUDA(cudaFuncSetAttribute(k_vcycle_tail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(kTailSmemMax * sizeof(double))));
    return true;
  });
  launch_k(k_vcycle_tail, 1, kTailThreads, (size_t)d.smem * sizeof(double), s, d);
  FDE_LAUNCH_CHECK();
}

}  // namespace fde_b200
