#include <algorithm>
#include <cmath>
#include <cstdint>

#include "csr.cuh"

namespace fde_b200 {

Csr Csr::from_triplets(size_t rows, size_t cols, std::vector<Triplet> t) {
  for (const Triplet& e : t)
    if (e.row >= rows || e.col >= cols) throw InvalidArgument("triplet index out of range");
  std::stable_sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  Csr m;
  m.rows = rows;
  m.cols = cols;
  m.ptr.assign(rows + 1, 0);
  m.idx.reserve(t.size());
  m.val.reserve(t.size());
  size_t i = 0;
  for (size_t r = 0; r < rows; ++r) {
    while (i < t.size() && t[i].row == r) {
      double v = t[i].value;
      const uint32_t c = t[i].col;
      ++i;
      while (i < t.size() && t[i].row == r && t[i].col == c) v += t[i++].value;  // duplicates
      m.idx.push_back(c);
      m.val.push_back(v);
    }
    m.ptr[r + 1] = (uint32_t)m.idx.size();
  }
  return m;
}

Csr Csr::transpose() const {
  Csr t;
  t.rows = cols;
  t.cols = rows;
  t.ptr.assign(cols + 1, 0);
  for (uint32_t c : idx) ++t.ptr[c + 1];
  for (size_t c = 0; c < cols; ++c) t.ptr[c + 1] += t.ptr[c];
  t.idx.resize(nnz());
  t.val.resize(nnz());
  std::vector<uint32_t> next(t.ptr.begin(), t.ptr.end() - 1);
  for (size_t r = 0; r < rows; ++r)
    for (uint32_t k = ptr[r]; k < ptr[r + 1]; ++k) {
      const uint32_t pos = next[idx[k]]++;
      t.idx[pos] = (uint32_t)r;
      t.val[pos] = val[k];
    }
  return t;
}

Csr Csr::multiply(const Csr& o) const {
  if (cols != o.rows) throw InvalidArgument("csr multiply shape mismatch");
  Csr out;
  out.rows = rows;
  out.cols = o.cols;
  out.ptr.assign(rows + 1, 0);
  std::vector<double> acc(o.cols, 0.0);
  std::vector<uint32_t> mark(o.cols, UINT32_MAX), live;
  for (size_t r = 0; r < rows; ++r) {
    live.clear();
    for (uint32_t k = ptr[r]; k < ptr[r + 1]; ++k) {
      const uint32_t mid = idx[k];
      const double va = val[k];
      for (uint32_t l = o.ptr[mid]; l < o.ptr[mid + 1]; ++l) {
        const uint32_t c = o.idx[l];
        if (mark[c] != r) {
          mark[c] = (uint32_t)r;
          acc[c] = va * o.val[l];
          live.push_back(c);
        } else {
          acc[c] += va * o.val[l];
        }
      }
    }
    std::sort(live.begin(), live.end());
    for (uint32_t c : live) {
      out.idx.push_back(c);
      out.val.push_back(acc[c]);
    }
    out.ptr[r + 1] = (uint32_t)out.idx.size();
  }
  return out;
}

std::vector<double> Csr::diag() const {
  if (rows != cols) throw InvalidArgument("diag of non-square csr");
  std::vector<double> d(rows, 0.0);
  for (size_t r = 0; r < rows; ++r)
    for (uint32_t k = ptr[r]; k < ptr[r + 1]; ++k) {
      if (idx[k] == r) {
        d[r] = val[k];
        break;
      }
      if (idx[k] > r) break;
    }
  return d;
}

Csr rap(const Csr& p, const Csr& a) {
  if (a.rows != a.cols || a.rows != p.rows) throw InvalidArgument("rap shape mismatch");
  return p.transpose().multiply(a.multiply(p));
}

Csr structured_to_csr(const StructuredOp& op) {
  const size_t n1 = op.n1(), n2 = op.n2(), n = n1 * n2;
  std::vector<Csr::Triplet> t;
  t.reserve(n * (n1 + n2 + 1));
  const auto& ax = op.block_x();
  const auto& ay = op.block_y();
  for (size_t j = 0; j < n2; ++j)
    for (size_t i = 0; i < n1; ++i) {
      const uint32_t p = (uint32_t)(i + j * n1);
      t.push_back({p, p, op.inv_r()});
      for (size_t ii = 0; ii < n1; ++ii) {
        const double v = op.dp()[p] * ax.entry(i, ii) + op.dm()[p] * ax.entry(ii, i);
        if (v != 0.0) t.push_back({p, (uint32_t)(ii + j * n1), v});
      }
      for (size_t jj = 0; jj < n2; ++jj) {
        const double v = op.s_over_r() * (op.ep()[p] * ay.entry(j, jj) + op.em()[p] * ay.entry(jj, j));
        if (v != 0.0) t.push_back({p, (uint32_t)(i + jj * n1), v});
      }
    }
  return Csr::from_triplets(n, n, std::move(t));
}

Csr prolong_matrix(const Xfer& x) {
  std::vector<Csr::Triplet> t;
  t.reserve(9 * (size_t)x.k1 * x.k2);
  const double wt[3] = {0.5, 1.0, 0.5};
  const int ri = x.cx ? 1 : 0, rj = x.cy ? 1 : 0;
  for (int b = 0; b < x.k2; ++b) {
    const int fb = x.cy ? 2 * b + 1 - x.par2 : b;
    for (int a = 0; a < x.k1; ++a) {
      const int fa = x.cx ? 2 * a + 1 - x.par1 : a;
      const uint32_t col = (uint32_t)(a + b * x.k1);
      for (int dj = -rj; dj <= rj; ++dj) {
        const int j = fb + dj;
        if (j < 0 || j >= x.n2) continue;
        for (int di = -ri; di <= ri; ++di) {
          const int i = fa + di;
          if (i < 0 || i >= x.n1) continue;
          t.push_back({(uint32_t)(i + j * x.n1), col, wt[di + 1] * wt[dj + 1]});
        }
      }
    }
  }
  return Csr::from_triplets((size_t)x.n1 * x.n2, (size_t)x.k1 * x.k2, std::move(t));
}

namespace {

// one warp per row; epilogues as the line passes (multigrid.cpp:358-364)
__global__ void k_csr(size_t rows, const uint32_t* __restrict__ ptr,
                      const uint32_t* __restrict__ idx, const double* __restrict__ val,
                      const double* __restrict__ x, double* __restrict__ out, int epi,
                      const double* __restrict__ b, const double* __restrict__ dinv,
                      double omega) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const size_t warps = (size_t)gridDim.x * (blockDim.x / 32);
  for (size_t r = blockIdx.x * (size_t)(blockDim.x / 32) + (threadIdx.x >> 5); r < rows;
       r += warps) {
    double s = 0.0;
    for (uint32_t k = ptr[r] + lane; k < ptr[r + 1]; k += 32) s = fma(val[k], x[idx[k]], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (epi == EPI_RESID) out[r] = b[r] - s;
      else if (epi == EPI_JACOBI) out[r] = x[r] + omega * dinv[r] * (b[r] - s);
      else out[r] = s;
    }
  }
}

// band row k: entries for columns k - bw .. k + bw at k * (2 bw + 1) + (c - k + bw).
// One warp; lane l owns band offsets d = l + 1 + 32 e (e < E).  The band
// entries of the next step are loaded while the current one updates y, so
// the substitution's serial chain does not wait on memory.
constexpr int kBandE = 8;  // bw <= 256
__global__ void k_band_solve(size_t n, int bw, const double* __restrict__ band,
                             const double* __restrict__ r, double* __restrict__ z) {
  pdl_enter();
  extern __shared__ double y[];
  const int lane = threadIdx.x;
  const size_t ld = 2 * (size_t)bw + 1;
  for (size_t i = lane; i < n; i += 32) y[i] = r[i];
  __syncwarp();
  // L y = r (unit lower): y_{k+d} -= l_{k+d,k} y_k
  auto lower = [&](size_t k, double (&v)[kBandE]) {
#pragma unroll
    for (int e = 0; e < kBandE; ++e) {
      const int d = lane + 1 + 32 * e;
      v[e] = (d <= bw && k + d < n) ? band[(k + d) * ld + (size_t)(bw - d)] : 0.0;
    }
  };
  double cur[kBandE], nxt[kBandE];
  lower(0, cur);
  for (size_t k = 0; k < n; ++k) {
    if (k + 1 < n) lower(k + 1, nxt);
    const double yk = y[k];
#pragma unroll
    for (int e = 0; e < kBandE; ++e) {
      const int d = lane + 1 + 32 * e;
      if (d <= bw && k + d < n) y[k + d] -= cur[e] * yk;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < kBandE; ++e) cur[e] = nxt[e];
  }
  // U z = y: z_k = y_k / u_kk, then y_{k-d} -= u_{k-d,k} z_k
  auto upper = [&](size_t k, double (&v)[kBandE], double& diag) {
#pragma unroll
    for (int e = 0; e < kBandE; ++e) {
      const int d = lane + 1 + 32 * e;
      v[e] = (d <= bw && (size_t)d <= k) ? band[(k - d) * ld + (size_t)(bw + d)] : 0.0;
    }
    diag = band[k * ld + bw];
  };
  double dcur = 0.0, dnxt = 0.0;
  upper(n - 1, cur, dcur);
  for (size_t k = n; k-- > 0;) {
    if (k > 0) upper(k - 1, nxt, dnxt);
    const double zk = y[k] / dcur;
    __syncwarp();
    if (lane == 0) y[k] = zk;
#pragma unroll
    for (int e = 0; e < kBandE; ++e) {
      const int d = lane + 1 + 32 * e;
      if (d <= bw && (size_t)d <= k) y[k - d] -= cur[e] * zk;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < kBandE; ++e) cur[e] = nxt[e];
    dcur = dnxt;
  }
  for (size_t i = lane; i < n; i += 32) z[i] = y[i];
}

}  // namespace

CsrOp::CsrOp(Csr m) : m_(std::move(m)), diag_(m_.diag()) {
  if (m_.rows != m_.cols) throw InvalidArgument("CsrOp needs a square matrix");
  d_ptr_.upload(m_.ptr.data(), m_.ptr.size());
  d_idx_.upload(m_.idx.data(), m_.idx.size());
  d_val_.upload(m_.val.data(), m_.val.size());
}

void CsrOp::run(const double* x, double* out, int epi, const EpiArgs& e, cudaStream_t s) const {
  if (x == out) throw InvalidArgument("CSR operator cannot run in place");
  const size_t rows = m_.rows;
  int blocks = (int)((rows + 7) / 8);
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(k_csr, blocks, 256, 0, s, rows, d_ptr_.get(), d_idx_.get(), d_val_.get(), x, out, epi,
           e.b, e.dinv, e.omega);
  FDE_LAUNCH_CHECK();
}

BandedLu::BandedLu(const Csr& a, size_t bw) : n_(a.rows), bw_(bw) {
  if (a.rows != a.cols) throw InvalidArgument("banded LU needs a square matrix");
  if (bw_ > 32 * (size_t)kBandE) throw InvalidArgument("p2-exact band wider than 256");
  if (n_ * sizeof(double) > 200 * 1024)
    throw InvalidArgument("p2-exact is limited to 25600 unknowns (substitution in shared memory)");
  const size_t ld = 2 * bw_ + 1;
  std::vector<double> band(n_ * ld, 0.0);
  auto at = [&](size_t i, size_t j) -> double& { return band[i * ld + (j + bw_ - i)]; };
  for (size_t r = 0; r < n_; ++r)
    for (uint32_t k = a.ptr[r]; k < a.ptr[r + 1]; ++k) {
      const size_t c = a.idx[k];
      if (c + bw_ < r || c > r + bw_) throw InvalidArgument("matrix exceeds the band");
      at(r, c) = a.val[k];
    }
  for (size_t k = 0; k < n_; ++k) {  // Doolittle LU in the band, no pivoting
    const double piv = at(k, k);
    if (piv == 0.0) throw RuntimeError("banded order-2 factorization failed");
    const size_t last = std::min(n_ - 1, k + bw_);
    for (size_t i = k + 1; i <= last; ++i) {
      const double l = at(i, k) / piv;
      at(i, k) = l;
      if (l == 0.0) continue;
      for (size_t j = k + 1; j <= last; ++j) at(i, j) -= l * at(k, j);
    }
  }
  d_band_.upload(band.data(), band.size());
}

void BandedLu::solve(const double* r, double* z, cudaStream_t s) const {
  static DeviceCache<bool> configured;  // per device
  configured.get([](int) {
    FDE_CUDA(cudaFuncSetAttribute(k_band_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  200 * 1024));
    return true;
  });
  launch_k(k_band_solve, 1, 32, n_ * sizeof(double), s, n_, (int)bw_, d_band_.get(), r, z);
  FDE_LAUNCH_CHECK();
}

}  // namespace fde_b200
