// Sparse (CSR) levels for the reference's Galerkin variants on 𝓜 and the
// exact banded P2 solve (reference: proj/src/sparse.cpp:8-140,
// proj/src/structured.cpp:168-192, proj/src/multigrid.cpp:229-253,443-475,
// proj/src/precond.cpp:90-133).  These are the oracle-size paths the
// reference itself limits to n <= 128 (`mgm-galerkin`) or small grids
// (`p2-exact`, a sparse direct factorisation): host-side assembly and R A P
// products, device-side SpMV / banded substitutions.
#pragma once
#include <cstdint>
#include <memory>
#include <vector>

#include "devbuf.cuh"
#include "operator.cuh"

namespace fde_b200 {

// sparse::Csr: rows sorted by column, duplicates collapsed (sparse.cpp:8-40)
struct Csr {
  size_t rows = 0, cols = 0;
  std::vector<uint32_t> ptr, idx;
  std::vector<double> val;
  struct Triplet {
    uint32_t row, col;
    double value;
  };
  static Csr from_triplets(size_t rows, size_t cols, std::vector<Triplet> t);
  Csr transpose() const;                    // sparse.cpp:51-70
  Csr multiply(const Csr& other) const;     // Gustavson, sparse.cpp:72-108
  std::vector<double> diag() const;         // sparse.cpp:110-123
  size_t nnz() const { return idx.size(); }
};
Csr rap(const Csr& p, const Csr& a);                 // P^T (A P), sparse.cpp:131-136
Csr structured_to_csr(const StructuredOp& op);       // StructuredFdeOperator::to_csr
Csr prolong_matrix(const Xfer& t);                   // GridTransfer::prolong_matrix

// A CSR level on the device (sparse::CsrOp): one warp per row.
class CsrOp {
 public:
  explicit CsrOp(Csr m);
  size_t size() const { return m_.rows; }
  const Csr& matrix() const { return m_; }
  const std::vector<double>& diagonal() const { return diag_; }
  // out = epilogue(A x) (EPI_STORE / EPI_RESID / EPI_JACOBI, out != x)
  void run(const double* x, double* out, int epi, const EpiArgs& e, cudaStream_t s) const;

 private:
  Csr m_;
  std::vector<double> diag_;
  DevBuf<uint32_t> d_ptr_, d_idx_;
  DevBuf<double> d_val_;
};

// Exact solve with the banded order-2 companion P2 (P2ExactPrecond,
// precond.cpp:90-101): LU without pivoting in band storage (P2 is a
// diagonally dominant M-matrix: no pivot is needed), factored on the host
// once, forward / backward substitution on the device (one CTA walks the
// rows; the band's updates of each row run across its threads).
class BandedLu {
 public:
  BandedLu(const Csr& a, size_t bandwidth);
  size_t size() const { return n_; }
  void solve(const double* r, double* z, cudaStream_t s) const;

 private:
  size_t n_, bw_;
  DevBuf<double> d_band_;  // row-major (2 bw + 1) entries per row, diagonal at bw
};

}  // namespace fde_b200
