// Clean-room, eager, dense subset of the Eigen 3 API -- just enough for the
// reference's hot-path translation units (proj/src/{structured,sparse,
// multigrid,precond,driver,problem}.cpp) to compile unmodified.
//
// TEST INFRASTRUCTURE ONLY (oracle build).  Not product code.
//
// Only PartialPivLU (the CoarseSolve::lu coarsest solve, multigrid.cpp:314-328)
// carries arithmetic that a BASELINE path can reach; it is a textbook
// row-pivoted Doolittle LU.  SparseLU is dense-backed (p2-exact only, off the
// hot path).  GeneralizedSelfAdjointEigenSolver throws (verify_tgm_theory only).
#pragma once
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <stdexcept>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum ComputationInfo { Success = 0, NumericalIssue = 1 };

class MatrixXd;
class VectorXd;
class DiagonalWrapper;

class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(Index r, Index c) : r_(r), c_(c), d_(static_cast<std::size_t>(r * c), 0.0) {}
  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
  static MatrixXd Identity(Index r, Index c) {
    MatrixXd m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double& operator()(Index i, Index j) { return d_[static_cast<std::size_t>(i + j * r_)]; }
  double operator()(Index i, Index j) const { return d_[static_cast<std::size_t>(i + j * r_)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  MatrixXd transpose() const {
    MatrixXd t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  MatrixXd eval() const { return *this; }
  inline VectorXd diagonal() const;
  inline class LdltLike ldlt() const;
  MatrixXd& operator+=(const MatrixXd& o) {
    for (std::size_t k = 0; k < d_.size(); ++k) d_[k] += o.d_[k];
    return *this;
  }

 protected:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

class VectorXd : public MatrixXd {
 public:
  VectorXd() = default;
  explicit VectorXd(Index n) : MatrixXd(n, 1) {}
  VectorXd(const MatrixXd& m) : MatrixXd(m) {
    if (m.cols() != 1) throw std::invalid_argument("eigen shim: not a vector");
  }
  double& operator[](Index i) { return d_[static_cast<std::size_t>(i)]; }
  double operator[](Index i) const { return d_[static_cast<std::size_t>(i)]; }
  double dot(const MatrixXd& o) const {
    double s = 0.0;
    for (Index i = 0; i < r_; ++i) s += d_[static_cast<std::size_t>(i)] * o.data()[i];
    return s;
  }
  double minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
  double maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
  VectorXd cwiseInverse() const {
    VectorXd v(r_);
    for (Index i = 0; i < r_; ++i) v[i] = 1.0 / (*this)[i];
    return v;
  }
  inline DiagonalWrapper asDiagonal() const;
};

class DiagonalWrapper {
 public:
  explicit DiagonalWrapper(VectorXd d) : d_(std::move(d)) {}
  const VectorXd& diag() const { return d_; }

 private:
  VectorXd d_;
};

inline DiagonalWrapper VectorXd::asDiagonal() const { return DiagonalWrapper(*this); }

inline VectorXd MatrixXd::diagonal() const {
  const Index n = std::min(r_, c_);
  VectorXd v(n);
  for (Index i = 0; i < n; ++i) v[i] = (*this)(i, i);
  return v;
}

inline MatrixXd operator*(const MatrixXd& a, const MatrixXd& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("eigen shim: product shape");
  MatrixXd c(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k) {
      const double bk = b(k, j);
      if (bk == 0.0) continue;
      for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, k) * bk;
    }
  return c;
}
inline MatrixXd operator*(double s, const MatrixXd& a) {
  MatrixXd c = a;
  for (Index k = 0; k < c.size(); ++k) c.data()[k] *= s;
  return c;
}
inline MatrixXd operator*(const DiagonalWrapper& d, const MatrixXd& a) {
  MatrixXd c = a;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) c(i, j) *= d.diag()[i];
  return c;
}
inline MatrixXd operator*(const MatrixXd& a, const DiagonalWrapper& d) {
  MatrixXd c = a;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) c(i, j) *= d.diag()[j];
  return c;
}
inline MatrixXd operator+(const MatrixXd& a, const MatrixXd& b) {
  MatrixXd c = a;
  c += b;
  return c;
}
inline MatrixXd operator-(const MatrixXd& a, const MatrixXd& b) {
  MatrixXd c = a;
  for (Index k = 0; k < c.size(); ++k) c.data()[k] -= b.data()[k];
  return c;
}

// Row-pivoted LU, P A = L U (partial pivoting on the largest magnitude).
template <class M>
class PartialPivLU {
 public:
  PartialPivLU() = default;
  explicit PartialPivLU(const MatrixXd& a) { compute(a); }
  PartialPivLU& compute(const MatrixXd& a) {
    if (a.rows() != a.cols()) throw std::invalid_argument("eigen shim: LU of non-square");
    lu_ = a;
    n_ = a.rows();
    perm_.resize(static_cast<std::size_t>(n_));
    sign_ = 1;
    for (Index i = 0; i < n_; ++i) perm_[static_cast<std::size_t>(i)] = i;
    for (Index k = 0; k < n_; ++k) {
      Index p = k;
      double best = std::fabs(lu_(k, k));
      for (Index i = k + 1; i < n_; ++i)
        if (std::fabs(lu_(i, k)) > best) { best = std::fabs(lu_(i, k)); p = i; }
      if (p != k) {
        for (Index j = 0; j < n_; ++j) std::swap(lu_(k, j), lu_(p, j));
        std::swap(perm_[static_cast<std::size_t>(k)], perm_[static_cast<std::size_t>(p)]);
        sign_ = -sign_;
      }
      const double piv = lu_(k, k);
      if (piv == 0.0) continue;
      for (Index i = k + 1; i < n_; ++i) {
        const double l = lu_(i, k) / piv;
        lu_(i, k) = l;
        if (l == 0.0) continue;
        for (Index j = k + 1; j < n_; ++j) lu_(i, j) -= l * lu_(k, j);
      }
    }
    return *this;
  }
  double determinant() const {
    double d = sign_;
    for (Index i = 0; i < n_; ++i) d *= lu_(i, i);
    return d;
  }
  MatrixXd solve(const MatrixXd& b) const {
    MatrixXd x(n_, b.cols());
    for (Index c = 0; c < b.cols(); ++c) {
      std::vector<double> y(static_cast<std::size_t>(n_));
      for (Index i = 0; i < n_; ++i) {
        double v = b(perm_[static_cast<std::size_t>(i)], c);
        for (Index j = 0; j < i; ++j) v -= lu_(i, j) * y[static_cast<std::size_t>(j)];
        y[static_cast<std::size_t>(i)] = v;
      }
      for (Index i = n_; i-- > 0;) {
        double v = y[static_cast<std::size_t>(i)];
        for (Index j = i + 1; j < n_; ++j) v -= lu_(i, j) * x(j, c);
        x(i, c) = v / lu_(i, i);
      }
    }
    return x;
  }

 private:
  MatrixXd lu_;
  Index n_ = 0;
  int sign_ = 1;
  std::vector<Index> perm_;
};

class LdltLike {
 public:
  explicit LdltLike(const MatrixXd& a) : lu_(a) {}
  MatrixXd solve(const MatrixXd& b) const { return lu_.solve(b); }

 private:
  PartialPivLU<MatrixXd> lu_;
};
inline LdltLike MatrixXd::ldlt() const { return LdltLike(*this); }

template <class T>
class Map;

template <>
class Map<const VectorXd> : public VectorXd {
 public:
  Map(const double* p, Index n) : VectorXd(n) { std::copy(p, p + n, data()); }
};

template <>
class Map<VectorXd> {
 public:
  Map(double* p, Index n) : p_(p), n_(n) {}
  Map& operator=(const MatrixXd& v) {
    if (v.size() != n_) throw std::invalid_argument("eigen shim: map size");
    std::copy(v.data(), v.data() + n_, p_);
    return *this;
  }

 private:
  double* p_;
  Index n_;
};

template <class M>
class GeneralizedSelfAdjointEigenSolver {
 public:
  GeneralizedSelfAdjointEigenSolver(const MatrixXd&, const MatrixXd&) {
    throw std::runtime_error("eigen shim: generalized eigensolver not provided (verify-only)");
  }
  VectorXd eigenvalues() const { return VectorXd(); }
};

template <class S>
struct Triplet {
  Triplet(Index r, Index c, S v) : r_(r), c_(c), v_(v) {}
  Index row() const { return r_; }
  Index col() const { return c_; }
  S value() const { return v_; }
  Index r_, c_;
  S v_;
};

template <class S>
class SparseMatrix {
 public:
  SparseMatrix() = default;
  SparseMatrix(Index r, Index c) : m_(r, c) {}
  template <class It>
  void setFromTriplets(It b, It e) {
    for (; b != e; ++b) m_(b->row(), b->col()) += b->value();
  }
  const MatrixXd& dense() const { return m_; }

 private:
  MatrixXd m_;
};

template <class Sp>
class SparseLU {
 public:
  void compute(const Sp& a) {
    lu_.compute(a.dense());
    info_ = lu_.determinant() == 0.0 ? NumericalIssue : Success;
  }
  ComputationInfo info() const { return info_; }
  VectorXd solve(const MatrixXd& b) const { return VectorXd(lu_.solve(b)); }

 private:
  PartialPivLU<MatrixXd> lu_;
  ComputationInfo info_ = Success;
};

}  // namespace Eigen
