// anisoq drop-in (B200): the slice of Eigen's dense API that the reference
// exposes through SelectorSystem (pq.hpp:71-74: Eigen::MatrixXd system_matrix,
// Eigen::VectorXd rhs) and that callers use on it — element access with
// Eigen::Index, rows()/cols()/size(), data(), Zero(), trace(),
// diagonal().array() += s, matrix * vector (incl. Eigen::Map<const VectorXd>),
// vector - vector, norm(). include/anisoq/pq.hpp includes this only when the
// real <Eigen/Dense> is not on the include path; with Eigen present the real
// types are used and this file is never seen. Storage is column-major like
// Eigen's default. No decompositions: the solves run on the device.
#pragma once

#include <cmath>
#include <cstddef>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;

class VectorXd {
 public:
  VectorXd() = default;
  explicit VectorXd(Index n) : v_(static_cast<std::size_t>(n), 0.0) {}
  static VectorXd Zero(Index n) { return VectorXd(n); }

  Index size() const { return static_cast<Index>(v_.size()); }
  Index rows() const { return size(); }
  Index cols() const { return 1; }
  double& operator()(Index i) { return v_[static_cast<std::size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<std::size_t>(i)]; }
  double& operator[](Index i) { return (*this)(i); }
  double operator[](Index i) const { return (*this)(i); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

  double squaredNorm() const {
    double s = 0.0;
    for (double x : v_) s += x * x;
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }

  friend VectorXd operator-(const VectorXd& a, const VectorXd& b) {
    VectorXd r(a.size());
    for (Index i = 0; i < a.size(); ++i) r(i) = a(i) - b(i);
    return r;
  }
  friend VectorXd operator+(const VectorXd& a, const VectorXd& b) {
    VectorXd r(a.size());
    for (Index i = 0; i < a.size(); ++i) r(i) = a(i) + b(i);
    return r;
  }

 private:
  std::vector<double> v_;
};

template <class T>
class Map;

// read-only view of n contiguous doubles as a column vector
template <>
class Map<const VectorXd> {
 public:
  Map(const double* p, Index n) : p_(p), n_(n) {}
  Index size() const { return n_; }
  double operator()(Index i) const { return p_[i]; }
  double operator[](Index i) const { return p_[i]; }
  const double* data() const { return p_; }

 private:
  const double* p_;
  Index n_;
};

class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(Index r, Index c) : r_(r), c_(c), v_(static_cast<std::size_t>(r * c), 0.0) {}
  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double& operator()(Index i, Index j) { return v_[static_cast<std::size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<std::size_t>(j * r_ + i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }

  double trace() const {
    double s = 0.0;
    for (Index i = 0; i < r_ && i < c_; ++i) s += (*this)(i, i);
    return s;
  }

  // m.diagonal().array() += s  (and -=, *=)
  class DiagonalArray {
   public:
    explicit DiagonalArray(MatrixXd& m) : m_(m) {}
    DiagonalArray& operator+=(double s) {
      for (Index i = 0; i < m_.r_ && i < m_.c_; ++i) m_(i, i) += s;
      return *this;
    }
    DiagonalArray& operator-=(double s) {
      for (Index i = 0; i < m_.r_ && i < m_.c_; ++i) m_(i, i) -= s;
      return *this;
    }
    DiagonalArray& operator*=(double s) {
      for (Index i = 0; i < m_.r_ && i < m_.c_; ++i) m_(i, i) *= s;
      return *this;
    }

   private:
    MatrixXd& m_;
  };
  class Diagonal {
   public:
    explicit Diagonal(MatrixXd& m) : m_(m) {}
    DiagonalArray array() { return DiagonalArray(m_); }
    Index size() const { return m_.r_ < m_.c_ ? m_.r_ : m_.c_; }
    double operator()(Index i) const { return m_(i, i); }

   private:
    MatrixXd& m_;
  };
  Diagonal diagonal() { return Diagonal(*this); }

  template <class V>
  VectorXd times(const V& x) const {
    VectorXd y(r_);
    for (Index j = 0; j < c_; ++j) {
      const double xj = x(j);
      for (Index i = 0; i < r_; ++i) y(i) += (*this)(i, j) * xj;
    }
    return y;
  }
  friend VectorXd operator*(const MatrixXd& a, const VectorXd& x) { return a.times(x); }
  friend VectorXd operator*(const MatrixXd& a, const Map<const VectorXd>& x) { return a.times(x); }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> v_;
};

}  // namespace Eigen
