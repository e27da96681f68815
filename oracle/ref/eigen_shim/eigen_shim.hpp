// eigen_shim.hpp -- ORACLE (test infrastructure): a from-scratch, eager,
// column-major subset of the Eigen3 API, only what the reference headers
// (/root/reference/proj/include/bfly) and tests use, so they compile
// UNMODIFIED here (Eigen is not vendored by the reference and is absent).
// Dense factorizations restate Eigen's published algorithms:
//   ColPivHouseholderQR  first max updated-norm pivot, Householder with
//                        beta = -sign(Re c0)||x||, LAWN-176 downdating;
//   HouseholderQR        the same reflectors without pivoting;
//   JacobiSVD            one-sided (Hestenes) Jacobi, singular values sorted
//                        decreasing (the SVD itself is unique up to phases);
//   PartialPivLU         row-pivoted Doolittle.
#pragma once

#include <algorithm>
#include <cassert>
#include <cfloat>
#include <cmath>
#include <complex>
#include <cstddef>
#include <initializer_list>
#include <limits>
#include <stdexcept>
#include <type_traits>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum DecompositionOptions { ComputeFullU = 4, ComputeThinU = 8, ComputeFullV = 16, ComputeThinV = 32 };

namespace internal {
template <class S> struct real_of { using type = S; };
template <class T> struct real_of<std::complex<T>> { using type = T; };
template <class S> inline S cj(const S& x) { return x; }
template <class T> inline std::complex<T> cj(const std::complex<T>& x) { return std::conj(x); }
template <class S> inline typename real_of<S>::type abs2(const S& x) { return x * x; }
template <class T> inline T abs2(const std::complex<T>& x) { return std::norm(x); }
template <class S> inline typename real_of<S>::type re(const S& x) { return x; }
template <class T> inline T re(const std::complex<T>& x) { return x.real(); }
template <class S> inline typename real_of<S>::type im(const S&) { return 0; }
template <class T> inline T im(const std::complex<T>& x) { return x.imag(); }
}  // namespace internal

template <class S, int R = Dynamic, int C = Dynamic, int Opt = 0, int MR = R, int MC = C> class Matrix;
template <class S> class Block;
template <class S> class ArrayView;
template <class S> class DiagonalWrapper;

template <class S> using MatrixX = Matrix<S, Dynamic, Dynamic>;

// ---------------------------------------------------------------- storage
template <class S>
class DenseBase {
 public:
  using Scalar = S;
  using RealScalar = typename internal::real_of<S>::type;
  Index rows_ = 0, cols_ = 0;
  std::vector<S> v_;

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  S* data() { return v_.data(); }
  const S* data() const { return v_.data(); }
  S& operator()(Index i, Index j) { return v_[i + j * rows_]; }
  const S& operator()(Index i, Index j) const { return v_[i + j * rows_]; }
  S& operator()(Index i) { return v_[i]; }
  const S& operator()(Index i) const { return v_[i]; }
  S& coeffRef(Index i, Index j) { return (*this)(i, j); }
  S coeff(Index i, Index j) const { return (*this)(i, j); }
  void resize(Index r, Index c) {
    if (r * c != size()) v_.assign((size_t)(r * c), S(0));
    rows_ = r;
    cols_ = c;
  }
};

// A read-write rectangular view into a Matrix.
template <class S>
class Block {
 public:
  using Scalar = S;
  using RealScalar = typename internal::real_of<S>::type;
  Block(DenseBase<S>& m, Index r0, Index c0, Index nr, Index nc) : m_(&m), r0_(r0), c0_(c0), nr_(nr), nc_(nc) {}
  Index rows() const { return nr_; }
  Index cols() const { return nc_; }
  Index size() const { return nr_ * nc_; }
  S& operator()(Index i, Index j) const { return (*m_)(r0_ + i, c0_ + j); }
  S& operator()(Index i) const { return nc_ == 1 ? (*this)(i, 0) : (*this)(0, i); }
  Matrix<S> eval() const;
  operator Matrix<S>() const { return eval(); }
  template <class E> Block& operator=(const E& e);
  Block& operator=(const Block& b) { return this->template operator=<Block>(b); }
  template <class E> Block& operator+=(const E& e);
  template <class E> Block& operator-=(const E& e);
  Block& operator*=(const S& s) {
    for (Index j = 0; j < nc_; ++j)
      for (Index i = 0; i < nr_; ++i) (*this)(i, j) *= s;
    return *this;
  }
  void setZero() {
    for (Index j = 0; j < nc_; ++j)
      for (Index i = 0; i < nr_; ++i) (*this)(i, j) = S(0);
  }
  RealScalar squaredNorm() const {
    RealScalar s = 0;
    for (Index j = 0; j < nc_; ++j)
      for (Index i = 0; i < nr_; ++i) s += internal::abs2((*this)(i, j));
    return s;
  }
  RealScalar norm() const { return std::sqrt(squaredNorm()); }
  void swap(Block other) {
    for (Index j = 0; j < nc_; ++j)
      for (Index i = 0; i < nr_; ++i) std::swap((*this)(i, j), other(i, j));
  }
  Block tail(Index n) const { return nc_ == 1 ? Block(*m_, r0_ + nr_ - n, c0_, n, 1) : Block(*m_, r0_, c0_ + nc_ - n, 1, n); }
  Block head(Index n) const { return nc_ == 1 ? Block(*m_, r0_, c0_, n, 1) : Block(*m_, r0_, c0_, 1, n); }
  Block segment(Index s, Index n) const {
    return nc_ == 1 ? Block(*m_, r0_ + s, c0_, n, 1) : Block(*m_, r0_, c0_ + s, 1, n);
  }
  Block topRows(Index n) const { return Block(*m_, r0_, c0_, n, nc_); }
  Block bottomRows(Index n) const { return Block(*m_, r0_ + nr_ - n, c0_, n, nc_); }
  Block middleRows(Index s, Index n) const { return Block(*m_, r0_ + s, c0_, n, nc_); }
  Block row(Index i) const { return Block(*m_, r0_ + i, c0_, 1, nc_); }
  Block col(Index j) const { return Block(*m_, r0_, c0_ + j, nr_, 1); }
  Block block(Index r, Index c, Index nr, Index nc) const { return Block(*m_, r0_ + r, c0_ + c, nr, nc); }
  Matrix<S> adjoint() const;
  Matrix<S> transpose() const;
  Matrix<S> conjugate() const;
  ArrayView<S> array() const;
  RealScalar maxAbs() const;

 private:
  DenseBase<S>* m_;
  Index r0_, c0_, nr_, nc_;
};

template <class S>
class DiagonalWrapper {
 public:
  using Scalar = S;
  std::vector<S> d;
};

template <class T> struct is_dense : std::false_type {};
template <class S, int R, int C, int O, int A, int B> struct is_dense<Matrix<S, R, C, O, A, B>> : std::true_type {};
template <class S> struct is_dense<Block<S>> : std::true_type {};

template <class E> inline auto evald(const E& e) { return e.eval(); }

// ------------------------------------------------------------------ matrix
template <class S, int R, int C, int Opt, int MR, int MC>
class Matrix : public DenseBase<S> {
  using Base = DenseBase<S>;

 public:
  using Scalar = S;
  using RealScalar = typename internal::real_of<S>::type;
  Matrix() {
    if (R > 0 && C > 0) this->resize(R, C);
    else if (C == 1) this->resize(0, 1);
  }
  Matrix(Index r, Index c) { this->resize(r, c); }
  explicit Matrix(Index n) { C == 1 ? this->resize(n, 1) : this->resize(1, n); }
  template <int R2, int C2, int O2, int A2, int B2>
  Matrix(const Matrix<S, R2, C2, O2, A2, B2>& o) {
    this->rows_ = o.rows();
    this->cols_ = o.cols();
    this->v_.assign(o.data(), o.data() + o.size());
  }
  Matrix(const Block<S>& b) { assign_from(b); }
  Matrix(const DiagonalWrapper<S>& d) {
    Index n = (Index)d.d.size();
    this->resize(n, n);
    for (Index i = 0; i < n; ++i) (*this)(i, i) = d.d[i];
  }
  template <class E, class = std::enable_if_t<is_dense<E>::value>>
  Matrix& operator=(const E& e) {
    Matrix tmp = e.eval();
    this->rows_ = tmp.rows_;
    this->cols_ = tmp.cols_;
    this->v_.swap(tmp.v_);
    return *this;
  }
  Matrix eval() const { return *this; }

  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  static Matrix Zero(Index n) { return Matrix(n); }
  static Matrix Identity(Index r, Index c) {
    Matrix m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = S(1);
    return m;
  }
  static Matrix Identity(Index n) { return Identity(n, n); }
  static Matrix Constant(Index r, Index c, const S& s) {
    Matrix m(r, c);
    std::fill(m.v_.begin(), m.v_.end(), s);
    return m;
  }
  void setZero() { std::fill(this->v_.begin(), this->v_.end(), S(0)); }
  void setIdentity() { *this = Identity(this->rows_, this->cols_); }
  Matrix& setZero(Index r, Index c) {
    this->resize(r, c);
    setZero();
    return *this;
  }

  // views
  Block<S> block(Index r, Index c, Index nr, Index nc) { return Block<S>(*this, r, c, nr, nc); }
  Block<S> row(Index i) { return Block<S>(*this, i, 0, 1, this->cols_); }
  Block<S> col(Index j) { return Block<S>(*this, 0, j, this->rows_, 1); }
  Block<S> topRows(Index n) { return Block<S>(*this, 0, 0, n, this->cols_); }
  Block<S> bottomRows(Index n) { return Block<S>(*this, this->rows_ - n, 0, n, this->cols_); }
  Block<S> middleRows(Index s, Index n) { return Block<S>(*this, s, 0, n, this->cols_); }
  Block<S> leftCols(Index n) { return Block<S>(*this, 0, 0, this->rows_, n); }
  Block<S> rightCols(Index n) { return Block<S>(*this, 0, this->cols_ - n, this->rows_, n); }
  Block<S> middleCols(Index s, Index n) { return Block<S>(*this, 0, s, this->rows_, n); }
  Block<S> bottomRightCorner(Index nr, Index nc) { return Block<S>(*this, this->rows_ - nr, this->cols_ - nc, nr, nc); }
  Block<S> topLeftCorner(Index nr, Index nc) { return Block<S>(*this, 0, 0, nr, nc); }
  Block<S> head(Index n) { return this->cols_ == 1 ? middleRows(0, n) : middleCols(0, n); }
  Block<S> tail(Index n) { return this->cols_ == 1 ? bottomRows(n) : rightCols(n); }
  Block<S> segment(Index s, Index n) { return this->cols_ == 1 ? middleRows(s, n) : middleCols(s, n); }
  // const views (copies suffice for read-only use)
  Matrix block(Index r, Index c, Index nr, Index nc) const { return const_cast<Matrix*>(this)->block(r, c, nr, nc).eval(); }
  Matrix row(Index i) const { return const_cast<Matrix*>(this)->row(i).eval(); }
  Matrix col(Index j) const { return const_cast<Matrix*>(this)->col(j).eval(); }
  Matrix topRows(Index n) const { return const_cast<Matrix*>(this)->topRows(n).eval(); }
  Matrix bottomRows(Index n) const { return const_cast<Matrix*>(this)->bottomRows(n).eval(); }
  Matrix middleRows(Index s, Index n) const { return const_cast<Matrix*>(this)->middleRows(s, n).eval(); }
  Matrix leftCols(Index n) const { return const_cast<Matrix*>(this)->leftCols(n).eval(); }
  Matrix head(Index n) const { return const_cast<Matrix*>(this)->head(n).eval(); }
  Matrix tail(Index n) const { return const_cast<Matrix*>(this)->tail(n).eval(); }
  Matrix segment(Index s, Index n) const { return const_cast<Matrix*>(this)->segment(s, n).eval(); }

  Matrix<S> adjoint() const {
    Matrix<S> t(this->cols_, this->rows_);
    for (Index j = 0; j < this->cols_; ++j)
      for (Index i = 0; i < this->rows_; ++i) t(j, i) = internal::cj((*this)(i, j));
    return t;
  }
  Matrix<S> transpose() const {
    Matrix<S> t(this->cols_, this->rows_);
    for (Index j = 0; j < this->cols_; ++j)
      for (Index i = 0; i < this->rows_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  Matrix<S> conjugate() const {
    Matrix<S> t(*this);
    for (auto& x : t.v_) x = internal::cj(x);
    return t;
  }
  Matrix<RealScalar> real() const {
    Matrix<RealScalar> t(this->rows_, this->cols_);
    for (Index i = 0; i < this->size(); ++i) t.data()[i] = internal::re(this->v_[i]);
    return t;
  }
  Matrix<RealScalar> imag() const {
    Matrix<RealScalar> t(this->rows_, this->cols_);
    for (Index i = 0; i < this->size(); ++i) t.data()[i] = internal::im(this->v_[i]);
    return t;
  }
  Matrix<RealScalar> cwiseAbs() const {
    Matrix<RealScalar> t(this->rows_, this->cols_);
    for (Index i = 0; i < this->size(); ++i) t.data()[i] = std::abs(this->v_[i]);
    return t;
  }
  RealScalar squaredNorm() const {
    RealScalar s = 0;
    for (const auto& x : this->v_) s += internal::abs2(x);
    return s;
  }
  RealScalar norm() const { return std::sqrt(squaredNorm()); }
  void normalize() {
    RealScalar n = norm();
    if (n > 0)
      for (auto& x : this->v_) x /= n;
  }
  Matrix normalized() const {
    Matrix t(*this);
    t.normalize();
    return t;
  }
  S sum() const {
    S s(0);
    for (const auto& x : this->v_) s += x;
    return s;
  }
  S mean() const { return sum() / S(RealScalar(this->size())); }
  S trace() const {
    S s(0);
    for (Index i = 0; i < std::min(this->rows_, this->cols_); ++i) s += (*this)(i, i);
    return s;
  }
  S minCoeff() const { return *std::min_element(this->v_.begin(), this->v_.end(), lt_); }
  S maxCoeff() const { return *std::max_element(this->v_.begin(), this->v_.end(), lt_); }
  S maxCoeff(Index* idx) const {
    Index b = 0;
    for (Index i = 1; i < this->size(); ++i)
      if (lt_(this->v_[b], this->v_[i])) b = i;
    *idx = b;
    return this->v_[b];
  }
  bool allFinite() const {
    for (const auto& x : this->v_)
      if (!std::isfinite(internal::re(x)) || !std::isfinite(internal::im(x))) return false;
    return true;
  }
  Matrix<S> diagonal() const {
    Index n = std::min(this->rows_, this->cols_);
    Matrix<S> d(n, 1);
    for (Index i = 0; i < n; ++i) d(i, 0) = (*this)(i, i);
    return d;
  }
  struct DiagView;
  DiagView diagonal();
  DiagonalWrapper<S> asDiagonal() const {
    DiagonalWrapper<S> w;
    w.d = this->v_;
    return w;
  }
  ArrayView<S> array();
  Matrix<S> array() const;
  Matrix<S> inverse() const;
  Matrix<S> eval_() const { return *this; }
  void swap(Matrix& o) {
    std::swap(this->rows_, o.rows_);
    std::swap(this->cols_, o.cols_);
    this->v_.swap(o.v_);
  }

  // comma initializer
  struct CommaInit {
    Matrix* m;
    Index row = 0, col = 0, blk_rows = 0;
    template <class E>
    CommaInit& put(const E& e) {
      auto x = evald(e);
      if (col == 0) blk_rows = x.rows();
      for (Index j = 0; j < x.cols(); ++j)
        for (Index i = 0; i < x.rows(); ++i) (*m)(row + i, col + j) = x(i, j);
      col += x.cols();
      if (col >= m->cols()) {
        row += blk_rows;
        col = 0;
      }
      return *this;
    }
    CommaInit& put_scalar(const S& s) {
      (*m)(row, col) = s;
      blk_rows = 1;
      if (++col >= m->cols()) {
        ++row;
        col = 0;
      }
      return *this;
    }
    template <class E, class = std::enable_if_t<is_dense<E>::value>>
    CommaInit& operator,(const E& e) { return put(e); }
    CommaInit& operator,(const S& s) { return put_scalar(s); }
  };
  template <class E, class = std::enable_if_t<is_dense<E>::value>>
  CommaInit operator<<(const E& e) {
    CommaInit ci{this};
    ci.put(e);
    return ci;
  }
  CommaInit operator<<(const S& s) {
    CommaInit ci{this};
    ci.put_scalar(s);
    return ci;
  }

  template <class E> Matrix& operator+=(const E& e);
  template <class E> Matrix& operator-=(const E& e);
  Matrix& operator*=(const S& s) {
    for (auto& x : this->v_) x *= s;
    return *this;
  }
  Matrix& operator/=(const S& s) {
    for (auto& x : this->v_) x /= s;
    return *this;
  }

 private:
  static bool lt_(const S& a, const S& b) { return internal::re(a) < internal::re(b); }
  void assign_from(const Block<S>& b) {
    this->resize(b.rows(), b.cols());
    for (Index j = 0; j < b.cols(); ++j)
      for (Index i = 0; i < b.rows(); ++i) (*this)(i, j) = b(i, j);
  }
};

template <class S> using VectorX = Matrix<S, Dynamic, 1>;

template <class S>
Matrix<S> Block<S>::eval() const {
  Matrix<S> m(nr_, nc_);
  for (Index j = 0; j < nc_; ++j)
    for (Index i = 0; i < nr_; ++i) m(i, j) = (*this)(i, j);
  return m;
}
template <class S> template <class E> Block<S>& Block<S>::operator=(const E& e) {
  Matrix<S> x = evald(e);
  if (x.rows() != nr_ || x.cols() != nc_) throw std::logic_error("eigen_shim: block assignment size mismatch");
  for (Index j = 0; j < nc_; ++j)
    for (Index i = 0; i < nr_; ++i) (*this)(i, j) = x(i, j);
  return *this;
}
template <class S> template <class E> Block<S>& Block<S>::operator+=(const E& e) {
  Matrix<S> x = evald(e);
  for (Index j = 0; j < nc_; ++j)
    for (Index i = 0; i < nr_; ++i) (*this)(i, j) += x(i, j);
  return *this;
}
template <class S> template <class E> Block<S>& Block<S>::operator-=(const E& e) {
  Matrix<S> x = evald(e);
  for (Index j = 0; j < nc_; ++j)
    for (Index i = 0; i < nr_; ++i) (*this)(i, j) -= x(i, j);
  return *this;
}
template <class S> Matrix<S> Block<S>::adjoint() const { return eval().adjoint(); }
template <class S> Matrix<S> Block<S>::transpose() const { return eval().transpose(); }
template <class S> Matrix<S> Block<S>::conjugate() const { return eval().conjugate(); }

template <class S, int R, int C, int O, int A, int B>
template <class E> Matrix<S, R, C, O, A, B>& Matrix<S, R, C, O, A, B>::operator+=(const E& e) {
  Matrix<S> x = evald(e);
  for (Index i = 0; i < this->size(); ++i) this->v_[i] += x.data()[i];
  return *this;
}
template <class S, int R, int C, int O, int A, int B>
template <class E> Matrix<S, R, C, O, A, B>& Matrix<S, R, C, O, A, B>::operator-=(const E& e) {
  Matrix<S> x = evald(e);
  for (Index i = 0; i < this->size(); ++i) this->v_[i] -= x.data()[i];
  return *this;
}

// ------------------------------------------------- array / diagonal views
template <class S>
class ArrayView {
 public:
  std::vector<S*> p;
  ArrayView& operator-=(const S& s) {
    for (auto* x : p) *x -= s;
    return *this;
  }
  ArrayView& operator+=(const S& s) {
    for (auto* x : p) *x += s;
    return *this;
  }
};

template <class S, int R, int C, int O, int A, int B>
struct Matrix<S, R, C, O, A, B>::DiagView {
  Matrix* m;
  ArrayView<S> array() {
    ArrayView<S> a;
    for (Index i = 0; i < std::min(m->rows(), m->cols()); ++i) a.p.push_back(&(*m)(i, i));
    return a;
  }
  operator Matrix<S>() const { return static_cast<const Matrix*>(m)->diagonal(); }
  Matrix<S> eval() const { return static_cast<const Matrix*>(m)->diagonal(); }
  typename Matrix::RealScalar minCoeff() const { return internal::re(eval().minCoeff()); }
  Matrix<typename Matrix::RealScalar> cwiseAbs() const { return eval().cwiseAbs(); }
};
template <class S, int R, int C, int O, int A, int B>
typename Matrix<S, R, C, O, A, B>::DiagView Matrix<S, R, C, O, A, B>::diagonal() {
  return DiagView{this};
}

// Arrays: element-wise expressions reduce to vectors of values
template <class S>
class ArrayExpr {
 public:
  using Scalar = S;
  std::vector<S> v;
  ArrayExpr square() const {
    ArrayExpr r{v};
    for (auto& x : r.v) x = x * x;
    return r;
  }
  ArrayExpr abs() const {
    ArrayExpr r{v};
    for (auto& x : r.v) x = std::abs(x);
    return r;
  }
  S sum() const {
    S s(0);
    for (const auto& x : v) s += x;
    return s;
  }
  S maxCoeff() const { return *std::max_element(v.begin(), v.end()); }
  S minCoeff() const { return *std::min_element(v.begin(), v.end()); }
  friend ArrayExpr operator-(const ArrayExpr& a, const S& s) {
    ArrayExpr r{a.v};
    for (auto& x : r.v) x -= s;
    return r;
  }
};
template <class S, int R, int C, int O, int A, int B>
ArrayView<S> Matrix<S, R, C, O, A, B>::array() {
  ArrayView<S> a;
  for (auto& x : this->v_) a.p.push_back(&x);
  return a;
}
template <class S, int R, int C, int O, int A, int B>
Matrix<S> Matrix<S, R, C, O, A, B>::array() const {
  return *this;
}
template <class S> inline ArrayExpr<S> operator-(const ArrayView<S>& a, const S& s) {
  ArrayExpr<S> r;
  for (auto* x : a.p) r.v.push_back(*x - s);
  return r;
}
template <class S> ArrayView<S> Block<S>::array() const {
  ArrayView<S> a;
  for (Index j = 0; j < nc_; ++j)
    for (Index i = 0; i < nr_; ++i) a.p.push_back(&(*this)(i, j));
  return a;
}

// ------------------------------------------------------------- arithmetic
template <class S>
Matrix<S> gemm(const Matrix<S>& a, const Matrix<S>& b) {
  if (a.cols() != b.rows()) throw std::logic_error("eigen_shim: product dimension mismatch");
  Matrix<S> c(a.rows(), b.cols());
  const Index m = a.rows(), n = b.cols(), k = a.cols();
  for (Index j = 0; j < n; ++j) {
    S* cj = c.data() + j * m;
    for (Index l = 0; l < k; ++l) {
      const S blj = b(l, j);
      if (blj == S(0)) continue;
      const S* al = a.data() + l * m;
      for (Index i = 0; i < m; ++i) cj[i] += al[i] * blj;
    }
  }
  return c;
}

template <class A, class B, class = std::enable_if_t<is_dense<A>::value && is_dense<B>::value>>
auto operator*(const A& a, const B& b) {
  return gemm<typename A::Scalar>(a.eval(), b.eval());
}
template <class A, class = std::enable_if_t<is_dense<A>::value>>
auto operator*(const A& a, const DiagonalWrapper<typename A::Scalar>& d) {
  Matrix<typename A::Scalar> r = a.eval();
  for (Index j = 0; j < r.cols(); ++j)
    for (Index i = 0; i < r.rows(); ++i) r(i, j) *= d.d[j];
  return r;
}
template <class A, class = std::enable_if_t<is_dense<A>::value>>
auto operator*(const DiagonalWrapper<typename A::Scalar>& d, const A& a) {
  Matrix<typename A::Scalar> r = a.eval();
  for (Index j = 0; j < r.cols(); ++j)
    for (Index i = 0; i < r.rows(); ++i) r(i, j) *= d.d[i];
  return r;
}
template <class A, class = std::enable_if_t<is_dense<A>::value>>
auto operator*(const A& a, const typename A::Scalar& s) {
  Matrix<typename A::Scalar> r = a.eval();
  r *= s;
  return r;
}
template <class A, class = std::enable_if_t<is_dense<A>::value>>
auto operator*(const typename A::Scalar& s, const A& a) {
  Matrix<typename A::Scalar> r = a.eval();
  r *= s;
  return r;
}
template <class A, class = std::enable_if_t<is_dense<A>::value &&
                                            !std::is_same<typename A::Scalar, typename A::RealScalar>::value>>
auto operator*(const typename A::RealScalar& s, const A& a) {
  Matrix<typename A::Scalar> r = a.eval();
  r *= typename A::Scalar(s);
  return r;
}
template <class A, class = std::enable_if_t<is_dense<A>::value>>
auto operator/(const A& a, const typename A::Scalar& s) {
  Matrix<typename A::Scalar> r = a.eval();
  r /= s;
  return r;
}
template <class A, class B, class = std::enable_if_t<is_dense<A>::value && is_dense<B>::value>>
auto operator+(const A& a, const B& b) {
  Matrix<typename A::Scalar> r = a.eval();
  r += b;
  return r;
}
template <class A, class B, class = std::enable_if_t<is_dense<A>::value && is_dense<B>::value>>
auto operator-(const A& a, const B& b) {
  Matrix<typename A::Scalar> r = a.eval();
  r -= b;
  return r;
}
template <class A, class = std::enable_if_t<is_dense<A>::value>>
auto operator-(const A& a) {
  Matrix<typename A::Scalar> r = a.eval();
  r *= typename A::Scalar(-1);
  return r;
}
template <class A, class B, class = std::enable_if_t<is_dense<A>::value && is_dense<B>::value>>
bool operator==(const A& a, const B& b) {
  auto x = a.eval();
  auto y = b.eval();
  return x.rows() == y.rows() && x.cols() == y.cols() && std::equal(x.data(), x.data() + x.size(), y.data());
}

// ---------------------------------------------------------- Householder
namespace internal {
// makeHouseholderInPlace on x[0..n): returns tau, writes beta, x[1..] <- essential
template <class S>
S make_householder(S* x, Index n, typename real_of<S>::type& beta) {
  using Rl = typename real_of<S>::type;
  Rl tail = 0;
  for (Index i = 1; i < n; ++i) tail += abs2(x[i]);
  S c0 = x[0];
  const Rl tiny = std::numeric_limits<Rl>::min();
  if (tail <= tiny && abs2(im(c0)) <= tiny) {
    beta = re(c0);
    for (Index i = 1; i < n; ++i) x[i] = S(0);
    return S(0);
  }
  beta = std::sqrt(abs2(c0) + tail);
  if (re(c0) >= Rl(0)) beta = -beta;
  S d = c0 - S(beta);
  for (Index i = 1; i < n; ++i) x[i] /= d;
  return cj((S(beta) - c0) / S(beta));
}
// (I - tau v v^H) on an (n x ncols) block (ld), v = (1; ess)
template <class S>
void apply_householder(S* m, Index ld, Index n, Index ncols, const S* ess, S tau) {
  if (n == 1) {
    for (Index j = 0; j < ncols; ++j) m[j * ld] *= (S(1) - tau);
    return;
  }
  if (tau == S(0)) return;
  for (Index j = 0; j < ncols; ++j) {
    S* col = m + j * ld;
    S tmp = col[0];
    for (Index i = 1; i < n; ++i) tmp += cj(ess[i - 1]) * col[i];
    S t = tau * tmp;
    col[0] -= t;
    for (Index i = 1; i < n; ++i) col[i] -= ess[i - 1] * t;
  }
}
}  // namespace internal

// Q = H_0 ... H_{n-1}, H_j = I - conj(tau_j) v_j v_j^H (householderQ())
template <class S>
class HouseholderSequence {
 public:
  Matrix<S> qr;
  std::vector<S> hc;
  Index len;
  template <class E>
  Matrix<S> operator*(const E& e) const {
    Matrix<S> x = evald(e);
    const Index rows = qr.rows();
    for (Index j = std::min(len, rows) - 1; j >= 0; --j)
      internal::apply_householder(x.data() + j, rows, rows - j, x.cols(), qr.data() + j + 1 + j * rows,
                                  internal::cj(hc[j]));
    return x;
  }
  operator Matrix<S>() const { return (*this) * Matrix<S>::Identity(qr.rows(), qr.rows()); }
};

template <class M>
class HouseholderQR {
 public:
  using S = typename M::Scalar;
  HouseholderQR() = default;
  explicit HouseholderQR(const M& a) { compute(a); }
  HouseholderQR& compute(const M& a) {
    qr_ = a;
    const Index rows = qr_.rows(), cols = qr_.cols(), size = std::min(rows, cols);
    hc_.assign(size, S(0));
    for (Index k = 0; k < size; ++k) {
      typename M::RealScalar beta;
      hc_[k] = internal::make_householder(qr_.data() + k + k * rows, rows - k, beta);
      qr_(k, k) = S(beta);
      internal::apply_householder(qr_.data() + k + (k + 1) * rows, rows, rows - k, cols - k - 1,
                                  qr_.data() + k + 1 + k * rows, hc_[k]);
    }
    return *this;
  }
  HouseholderSequence<S> householderQ() const { return HouseholderSequence<S>{qr_, hc_, (Index)hc_.size()}; }
  const Matrix<S>& matrixQR() const { return qr_; }

 private:
  Matrix<S> qr_;
  std::vector<S> hc_;
};

template <class M>
class ColPivHouseholderQR {
 public:
  using S = typename M::Scalar;
  using Rl = typename M::RealScalar;
  ColPivHouseholderQR() = default;
  explicit ColPivHouseholderQR(const M& a) { compute(a); }
  ColPivHouseholderQR& compute(const M& a) {
    qr_ = a;
    const Index rows = qr_.rows(), cols = qr_.cols(), size = std::min(rows, cols);
    hc_.assign(size, S(0));
    std::vector<Rl> nu(cols), nd(cols);
    perm_.resize(cols);
    for (Index j = 0; j < cols; ++j) {
      nu[j] = nd[j] = qr_.col(j).norm();
      perm_[j] = j;
    }
    const Rl thresh = std::sqrt(std::numeric_limits<Rl>::epsilon());
    for (Index k = 0; k < size; ++k) {
      Index big = k;
      for (Index j = k + 1; j < cols; ++j)
        if (nu[j] > nu[big]) big = j;
      if (big != k) {
        for (Index i = 0; i < rows; ++i) std::swap(qr_(i, k), qr_(i, big));
        std::swap(nu[k], nu[big]);
        std::swap(nd[k], nd[big]);
        std::swap(perm_[k], perm_[big]);
      }
      Rl beta;
      hc_[k] = internal::make_householder(qr_.data() + k + k * rows, rows - k, beta);
      qr_(k, k) = S(beta);
      internal::apply_householder(qr_.data() + k + (k + 1) * rows, rows, rows - k, cols - k - 1,
                                  qr_.data() + k + 1 + k * rows, hc_[k]);
      for (Index j = k + 1; j < cols; ++j) {
        if (nu[j] != Rl(0)) {
          Rl temp = std::abs(qr_(k, j)) / nu[j];
          temp = (Rl(1) + temp) * (Rl(1) - temp);
          if (temp < Rl(0)) temp = 0;
          Rl ratio = nu[j] / nd[j];
          Rl temp2 = temp * ratio * ratio;
          if (temp2 <= thresh) {
            Rl s = 0;
            for (Index i = k + 1; i < rows; ++i) s += internal::abs2(qr_(i, j));
            nd[j] = std::sqrt(s);
            nu[j] = nd[j];
          } else {
            nu[j] *= std::sqrt(temp);
          }
        }
      }
    }
    return *this;
  }
  // upper triangle of the factored matrix (matrixR)
  const Matrix<S>& matrixR() const { return qr_; }
  HouseholderSequence<S> householderQ() const { return HouseholderSequence<S>{qr_, hc_, (Index)hc_.size()}; }
  Index rank() const;

 private:
  Matrix<S> qr_;
  std::vector<S> hc_;
  std::vector<Index> perm_;
};

// --------------------------------------------------------------- JacobiSVD
template <class M>
class JacobiSVD {
 public:
  using S = typename M::Scalar;
  using Rl = typename M::RealScalar;
  JacobiSVD() = default;
  explicit JacobiSVD(const M& a, unsigned opts = 0) { compute(a, opts); }
  JacobiSVD& compute(const M& a, unsigned opts = 0) {
    const bool wide = a.rows() < a.cols();
    Matrix<S> t = wide ? a.adjoint() : Matrix<S>(a);  // tall p x q
    const Index p = t.rows(), q = t.cols();
    Matrix<S> v = Matrix<S>::Identity(q, q);
    for (int sweep = 0; sweep < 80; ++sweep) {
      bool rotated = false;
      for (Index i = 0; i + 1 < q; ++i)
        for (Index j = i + 1; j < q; ++j) {
          Rl alpha = 0, beta = 0;
          S gamma(0);
          for (Index r = 0; r < p; ++r) {
            alpha += internal::abs2(t(r, i));
            beta += internal::abs2(t(r, j));
            gamma += internal::cj(t(r, i)) * t(r, j);
          }
          Rl g = std::abs(gamma);
          if (g == Rl(0) || g <= Rl(1e-15) * std::sqrt(alpha * beta)) continue;
          rotated = true;
          S ph = gamma / S(g);
          Rl zeta = (beta - alpha) / (Rl(2) * g);
          Rl tt = (zeta >= 0 ? Rl(1) : Rl(-1)) / (std::abs(zeta) + std::sqrt(Rl(1) + zeta * zeta));
          Rl c = Rl(1) / std::sqrt(Rl(1) + tt * tt), s = c * tt;
          S cph = internal::cj(ph);
          for (Index r = 0; r < p; ++r) {
            S x = t(r, i), y = t(r, j) * cph;
            t(r, i) = S(c) * x - S(s) * y;
            t(r, j) = S(s) * x + S(c) * y;
          }
          for (Index r = 0; r < q; ++r) {
            S x = v(r, i), y = v(r, j) * cph;
            v(r, i) = S(c) * x - S(s) * y;
            v(r, j) = S(s) * x + S(c) * y;
          }
        }
      if (!rotated) break;
    }
    // sort by decreasing singular value
    std::vector<Rl> sv(q);
    for (Index i = 0; i < q; ++i) sv[i] = t.col(i).norm();
    std::vector<Index> order(q);
    for (Index i = 0; i < q; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) { return sv[x] > sv[y]; });
    sv_ = Matrix<Rl, Dynamic, 1>(q);
    Matrix<S> u(p, q), vv(q, q);
    for (Index c = 0; c < q; ++c) {
      const Index o = order[c];
      sv_(c) = sv[o];
      for (Index r = 0; r < p; ++r) u(r, c) = sv[o] > 0 ? t(r, o) / S(sv[o]) : (r == c ? S(1) : S(0));
      for (Index r = 0; r < q; ++r) vv(r, c) = v(r, o);
    }
    // A = U S V^H for tall A; for wide A (= T^H) swap the roles
    u_ = wide ? vv : u;
    v_ = wide ? u : vv;
    (void)opts;
    return *this;
  }
  const Matrix<Rl, Dynamic, 1>& singularValues() const { return sv_; }
  const Matrix<S>& matrixU() const { return u_; }
  const Matrix<S>& matrixV() const { return v_; }

 private:
  Matrix<Rl, Dynamic, 1> sv_;
  Matrix<S> u_, v_;
};

// ------------------------------------------------------------ PartialPivLU
template <class M>
class PartialPivLU {
 public:
  using S = typename M::Scalar;
  PartialPivLU() = default;
  explicit PartialPivLU(const M& a) { compute(a); }
  PartialPivLU& compute(const M& a) {
    lu_ = a;
    const Index n = lu_.rows();
    perm_.resize(n);
    for (Index i = 0; i < n; ++i) perm_[i] = i;
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(lu_(i, k)) > std::abs(lu_(p, k))) p = i;
      if (p != k) {
        for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(p, j));
        std::swap(perm_[k], perm_[p]);
      }
      if (lu_(k, k) == S(0)) continue;
      for (Index i = k + 1; i < n; ++i) {
        lu_(i, k) /= lu_(k, k);
        const S f = lu_(i, k);
        for (Index j = k + 1; j < n; ++j) lu_(i, j) -= f * lu_(k, j);
      }
    }
    return *this;
  }
  const Matrix<S>& matrixLU() const { return lu_; }
  template <class E>
  Matrix<S> solve(const E& e) const {
    Matrix<S> b = evald(e);
    const Index n = lu_.rows();
    Matrix<S> x(n, b.cols());
    for (Index c = 0; c < b.cols(); ++c) {
      for (Index i = 0; i < n; ++i) x(i, c) = b(perm_[i], c);
      for (Index i = 0; i < n; ++i)
        for (Index j = 0; j < i; ++j) x(i, c) -= lu_(i, j) * x(j, c);
      for (Index i = n - 1; i >= 0; --i) {
        for (Index j = i + 1; j < n; ++j) x(i, c) -= lu_(i, j) * x(j, c);
        x(i, c) /= lu_(i, i);
      }
    }
    return x;
  }
  struct Transposed {
    const PartialPivLU* lu;
    // A^T x = b with P A = L U  =>  U^T L^T P x = b
    template <class E>
    Matrix<S> solve(const E& e) const {
      Matrix<S> b = evald(e);
      const Matrix<S>& f = lu->lu_;
      const Index n = f.rows();
      Matrix<S> x(n, b.cols());
      for (Index c = 0; c < b.cols(); ++c) {
        std::vector<S> y(n);
        for (Index i = 0; i < n; ++i) {  // U^T y = b
          S s = b(i, c);
          for (Index j = 0; j < i; ++j) s -= f(j, i) * y[j];
          y[i] = s / f(i, i);
        }
        for (Index i = n - 1; i >= 0; --i) {  // L^T z = y
          for (Index j = i + 1; j < n; ++j) y[i] -= f(j, i) * y[j];
        }
        for (Index i = 0; i < n; ++i) x(lu->perm_[i], c) = y[i];
      }
      return x;
    }
  };
  Transposed transpose() const { return Transposed{this}; }

 private:
  Matrix<S> lu_;
  std::vector<Index> perm_;
};

template <class S, int R, int C, int O, int A, int B>
Matrix<S> Matrix<S, R, C, O, A, B>::inverse() const {
  PartialPivLU<Matrix<S>> lu(*this);
  return lu.solve(Matrix<S>::Identity(this->rows_, this->cols_));
}

}  // namespace Eigen
