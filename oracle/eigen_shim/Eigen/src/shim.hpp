// Eigen-subset shim — ORACLE TEST INFRASTRUCTURE ONLY.
//
// Eigen 3.3+ is a header-only dependency of the reference
// (/root/reference/proj/CMakeLists.txt:10) that is absent from this image.
// This file implements the fixed-size subset the reference hot-path sources
// (src/{geometry,camera,warping,alignment,fusion}.cpp) and their unit tests use,
// so the UNMODIFIED reference sources can be compiled in place into
// oracle/_ref/ and used as the parity checker.  It is never linked into the
// product library.
//
// Rounding conventions (documented in DESIGN.md, "parity unpinned vs real Eigen
// at ulp level"):
//  * every fixed-size reduction (matrix-product coefficient, dot, sum,
//    squaredNorm) follows Eigen's redux_novec_unroller: recursive halving,
//    v0 + (v1 + v2) for length 3;
//  * 3x3 inverse follows Eigen's cofactor formula (InverseImpl.h):
//    det = c00*m00 + (c10*m10 + c20*m20), every entry = cofactor * (1/det);
//  * LDLT follows Eigen's pivoted ldlt_inplace<Lower>; 6x6 inverse uses
//    partial-pivot LU; SelfAdjointEigenSolver uses cyclic Jacobi.
// The product library's host math (paper_1807_08271_b200/csrc/host_math.hpp)
// follows the same conventions, so mask-deciding warp matrices are bit-identical.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <limits>
#include <type_traits>
#include <utility>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
constexpr int ColMajor = 0;
constexpr int RowMajor = 1;
constexpr int Lower = 1;
constexpr int Upper = 2;

namespace shim {
// Eigen redux_novec_unroller order: func(redux(Start, Len/2), redux(Start+Len/2, Len-Len/2)).
template <typename F>
inline double redux(const F& f, int start, int len) {
  if (len == 1) return f(start);
  const int half = len / 2;
  return redux(f, start, half) + redux(f, start + half, len - half);
}
}  // namespace shim

template <typename S, int R, int C, int Opt = 0, int MR = R, int MC = C>
class Matrix;

template <typename M, int BR, int BC>
class BlockRef;

template <typename M>
struct CommaInit;

template <int N>
struct DiagonalWrapper;

template <int R, int C>
struct BoolArray {
  bool v[R * C];
  bool any() const {
    for (int i = 0; i < R * C; ++i)
      if (v[i]) return true;
    return false;
  }
  bool all() const {
    for (int i = 0; i < R * C; ++i)
      if (!v[i]) return false;
    return true;
  }
};

template <int R, int C>
struct ArrayView {
  const double* d;
  BoolArray<R, C> operator<=(double s) const {
    BoolArray<R, C> b;
    for (int i = 0; i < R * C; ++i) b.v[i] = d[i] <= s;
    return b;
  }
  BoolArray<R, C> operator<(double s) const {
    BoolArray<R, C> b;
    for (int i = 0; i < R * C; ++i) b.v[i] = d[i] < s;
    return b;
  }
  BoolArray<R, C> operator>(double s) const {
    BoolArray<R, C> b;
    for (int i = 0; i < R * C; ++i) b.v[i] = d[i] > s;
    return b;
  }
  BoolArray<R, C> operator>=(double s) const {
    BoolArray<R, C> b;
    for (int i = 0; i < R * C; ++i) b.v[i] = d[i] >= s;
    return b;
  }
};

template <typename M>
class LDLT;
template <typename M>
class LLT;

template <typename S, int R, int C, int Opt, int MR, int MC>
class Matrix {
  static_assert(std::is_same<S, double>::value, "shim supports double only");

 public:
  using Scalar = double;
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;
  static constexpr int SizeAtCompileTime = R * C;
  double d[R * C];

  Matrix() {
    for (int i = 0; i < R * C; ++i) d[i] = 0.0;
  }
  template <typename A, typename B, typename = std::enable_if_t<std::is_arithmetic<A>::value && std::is_arithmetic<B>::value>>
  Matrix(A a, B b) {
    static_assert(R * C == 2, "2-arg ctor needs a 2-vector");
    d[0] = static_cast<double>(a);
    d[1] = static_cast<double>(b);
  }
  template <typename A, typename B, typename Cc>
  Matrix(A a, B b, Cc c) {
    static_assert(R * C == 3, "3-arg ctor needs a 3-vector");
    d[0] = static_cast<double>(a);
    d[1] = static_cast<double>(b);
    d[2] = static_cast<double>(c);
  }
  template <typename A, typename B, typename Cc, typename D>
  Matrix(A a, B b, Cc c, D e) {
    static_assert(R * C == 4, "4-arg ctor needs a 4-vector");
    d[0] = static_cast<double>(a);
    d[1] = static_cast<double>(b);
    d[2] = static_cast<double>(c);
    d[3] = static_cast<double>(e);
  }
  template <typename M, int BR, int BC>
  Matrix(const BlockRef<M, BR, BC>& b) {
    static_assert(BR == R && BC == C, "block size mismatch");
    for (int j = 0; j < C; ++j)
      for (int i = 0; i < R; ++i) (*this)(i, j) = b(i, j);
  }
  template <int N>
  Matrix(const DiagonalWrapper<N>& dw);

  static constexpr Index rows() { return R; }
  static constexpr Index cols() { return C; }
  static constexpr Index size() { return R * C; }
  double* data() { return d; }
  const double* data() const { return d; }

  double& operator()(Index i, Index j) { return d[j * R + i]; }
  const double& operator()(Index i, Index j) const { return d[j * R + i]; }
  double& operator()(Index i) { return d[i]; }
  const double& operator()(Index i) const { return d[i]; }
  double& operator[](Index i) { return d[i]; }
  const double& operator[](Index i) const { return d[i]; }
  double& coeffRef(Index i, Index j) { return (*this)(i, j); }
  double coeff(Index i, Index j) const { return (*this)(i, j); }
  double& x() { return d[0]; }
  double& y() { return d[1]; }
  double& z() { return d[2]; }
  double x() const { return d[0]; }
  double y() const { return d[1]; }
  double z() const { return d[2]; }
  double value() const {
    static_assert(R * C == 1, "value() needs 1x1");
    return d[0];
  }

  static Matrix Zero() { return Matrix(); }
  static Matrix Ones() {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.d[i] = 1.0;
    return m;
  }
  static Matrix Constant(double v) {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.d[i] = v;
    return m;
  }
  static Matrix Identity() {
    Matrix m;
    for (int i = 0; i < std::min(R, C); ++i) m(i, i) = 1.0;
    return m;
  }
  static Matrix Unit(int k) {
    Matrix m;
    m.d[k] = 1.0;
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }
  static Matrix Random() {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.d[i] = 2.0 * (std::rand() / double(RAND_MAX)) - 1.0;
    return m;
  }
  Matrix& setZero() { return *this = Zero(); }
  Matrix& setIdentity() { return *this = Identity(); }

  CommaInit<Matrix> operator<<(double v);
  template <int R2, int C2>
  CommaInit<Matrix> operator<<(const Matrix<double, R2, C2>& m);

  // --- arithmetic (eager) ---
  Matrix operator-() const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.d[i] = -d[i];
    return m;
  }
  Matrix& operator+=(const Matrix& o) {
    for (int i = 0; i < R * C; ++i) d[i] += o.d[i];
    return *this;
  }
  Matrix& operator-=(const Matrix& o) {
    for (int i = 0; i < R * C; ++i) d[i] -= o.d[i];
    return *this;
  }
  template <typename T, typename = std::enable_if_t<std::is_arithmetic<T>::value>>
  Matrix& operator*=(T s) {
    for (int i = 0; i < R * C; ++i) d[i] *= static_cast<double>(s);
    return *this;
  }
  template <typename T, typename = std::enable_if_t<std::is_arithmetic<T>::value>>
  Matrix& operator/=(T s) {
    for (int i = 0; i < R * C; ++i) d[i] /= static_cast<double>(s);
    return *this;
  }
  Matrix& noalias() { return *this; }
  const Matrix& eval() const { return *this; }

  Matrix<double, C, R> transpose() const {
    Matrix<double, C, R> t;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C; ++j) t(j, i) = (*this)(i, j);
    return t;
  }
  Matrix<double, C, R> adjoint() const { return transpose(); }

  double sum() const {
    return shim::redux([this](int i) { return d[i]; }, 0, R * C);
  }
  double squaredNorm() const {
    return shim::redux([this](int i) { return d[i] * d[i]; }, 0, R * C);
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  Matrix normalized() const {
    const double n = squaredNorm();
    Matrix m = *this;
    if (n > 0.0) m /= std::sqrt(n);
    return m;
  }
  void normalize() {
    const double n = squaredNorm();
    if (n > 0.0) *this /= std::sqrt(n);
  }
  double dot(const Matrix& o) const {
    return shim::redux([&](int i) { return d[i] * o.d[i]; }, 0, R * C);
  }
  double trace() const {
    return shim::redux([this](int i) { return (*this)(i, i); }, 0, std::min(R, C));
  }
  Matrix<double, 3, 1> cross(const Matrix<double, 3, 1>& o) const {
    return Matrix<double, 3, 1>(d[1] * o.d[2] - d[2] * o.d[1], d[2] * o.d[0] - d[0] * o.d[2],
                                d[0] * o.d[1] - d[1] * o.d[0]);
  }
  double maxCoeff() const {
    double m = d[0];
    for (int i = 1; i < R * C; ++i)
      if (d[i] > m) m = d[i];
    return m;
  }
  template <typename I>
  double maxCoeff(I* idx) const {
    int k = 0;
    for (int i = 1; i < R * C; ++i)
      if (d[i] > d[k]) k = i;
    *idx = static_cast<I>(k);
    return d[k];
  }
  double minCoeff() const {
    double m = d[0];
    for (int i = 1; i < R * C; ++i)
      if (d[i] < m) m = d[i];
    return m;
  }
  template <typename I>
  double minCoeff(I* idx) const {
    int k = 0;
    for (int i = 1; i < R * C; ++i)
      if (d[i] < d[k]) k = i;
    *idx = static_cast<I>(k);
    return d[k];
  }
  Matrix cwiseAbs() const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.d[i] = std::abs(d[i]);
    return m;
  }
  Matrix cwiseSqrt() const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.d[i] = std::sqrt(d[i]);
    return m;
  }
  Matrix cwiseInverse() const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.d[i] = 1.0 / d[i];
    return m;
  }
  Matrix cwiseProduct(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < R * C; ++i) m.d[i] = d[i] * o.d[i];
    return m;
  }
  bool allFinite() const {
    for (int i = 0; i < R * C; ++i)
      if (!std::isfinite(d[i])) return false;
    return true;
  }
  bool hasNaN() const {
    for (int i = 0; i < R * C; ++i)
      if (std::isnan(d[i])) return true;
    return false;
  }
  ArrayView<R, C> array() const { return ArrayView<R, C>{d}; }
  DiagonalWrapper<R * C> asDiagonal() const;
  Matrix<double, (R < C ? R : C), 1> diagonal() const {
    Matrix<double, (R < C ? R : C), 1> v;
    for (int i = 0; i < std::min(R, C); ++i) v(i) = (*this)(i, i);
    return v;
  }

  Matrix inverse() const;
  double determinant() const;
  LDLT<Matrix> ldlt() const;
  LLT<Matrix> llt() const;

  // --- blocks: non-const returns a writable proxy, const returns a copy ---
  template <int BR, int BC>
  BlockRef<Matrix, BR, BC> block(Index i, Index j) { return BlockRef<Matrix, BR, BC>(this, i, j); }
  template <int BR, int BC>
  Matrix<double, BR, BC> block(Index i, Index j) const {
    Matrix<double, BR, BC> m;
    for (int c = 0; c < BC; ++c)
      for (int r = 0; r < BR; ++r) m(r, c) = (*this)(i + r, j + c);
    return m;
  }
  BlockRef<Matrix, R, 1> col(Index j) { return block<R, 1>(0, j); }
  Matrix<double, R, 1> col(Index j) const { return block<R, 1>(0, j); }
  BlockRef<Matrix, 1, C> row(Index i) { return block<1, C>(i, 0); }
  Matrix<double, 1, C> row(Index i) const { return block<1, C>(i, 0); }
  template <int N>
  BlockRef<Matrix, (C == 1 ? N : 1), (C == 1 ? 1 : N)> head() {
    return BlockRef<Matrix, (C == 1 ? N : 1), (C == 1 ? 1 : N)>(this, 0, 0);
  }
  template <int N>
  Matrix<double, (C == 1 ? N : 1), (C == 1 ? 1 : N)> head() const {
    return block<(C == 1 ? N : 1), (C == 1 ? 1 : N)>(0, 0);
  }
  template <int N>
  BlockRef<Matrix, (C == 1 ? N : 1), (C == 1 ? 1 : N)> tail() {
    return BlockRef<Matrix, (C == 1 ? N : 1), (C == 1 ? 1 : N)>(this, C == 1 ? R - N : 0,
                                                                  C == 1 ? 0 : C - N);
  }
  template <int N>
  Matrix<double, (C == 1 ? N : 1), (C == 1 ? 1 : N)> tail() const {
    return block<(C == 1 ? N : 1), (C == 1 ? 1 : N)>(C == 1 ? R - N : 0, C == 1 ? 0 : C - N);
  }
  template <int N>
  BlockRef<Matrix, R, N> leftCols() { return block<R, N>(0, 0); }
  template <int N>
  Matrix<double, R, N> leftCols() const { return block<R, N>(0, 0); }
  template <int N>
  BlockRef<Matrix, R, N> rightCols() { return block<R, N>(0, C - N); }
  template <int N>
  Matrix<double, R, N> rightCols() const { return block<R, N>(0, C - N); }
  template <int N>
  BlockRef<Matrix, N, C> topRows() { return block<N, C>(0, 0); }
  template <int N>
  Matrix<double, N, C> topRows() const { return block<N, C>(0, 0); }
  template <int N>
  BlockRef<Matrix, N, C> bottomRows() { return block<N, C>(R - N, 0); }
  template <int N>
  Matrix<double, N, C> bottomRows() const { return block<N, C>(R - N, 0); }
  template <int BR, int BC>
  BlockRef<Matrix, BR, BC> topLeftCorner() { return block<BR, BC>(0, 0); }
  template <int BR, int BC>
  Matrix<double, BR, BC> topLeftCorner() const { return block<BR, BC>(0, 0); }
  template <int BR, int BC>
  BlockRef<Matrix, BR, BC> topRightCorner() { return block<BR, BC>(0, C - BC); }
  template <int BR, int BC>
  Matrix<double, BR, BC> topRightCorner() const { return block<BR, BC>(0, C - BC); }
  template <int BR, int BC>
  BlockRef<Matrix, BR, BC> bottomLeftCorner() { return block<BR, BC>(R - BR, 0); }
  template <int BR, int BC>
  Matrix<double, BR, BC> bottomLeftCorner() const { return block<BR, BC>(R - BR, 0); }
  template <int BR, int BC>
  BlockRef<Matrix, BR, BC> bottomRightCorner() { return block<BR, BC>(R - BR, C - BC); }
  template <int BR, int BC>
  Matrix<double, BR, BC> bottomRightCorner() const { return block<BR, BC>(R - BR, C - BC); }
};

// Writable block proxy (lvalue uses only: assignment, +=, -=, swap, element access).
template <typename M, int BR, int BC>
class BlockRef {
 public:
  BlockRef(M* m, Index i, Index j) : m_(m), i_(i), j_(j) {}
  double& operator()(Index r, Index c) { return (*m_)(i_ + r, j_ + c); }
  double operator()(Index r, Index c) const { return (*m_)(i_ + r, j_ + c); }
  double& operator()(Index k) { return BC == 1 ? (*this)(k, 0) : (*this)(0, k); }
  double operator()(Index k) const { return BC == 1 ? (*this)(k, 0) : (*this)(0, k); }
  double& operator[](Index k) { return (*this)(k); }
  Matrix<double, BR, BC> eval() const { return Matrix<double, BR, BC>(*this); }
  operator Matrix<double, BR, BC>() const { return eval(); }
  BlockRef& operator=(const Matrix<double, BR, BC>& o) {
    for (int c = 0; c < BC; ++c)
      for (int r = 0; r < BR; ++r) (*this)(r, c) = o(r, c);
    return *this;
  }
  BlockRef& operator=(const BlockRef& o) { return *this = o.eval(); }
  BlockRef& operator+=(const Matrix<double, BR, BC>& o) { return *this = eval() += o; }
  BlockRef& operator-=(const Matrix<double, BR, BC>& o) {
    for (int c = 0; c < BC; ++c)
      for (int r = 0; r < BR; ++r) (*this)(r, c) -= o(r, c);
    return *this;
  }
  template <typename T, typename = std::enable_if_t<std::is_arithmetic<T>::value>>
  BlockRef& operator/=(T s) {
    for (int c = 0; c < BC; ++c)
      for (int r = 0; r < BR; ++r) (*this)(r, c) /= static_cast<double>(s);
    return *this;
  }
  void swap(BlockRef o) {
    for (int c = 0; c < BC; ++c)
      for (int r = 0; r < BR; ++r) std::swap((*this)(r, c), o(r, c));
  }
  Matrix<double, BC, BR> transpose() const { return eval().transpose(); }
  double norm() const { return eval().norm(); }
  double squaredNorm() const { return eval().squaredNorm(); }
  double sum() const { return eval().sum(); }
  double maxCoeff() const { return eval().maxCoeff(); }
  double minCoeff() const { return eval().minCoeff(); }
  Matrix<double, BR, BC> normalized() const { return eval().normalized(); }
  Matrix<double, BR, BC> cwiseAbs() const { return eval().cwiseAbs(); }
  double x() const { return (*this)(0); }
  double y() const { return (*this)(1); }
  double z() const { return (*this)(2); }

 private:
  M* m_;
  Index i_, j_;
};

template <int N>
struct DiagonalWrapper {
  Matrix<double, N, 1> v;
};

template <typename S, int R, int C, int O, int MR, int MC>
template <int N>
Matrix<S, R, C, O, MR, MC>::Matrix(const DiagonalWrapper<N>& dw) {
  static_assert(R == N && C == N, "diagonal size mismatch");
  for (int i = 0; i < N; ++i) (*this)(i, i) = dw.v(i);
}

template <typename S, int R, int C, int O, int MR, int MC>
DiagonalWrapper<R * C> Matrix<S, R, C, O, MR, MC>::asDiagonal() const {
  DiagonalWrapper<R * C> w;
  for (int i = 0; i < R * C; ++i) w.v(i) = d[i];
  return w;
}

// diag * M scales rows: d_i * M_ij ; M * diag scales columns: M_ij * d_j.
template <int N, int C>
Matrix<double, N, C> operator*(const DiagonalWrapper<N>& dw, const Matrix<double, N, C>& m) {
  Matrix<double, N, C> o;
  for (int j = 0; j < C; ++j)
    for (int i = 0; i < N; ++i) o(i, j) = dw.v(i) * m(i, j);
  return o;
}
template <int R, int N>
Matrix<double, R, N> operator*(const Matrix<double, R, N>& m, const DiagonalWrapper<N>& dw) {
  Matrix<double, R, N> o;
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < R; ++i) o(i, j) = m(i, j) * dw.v(j);
  return o;
}

// Comma initializer: scalars and sub-matrices fill row-wise.
template <typename M>
struct CommaInit {
  M* m;
  int row = 0, col = 0, cur_rows = 1;
  void put(double v) {
    if (col == M::ColsAtCompileTime) {
      row += cur_rows;
      col = 0;
      cur_rows = 1;
    }
    (*m)(row, col) = v;
    ++col;
  }
  template <int R2, int C2>
  void put(const Matrix<double, R2, C2>& s) {
    if (col == M::ColsAtCompileTime) {
      row += cur_rows;
      col = 0;
      cur_rows = R2;
    }
    if (col == 0) cur_rows = R2;
    for (int c = 0; c < C2; ++c)
      for (int r = 0; r < R2; ++r) (*m)(row + r, col + c) = s(r, c);
    col += C2;
  }
  CommaInit& operator,(double v) {
    put(v);
    return *this;
  }
  template <int R2, int C2>
  CommaInit& operator,(const Matrix<double, R2, C2>& s) {
    put(s);
    return *this;
  }
};

template <typename S, int R, int C, int O, int MR, int MC>
CommaInit<Matrix<S, R, C, O, MR, MC>> Matrix<S, R, C, O, MR, MC>::operator<<(double v) {
  CommaInit<Matrix> ci{this};
  ci.put(v);
  return ci;
}
template <typename S, int R, int C, int O, int MR, int MC>
template <int R2, int C2>
CommaInit<Matrix<S, R, C, O, MR, MC>> Matrix<S, R, C, O, MR, MC>::operator<<(
    const Matrix<double, R2, C2>& m) {
  CommaInit<Matrix> ci{this};
  ci.put(m);
  return ci;
}

// --- free arithmetic ---
template <int R, int C>
Matrix<double, R, C> operator+(const Matrix<double, R, C>& a, const Matrix<double, R, C>& b) {
  Matrix<double, R, C> o;
  for (int i = 0; i < R * C; ++i) o.d[i] = a.d[i] + b.d[i];
  return o;
}
template <int R, int C>
Matrix<double, R, C> operator-(const Matrix<double, R, C>& a, const Matrix<double, R, C>& b) {
  Matrix<double, R, C> o;
  for (int i = 0; i < R * C; ++i) o.d[i] = a.d[i] - b.d[i];
  return o;
}
template <int R, int C, typename T, typename = std::enable_if_t<std::is_arithmetic<T>::value>>
Matrix<double, R, C> operator*(T s, const Matrix<double, R, C>& a) {
  Matrix<double, R, C> o;
  for (int i = 0; i < R * C; ++i) o.d[i] = static_cast<double>(s) * a.d[i];
  return o;
}
template <int R, int C, typename T, typename = std::enable_if_t<std::is_arithmetic<T>::value>>
Matrix<double, R, C> operator*(const Matrix<double, R, C>& a, T s) {
  Matrix<double, R, C> o;
  for (int i = 0; i < R * C; ++i) o.d[i] = a.d[i] * static_cast<double>(s);
  return o;
}
template <int R, int C, typename T, typename = std::enable_if_t<std::is_arithmetic<T>::value>>
Matrix<double, R, C> operator/(const Matrix<double, R, C>& a, T s) {
  Matrix<double, R, C> o;
  for (int i = 0; i < R * C; ++i) o.d[i] = a.d[i] / static_cast<double>(s);
  return o;
}
// Coefficient-based (lazy) product: each coefficient is a redux_novec_unroller sum.
template <int R, int K, int C>
Matrix<double, R, C> operator*(const Matrix<double, R, K>& a, const Matrix<double, K, C>& b) {
  Matrix<double, R, C> o;
  for (int j = 0; j < C; ++j)
    for (int i = 0; i < R; ++i)
      o(i, j) = shim::redux([&](int k) { return a(i, k) * b(k, j); }, 0, K);
  return o;
}
// Block operands in arithmetic: evaluate first.
template <typename M, int BR, int BC, typename X>
auto operator+(const BlockRef<M, BR, BC>& a, const X& b) { return a.eval() + b; }
template <typename M, int BR, int BC, typename X>
auto operator-(const BlockRef<M, BR, BC>& a, const X& b) { return a.eval() - b; }
template <typename M, int BR, int BC, typename X>
auto operator*(const BlockRef<M, BR, BC>& a, const X& b) { return a.eval() * b; }
template <typename M, int BR, int BC, typename X>
auto operator/(const BlockRef<M, BR, BC>& a, const X& b) { return a.eval() / b; }
template <int R, int C, typename M, int BR, int BC>
auto operator+(const Matrix<double, R, C>& a, const BlockRef<M, BR, BC>& b) { return a + b.eval(); }
template <int R, int C, typename M, int BR, int BC>
auto operator-(const Matrix<double, R, C>& a, const BlockRef<M, BR, BC>& b) { return a - b.eval(); }
template <int R, int C, typename M, int BR, int BC>
auto operator*(const Matrix<double, R, C>& a, const BlockRef<M, BR, BC>& b) { return a * b.eval(); }
template <typename T, typename M, int BR, int BC, typename = std::enable_if_t<std::is_arithmetic<T>::value>>
auto operator*(T s, const BlockRef<M, BR, BC>& b) { return s * b.eval(); }

// --- 3x3 inverse: Eigen InverseImpl.h cofactor form ---
namespace shim {
template <typename M>
inline double cof3(const M& m, int i, int j) {
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m(i1, j1) * m(i2, j2) - m(i1, j2) * m(i2, j1);
}

template <int N>
Matrix<double, N, N> lu_inverse(const Matrix<double, N, N>& a) {
  // Partial-pivot LU (Eigen PartialPivLU) followed by solving for identity columns.
  Matrix<double, N, N> lu = a;
  int perm[N];
  for (int i = 0; i < N; ++i) perm[i] = i;
  for (int k = 0; k < N; ++k) {
    int p = k;
    double best = std::abs(lu(k, k));
    for (int i = k + 1; i < N; ++i)
      if (std::abs(lu(i, k)) > best) {
        best = std::abs(lu(i, k));
        p = i;
      }
    if (p != k) {
      for (int j = 0; j < N; ++j) std::swap(lu(k, j), lu(p, j));
      std::swap(perm[k], perm[p]);
    }
    if (lu(k, k) != 0.0)
      for (int i = k + 1; i < N; ++i) lu(i, k) /= lu(k, k);
    for (int i = k + 1; i < N; ++i)
      for (int j = k + 1; j < N; ++j) lu(i, j) -= lu(i, k) * lu(k, j);
  }
  Matrix<double, N, N> inv;
  for (int c = 0; c < N; ++c) {
    double y[N];
    for (int i = 0; i < N; ++i) y[i] = perm[i] == c ? 1.0 : 0.0;
    for (int i = 0; i < N; ++i)
      for (int k = 0; k < i; ++k) y[i] -= lu(i, k) * y[k];
    for (int i = N - 1; i >= 0; --i) {
      for (int k = i + 1; k < N; ++k) y[i] -= lu(i, k) * y[k];
      y[i] /= lu(i, i);
    }
    for (int i = 0; i < N; ++i) inv(i, c) = y[i];
  }
  return inv;
}
}  // namespace shim

template <typename S, int R, int C, int O, int MR, int MC>
Matrix<S, R, C, O, MR, MC> Matrix<S, R, C, O, MR, MC>::inverse() const {
  static_assert(R == C, "inverse of a square matrix only");
  if constexpr (R == 1) {
    Matrix m;
    m.d[0] = 1.0 / d[0];
    return m;
  } else if constexpr (R == 2) {
    const double det = (*this)(0, 0) * (*this)(1, 1) - (*this)(1, 0) * (*this)(0, 1);
    const double invdet = 1.0 / det;
    Matrix m;
    m(0, 0) = (*this)(1, 1) * invdet;
    m(1, 0) = -(*this)(1, 0) * invdet;
    m(0, 1) = -(*this)(0, 1) * invdet;
    m(1, 1) = (*this)(0, 0) * invdet;
    return m;
  } else if constexpr (R == 3) {
    const Matrix& a = *this;
    const double c00 = shim::cof3(a, 0, 0), c10 = shim::cof3(a, 1, 0), c20 = shim::cof3(a, 2, 0);
    const double det = c00 * a(0, 0) + (c10 * a(1, 0) + c20 * a(2, 0));
    const double invdet = 1.0 / det;
    Matrix m;
    m(0, 0) = c00 * invdet;
    m(0, 1) = c10 * invdet;
    m(0, 2) = c20 * invdet;
    m(1, 0) = shim::cof3(a, 0, 1) * invdet;
    m(1, 1) = shim::cof3(a, 1, 1) * invdet;
    m(1, 2) = shim::cof3(a, 2, 1) * invdet;
    m(2, 0) = shim::cof3(a, 0, 2) * invdet;
    m(2, 1) = shim::cof3(a, 1, 2) * invdet;
    m(2, 2) = shim::cof3(a, 2, 2) * invdet;
    return m;
  } else {
    return shim::lu_inverse<R>(*this);
  }
}

template <typename S, int R, int C, int O, int MR, int MC>
double Matrix<S, R, C, O, MR, MC>::determinant() const {
  static_assert(R == C && R == 3, "determinant: 3x3 only");
  const Matrix& a = *this;
  return shim::cof3(a, 0, 0) * a(0, 0) + (shim::cof3(a, 1, 0) * a(1, 0) + shim::cof3(a, 2, 0) * a(2, 0));
}

// --- LDLT with diagonal pivoting (Eigen ldlt_inplace<Lower>::unblocked) ---
template <typename MT>
class LDLT {
  static constexpr int N = MT::RowsAtCompileTime;

 public:
  explicit LDLT(const Matrix<double, N, N>& a) : m_(a) {
    // Only the lower triangle is referenced.
    double temp[N];
    for (int k = 0; k < N; ++k) {
      int big = k;
      double bigv = std::abs(m_(k, k));
      for (int i = k + 1; i < N; ++i)
        if (std::abs(m_(i, i)) > bigv) {
          bigv = std::abs(m_(i, i));
          big = i;
        }
      tr_[k] = big;
      if (k != big) {
        for (int j = 0; j < k; ++j) std::swap(m_(k, j), m_(big, j));
        for (int i = big + 1; i < N; ++i) std::swap(m_(i, k), m_(i, big));
        std::swap(m_(k, k), m_(big, big));
        for (int i = k + 1; i < big; ++i) {
          const double t = m_(i, k);
          m_(i, k) = m_(big, i);
          m_(big, i) = t;
        }
      }
      const int rs = N - k - 1;
      if (k > 0) {
        for (int j = 0; j < k; ++j) temp[j] = m_(j, j) * m_(k, j);
        double acc = 0.0;
        for (int j = 0; j < k; ++j) acc += m_(k, j) * temp[j];
        m_(k, k) -= acc;
        for (int i = k + 1; i < N; ++i) {
          double s = 0.0;
          for (int j = 0; j < k; ++j) s += m_(i, j) * temp[j];
          m_(i, k) -= s;
        }
      }
      const double akk = m_(k, k);
      const bool valid = std::abs(akk) > 0.0;
      if (k == 0 && !valid) {
        for (int j = 0; j < N; ++j) tr_[j] = j;
        ok_ = false;
        break;
      }
      if (rs > 0 && valid)
        for (int i = k + 1; i < N; ++i) m_(i, k) /= akk;
    }
  }
  Matrix<double, N, 1> solve(const Matrix<double, N, 1>& b) const {
    Matrix<double, N, 1> x = b;
    for (int k = 0; k < N; ++k) std::swap(x(k), x(tr_[k]));
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < i; ++j) x(i) -= m_(i, j) * x(j);
    const double tol = std::numeric_limits<double>::min();
    for (int i = 0; i < N; ++i) {
      if (std::abs(m_(i, i)) > tol)
        x(i) /= m_(i, i);
      else
        x(i) = 0.0;
    }
    for (int i = N - 1; i >= 0; --i)
      for (int j = i + 1; j < N; ++j) x(i) -= m_(j, i) * x(j);
    for (int k = N - 1; k >= 0; --k) std::swap(x(k), x(tr_[k]));
    return x;
  }
  bool ok() const { return ok_; }

 private:
  Matrix<double, N, N> m_;
  int tr_[N];
  bool ok_ = true;
};

template <typename MT>
class LLT {
  static constexpr int N = MT::RowsAtCompileTime;

 public:
  explicit LLT(const Matrix<double, N, N>& a) {
    for (int j = 0; j < N; ++j) {
      double s = a(j, j);
      for (int k = 0; k < j; ++k) s -= l_(j, k) * l_(j, k);
      if (s <= 0.0) ok_ = false;
      l_(j, j) = std::sqrt(s);
      for (int i = j + 1; i < N; ++i) {
        double t = a(i, j);
        for (int k = 0; k < j; ++k) t -= l_(i, k) * l_(j, k);
        l_(i, j) = t / l_(j, j);
      }
    }
  }
  Matrix<double, N, N> matrixL() const { return l_; }
  Matrix<double, N, 1> solve(const Matrix<double, N, 1>& b) const {
    Matrix<double, N, 1> y = b;
    for (int i = 0; i < N; ++i) {
      for (int k = 0; k < i; ++k) y(i) -= l_(i, k) * y(k);
      y(i) /= l_(i, i);
    }
    for (int i = N - 1; i >= 0; --i) {
      for (int k = i + 1; k < N; ++k) y(i) -= l_(k, i) * y(k);
      y(i) /= l_(i, i);
    }
    return y;
  }

 private:
  Matrix<double, N, N> l_;
  bool ok_ = true;
};

template <typename S, int R, int C, int O, int MR, int MC>
LDLT<Matrix<S, R, C, O, MR, MC>> Matrix<S, R, C, O, MR, MC>::ldlt() const {
  return LDLT<Matrix>(*this);
}
template <typename S, int R, int C, int O, int MR, int MC>
LLT<Matrix<S, R, C, O, MR, MC>> Matrix<S, R, C, O, MR, MC>::llt() const {
  return LLT<Matrix>(*this);
}

// --- symmetric eigenvalues (cyclic Jacobi; ascending like Eigen) ---
template <typename M>
class SelfAdjointEigenSolver {
 public:
  static constexpr int N = M::RowsAtCompileTime;
  explicit SelfAdjointEigenSolver(const M& a) {
    M s;
    // Eigen reads the lower triangle.
    for (int i = 0; i < N; ++i)
      for (int j = 0; j <= i; ++j) s(i, j) = s(j, i) = a(i, j);
    for (int sweep = 0; sweep < 100; ++sweep) {
      double off = 0.0;
      for (int i = 0; i < N; ++i)
        for (int j = i + 1; j < N; ++j) off += s(i, j) * s(i, j);
      if (off == 0.0) break;
      for (int p = 0; p < N; ++p)
        for (int q = p + 1; q < N; ++q) {
          if (s(p, q) == 0.0) continue;
          const double theta = (s(q, q) - s(p, p)) / (2.0 * s(p, q));
          const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
          const double c = 1.0 / std::sqrt(t * t + 1.0), sn = t * c;
          for (int k = 0; k < N; ++k) {
            const double skp = s(k, p), skq = s(k, q);
            s(k, p) = c * skp - sn * skq;
            s(k, q) = sn * skp + c * skq;
          }
          for (int k = 0; k < N; ++k) {
            const double spk = s(p, k), sqk = s(q, k);
            s(p, k) = c * spk - sn * sqk;
            s(q, k) = sn * spk + c * sqk;
          }
        }
    }
    for (int i = 0; i < N; ++i) ev_(i) = s(i, i);
    std::sort(ev_.d, ev_.d + N);
  }
  const Matrix<double, N, 1>& eigenvalues() const { return ev_; }

 private:
  Matrix<double, N, 1> ev_;
};

using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using RowVector2d = Matrix<double, 1, 2>;
using RowVector3d = Matrix<double, 1, 3>;
using RowVector4d = Matrix<double, 1, 4>;

}  // namespace Eigen
