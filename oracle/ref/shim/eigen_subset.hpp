// ORACLE (test infrastructure): Eigen-subset shim used ONLY to compile the
// unmodified reference sources (/root/reference/proj/src/*.cpp and its tests)
// into oracle/_ref/.  Eigen is not installed in this image and there is no
// network; the reference's CMake asks for an unpinned Eigen3
// (proj/CMakeLists.txt:13).  This header covers exactly the API the reference
// uses (SURVEY.md §8(c) enumerates it) with eager evaluation in Eigen 3.4's
// per-coefficient operation order:
//   * coefficient-wise ops and scalar ops as written (x / s divides, it does
//     not multiply by a reciprocal: scalar_quotient_op);
//   * products res(i,j) = ((a(i,0) b(0,j) + a(i,1) b(1,j)) + a(i,2) b(2,j)),
//     the order of both the coefficient-based lazy product and its packet
//     form (pmul then pmadd, no FMA contraction: -ffp-contract=off);
//   * sum / dot / squaredNorm as left-to-right reductions (the unrolled
//     redux for fixed sizes; dynamic-size vectors only appear in tests);
//   * norm = sqrt(squaredNorm), normalized = x / sqrt(squaredNorm) (0 stays);
//   * cross as in Eigen's cross3_impl, 3x3 determinant as
//     bruteforce_det3_helper (expansion along column 0);
//   * JacobiSVD<Matrix3d> (two-sided Jacobi, real_2x2_jacobi_svd +
//     makeJacobi, singular values sorted descending with U/V columns),
//     LDLT (ldlt_inplace<Lower>::unblocked, pseudo-inverse of D with the
//     smallest-normal tolerance), PartialPivLU (unblocked_lu, row swaps),
//     AngleAxis / Quaternion toRotationMatrix — restated from Eigen 3.4's
//     published algorithms (the same restatements as oracle/wf_oracle.cpp).
// Bitwise identity with a real Eigen build is NOT pinned (no Eigen here); the
// orders above are the ones Eigen 3.4 uses for these fixed sizes on x86-64
// without FMA.  Like Eigen/Core, it pulls in the C/C++ headers Eigen
// includes transitively (<cstdint>, <cstring>, <string>, ...), which the
// reference headers rely on.
#pragma once

// Reduction order of small products and traces (see the product section):
// 0 = natural left-to-right (the order oracle/wf_oracle.cpp and the CUDA
// path use; default), 1 = Eigen 3.4 as read from its source (tree order for
// strided lhs rows, packet order for a transposed lhs), 2 = tree order for
// every product and trace.
#ifndef WF_SHIM_ORDER
#define WF_SHIM_ORDER 0
#endif

#include <algorithm>
#include <array>
#include <cassert>
#include <cfloat>
#include <climits>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <iosfwd>
#include <string>
#include <initializer_list>
#include <limits>
#include <ostream>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum DecompositionOptions { ComputeFullU = 0x04, ComputeThinU = 0x08, ComputeFullV = 0x10, ComputeThinV = 0x20 };

template <typename T, int R, int C>
class Matrix;
template <typename T, int R, int C>
class ArrayW;
template <typename T, int R, int C>
struct TransposeView;

namespace detail {
template <typename T, int R, int C>
struct Storage {  // fixed size
  std::array<T, std::size_t(R * C)> d{};
  static constexpr Index rows() { return R; }
  static constexpr Index cols() { return C; }
  void resize(Index r, Index c) { (void)r, (void)c; assert(r == R && c == C); }
};
template <typename T, int R, int C>
struct DynStorage {
  std::vector<T> d;
  Index r = (R > 0 ? R : 0), c = (C > 0 ? C : 0);
  Index rows() const { return r; }
  Index cols() const { return c; }
  void resize(Index rr, Index cc) {
    r = rr;
    c = cc;
    d.assign(std::size_t(rr * cc), T(0));
  }
};
template <typename T, int R, int C>
using StorageFor = std::conditional_t<(R > 0 && C > 0), Storage<T, R, C>, DynStorage<T, R, C>>;

template <typename S>
using EnableScalar = std::enable_if_t<std::is_arithmetic_v<S>, int>;

// Eigen 3.4 redux_novec_unroller: sum(start, n) = sum(start, n/2) +
// sum(start + n/2, n - n/2) — the order of every unrolled reduction over
// coefficients without packet access (e.g. a row of a column-major matrix)
template <typename T, typename F>
T tree_sum_at(Index start, Index n, const F& f) {
  if (n == 1) return f(start);
  const Index h = n / 2;
  return tree_sum_at<T>(start, h, f) + tree_sum_at<T>(start + h, n - h, f);
}
template <typename T, typename F>
T tree_sum(Index n, const F& f) {
  return tree_sum_at<T>(0, n, f);
}
}  // namespace detail

// lazy transpose: Eigen keeps `m.transpose()` as an expression inside a
// product, so its rows are contiguous and the product's coefficient
// reduction is packet-vectorised ((t0 + t1) + t2); assigned to a matrix it
// is a plain transposed copy
template <typename T, int R, int C>
struct TransposeView {
  Matrix<T, R, C> m;
  operator Matrix<T, R, C>() const { return m; }
  T operator()(Index i, Index j) const { return m(i, j); }
  Index rows() const { return m.rows(); }
  Index cols() const { return m.cols(); }
  Matrix<T, C, R> transpose() const { return m.transposed(); }
  T trace() const { return m.trace(); }
  Matrix<T, R, C> eval() const { return m; }
};

// writable view of a sub-block (col, block<>, head<>, segment<> on a
// non-const matrix); reads convert to an owning Matrix
template <typename T, int R, int C, typename Parent>
class BlockRef {
 public:
  BlockRef(Parent& p, Index r0, Index c0) : p_(p), r0_(r0), c0_(c0) {}
  T& operator()(Index i, Index j) { return p_(r0_ + i, c0_ + j); }
  T operator()(Index i, Index j) const { return p_(r0_ + i, c0_ + j); }
  Matrix<T, R, C> eval() const {
    Matrix<T, R, C> m;
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) m(i, j) = (*this)(i, j);
    return m;
  }
  operator Matrix<T, R, C>() const { return eval(); }
  BlockRef& operator=(const Matrix<T, R, C>& m) {
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) (*this)(i, j) = m(i, j);
    return *this;
  }
  BlockRef& operator=(const BlockRef& o) { return *this = o.eval(); }
  BlockRef& operator+=(const Matrix<T, R, C>& m) {
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) (*this)(i, j) = (*this)(i, j) + m(i, j);
    return *this;
  }
  BlockRef& operator-=(const Matrix<T, R, C>& m) {
    for (Index j = 0; j < C; ++j)
      for (Index i = 0; i < R; ++i) (*this)(i, j) = (*this)(i, j) - m(i, j);
    return *this;
  }
  T squaredNorm() const { return eval().squaredNorm(); }
  T norm() const { return eval().norm(); }

 private:
  Parent& p_;
  Index r0_, c0_;
};

template <typename T, int R, int C>
class Matrix {
  detail::StorageFor<T, R, C> s_;

 public:
  using Scalar = T;
  static constexpr int RowsAtCompileTime = R, ColsAtCompileTime = C;
  static constexpr bool IsVector = (R == 1 || C == 1);

  Matrix() {
    if constexpr (R > 0 && C > 0) s_.d.fill(T(0));
  }
  // dynamic: VectorXd b(n) / MatrixXd a(r, c)
  template <int RR = R, int CC = C, std::enable_if_t<(RR < 0 || CC < 0), int> = 0>
  explicit Matrix(Index n) {
    if constexpr (C == 1)
      s_.resize(n, 1);
    else if constexpr (R == 1)
      s_.resize(1, n);
    else
      s_.resize(n, n);
  }
  template <int RR = R, int CC = C, std::enable_if_t<(RR < 0 || CC < 0), int> = 0>
  Matrix(Index r, Index c) {
    s_.resize(r, c);
  }
  // fixed-size vector constructors (Vector2d(x, y), Vector3d(x, y, z)); like
  // Eigen they accept any arithmetic arguments and cast to the scalar
  template <typename A, typename B, int RR = R, int CC = C,
            std::enable_if_t<(RR * CC == 2 && std::is_arithmetic_v<A> && std::is_arithmetic_v<B>), int> = 0>
  Matrix(A x, B y) {
    s_.d[0] = T(x);
    s_.d[1] = T(y);
  }
  template <typename A, typename B, typename D, int RR = R, int CC = C,
            std::enable_if_t<(RR * CC == 3 && std::is_arithmetic_v<A>), int> = 0>
  Matrix(A x, B y, D z) {
    s_.d[0] = T(x);
    s_.d[1] = T(y);
    s_.d[2] = T(z);
  }
  template <typename A, typename B, typename D, typename E, int RR = R, int CC = C,
            std::enable_if_t<(RR * CC == 4 && std::is_arithmetic_v<A>), int> = 0>
  Matrix(A x, B y, D z, E w) {
    s_.d[0] = T(x);
    s_.d[1] = T(y);
    s_.d[2] = T(z);
    s_.d[3] = T(w);
  }
  // conversion between fixed and dynamic shapes (VectorXd <-> Vector3d)
  template <int R2, int C2, std::enable_if_t<(R2 != R || C2 != C), int> = 0>
  Matrix(const Matrix<T, R2, C2>& o) {
    if constexpr (!(R > 0 && C > 0)) s_.resize(o.rows(), o.cols());
    assert(o.rows() == rows() && o.cols() == cols());
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) (*this)(i, j) = o(i, j);
  }
  template <int R2, int C2, typename P>
  Matrix(const BlockRef<T, R2, C2, P>& b) : Matrix(b.eval()) {}
  Matrix(const ArrayW<T, R, C>& a);  // array -> matrix (Eigen allows on construction)

  Index rows() const { return s_.rows(); }
  Index cols() const { return s_.cols(); }
  Index size() const { return rows() * cols(); }
  T* data() { return s_.d.data(); }
  const T* data() const { return s_.d.data(); }

  // column-major, as Eigen's default
  T& operator()(Index i, Index j) { return s_.d[std::size_t(i + j * rows())]; }
  const T& operator()(Index i, Index j) const { return s_.d[std::size_t(i + j * rows())]; }
  T& operator()(Index i) { return s_.d[std::size_t(i)]; }
  const T& operator()(Index i) const { return s_.d[std::size_t(i)]; }
  T& operator[](Index i) { return s_.d[std::size_t(i)]; }
  const T& operator[](Index i) const { return s_.d[std::size_t(i)]; }
  T& coeffRef(Index i, Index j) { return (*this)(i, j); }
  T coeff(Index i, Index j) const { return (*this)(i, j); }
  T coeff(Index i) const { return (*this)(i); }
  T& x() { return s_.d[0]; }
  T& y() { return s_.d[1]; }
  T& z() { return s_.d[2]; }
  T& w() { return s_.d[3]; }
  const T& x() const { return s_.d[0]; }
  const T& y() const { return s_.d[1]; }
  const T& z() const { return s_.d[2]; }
  const T& w() const { return s_.d[3]; }

  static Matrix Zero() { return Constant(T(0)); }
  static Matrix Zero(Index n) {
    Matrix m(n);
    return m;
  }
  static Matrix Zero(Index r, Index c) { return Matrix(r, c); }
  static Matrix Ones() { return Constant(T(1)); }
  static Matrix Constant(T v) {
    Matrix m;
    for (auto& e : m.s_.d) e = v;
    return m;
  }
  static Matrix Identity() {
    Matrix m = Zero();
    for (Index i = 0; i < std::min(m.rows(), m.cols()); ++i) m(i, i) = T(1);
    return m;
  }
  static Matrix Unit(Index k) {
    Matrix m = Zero();
    m(k) = T(1);
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }

  Matrix& setZero() {
    for (auto& e : s_.d) e = T(0);
    return *this;
  }
  Matrix& setIdentity() { return *this = Identity(); }
  Matrix& setConstant(T v) {
    for (auto& e : s_.d) e = v;
    return *this;
  }
  void fill(T v) { setConstant(v); }

  // ---- comma initializer (fills row by row) ----
  struct CommaInit {
    Matrix& m;
    Index k;
    CommaInit& operator,(T v) {
      m(k / m.cols(), k % m.cols()) = v;
      ++k;
      return *this;
    }
  };
  template <typename S, detail::EnableScalar<S> = 0>
  CommaInit operator<<(S v) {
    (*this)(0, 0) = T(v);
    return CommaInit{*this, 1};
  }

  // ---- coefficient-wise arithmetic ----
  Matrix operator-() const {
    Matrix r = *this;
    for (auto& e : r.s_.d) e = -e;
    return r;
  }
  Matrix& operator+=(const Matrix& o) {
    for (std::size_t i = 0; i < s_.d.size(); ++i) s_.d[i] = s_.d[i] + o.s_.d[i];
    return *this;
  }
  Matrix& operator-=(const Matrix& o) {
    for (std::size_t i = 0; i < s_.d.size(); ++i) s_.d[i] = s_.d[i] - o.s_.d[i];
    return *this;
  }
  template <typename S, detail::EnableScalar<S> = 0>
  Matrix& operator*=(S s) {
    for (auto& e : s_.d) e = e * T(s);
    return *this;
  }
  template <typename S, detail::EnableScalar<S> = 0>
  Matrix& operator/=(S s) {
    for (auto& e : s_.d) e = e / T(s);
    return *this;
  }
  friend Matrix operator+(Matrix a, const Matrix& b) { return a += b; }
  friend Matrix operator-(Matrix a, const Matrix& b) { return a -= b; }
  template <typename S, detail::EnableScalar<S> = 0>
  friend Matrix operator*(Matrix a, S s) {
    for (auto& e : a.s_.d) e = e * T(s);
    return a;
  }
  template <typename S, detail::EnableScalar<S> = 0>
  friend Matrix operator*(S s, Matrix a) {
    for (auto& e : a.s_.d) e = T(s) * e;
    return a;
  }
  template <typename S, detail::EnableScalar<S> = 0>
  friend Matrix operator/(Matrix a, S s) {
    for (auto& e : a.s_.d) e = e / T(s);
    return a;
  }
  friend bool operator==(const Matrix& a, const Matrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
    for (std::size_t i = 0; i < a.s_.d.size(); ++i)
      if (!(a.s_.d[i] == b.s_.d[i])) return false;
    return true;
  }
  friend bool operator!=(const Matrix& a, const Matrix& b) { return !(a == b); }

  Matrix cwiseProduct(const Matrix& o) const {
    Matrix r = *this;
    for (std::size_t i = 0; i < s_.d.size(); ++i) r.s_.d[i] = s_.d[i] * o.s_.d[i];
    return r;
  }
  Matrix cwiseQuotient(const Matrix& o) const {
    Matrix r = *this;
    for (std::size_t i = 0; i < s_.d.size(); ++i) r.s_.d[i] = s_.d[i] / o.s_.d[i];
    return r;
  }
  Matrix cwiseAbs() const {
    Matrix r = *this;
    for (auto& e : r.s_.d) e = std::abs(e);
    return r;
  }
  // Eigen's scalar_max_op: (a < b) ? b : a
  Matrix cwiseMax(T v) const {
    Matrix r = *this;
    for (auto& e : r.s_.d) e = (e < v) ? v : e;
    return r;
  }
  Matrix cwiseMax(const Matrix& o) const {
    Matrix r = *this;
    for (std::size_t i = 0; i < s_.d.size(); ++i) r.s_.d[i] = (s_.d[i] < o.s_.d[i]) ? o.s_.d[i] : s_.d[i];
    return r;
  }
  Matrix cwiseMin(T v) const {
    Matrix r = *this;
    for (auto& e : r.s_.d) e = (v < e) ? v : e;
    return r;
  }
  Matrix cwiseMin(const Matrix& o) const {
    Matrix r = *this;
    for (std::size_t i = 0; i < s_.d.size(); ++i) r.s_.d[i] = (o.s_.d[i] < s_.d[i]) ? o.s_.d[i] : s_.d[i];
    return r;
  }

  // ---- reductions (left to right, as the unrolled redux) ----
  T sum() const {
    T acc = s_.d[0];
    for (std::size_t i = 1; i < s_.d.size(); ++i) acc = acc + s_.d[i];
    return acc;
  }
  T prod() const {
    T acc = s_.d[0];
    for (std::size_t i = 1; i < s_.d.size(); ++i) acc = acc * s_.d[i];
    return acc;
  }
  T mean() const { return sum() / T(size()); }
  T maxCoeff() const {
    T m = s_.d[0];
    for (std::size_t i = 1; i < s_.d.size(); ++i)
      if (s_.d[i] > m) m = s_.d[i];
    return m;
  }
  T minCoeff() const {
    T m = s_.d[0];
    for (std::size_t i = 1; i < s_.d.size(); ++i)
      if (s_.d[i] < m) m = s_.d[i];
    return m;
  }
  T maxCoeff(Index* at) const {
    Index k = 0;
    for (Index i = 1; i < size(); ++i)
      if (s_.d[i] > s_.d[k]) k = i;
    *at = k;
    return s_.d[k];
  }
  T dot(const Matrix& o) const {
    T acc = s_.d[0] * o.s_.d[0];
    for (std::size_t i = 1; i < s_.d.size(); ++i) acc = acc + s_.d[i] * o.s_.d[i];
    return acc;
  }
  T squaredNorm() const { return dot(*this); }
  T norm() const { return std::sqrt(squaredNorm()); }
  Matrix normalized() const {
    const T n = squaredNorm();
    if (n == T(0)) return *this;
    return *this / std::sqrt(n);
  }
  void normalize() {
    const T n = squaredNorm();
    if (n > T(0)) *this /= std::sqrt(n);
  }
  // the diagonal is strided (no packet access): redux_novec_unroller order
  T trace() const {
#if WF_SHIM_ORDER == 0
    T acc = (*this)(0, 0);
    for (Index i = 1; i < std::min(rows(), cols()); ++i) acc = acc + (*this)(i, i);
    return acc;
#else
    return detail::tree_sum<T>(std::min(rows(), cols()), [&](Index i) { return (*this)(i, i); });
#endif
  }
  Matrix<T, (R > 0 && C > 0 ? (R < C ? R : C) : Dynamic), 1> diagonal() const {
    Matrix<T, (R > 0 && C > 0 ? (R < C ? R : C) : Dynamic), 1> d;
    if constexpr (!(R > 0 && C > 0)) d = Matrix<T, Dynamic, 1>(std::min(rows(), cols()));
    for (Index i = 0; i < std::min(rows(), cols()); ++i) d(i) = (*this)(i, i);
    return d;
  }
  Matrix<T, C, R> transposed() const {
    Matrix<T, C, R> t;
    if constexpr (!(R > 0 && C > 0)) t = Matrix<T, C, R>(cols(), rows());
    for (Index j = 0; j < cols(); ++j)
      for (Index i = 0; i < rows(); ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  TransposeView<T, C, R> transpose() const { return TransposeView<T, C, R>{transposed()}; }
  Matrix cross(const Matrix& b) const {
    static_assert(R * C == 3, "cross needs 3-vectors");
    const Matrix& a = *this;
    return Matrix(a(1) * b(2) - a(2) * b(1), a(2) * b(0) - a(0) * b(2), a(0) * b(1) - a(1) * b(0));
  }
  T determinant() const;
  Matrix inverse() const;

  template <typename U>
  Matrix<U, R, C> cast() const {
    Matrix<U, R, C> r;
    if constexpr (!(R > 0 && C > 0)) r = Matrix<U, R, C>(rows(), cols());
    for (Index i = 0; i < size(); ++i) r(i) = U(s_.d[std::size_t(i)]);
    return r;
  }

  ArrayW<T, R, C> array() const;

  // ---- blocks ----
  Matrix<T, R, 1> col(Index j) const {
    Matrix<T, R, 1> c;
    for (Index i = 0; i < R; ++i) c(i) = (*this)(i, j);
    return c;
  }
  BlockRef<T, R, 1, Matrix> col(Index j) { return BlockRef<T, R, 1, Matrix>(*this, 0, j); }
  Matrix<T, 1, C> row(Index i) const {
    Matrix<T, 1, C> r;
    for (Index j = 0; j < C; ++j) r(j) = (*this)(i, j);
    return r;
  }
  BlockRef<T, 1, C, Matrix> row(Index i) { return BlockRef<T, 1, C, Matrix>(*this, i, 0); }
  template <int BR, int BC>
  Matrix<T, BR, BC> block(Index i, Index j) const {
    Matrix<T, BR, BC> b;
    for (Index c = 0; c < BC; ++c)
      for (Index r = 0; r < BR; ++r) b(r, c) = (*this)(i + r, j + c);
    return b;
  }
  template <int BR, int BC>
  BlockRef<T, BR, BC, Matrix> block(Index i, Index j) {
    return BlockRef<T, BR, BC, Matrix>(*this, i, j);
  }
  // vector segments
  template <int N>
  Matrix<T, N, 1> segment(Index i) const {
    Matrix<T, N, 1> v;
    for (Index k = 0; k < N; ++k) v(k) = (*this)(i + k);
    return v;
  }
  template <int N>
  BlockRef<T, N, 1, Matrix> segment(Index i) {
    static_assert(C == 1, "segment on column vectors");
    return BlockRef<T, N, 1, Matrix>(*this, i, 0);
  }
  template <int N>
  Matrix<T, N, 1> head() const {
    return segment<N>(0);
  }
  template <int N>
  BlockRef<T, N, 1, Matrix> head() {
    return segment<N>(0);
  }
  template <int N>
  Matrix<T, N, 1> tail() const {
    return segment<N>(size() - N);
  }
  template <int N>
  BlockRef<T, N, 1, Matrix> tail() {
    return segment<N>(size() - N);
  }

  struct LDLTd;
  struct PartialPivLUd;
  LDLTd ldlt() const { return LDLTd(*this); }
  PartialPivLUd partialPivLu() const { return PartialPivLUd(*this); }

  template <typename U, int R2, int C2>
  friend class Matrix;
};

// ---- products -----------------------------------------------------------------
// Small fixed-size products are Eigen's lazy coefficient-based product:
// res(i,j) = (lhs.row(i)^T .cwiseProduct(rhs.col(j))).sum().  The 3x3 / 3x1
// destinations are not vectorised (size 3 is not a packet multiple), so the
// reduction order depends on whether lhs.row(i) is contiguous:
//  * plain (column-major) lhs: strided row, no packet access ->
//    redux_novec_unroller: t0 + (t1 + t2);
//  * lhs = m.transpose() (a view): contiguous row and column ->
//    LinearVectorized redux: predux(t0, t1) + t2 = (t0 + t1) + t2.
template <bool Packet, typename T, int R, int K, int K2, int C>
Matrix<T, R, C> product(const Matrix<T, R, K>& a, const Matrix<T, K2, C>& b) {
  static_assert(K == K2 || K < 0 || K2 < 0, "inner dimensions");
  Matrix<T, R, C> r;
  if constexpr (!(R > 0 && C > 0)) r = Matrix<T, R, C>(a.rows(), b.cols());
  const Index kk = a.cols();
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) {
      const bool natural = WF_SHIM_ORDER == 0 || (WF_SHIM_ORDER == 1 && Packet);
      if (natural || kk < 3) {
        T acc = a(i, 0) * b(0, j);
        for (Index k = 1; k < kk; ++k) acc = acc + a(i, k) * b(k, j);
        r(i, j) = acc;
      } else {
        r(i, j) = detail::tree_sum<T>(kk, [&](Index k) { return a(i, k) * b(k, j); });
      }
    }
  return r;
}
template <typename T, int R, int K, int K2, int C>
Matrix<T, R, C> operator*(const Matrix<T, R, K>& a, const Matrix<T, K2, C>& b) {
  return product<false>(a, b);
}
template <typename T, int R, int K, int K2, int C>
Matrix<T, R, C> operator*(const TransposeView<T, R, K>& a, const Matrix<T, K2, C>& b) {
  return product<true>(a.m, b);
}
template <typename T, int R, int K, int K2, int C>
Matrix<T, R, C> operator*(const Matrix<T, R, K>& a, const TransposeView<T, K2, C>& b) {
  return product<false>(a, b.m);
}
template <typename T, int R, int K, int K2, int C>
Matrix<T, R, C> operator*(const TransposeView<T, R, K>& a, const TransposeView<T, K2, C>& b) {
  return product<false>(a.m, b.m);
}
template <typename T, int R, int C, typename S, detail::EnableScalar<S> = 0>
Matrix<T, R, C> operator*(S s, const TransposeView<T, R, C>& a) {
  return s * a.m;
}
template <typename T, int R, int C, typename S, detail::EnableScalar<S> = 0>
Matrix<T, R, C> operator*(const TransposeView<T, R, C>& a, S s) {
  return a.m * s;
}
template <typename T, int R, int C, typename P>
Matrix<T, R, C> operator+(const BlockRef<T, R, C, P>& a, const Matrix<T, R, C>& b) {
  return a.eval() + b;
}
template <typename T, int R, int C, typename P>
Matrix<T, R, C> operator+(const Matrix<T, R, C>& a, const BlockRef<T, R, C, P>& b) {
  return a + b.eval();
}
template <typename T, int R, int C, typename P>
Matrix<T, R, C> operator-(const BlockRef<T, R, C, P>& a, const Matrix<T, R, C>& b) {
  return a.eval() - b;
}
template <typename T, int R, int C, typename P>
Matrix<T, R, C> operator-(const Matrix<T, R, C>& a, const BlockRef<T, R, C, P>& b) {
  return a - b.eval();
}

// bruteforce_det3_helper(m, a, b, c) = m(a,0) * (m(b,1) m(c,2) - m(b,2) m(c,1))
template <typename T, int R, int C>
T Matrix<T, R, C>::determinant() const {
  const Matrix& m = *this;
  if (rows() == 1) return m(0, 0);
  if (rows() == 2) return m(0, 0) * m(1, 1) - m(1, 0) * m(0, 1);
  assert(rows() == 3 && cols() == 3);
  auto h = [&](int a, int b, int c) { return m(a, 0) * (m(b, 1) * m(c, 2) - m(b, 2) * m(c, 1)); };
  return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
}

// compute_inverse<3x3>: cofactors / determinant
template <typename T, int R, int C>
Matrix<T, R, C> Matrix<T, R, C>::inverse() const {
  const Matrix& m = *this;
  assert(rows() == 3 && cols() == 3);
  auto cof = [&](int i, int j) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
    return m(i1, j1) * m(i2, j2) - m(i1, j2) * m(i2, j1);
  };
  Matrix c;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) c(j, i) = cof(i, j);  // adjugate
  const T det = m(0, 0) * c(0, 0) + m(0, 1) * c(1, 0) + m(0, 2) * c(2, 0);
  return c / det;
}

// ---- Array view: coefficient-wise comparisons, floor, scalar offsets ------
template <typename T, int R, int C>
class ArrayW {
 public:
  Matrix<T, R, C> m;
  explicit ArrayW(const Matrix<T, R, C>& x) : m(x) {}
  struct Bools {
    std::vector<bool> b;
    bool all() const { return std::all_of(b.begin(), b.end(), [](bool v) { return v; }); }
    bool any() const { return std::any_of(b.begin(), b.end(), [](bool v) { return v; }); }
    Index count() const { return Index(std::count(b.begin(), b.end(), true)); }
  };
  template <typename F>
  Bools cmp(F f) const {
    Bools r;
    for (Index i = 0; i < m.size(); ++i) r.b.push_back(f(i));
    return r;
  }
#define WF_SHIM_CMP(OP)                                                                       \
  template <typename S, detail::EnableScalar<S> = 0>                                          \
  Bools operator OP(S s) const {                                                              \
    return cmp([&](Index i) { return m(i) OP T(s); });                                        \
  }                                                                                           \
  Bools operator OP(const ArrayW& o) const { return cmp([&](Index i) { return m(i) OP o.m(i); }); }
  WF_SHIM_CMP(<)
  WF_SHIM_CMP(<=)
  WF_SHIM_CMP(>)
  WF_SHIM_CMP(>=)
  WF_SHIM_CMP(==)
  WF_SHIM_CMP(!=)
#undef WF_SHIM_CMP
  template <typename S, detail::EnableScalar<S> = 0>
  ArrayW operator+(S s) const {
    ArrayW r = *this;
    for (Index i = 0; i < m.size(); ++i) r.m(i) = m(i) + T(s);
    return r;
  }
  template <typename S, detail::EnableScalar<S> = 0>
  ArrayW operator-(S s) const {
    ArrayW r = *this;
    for (Index i = 0; i < m.size(); ++i) r.m(i) = m(i) - T(s);
    return r;
  }
  ArrayW operator*(const ArrayW& o) const { return ArrayW(m.cwiseProduct(o.m)); }
  ArrayW operator/(const ArrayW& o) const { return ArrayW(m.cwiseQuotient(o.m)); }
  ArrayW operator+(const ArrayW& o) const { return ArrayW(m + o.m); }
  ArrayW operator-(const ArrayW& o) const { return ArrayW(m - o.m); }
  ArrayW floor() const {
    ArrayW r = *this;
    for (Index i = 0; i < m.size(); ++i) r.m(i) = std::floor(m(i));
    return r;
  }
  ArrayW abs() const { return ArrayW(m.cwiseAbs()); }
  ArrayW square() const { return ArrayW(m.cwiseProduct(m)); }
  ArrayW sqrt() const {
    ArrayW r = *this;
    for (Index i = 0; i < m.size(); ++i) r.m(i) = std::sqrt(m(i));
    return r;
  }
  ArrayW max(T v) const { return ArrayW(m.cwiseMax(v)); }
  ArrayW min(T v) const { return ArrayW(m.cwiseMin(v)); }
  T sum() const { return m.sum(); }
  T maxCoeff() const { return m.maxCoeff(); }
  T minCoeff() const { return m.minCoeff(); }
  Matrix<T, R, C> matrix() const { return m; }
  template <typename U>
  ArrayW<U, R, C> cast() const {
    return ArrayW<U, R, C>(m.template cast<U>());
  }
};
template <typename T, int R, int C>
Matrix<T, R, C>::Matrix(const ArrayW<T, R, C>& a) : Matrix(a.m) {}
template <typename T, int R, int C>
ArrayW<T, R, C> Matrix<T, R, C>::array() const {
  return ArrayW<T, R, C>(*this);
}

// ---- LDLT (Eigen 3.4 ldlt_inplace<Lower>::unblocked + _solve_impl) --------
template <typename T, int R, int C>
struct Matrix<T, R, C>::LDLTd {
  Matrix a;
  std::vector<Index> tr;
  explicit LDLTd(const Matrix& m) : a(m) {
    const Index n = a.rows();
    tr.assign(std::size_t(n), 0);
    std::vector<T> temp(static_cast<std::size_t>(n) + 0);
    for (Index k = 0; k < n; ++k) {
      Index big = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(a(i, i)) > std::abs(a(big, big))) big = i;
      tr[std::size_t(k)] = big;
      if (big != k) {
        for (Index j = 0; j < k; ++j) std::swap(a(k, j), a(big, j));
        for (Index i = big + 1; i < n; ++i) std::swap(a(i, k), a(i, big));
        std::swap(a(k, k), a(big, big));
        for (Index i = k + 1; i < big; ++i) {
          const T t = a(i, k);
          a(i, k) = a(big, i);
          a(big, i) = t;
        }
      }
      if (k > 0) {
        for (Index j = 0; j < k; ++j) temp[std::size_t(j)] = a(j, j) * a(k, j);
        T d = T(0);
        for (Index j = 0; j < k; ++j) d += a(k, j) * temp[std::size_t(j)];
        a(k, k) -= d;
        for (Index i = k + 1; i < n; ++i) {
          T s = T(0);
          for (Index j = 0; j < k; ++j) s += a(i, j) * temp[std::size_t(j)];
          a(i, k) -= s;
        }
      }
      const T akk = a(k, k);
      if (std::abs(akk) > T(0))
        for (Index i = k + 1; i < n; ++i) a(i, k) /= akk;
    }
  }
  template <int RB>
  Matrix<T, RB, 1> solve(const Matrix<T, RB, 1>& b) const {
    const Index n = a.rows();
    Matrix<T, RB, 1> x = b;
    for (Index k = 0; k < n; ++k) std::swap(x(k), x(tr[std::size_t(k)]));
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < i; ++j) x(i) -= a(i, j) * x(j);
    for (Index i = 0; i < n; ++i) {
      const T d = a(i, i);
      x(i) = std::abs(d) > std::numeric_limits<T>::min() ? x(i) / d : T(0);
    }
    for (Index i = n - 1; i >= 0; --i)
      for (Index j = i + 1; j < n; ++j) x(i) -= a(j, i) * x(j);
    for (Index k = n - 1; k >= 0; --k) std::swap(x(k), x(tr[std::size_t(k)]));
    return x;
  }
};

// ---- PartialPivLU (Eigen 3.4 partial_lu_impl::unblocked_lu) -----------------
template <typename T, int R, int C>
struct Matrix<T, R, C>::PartialPivLUd {
  Matrix a;
  std::vector<Index> perm;
  explicit PartialPivLUd(const Matrix& m) : a(m) {
    const Index n = a.rows();
    perm.resize(std::size_t(n));
    for (Index i = 0; i < n; ++i) perm[std::size_t(i)] = i;
    for (Index k = 0; k < n; ++k) {
      Index p = k;
      for (Index i = k + 1; i < n; ++i)
        if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
      if (a(p, k) != T(0)) {
        if (p != k) {
          for (Index c = 0; c < n; ++c) std::swap(a(k, c), a(p, c));
          std::swap(perm[std::size_t(k)], perm[std::size_t(p)]);
        }
        for (Index i = k + 1; i < n; ++i) a(i, k) /= a(k, k);
      }
      for (Index i = k + 1; i < n; ++i)
        for (Index c = k + 1; c < n; ++c) a(i, c) -= a(i, k) * a(k, c);
    }
  }
  template <int RB>
  Matrix<T, RB, 1> solve(const Matrix<T, RB, 1>& b) const {
    const Index n = a.rows();
    Matrix<T, RB, 1> x = b;
    for (Index i = 0; i < n; ++i) x(i) = b(perm[std::size_t(i)]);
    for (Index i = 1; i < n; ++i)
      for (Index j = 0; j < i; ++j) x(i) -= a(i, j) * x(j);
    for (Index i = n - 1; i >= 0; --i) {
      for (Index j = n - 1; j > i; --j) x(i) -= a(i, j) * x(j);
      x(i) /= a(i, i);
    }
    return x;
  }
};

using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Vector3f = Matrix<float, 3, 1>;
using Vector3i = Matrix<int, 3, 1>;
using Vector2i = Matrix<int, 2, 1>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix3f = Matrix<float, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXf = Matrix<float, Dynamic, 1>;

template <typename T, int R, int C>
std::ostream& operator<<(std::ostream& os, const Matrix<T, R, C>& m) {
  for (Index i = 0; i < m.rows(); ++i) {
    for (Index j = 0; j < m.cols(); ++j) os << (j ? " " : "") << m(i, j);
    if (i + 1 < m.rows()) os << '\n';
  }
  return os;
}

// ---- JacobiSVD<Matrix3d> (ComputeFullU | ComputeFullV) ---------------------
namespace detail {
struct Rot {  // JacobiRotation<double>: J = [c s; -s c]
  double c = 1, s = 0;
  Rot transpose() const { return {c, -s}; }
};
inline Rot operator*(const Rot& a, const Rot& b) { return {a.c * b.c - a.s * b.s, a.c * b.s + a.s * b.c}; }
// applyOnTheLeft(p, q, j): rows p, q
inline void rot_rows(Matrix3d& m, int p, int q, const Rot& j) {
  for (int i = 0; i < 3; ++i) {
    const double xi = m(p, i), yi = m(q, i);
    m(p, i) = j.c * xi + j.s * yi;
    m(q, i) = -j.s * xi + j.c * yi;
  }
}
// applyOnTheRight(p, q, j): columns p, q with j^T
inline void rot_cols(Matrix3d& m, int p, int q, const Rot& j) {
  const Rot t = j.transpose();
  for (int i = 0; i < 3; ++i) {
    const double xi = m(i, p), yi = m(i, q);
    m(i, p) = t.c * xi + t.s * yi;
    m(i, q) = -t.s * xi + t.c * yi;
  }
}
inline Rot make_jacobi(double x, double y, double z) {
  Rot r;
  const double deno = 2.0 * std::abs(y);
  if (deno < DBL_MIN) return r;
  const double tau = (x - z) / deno;
  const double w = std::sqrt(tau * tau + 1.0);
  const double t = tau > 0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
  const double sign_t = t > 0 ? 1.0 : -1.0;
  const double n = 1.0 / std::sqrt(t * t + 1.0);
  r.s = -sign_t * (y / std::abs(y)) * std::abs(t) * n;
  r.c = n;
  return r;
}
inline void real_2x2_jacobi_svd(const Matrix3d& w, int p, int q, Rot& jl, Rot& jr) {
  const double m00 = w(p, p), m01 = w(p, q), m10 = w(q, p), m11 = w(q, q);
  Rot rot1;
  const double t = m00 + m11;
  const double d = m10 - m01;
  if (std::abs(d) < DBL_MIN) {
    rot1.s = 0;
    rot1.c = 1;
  } else {
    const double u = t / d;
    const double tmp = std::sqrt(1.0 + u * u);
    rot1.s = 1.0 / tmp;
    rot1.c = u / tmp;
  }
  const double n00 = rot1.c * m00 + rot1.s * m10, n01 = rot1.c * m01 + rot1.s * m11;
  const double n11 = -rot1.s * m01 + rot1.c * m11;
  jr = make_jacobi(n00, n01, n11);
  jl = rot1 * jr.transpose();
}
}  // namespace detail

template <typename M>
class JacobiSVD {
  static_assert(std::is_same_v<M, Matrix3d>, "shim: JacobiSVD<Matrix3d> only");

 public:
  JacobiSVD(const Matrix3d& a, int /*options*/ = ComputeFullU | ComputeFullV) {
    using detail::Rot;
    double scale = 0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) scale = std::max(scale, std::abs(a(i, j)));
    if (!std::isfinite(scale)) {
      u_ = Matrix3d::Identity();
      v_ = Matrix3d::Identity();
      s_ = Vector3d::Zero();
      return;
    }
    if (scale == 0) scale = 1;
    Matrix3d w = a / scale;
    u_ = Matrix3d::Identity();
    v_ = Matrix3d::Identity();
    const double considerAsZero = DBL_MIN;
    const double precision = 2.0 * DBL_EPSILON;
    double maxDiag = std::max(std::abs(w(0, 0)), std::max(std::abs(w(1, 1)), std::abs(w(2, 2))));
    bool finished = false;
    while (!finished) {
      finished = true;
      for (int p = 1; p < 3; ++p)
        for (int q = 0; q < p; ++q) {
          const double threshold = std::max(considerAsZero, precision * maxDiag);
          if (std::abs(w(p, q)) > threshold || std::abs(w(q, p)) > threshold) {
            finished = false;
            Rot jl, jr;
            detail::real_2x2_jacobi_svd(w, p, q, jl, jr);
            detail::rot_rows(w, p, q, jl);
            detail::rot_cols(u_, p, q, jl.transpose());
            detail::rot_cols(w, p, q, jr);
            detail::rot_cols(v_, p, q, jr);
            maxDiag = std::max(maxDiag, std::max(std::abs(w(p, p)), std::abs(w(q, q))));
          }
        }
    }
    for (int i = 0; i < 3; ++i) {
      const double d = w(i, i);
      s_(i) = std::abs(d);
      if (d < 0)
        for (int k = 0; k < 3; ++k) u_(k, i) = -u_(k, i);
    }
    s_ *= scale;
    for (int i = 0; i < 3; ++i) {
      int pos = i;
      double best = s_(i);
      for (int k = i + 1; k < 3; ++k)
        if (s_(k) > best) {
          best = s_(k);
          pos = k;
        }
      if (best == 0) break;
      if (pos != i) {
        std::swap(s_(i), s_(pos));
        for (int k = 0; k < 3; ++k) {
          std::swap(u_(k, i), u_(k, pos));
          std::swap(v_(k, i), v_(k, pos));
        }
      }
    }
  }
  const Matrix3d& matrixU() const { return u_; }
  const Matrix3d& matrixV() const { return v_; }
  const Vector3d& singularValues() const { return s_; }

 private:
  Matrix3d u_, v_;
  Vector3d s_;
};

// ---- geometry ----------------------------------------------------------------
template <typename T>
class AngleAxis {
 public:
  AngleAxis(T angle, const Matrix<T, 3, 1>& axis) : a_(angle), n_(axis) {}
  Matrix<T, 3, 3> toRotationMatrix() const {
    Matrix<T, 3, 3> res;
    const Matrix<T, 3, 1> sin_axis = std::sin(a_) * n_;
    const T c = std::cos(a_);
    const Matrix<T, 3, 1> cos1_axis = (T(1) - c) * n_;
    T tmp;
    tmp = cos1_axis.x() * n_.y();
    res(0, 1) = tmp - sin_axis.z();
    res(1, 0) = tmp + sin_axis.z();
    tmp = cos1_axis.x() * n_.z();
    res(0, 2) = tmp + sin_axis.y();
    res(2, 0) = tmp - sin_axis.y();
    tmp = cos1_axis.y() * n_.z();
    res(1, 2) = tmp - sin_axis.x();
    res(2, 1) = tmp + sin_axis.x();
    const Matrix<T, 3, 1> dg = cos1_axis.cwiseProduct(n_);
    for (int i = 0; i < 3; ++i) res(i, i) = dg(i) + c;
    return res;
  }
  T angle() const { return a_; }
  const Matrix<T, 3, 1>& axis() const { return n_; }

 private:
  T a_;
  Matrix<T, 3, 1> n_;
};
using AngleAxisd = AngleAxis<double>;

template <typename T>
class Quaternion {
 public:
  Quaternion(T w, T x, T y, T z) : w_(w), x_(x), y_(y), z_(z) {}
  T w() const { return w_; }
  T x() const { return x_; }
  T y() const { return y_; }
  T z() const { return z_; }
  T squaredNorm() const { return ((x_ * x_ + y_ * y_) + z_ * z_) + w_ * w_; }  // coeffs() = (x, y, z, w)
  T norm() const { return std::sqrt(squaredNorm()); }
  void normalize() {
    const T n = squaredNorm();
    if (n > T(0)) {
      const T s = std::sqrt(n);
      x_ /= s;
      y_ /= s;
      z_ /= s;
      w_ /= s;
    }
  }
  Quaternion normalized() const {
    Quaternion q = *this;
    q.normalize();
    return q;
  }
  Matrix<T, 3, 3> toRotationMatrix() const {
    Matrix<T, 3, 3> res;
    const T tx = T(2) * x_, ty = T(2) * y_, tz = T(2) * z_;
    const T twx = tx * w_, twy = ty * w_, twz = tz * w_;
    const T txx = tx * x_, txy = ty * x_, txz = tz * x_;
    const T tyy = ty * y_, tyz = tz * y_, tzz = tz * z_;
    res(0, 0) = T(1) - (tyy + tzz);
    res(0, 1) = txy - twz;
    res(0, 2) = txz + twy;
    res(1, 0) = txy + twz;
    res(1, 1) = T(1) - (txx + tzz);
    res(1, 2) = tyz - twx;
    res(2, 0) = txz - twy;
    res(2, 1) = tyz + twx;
    res(2, 2) = T(1) - (txx + tyy);
    return res;
  }

 private:
  T w_, x_, y_, z_;
};
using Quaterniond = Quaternion<double>;

}  // namespace Eigen
