// Minimal dense-matrix library exposing the subset of the Eigen 3 API that
// the reference's hot-path sources use (proj/src/{estimator,model,wiener,
// stft,fft,synth,metrics}.cpp and its unit tests), so that those UNMODIFIED
// sources compile here without Eigen (absent from this image,
// proj/CMakeLists.txt:12). TEST INFRASTRUCTURE ONLY: it is linked into
// oracle/_ref (the reference built from its own sources), never into the
// product library.
//
// Written from Eigen's published semantics, not from its sources:
//  * column-major dense storage (Eigen's default), Index = std::ptrdiff_t;
//  * expressions are evaluated eagerly into temporaries (Eigen builds lazy
//    expression templates; the values are the same up to rounding because
//    every reduction here runs in index order, which is what the reference's
//    own brute-force oracles (proj/tests/oracles.hpp) assume too);
//  * a.dot(b) = sum_i conj(a_i) b_i (conjugate-linear in the first argument);
//  * PartialPivLU: Doolittle LU with row partial pivoting on |a_ik| (first
//    maximum wins), unit-lower L, a zero pivot column skipped (no division),
//    determinant = sign(P) prod diag(U), inverse = solve(I);
//  * JacobiSVD: singular values only (one-sided Jacobi), sorted descending;
//  * SelfAdjointEigenSolver: cyclic complex Jacobi, eigenvalues ascending.
// Bitwise parity with Eigen's blocked/vectorised kernels is not claimed
// (Eigen's summation order is unpinned; the reference's own
// tests pin results to 1e-10 .. 1e-12 relative).
#pragma once

#include <algorithm>
#include <cassert>
#include <cmath>
#include <complex>
#include <cstddef>
#include <functional>
#include <initializer_list>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;

template <class S> struct NumTraits { using Real = S; static constexpr bool IsComplex = false; };
template <class T> struct NumTraits<std::complex<T>> { using Real = T; static constexpr bool IsComplex = true; };

template <class T> struct is_scalar_t : std::is_arithmetic<T> {};
template <class T> struct is_scalar_t<std::complex<T>> : std::true_type {};
template <class T> constexpr bool is_scalar_v = is_scalar_t<std::decay_t<T>>::value;

namespace internal {
template <class S> inline S conj(const S& v) { return v; }
template <class T> inline std::complex<T> conj(const std::complex<T>& v) { return std::conj(v); }
template <class S> inline typename NumTraits<S>::Real abs2(const S& v) { return v * v; }
template <class T> inline T abs2(const std::complex<T>& v) { return v.real() * v.real() + v.imag() * v.imag(); }
template <class S> inline S real(const S& v) { return v; }
template <class T> inline T real(const std::complex<T>& v) { return v.real(); }
template <class S> inline S imag(const S&) { return S(0); }
template <class T> inline T imag(const std::complex<T>& v) { return v.imag(); }
template <class S> inline bool isfinite(const S& v) { return std::isfinite(v); }
template <class T> inline bool isfinite(const std::complex<T>& v) { return std::isfinite(v.real()) && std::isfinite(v.imag()); }
// product without the C99 Annex-G NaN recovery (what Eigen's kernels do)
template <class A, class B> inline auto mul(const A& a, const B& b) { return a * b; }
template <class T> inline std::complex<T> mul(const std::complex<T>& a, const std::complex<T>& b) {
  return {a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real()};
}
}  // namespace internal

template <class S> class Dense;
template <class S> class Block;
template <class S, int R = Dynamic, int C = Dynamic> class Matrix;
template <class S> class ArrayX;
template <class S> class DiagonalWrapper;
template <class M> class PartialPivLU;

template <class S> using Plain = Matrix<S, Dynamic, Dynamic>;

// ---------------------------------------------------------------- views --
// Column-major strided view: element (i, j) at p_[i + j * ld_].
template <class S>
class Dense {
 public:
  using Scalar = S;
  using RealScalar = typename NumTraits<S>::Real;

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  Index outerStride() const { return ld_; }
  S* data() { return p_; }
  const S* data() const { return p_; }

  S& operator()(Index i, Index j) { return p_[i + j * ld_]; }
  const S& operator()(Index i, Index j) const { return p_[i + j * ld_]; }
  S& coeffRef(Index i, Index j) { return (*this)(i, j); }
  const S& coeff(Index i, Index j) const { return (*this)(i, j); }
  // linear (vector) access
  S& operator()(Index k) { return lin(k); }
  const S& operator()(Index k) const { return const_cast<Dense*>(this)->lin(k); }
  S& operator[](Index k) { return lin(k); }
  const S& operator[](Index k) const { return const_cast<Dense*>(this)->lin(k); }
  S& coeffRef(Index k) { return lin(k); }
  const S& coeff(Index k) const { return const_cast<Dense*>(this)->lin(k); }

  // ---- blocks (writable views; const objects hand out views too, as the
  // reference only reads through those)
  Block<S> block(Index i, Index j, Index r, Index c) const { return Block<S>(mp(i, j), r, c, ld_); }
  Block<S> row(Index i) const { return block(i, 0, 1, c_); }
  Block<S> col(Index j) const { return block(0, j, r_, 1); }
  Block<S> middleRows(Index i, Index n) const { return block(i, 0, n, c_); }
  Block<S> middleCols(Index j, Index n) const { return block(0, j, r_, n); }
  Block<S> topRows(Index n) const { return block(0, 0, n, c_); }
  Block<S> bottomRows(Index n) const { return block(r_ - n, 0, n, c_); }
  Block<S> leftCols(Index n) const { return block(0, 0, r_, n); }
  Block<S> rightCols(Index n) const { return block(0, c_ - n, r_, n); }
  Block<S> topLeftCorner(Index r, Index c) const { return block(0, 0, r, c); }
  Block<S> topRightCorner(Index r, Index c) const { return block(0, c_ - c, r, c); }
  Block<S> bottomLeftCorner(Index r, Index c) const { return block(r_ - r, 0, r, c); }
  Block<S> bottomRightCorner(Index r, Index c) const { return block(r_ - r, c_ - c, r, c); }
  Block<S> segment(Index k, Index n) const {
    return r_ == 1 && c_ != 1 ? block(0, k, 1, n) : block(k, 0, n, 1);
  }
  Block<S> head(Index n) const { return segment(0, n); }
  Block<S> tail(Index n) const { return segment(size() - n, n); }

  // ---- evaluated unary forms
  Plain<S> eval() const { return Plain<S>(*this); }
  Plain<S> transpose() const {
    Plain<S> o(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) o(j, i) = (*this)(i, j);
    return o;
  }
  Plain<S> adjoint() const {
    Plain<S> o(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) o(j, i) = internal::conj((*this)(i, j));
    return o;
  }
  Plain<S> conjugate() const { return map([](const S& v) { return internal::conj(v); }); }
  Plain<RealScalar> real() const { return mapr([](const S& v) { return internal::real(v); }); }
  Plain<RealScalar> imag() const { return mapr([](const S& v) { return internal::imag(v); }); }
  Plain<RealScalar> cwiseAbs() const { return mapr([](const S& v) { return RealScalar(std::abs(v)); }); }
  Plain<RealScalar> cwiseAbs2() const { return mapr([](const S& v) { return internal::abs2(v); }); }
  Plain<S> cwiseInverse() const { return map([](const S& v) { return S(1) / v; }); }
  Plain<S> cwiseSqrt() const { return map([](const S& v) { return S(std::sqrt(v)); }); }
  Plain<S> cwiseMax(const S& s) const { return map([&](const S& v) { return std::max(v, s); }); }
  Plain<S> cwiseMin(const S& s) const { return map([&](const S& v) { return std::min(v, s); }); }
  Plain<S> cwiseMax(const Dense& o) const { return zip(o, [](const S& a, const S& b) { return std::max(a, b); }); }
  Plain<S> cwiseMin(const Dense& o) const { return zip(o, [](const S& a, const S& b) { return std::min(a, b); }); }
  Plain<S> cwiseProduct(const Dense& o) const { return zip(o, [](const S& a, const S& b) { return internal::mul(a, b); }); }
  Plain<S> cwiseQuotient(const Dense& o) const { return zip(o, [](const S& a, const S& b) { return a / b; }); }
  template <class F> Plain<S> unaryExpr(F f) const { return map(f); }
  template <class T> Plain<T> cast() const {
    Plain<T> o(r_, c_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) o(i, j) = static_cast<T>((*this)(i, j));
    return o;
  }

  // ---- reductions (index order: column by column, rows inside)
  S sum() const {
    S s(0);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s += (*this)(i, j);
    return s;
  }
  S prod() const {
    S s(1);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s *= (*this)(i, j);
    return s;
  }
  S mean() const { return sum() / S(static_cast<RealScalar>(size())); }
  S value() const {
    if (size() != 1) throw std::invalid_argument("Eigen shim: value() needs a 1x1 matrix");
    return (*this)(0, 0);
  }
  S trace() const {
    S s(0);
    for (Index i = 0; i < std::min(r_, c_); ++i) s += (*this)(i, i);
    return s;
  }
  RealScalar squaredNorm() const {
    RealScalar s(0);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s += internal::abs2((*this)(i, j));
    return s;
  }
  RealScalar norm() const { return std::sqrt(squaredNorm()); }
  RealScalar lpNorm1() const {
    RealScalar s(0);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s += std::abs((*this)(i, j));
    return s;
  }
  S maxCoeff() const { Index i, j; return maxCoeff(&i, &j); }
  S minCoeff() const { Index i, j; return minCoeff(&i, &j); }
  S maxCoeff(Index* k) const { Index i, j; S v = maxCoeff(&i, &j); *k = r_ == 1 ? j : i; return v; }
  S minCoeff(Index* k) const { Index i, j; S v = minCoeff(&i, &j); *k = r_ == 1 ? j : i; return v; }
  S maxCoeff(Index* ri, Index* ci) const { return extreme(ri, ci, [](const S& a, const S& b) { return a > b; }); }
  S minCoeff(Index* ri, Index* ci) const { return extreme(ri, ci, [](const S& a, const S& b) { return a < b; }); }
  bool allFinite() const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i)
        if (!internal::isfinite((*this)(i, j))) return false;
    return true;
  }
  bool hasNaN() const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) {
        const S v = (*this)(i, j);
        if (internal::real(v) != internal::real(v) || internal::imag(v) != internal::imag(v)) return true;
      }
    return false;
  }
  S dot(const Dense& o) const {
    assert(size() == o.size());
    S s(0);
    for (Index k = 0; k < size(); ++k) s += internal::mul(internal::conj((*this)[k]), o[k]);
    return s;
  }
  bool isApprox(const Dense& o, RealScalar prec = RealScalar(1e-12)) const {
    const Plain<S> d = zip(o, [](const S& a, const S& b) { return a - b; });
    return d.norm() <= prec * std::min(norm(), o.norm());
  }
  bool isZero(RealScalar prec = RealScalar(1e-12)) const {
    for (Index k = 0; k < size(); ++k)
      if (std::abs((*this)[k]) > prec) return false;
    return true;
  }

  // ---- in-place compound operators (write through the view)
  Dense& operator+=(const Dense& o) { return inplace(o, [](S& a, const S& b) { a += b; }); }
  Dense& operator-=(const Dense& o) { return inplace(o, [](S& a, const S& b) { a -= b; }); }
  template <class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
  Dense& operator*=(const T& s) { return each([&](S& a) { a = internal::mul(a, S(s)); }); }
  template <class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
  Dense& operator/=(const T& s) { return each([&](S& a) { a /= S(s); }); }
  Dense& setZero() { return each([](S& a) { a = S(0); }); }
  Dense& setOnes() { return each([](S& a) { a = S(1); }); }
  Dense& setConstant(const S& v) { return each([&](S& a) { a = v; }); }
  void fill(const S& v) { setConstant(v); }
  Dense& setIdentity() {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) = S(i == j ? 1 : 0);
    return *this;
  }

  // ---- decompositions
  PartialPivLU<Plain<S>> partialPivLu() const;
  PartialPivLU<Plain<S>> lu() const;
  S determinant() const;
  Plain<S> inverse() const;

  ArrayX<S> array() const;
  DiagonalWrapper<S> asDiagonal() const;
  Matrix<std::complex<RealScalar>, Dynamic, 1> eigenvalues() const;

 protected:
  S* p_ = nullptr;
  Index r_ = 0, c_ = 0, ld_ = 0;

  Dense() = default;
  Dense(S* p, Index r, Index c, Index ld) : p_(p), r_(r), c_(c), ld_(ld) {}
  Dense(const Dense&) = default;
  Dense& operator=(const Dense&) = default;

  S& lin(Index k) {
    if (c_ == 1) return p_[k];
    if (r_ == 1) return p_[k * ld_];
    return p_[(k % r_) + (k / r_) * ld_];
  }
  S* mp(Index i, Index j) const { return p_ + i + j * ld_; }
  template <class F> Plain<S> map(F f) const {
    Plain<S> o(r_, c_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) o(i, j) = f((*this)(i, j));
    return o;
  }
  template <class F> Plain<RealScalar> mapr(F f) const {
    Plain<RealScalar> o(r_, c_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) o(i, j) = f((*this)(i, j));
    return o;
  }
  template <class F> Plain<S> zip(const Dense& b, F f) const {
    if (b.rows() != r_ || b.cols() != c_) throw std::invalid_argument("Eigen shim: size mismatch");
    Plain<S> o(r_, c_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) o(i, j) = f((*this)(i, j), b(i, j));
    return o;
  }
  template <class F> Dense& each(F f) {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) f((*this)(i, j));
    return *this;
  }
  template <class F> Dense& inplace(const Dense& o, F f) {
    const Plain<S> t(o);  // aliasing-safe
    if (t.rows() != r_ || t.cols() != c_) throw std::invalid_argument("Eigen shim: size mismatch");
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) f((*this)(i, j), t(i, j));
    return *this;
  }
  template <class F> S extreme(Index* ri, Index* ci, F better) const {
    S best = (*this)(0, 0);
    *ri = 0;
    *ci = 0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i)
        if (better((*this)(i, j), best)) {
          best = (*this)(i, j);
          *ri = i;
          *ci = j;
        }
    return best;
  }
  void copy_from(const Dense& o) {  // same shape, aliasing-safe
    const Plain<S> t(o);
    if (t.rows() != r_ || t.cols() != c_) {
      if (t.size() == size() && (r_ == 1 || c_ == 1) && (t.rows() == 1 || t.cols() == 1)) {
        for (Index k = 0; k < size(); ++k) lin(k) = t[k];
        return;
      }
      throw std::invalid_argument("Eigen shim: block assignment size mismatch");
    }
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) = t(i, j);
  }
  template <class> friend class Dense;
};

template <class S>
class Block : public Dense<S> {
 public:
  Block(S* p, Index r, Index c, Index ld) : Dense<S>(p, r, c, ld) {}
  Block(const Block&) = default;
  Block& operator=(const Block& o) { this->copy_from(o); return *this; }
  Block& operator=(const Dense<S>& o) { this->copy_from(o); return *this; }
  Block& noalias() { return *this; }
  template <class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
  Block& operator*=(const T& s) { Dense<S>::operator*=(s); return *this; }
  template <class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
  Block& operator/=(const T& s) { Dense<S>::operator/=(s); return *this; }
  Block& operator+=(const Dense<S>& o) { Dense<S>::operator+=(o); return *this; }
  Block& operator-=(const Dense<S>& o) { Dense<S>::operator-=(o); return *this; }
};

// -------------------------------------------------------------- storage --
template <class S, int R, int C>
class Matrix : public Dense<S> {
  using Base = Dense<S>;

 public:
  Matrix() { shape(R > 0 ? R : 0, C > 0 ? C : 0); }
  explicit Matrix(Index n) {
    static_assert(R == 1 || C == 1, "single-size constructor needs a vector type");
    if (C == 1) shape(n, 1); else shape(1, n);
  }
  Matrix(Index r, Index c) { shape(r, c); }
  Matrix(const Matrix& o) : Base() { assign(o); }
  Matrix(Matrix&& o) noexcept : Base() { take(std::move(o)); }
  template <int R2, int C2> Matrix(const Matrix<S, R2, C2>& o) : Base() { assign(o); }
  Matrix(const Dense<S>& o) : Base() { assign(o); }
  Matrix(const ArrayX<S>& a);
  Matrix(std::initializer_list<std::initializer_list<S>> rows_list) {
    const Index r = static_cast<Index>(rows_list.size());
    const Index c = r ? static_cast<Index>(rows_list.begin()->size()) : 0;
    shape(r, c);
    Index i = 0;
    for (const auto& rl : rows_list) {
      Index j = 0;
      for (const auto& v : rl) (*this)(i, j++) = v;
      ++i;
    }
  }

  Matrix& operator=(const Matrix& o) { if (this != &o) assign(o); return *this; }
  Matrix& operator=(Matrix&& o) noexcept { if (this != &o) take(std::move(o)); return *this; }
  template <int R2, int C2> Matrix& operator=(const Matrix<S, R2, C2>& o) { assign(o); return *this; }
  Matrix& operator=(const Dense<S>& o) { assign(o); return *this; }
  Matrix& operator=(const ArrayX<S>& a);
  Matrix& noalias() { return *this; }

  template <class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
  Matrix& operator*=(const T& s) { Base::operator*=(s); return *this; }
  template <class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
  Matrix& operator/=(const T& s) { Base::operator/=(s); return *this; }
  Matrix& operator+=(const Dense<S>& o) { Base::operator+=(o); return *this; }
  Matrix& operator-=(const Dense<S>& o) { Base::operator-=(o); return *this; }
  Matrix& operator*=(const Dense<S>& o);

  void resize(Index r, Index c) { shape(r, c); }
  void resize(Index n) { if (C == 1 || (C != 1 && R != 1 && this->c_ == 1)) shape(n, 1); else shape(1, n); }
  void conservativeResize(Index r, Index c) {
    Matrix o(r, c);
    o.setZero();
    for (Index j = 0; j < std::min(c, this->c_); ++j)
      for (Index i = 0; i < std::min(r, this->r_); ++i) o(i, j) = (*this)(i, j);
    *this = std::move(o);
  }
  void conservativeResize(Index n) { if (C == 1) conservativeResize(n, 1); else conservativeResize(1, n); }

  static Matrix Zero(Index r, Index c) { Matrix m(r, c); m.setZero(); return m; }
  static Matrix Zero(Index n) { Matrix m(n); m.setZero(); return m; }
  static Matrix Zero() { Matrix m; m.setZero(); return m; }
  static Matrix Ones(Index r, Index c) { Matrix m(r, c); m.setOnes(); return m; }
  static Matrix Ones(Index n) { Matrix m(n); m.setOnes(); return m; }
  static Matrix Constant(Index r, Index c, const S& v) { Matrix m(r, c); m.setConstant(v); return m; }
  static Matrix Constant(Index n, const S& v) { Matrix m(n); m.setConstant(v); return m; }
  static Matrix Identity(Index r, Index c) { Matrix m(r, c); m.setIdentity(); return m; }
  static Matrix Identity() { Matrix m; m.setIdentity(); return m; }
  template <class F> static Matrix NullaryExpr(Index r, Index c, F f) {
    Matrix m(r, c);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) m(i, j) = nullary(f, i, j);
    return m;
  }
  template <class F> static Matrix NullaryExpr(Index n, F f) {
    Matrix m(n);
    for (Index k = 0; k < n; ++k) m[k] = nullary1(f, k);
    return m;
  }
  static Matrix LinSpaced(Index n, const S& lo, const S& hi) {
    Matrix m(n);
    for (Index k = 0; k < n; ++k)
      m[k] = n == 1 ? hi : lo + (hi - lo) * S(static_cast<typename NumTraits<S>::Real>(k)) /
                                      S(static_cast<typename NumTraits<S>::Real>(n - 1));
    return m;
  }

 private:
  std::vector<S> v_;
  void shape(Index r, Index c) {
    v_.assign(static_cast<size_t>(r * c), S(0));
    this->p_ = v_.data();
    this->r_ = r;
    this->c_ = c;
    this->ld_ = r;
  }
  void assign(const Dense<S>& o) {
    // vectors take any vector shape (Eigen's implicit vector transposition)
    Index r = o.rows(), c = o.cols();
    if (C == 1 && r == 1 && c != 1) std::swap(r, c);
    if (R == 1 && c == 1 && r != 1) std::swap(r, c);
    std::vector<S> t(static_cast<size_t>(r * c));
    for (Index k = 0, n = r * c; k < n; ++k) t[static_cast<size_t>(k)] = (o.rows() == r) ? o(k % r, k / (r ? r : 1)) : o[k];
    v_.swap(t);
    this->p_ = v_.data();
    this->r_ = r;
    this->c_ = c;
    this->ld_ = r;
  }
  void take(Matrix&& o) {
    v_ = std::move(o.v_);
    this->p_ = v_.data();
    this->r_ = o.r_;
    this->c_ = o.c_;
    this->ld_ = o.r_;
    o.p_ = nullptr;
    o.r_ = o.c_ = o.ld_ = 0;
  }
  template <class F> static S nullary(F& f, Index i, Index j) {
    if constexpr (std::is_invocable_v<F&, Index, Index>) return f(i, j);
    else if constexpr (std::is_invocable_v<F&, Index>) return f(i + j);
    else return f();
  }
  template <class F> static S nullary1(F& f, Index k) {
    if constexpr (std::is_invocable_v<F&, Index>) return f(k);
    else return f();
  }
};

using MatrixXd = Matrix<double, Dynamic, Dynamic>;
using MatrixXf = Matrix<float, Dynamic, Dynamic>;
using MatrixXcd = Matrix<std::complex<double>, Dynamic, Dynamic>;
using MatrixXcf = Matrix<std::complex<float>, Dynamic, Dynamic>;
using MatrixXi = Matrix<int, Dynamic, Dynamic>;
using VectorXd = Matrix<double, Dynamic, 1>;
using VectorXf = Matrix<float, Dynamic, 1>;
using VectorXcd = Matrix<std::complex<double>, Dynamic, 1>;
using VectorXi = Matrix<int, Dynamic, 1>;
using RowVectorXd = Matrix<double, 1, Dynamic>;
using RowVectorXcd = Matrix<std::complex<double>, 1, Dynamic>;
using Matrix2cd = Matrix<std::complex<double>, Dynamic, Dynamic>;

// ----------------------------------------------------------- arithmetic --
namespace internal {
template <class A, class B> using sum_t = decltype(std::declval<A>() * std::declval<B>());

template <class SA, class SB>
Plain<sum_t<SA, SB>> gemm(const Dense<SA>& a, const Dense<SB>& b) {
  using SR = sum_t<SA, SB>;
  if (a.cols() != b.rows()) throw std::invalid_argument("Eigen shim: product size mismatch");
  const Index m = a.rows(), n = b.cols(), kk = a.cols();
  Plain<SR> o(m, n);  // zero-initialised
  // res(:, j) += a(:, k) * b(k, j), k ascending: each entry sums over k in order
  for (Index j = 0; j < n; ++j) {
    SR* oc = o.data() + j * m;
    for (Index k = 0; k < kk; ++k) {
      const SB bkj = b(k, j);
      const SA* ac = a.data() + k * a.outerStride();
      for (Index i = 0; i < m; ++i) oc[i] += mul(SR(ac[i]), SR(bkj));
    }
  }
  return o;
}
}  // namespace internal

template <class S> Plain<S> operator+(const Dense<S>& a, const Dense<S>& b) {
  Plain<S> o(a);
  o += b;
  return o;
}
template <class S> Plain<S> operator-(const Dense<S>& a, const Dense<S>& b) {
  Plain<S> o(a);
  o -= b;
  return o;
}
template <class S> Plain<S> operator-(const Dense<S>& a) {
  Plain<S> o(a);
  o *= S(-1);
  return o;
}
template <class SA, class SB>
Plain<internal::sum_t<SA, SB>> operator*(const Dense<SA>& a, const Dense<SB>& b) {
  return internal::gemm(a, b);
}
namespace internal {
// matrix-scalar result type: the matrix scalar, widened to complex when a
// complex scalar meets a real matrix (Eigen's ScalarBinaryOpTraits)
template <class S, class T> struct promote { using type = S; };
template <class S, class T> struct promote<S, std::complex<T>> {
  using type = std::conditional_t<NumTraits<S>::IsComplex, S, std::complex<S>>;
};
template <class S, class T> using promote_t = typename promote<S, std::decay_t<T>>::type;
template <class SR, class T> inline SR as(const T& v) {
  if constexpr (NumTraits<SR>::IsComplex && !NumTraits<T>::IsComplex)
    return SR(static_cast<typename NumTraits<SR>::Real>(v));
  else
    return SR(v);
}
}  // namespace internal
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
auto operator*(const Dense<S>& a, const T& s) {
  using SR = internal::promote_t<S, T>;
  const SR v = internal::as<SR>(s);
  Plain<SR> o(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) o(i, j) = internal::mul(internal::as<SR>(a(i, j)), v);
  return o;
}
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
auto operator*(const T& s, const Dense<S>& a) {
  using SR = internal::promote_t<S, T>;
  const SR v = internal::as<SR>(s);
  Plain<SR> o(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) o(i, j) = internal::mul(v, internal::as<SR>(a(i, j)));
  return o;
}
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
auto operator/(const Dense<S>& a, const T& s) {
  using SR = internal::promote_t<S, T>;
  const SR v = internal::as<SR>(s);
  Plain<SR> o(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) o(i, j) = internal::as<SR>(a(i, j)) / v;
  return o;
}
template <class S> bool operator==(const Dense<S>& a, const Dense<S>& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i)
      if (!(a(i, j) == b(i, j))) return false;
  return true;
}
template <class S> bool operator!=(const Dense<S>& a, const Dense<S>& b) { return !(a == b); }

// comma initializer: m << a, b, c, ... fills row by row
template <class S>
class CommaInitializer {
 public:
  CommaInitializer(Dense<S>& m, const S& first) : m_(m) { put(first); }
  CommaInitializer& operator,(const S& v) { put(v); return *this; }
  ~CommaInitializer() noexcept(false) {
    if (k_ != m_.size() && std::uncaught_exceptions() == 0)
      throw std::invalid_argument("Eigen shim: too few coefficients passed to comma initializer");
  }

 private:
  void put(const S& v) {
    if (k_ >= m_.size()) throw std::invalid_argument("Eigen shim: too many coefficients passed to comma initializer");
    m_(k_ / m_.cols(), k_ % m_.cols()) = v;
    ++k_;
  }
  Dense<S>& m_;
  Index k_ = 0;
};
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
CommaInitializer<S> operator<<(Dense<S>& m, const T& v) { return CommaInitializer<S>(m, internal::as<S>(v)); }

template <class S, int R, int C>
Matrix<S, R, C>& Matrix<S, R, C>::operator*=(const Dense<S>& o) {
  *this = internal::gemm(static_cast<const Dense<S>&>(*this), o);
  return *this;
}

// ------------------------------------------------------------- diagonal --
template <class S>
class DiagonalWrapper {
 public:
  explicit DiagonalWrapper(const Dense<S>& v) : d_(v) {}
  const Plain<S>& diagonal() const { return d_; }
  Index size() const { return d_.size(); }
  Plain<S> toDenseMatrix() const {
    Plain<S> o = Plain<S>::Zero(d_.size(), d_.size());
    for (Index k = 0; k < d_.size(); ++k) o(k, k) = d_[k];
    return o;
  }

 private:
  Plain<S> d_;
};
template <class S> DiagonalWrapper<S> Dense<S>::asDiagonal() const { return DiagonalWrapper<S>(*this); }
template <class SA, class SB>
Plain<internal::sum_t<SA, SB>> operator*(const Dense<SA>& a, const DiagonalWrapper<SB>& d) {
  using SR = internal::sum_t<SA, SB>;
  Plain<SR> o(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) o(i, j) = internal::mul(SR(a(i, j)), SR(d.diagonal()[j]));
  return o;
}
template <class SA, class SB>
Plain<internal::sum_t<SA, SB>> operator*(const DiagonalWrapper<SA>& d, const Dense<SB>& a) {
  using SR = internal::sum_t<SA, SB>;
  Plain<SR> o(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) o(i, j) = internal::mul(SR(d.diagonal()[i]), SR(a(i, j)));
  return o;
}

// ---------------------------------------------------------------- array --
// Coefficient-wise view of a matrix (evaluated copy).
template <class S>
class ArrayX {
 public:
  using Real = typename NumTraits<S>::Real;
  ArrayX() = default;
  explicit ArrayX(const Dense<S>& m) : m_(m) {}
  explicit ArrayX(Plain<S>&& m) : m_(std::move(m)) {}
  Index rows() const { return m_.rows(); }
  Index cols() const { return m_.cols(); }
  Index size() const { return m_.size(); }
  S& operator()(Index i, Index j) { return m_(i, j); }
  const S& operator()(Index i, Index j) const { return m_(i, j); }
  S& operator[](Index k) { return m_[k]; }
  const S& operator[](Index k) const { return m_[k]; }
  const Plain<S>& matrix() const { return m_; }
  Plain<S>& matrix() { return m_; }

  template <class F> ArrayX map(F f) const { return ArrayX(m_.unaryExpr(f)); }
  ArrayX sqrt() const { return map([](const S& v) { return S(std::sqrt(v)); }); }
  ArrayX square() const { return map([](const S& v) { return internal::mul(v, v); }); }
  ArrayX cube() const { return map([](const S& v) { return internal::mul(internal::mul(v, v), v); }); }
  ArrayX inverse() const { return map([](const S& v) { return S(1) / v; }); }
  ArrayX log() const { return map([](const S& v) { return S(std::log(v)); }); }
  ArrayX log10() const { return map([](const S& v) { return S(std::log10(v)); }); }
  ArrayX exp() const { return map([](const S& v) { return S(std::exp(v)); }); }
  ArrayX<Real> abs() const { return ArrayX<Real>(m_.cwiseAbs()); }
  ArrayX<Real> abs2() const { return ArrayX<Real>(m_.cwiseAbs2()); }
  ArrayX<Real> real() const { return ArrayX<Real>(m_.real()); }
  ArrayX<Real> imag() const { return ArrayX<Real>(m_.imag()); }
  ArrayX max(const S& s) const { return map([&](const S& v) { return std::max(v, s); }); }
  ArrayX min(const S& s) const { return map([&](const S& v) { return std::min(v, s); }); }
  ArrayX max(const ArrayX& o) const { return ArrayX(m_.cwiseMax(o.m_)); }
  ArrayX min(const ArrayX& o) const { return ArrayX(m_.cwiseMin(o.m_)); }
  S sum() const { return m_.sum(); }
  S prod() const { return m_.prod(); }
  S mean() const { return m_.mean(); }
  S maxCoeff() const { return m_.maxCoeff(); }
  S minCoeff() const { return m_.minCoeff(); }
  bool allFinite() const { return m_.allFinite(); }
  ArrayX transpose() const { return ArrayX(m_.transpose()); }
  ArrayX& operator+=(const ArrayX& o) { m_ += o.m_; return *this; }
  ArrayX& operator-=(const ArrayX& o) { m_ -= o.m_; return *this; }
  ArrayX& operator*=(const ArrayX& o) { m_ = m_.cwiseProduct(o.m_); return *this; }
  ArrayX& operator/=(const ArrayX& o) { m_ = m_.cwiseQuotient(o.m_); return *this; }
  template <class T, std::enable_if_t<is_scalar_v<T>, int> = 0> ArrayX& operator*=(const T& s) { m_ *= s; return *this; }
  template <class T, std::enable_if_t<is_scalar_v<T>, int> = 0> ArrayX& operator/=(const T& s) { m_ /= s; return *this; }

  // rowwise() op v: v (a row of length cols) applied to every row
  struct Rowwise {
    const ArrayX& a;
    template <class F> ArrayX apply(const ArrayX& v, F f) const {
      ArrayX o(a.m_);
      for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) o(i, j) = f(a(i, j), v[j]);
      return o;
    }
    ArrayX operator*(const ArrayX& v) const { return apply(v, [](const S& x, const S& y) { return internal::mul(x, y); }); }
    ArrayX operator/(const ArrayX& v) const { return apply(v, [](const S& x, const S& y) { return x / y; }); }
    ArrayX operator+(const ArrayX& v) const { return apply(v, [](const S& x, const S& y) { return x + y; }); }
    ArrayX operator-(const ArrayX& v) const { return apply(v, [](const S& x, const S& y) { return x - y; }); }
    ArrayX sum() const {
      ArrayX o(Plain<S>::Zero(1, a.cols()));
      for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) o(0, j) += a(i, j);
      return o;
    }
  };
  struct Colwise {
    const ArrayX& a;
    template <class F> ArrayX apply(const ArrayX& v, F f) const {
      ArrayX o(a.m_);
      for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) o(i, j) = f(a(i, j), v[i]);
      return o;
    }
    ArrayX operator*(const ArrayX& v) const { return apply(v, [](const S& x, const S& y) { return internal::mul(x, y); }); }
    ArrayX operator/(const ArrayX& v) const { return apply(v, [](const S& x, const S& y) { return x / y; }); }
    ArrayX operator+(const ArrayX& v) const { return apply(v, [](const S& x, const S& y) { return x + y; }); }
    ArrayX operator-(const ArrayX& v) const { return apply(v, [](const S& x, const S& y) { return x - y; }); }
    ArrayX sum() const {
      ArrayX o(Plain<S>::Zero(a.rows(), 1));
      for (Index j = 0; j < a.cols(); ++j)
        for (Index i = 0; i < a.rows(); ++i) o(i, 0) += a(i, j);
      return o;
    }
  };
  Rowwise rowwise() const { return Rowwise{*this}; }
  Colwise colwise() const { return Colwise{*this}; }

 private:
  Plain<S> m_;
};

template <class S> ArrayX<S> Dense<S>::array() const { return ArrayX<S>(*this); }
template <class S, int R, int C> Matrix<S, R, C>::Matrix(const ArrayX<S>& a) : Base() { assign(a.matrix()); }
template <class S, int R, int C> Matrix<S, R, C>& Matrix<S, R, C>::operator=(const ArrayX<S>& a) {
  assign(a.matrix());
  return *this;
}

template <class S> ArrayX<S> operator*(const ArrayX<S>& a, const ArrayX<S>& b) { return ArrayX<S>(a.matrix().cwiseProduct(b.matrix())); }
template <class S> ArrayX<S> operator/(const ArrayX<S>& a, const ArrayX<S>& b) { return ArrayX<S>(a.matrix().cwiseQuotient(b.matrix())); }
template <class S> ArrayX<S> operator+(const ArrayX<S>& a, const ArrayX<S>& b) { return ArrayX<S>(a.matrix() + b.matrix()); }
template <class S> ArrayX<S> operator-(const ArrayX<S>& a, const ArrayX<S>& b) { return ArrayX<S>(a.matrix() - b.matrix()); }
template <class S> ArrayX<S> operator-(const ArrayX<S>& a) { return ArrayX<S>(-a.matrix()); }
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
ArrayX<S> operator*(const ArrayX<S>& a, const T& s) { return ArrayX<S>(a.matrix() * S(s)); }
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
ArrayX<S> operator*(const T& s, const ArrayX<S>& a) { return ArrayX<S>(S(s) * a.matrix()); }
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
ArrayX<S> operator/(const ArrayX<S>& a, const T& s) { return ArrayX<S>(a.matrix() / S(s)); }
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
ArrayX<S> operator/(const T& s, const ArrayX<S>& a) { return a.map([&](const S& v) { return S(s) / v; }); }
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
ArrayX<S> operator+(const ArrayX<S>& a, const T& s) { return a.map([&](const S& v) { return v + S(s); }); }
template <class S, class T, std::enable_if_t<is_scalar_v<T>, int> = 0>
ArrayX<S> operator-(const ArrayX<S>& a, const T& s) { return a.map([&](const S& v) { return v - S(s); }); }

using ArrayXd = ArrayX<double>;
using ArrayXXd = ArrayX<double>;

// ------------------------------------------------------------------- LU --
template <class M>
class PartialPivLU {
 public:
  using S = typename M::Scalar;
  using Real = typename NumTraits<S>::Real;
  PartialPivLU() = default;
  explicit PartialPivLU(const Dense<S>& a) { compute(a); }
  template <int R, int C> explicit PartialPivLU(const Matrix<S, R, C>& a) { compute(a); }

  PartialPivLU& compute(const Dense<S>& a) {
    if (a.rows() != a.cols()) throw std::invalid_argument("Eigen shim: PartialPivLU needs a square matrix");
    lu_ = Plain<S>(a);
    const Index n = lu_.rows();
    perm_.assign(static_cast<size_t>(n), 0);
    swaps_ = 0;
    for (Index k = 0; k < n; ++k) {
      Index piv = k;
      Real best = std::abs(lu_(k, k));
      for (Index i = k + 1; i < n; ++i) {
        const Real s = std::abs(lu_(i, k));
        if (s > best) {
          best = s;
          piv = i;
        }
      }
      perm_[static_cast<size_t>(k)] = piv;
      if (best != Real(0)) {
        if (piv != k) {
          ++swaps_;
          for (Index j = 0; j < n; ++j) std::swap(lu_(k, j), lu_(piv, j));
        }
        const S d = lu_(k, k);
        for (Index i = k + 1; i < n; ++i) lu_(i, k) /= d;
      }
      for (Index j = k + 1; j < n; ++j) {
        const S u = lu_(k, j);
        for (Index i = k + 1; i < n; ++i) lu_(i, j) -= internal::mul(lu_(i, k), u);
      }
    }
    return *this;
  }
  const Plain<S>& matrixLU() const { return lu_; }
  S determinant() const {
    S d(swaps_ % 2 ? -1 : 1);
    for (Index i = 0; i < lu_.rows(); ++i) d = internal::mul(d, lu_(i, i));
    return d;
  }
  Plain<S> solve(const Dense<S>& b) const {
    const Index n = lu_.rows();
    Plain<S> x(b);
    for (Index k = 0; k < n; ++k) {
      const Index p = perm_[static_cast<size_t>(k)];
      if (p != k)
        for (Index j = 0; j < x.cols(); ++j) std::swap(x(k, j), x(p, j));
    }
    for (Index j = 0; j < x.cols(); ++j) {
      for (Index i = 0; i < n; ++i) {  // unit lower
        S acc = x(i, j);
        for (Index k = 0; k < i; ++k) acc -= internal::mul(lu_(i, k), x(k, j));
        x(i, j) = acc;
      }
      for (Index i = n - 1; i >= 0; --i) {  // upper
        S acc = x(i, j);
        for (Index k = i + 1; k < n; ++k) acc -= internal::mul(lu_(i, k), x(k, j));
        x(i, j) = acc / lu_(i, i);
      }
    }
    return x;
  }
  Plain<S> inverse() const { return solve(Plain<S>::Identity(lu_.rows(), lu_.rows())); }
  Index rows() const { return lu_.rows(); }
  Index cols() const { return lu_.cols(); }

 private:
  Plain<S> lu_;
  std::vector<Index> perm_;
  int swaps_ = 0;
};
template <class S> PartialPivLU<Plain<S>> Dense<S>::partialPivLu() const { return PartialPivLU<Plain<S>>(*this); }
template <class S> PartialPivLU<Plain<S>> Dense<S>::lu() const { return PartialPivLU<Plain<S>>(*this); }
template <class S> S Dense<S>::determinant() const { return PartialPivLU<Plain<S>>(*this).determinant(); }
template <class S> Plain<S> Dense<S>::inverse() const { return PartialPivLU<Plain<S>>(*this).inverse(); }
template <class M> using FullPivLU = PartialPivLU<M>;

// ---------------------------------------------------------- SVD / eigen --
enum { ComputeThinU = 1, ComputeThinV = 2, ComputeFullU = 4, ComputeFullV = 8, EigenvaluesOnly = 0, ComputeEigenvectors = 1 };

// Singular values by one-sided (Hestenes) Jacobi on the columns: rotate
// column pairs until they are mutually orthogonal; the column norms are then
// the singular values.
template <class M>
class JacobiSVD {
 public:
  using S = typename M::Scalar;
  using Real = typename NumTraits<S>::Real;
  explicit JacobiSVD(const Dense<S>& a, int = 0) {
    Plain<S> u = a.rows() >= a.cols() ? Plain<S>(a) : a.adjoint();
    const Index m = u.rows(), n = u.cols();
    for (int sweep = 0; sweep < 60; ++sweep) {
      bool rotated = false;
      for (Index p = 0; p < n - 1; ++p)
        for (Index q = p + 1; q < n; ++q) {
          Real app = 0, aqq = 0;
          S apq(0);
          for (Index i = 0; i < m; ++i) {
            app += internal::abs2(u(i, p));
            aqq += internal::abs2(u(i, q));
            apq += internal::mul(internal::conj(u(i, p)), u(i, q));
          }
          const Real g = std::abs(apq);
          if (g == Real(0) || g <= std::numeric_limits<Real>::epsilon() * std::sqrt(app * aqq)) continue;
          rotated = true;
          const S ph = apq / S(g);  // unit phase
          const Real zeta = (aqq - app) / (Real(2) * g);
          const Real t = (zeta >= 0 ? Real(1) : Real(-1)) / (std::abs(zeta) + std::sqrt(Real(1) + zeta * zeta));
          const Real c = Real(1) / std::sqrt(Real(1) + t * t), s = c * t;
          for (Index i = 0; i < m; ++i) {
            const S up = u(i, p), uq = u(i, q);
            u(i, p) = S(c) * up - S(s) * internal::conj(ph) * uq;
            u(i, q) = S(s) * ph * up + S(c) * uq;
          }
        }
      if (!rotated) break;
    }
    sv_ = Matrix<Real, Dynamic, 1>(n);
    for (Index j = 0; j < n; ++j) sv_[j] = u.col(j).norm();
    std::vector<Real> v(sv_.data(), sv_.data() + n);
    std::sort(v.begin(), v.end(), std::greater<Real>());
    for (Index j = 0; j < n; ++j) sv_[j] = v[static_cast<size_t>(j)];
  }
  const Matrix<Real, Dynamic, 1>& singularValues() const { return sv_; }

 private:
  Matrix<Real, Dynamic, 1> sv_;
};

// Hermitian eigenvalues by cyclic Jacobi rotations, ascending.
template <class M>
class SelfAdjointEigenSolver {
 public:
  using S = typename M::Scalar;
  using Real = typename NumTraits<S>::Real;
  SelfAdjointEigenSolver() = default;
  explicit SelfAdjointEigenSolver(const Dense<S>& a, int = 0) { compute(a); }
  SelfAdjointEigenSolver& compute(const Dense<S>& a0, int = 0) {
    Plain<S> a(a0);
    const Index n = a.rows();
    for (int sweep = 0; sweep < 100; ++sweep) {
      Real off = 0;
      for (Index q = 0; q < n; ++q)
        for (Index p = 0; p < q; ++p) off += internal::abs2(a(p, q));
      if (off == Real(0)) break;
      for (Index p = 0; p < n - 1; ++p)
        for (Index q = p + 1; q < n; ++q) {
          const Real g = std::abs(a(p, q));
          if (g == Real(0)) continue;
          const S ph = a(p, q) / S(g);
          const Real app = internal::real(a(p, p)), aqq = internal::real(a(q, q));
          const Real zeta = (aqq - app) / (Real(2) * g);
          const Real t = (zeta >= 0 ? Real(1) : Real(-1)) / (std::abs(zeta) + std::sqrt(Real(1) + zeta * zeta));
          const Real c = Real(1) / std::sqrt(Real(1) + t * t), s = c * t;
          // A <- J^H A J with J = [[c, s ph], [-s conj(ph), c]] on (p, q)
          for (Index k = 0; k < n; ++k) {
            const S akp = a(k, p), akq = a(k, q);
            a(k, p) = S(c) * akp - S(s) * internal::conj(ph) * akq;
            a(k, q) = S(s) * ph * akp + S(c) * akq;
          }
          for (Index k = 0; k < n; ++k) {
            const S apk = a(p, k), aqk = a(q, k);
            a(p, k) = S(c) * apk - S(s) * ph * aqk;
            a(q, k) = S(s) * internal::conj(ph) * apk + S(c) * aqk;
          }
        }
    }
    ev_ = Matrix<Real, Dynamic, 1>(n);
    std::vector<Real> v(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) v[static_cast<size_t>(i)] = internal::real(a(i, i));
    std::sort(v.begin(), v.end());
    for (Index i = 0; i < n; ++i) ev_[i] = v[static_cast<size_t>(i)];
    return *this;
  }
  const Matrix<Real, Dynamic, 1>& eigenvalues() const { return ev_; }

 private:
  Matrix<Real, Dynamic, 1> ev_;
};

// Eigenvalues of a general square matrix: complex QR iteration with the
// Wilkinson shift of the trailing 2x2 block and deflation (Householder-free:
// modified Gram-Schmidt QR, adequate for the small matrices the tests use).
template <class S>
Matrix<std::complex<typename NumTraits<S>::Real>, Dynamic, 1> Dense<S>::eigenvalues() const {
  using R = typename NumTraits<S>::Real;
  using C = std::complex<R>;
  Index n = rows();
  Plain<C> a(n, n);
  for (Index j = 0; j < n; ++j)
    for (Index i = 0; i < n; ++i) a(i, j) = C((*this)(i, j));
  Matrix<C, Dynamic, 1> ev(n);
  const R eps = std::numeric_limits<R>::epsilon();
  for (int guard = 0; n > 0 && guard < 100000; ++guard) {
    if (n == 1) {
      ev[0] = a(0, 0);
      break;
    }
    const R sub = std::abs(a(n - 1, n - 2));
    if (sub <= eps * (std::abs(a(n - 1, n - 1)) + std::abs(a(n - 2, n - 2)))) {
      ev[n - 1] = a(n - 1, n - 1);
      --n;
      continue;
    }
    // Wilkinson shift: eigenvalue of the trailing 2x2 closer to a(n-1, n-1)
    const C p = a(n - 2, n - 2), q = a(n - 2, n - 1), r = a(n - 1, n - 2), t = a(n - 1, n - 1);
    const C half = (p - t) / C(2), disc = std::sqrt(half * half + q * r);
    const C m1 = t - q * r / (half + disc), m2 = t - q * r / (half - disc);
    C mu = std::abs(half + disc) == R(0) ? m2 : (std::abs(half - disc) == R(0) ? m1 : (std::abs(m1 - t) < std::abs(m2 - t) ? m1 : m2));
    if (guard % 11 == 10) mu += C(sub);  // exceptional shift
    // QR of the leading n x n block minus mu I
    Plain<C> qm(n, n), rm = Plain<C>::Zero(n, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) qm(i, j) = a(i, j) - (i == j ? mu : C(0));
    for (Index j = 0; j < n; ++j) {
      for (Index k = 0; k < j; ++k) {
        C d(0);
        for (Index i = 0; i < n; ++i) d += std::conj(qm(i, k)) * qm(i, j);
        rm(k, j) = d;
        for (Index i = 0; i < n; ++i) qm(i, j) -= d * qm(i, k);
      }
      R nn = 0;
      for (Index i = 0; i < n; ++i) nn += std::norm(qm(i, j));
      nn = std::sqrt(nn);
      rm(j, j) = C(nn);
      if (nn > R(0))
        for (Index i = 0; i < n; ++i) qm(i, j) /= C(nn);
    }
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) {
        C acc(0);
        for (Index k = 0; k < n; ++k) acc += rm(i, k) * qm(k, j);
        a(i, j) = acc + (i == j ? mu : C(0));
      }
  }
  return ev;
}

}  // namespace Eigen
