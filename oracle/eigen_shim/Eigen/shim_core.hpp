// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Minimal Eigen-API shim so the UNMODIFIED reference headers
// (/root/reference/proj/include/hexmg/{cg,coarse_solver}.hpp) compile without
// Eigen, which the reference pins only as "Eigen3 >= 3.3"
// (proj/CMakeLists.txt:11, find_package(Eigen3 3.3 REQUIRED NO_MODULE)) and
// does not vendor (proj/.gitignore:2).  Only the entry points the reference
// calls are provided:
//   - Eigen::MatrixXd::Zero / operator()                      cg.hpp:63-69
//   - SelfAdjointEigenSolver<MatrixXd>(t, EigenvaluesOnly)   cg.hpp:70-72
//       restated: Eigen computes all eigenvalues of a dense symmetric matrix
//       (Householder tridiagonalisation + implicit symmetric QR).  The matrix
//       the reference passes is already tridiagonal (the CG/Lanczos T), so we
//       compute every eigenvalue by Sturm-sequence bisection to full
//       precision; a non-tridiagonal input falls back to cyclic Jacobi.
//   - Map<const SparseMatrix<double,RowMajor,int>> -> SparseMatrix<double>
//                                                             coarse_solver.hpp:19-22
//   - SimplicialLLT::{analyzePattern,factorize,info,solve}    coarse_solver.hpp:23-40
//       restated: Eigen's SimplicialLLT is an up-looking simplicial sparse
//       LL^T after a fill-reducing permutation (AMD by default).  We use the
//       same up-looking LL^T (elimination tree + row patterns) with a
//       graph nested-dissection ordering instead of AMD; the permutation
//       changes only roundoff.
//   - Map<const VectorXd>, Map<VectorXd>::operator=           coarse_solver.hpp:37-39
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
enum StorageOptions { ColMajor = 0, RowMajor = 0x1 };
enum DecompositionOptions { EigenvaluesOnly = 0x40, ComputeEigenvectors = 0x80 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

class VectorXd {
 public:
  VectorXd() = default;
  explicit VectorXd(Index n) : v_((size_t)n, 0.0) {}
  Index size() const { return (Index)v_.size(); }
  double& operator()(Index i) { return v_[(size_t)i]; }
  double operator()(Index i) const { return v_[(size_t)i]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }
  double maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }

 private:
  std::vector<double> v_;
};

class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(Index r, Index c) : r_(r), c_(c), a_((size_t)(r * c), 0.0) {}
  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double& operator()(Index i, Index j) { return a_[(size_t)(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return a_[(size_t)(j * r_ + i)]; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> a_;
};

namespace shim {

// Number of eigenvalues of the symmetric tridiagonal (d, e) strictly below x
// (Sturm sequence count via the LDL^T pivots).
inline int sturm_count(const std::vector<double>& d, const std::vector<double>& e, double x) {
  int count = 0;
  double q = 1.0;
  const double tiny = 1e-300;
  for (size_t i = 0; i < d.size(); ++i) {
    double off = i ? e[i - 1] * e[i - 1] : 0.0;
    q = d[i] - x - (i ? off / q : 0.0);
    if (q == 0.0) q = -tiny;
    if (q < 0.0) ++count;
  }
  return count;
}

inline std::vector<double> tridiag_eigenvalues(const std::vector<double>& d,
                                               const std::vector<double>& e) {
  int n = (int)d.size();
  double lo = d[0], hi = d[0];
  for (int i = 0; i < n; ++i) {
    double r = (i > 0 ? std::abs(e[i - 1]) : 0.0) + (i + 1 < n ? std::abs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
  }
  double scale = std::max(std::abs(lo), std::abs(hi));
  lo -= 1e-14 * scale + 1e-300;
  hi += 1e-14 * scale + 1e-300;
  std::vector<double> ev(n);
  for (int k = 0; k < n; ++k) {
    // k-th smallest eigenvalue: smallest x with count(x) > k.
    double a = lo, b = hi;
    for (int it = 0; it < 200; ++it) {
      double mid = 0.5 * (a + b);
      if (mid <= a || mid >= b) break;
      if (sturm_count(d, e, mid) > k)
        b = mid;
      else
        a = mid;
    }
    ev[k] = 0.5 * (a + b);
  }
  return ev;
}

inline std::vector<double> jacobi_eigenvalues(MatrixXd m) {
  int n = (int)m.rows();
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += m(i, j) * m(i, j);
    if (off < 1e-30) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (m(p, q) == 0.0) continue;
        double theta = (m(q, q) - m(p, p)) / (2.0 * m(p, q));
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          double mkp = m(k, p), mkq = m(k, q);
          m(k, p) = c * mkp - s * mkq;
          m(k, q) = s * mkp + c * mkq;
        }
        for (int k = 0; k < n; ++k) {
          double mpk = m(p, k), mqk = m(q, k);
          m(p, k) = c * mpk - s * mqk;
          m(q, k) = s * mpk + c * mqk;
        }
      }
  }
  std::vector<double> ev(n);
  for (int i = 0; i < n; ++i) ev[i] = m(i, i);
  std::sort(ev.begin(), ev.end());
  return ev;
}

}  // namespace shim

template <class MatrixType>
class SelfAdjointEigenSolver {
 public:
  SelfAdjointEigenSolver(const MatrixXd& m, int /*options*/ = EigenvaluesOnly) {
    Index n = m.rows();
    bool tridiagonal = true;
    for (Index j = 0; j < n && tridiagonal; ++j)
      for (Index i = 0; i < n; ++i)
        if (std::abs(i - j) > 1 && m(i, j) != 0.0) {
          tridiagonal = false;
          break;
        }
    std::vector<double> ev;
    if (n == 0) {
    } else if (tridiagonal) {
      std::vector<double> d((size_t)n), e((size_t)std::max<Index>(n - 1, 0));
      for (Index i = 0; i < n; ++i) d[(size_t)i] = m(i, i);
      for (Index i = 0; i + 1 < n; ++i) e[(size_t)i] = m(i + 1, i);
      ev = shim::tridiag_eigenvalues(d, e);
    } else {
      ev = shim::jacobi_eigenvalues(m);
    }
    evals_ = VectorXd(n);
    for (Index i = 0; i < n; ++i) evals_(i) = ev[(size_t)i];
  }
  const VectorXd& eigenvalues() const { return evals_; }

 private:
  VectorXd evals_;
};

template <class Scalar, int Options = ColMajor, class StorageIndex = int>
class SparseMatrix;

template <class T>
class Map;

// Read-only view of a compressed sparse matrix (row-major in the reference).
template <class Scalar, int Options, class StorageIndex>
class Map<const SparseMatrix<Scalar, Options, StorageIndex>> {
 public:
  Map(Index rows, Index cols, Index nnz, const StorageIndex* outer, const StorageIndex* inner,
      const Scalar* values)
      : rows_(rows), cols_(cols), nnz_(nnz), outer_(outer), inner_(inner), values_(values) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index nonZeros() const { return nnz_; }
  const StorageIndex* outerIndexPtr() const { return outer_; }
  const StorageIndex* innerIndexPtr() const { return inner_; }
  const Scalar* valuePtr() const { return values_; }

 private:
  Index rows_, cols_, nnz_;
  const StorageIndex* outer_;
  const StorageIndex* inner_;
  const Scalar* values_;
};

// Column-major (CSC) owning sparse matrix.
template <class Scalar, int Options, class StorageIndex>
class SparseMatrix {
 public:
  SparseMatrix() = default;
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  template <int O2, class I2>
  SparseMatrix& operator=(const Map<const SparseMatrix<Scalar, O2, I2>>& m) {
    rows_ = m.rows();
    cols_ = m.cols();
    std::vector<Index> ptr((size_t)cols_ + 1, 0);
    Index outer = (O2 & RowMajor) ? rows_ : cols_;
    for (Index o = 0; o < outer; ++o)
      for (I2 p = m.outerIndexPtr()[o]; p < m.outerIndexPtr()[o + 1]; ++p) {
        Index r = (O2 & RowMajor) ? o : (Index)m.innerIndexPtr()[p];
        Index c = (O2 & RowMajor) ? (Index)m.innerIndexPtr()[p] : o;
        (void)r;
        ++ptr[(size_t)c + 1];
      }
    for (Index c = 0; c < cols_; ++c) ptr[(size_t)c + 1] += ptr[(size_t)c];
    col_ptr_.assign(ptr.begin(), ptr.end());
    row_idx_.assign((size_t)ptr.back(), 0);
    vals_.assign((size_t)ptr.back(), 0.0);
    std::vector<Index> pos(ptr.begin(), ptr.end() - 1);
    // Row-major traversal in ascending row order keeps CSC rows sorted.
    for (Index o = 0; o < outer; ++o)
      for (I2 p = m.outerIndexPtr()[o]; p < m.outerIndexPtr()[o + 1]; ++p) {
        Index r = (O2 & RowMajor) ? o : (Index)m.innerIndexPtr()[p];
        Index c = (O2 & RowMajor) ? (Index)m.innerIndexPtr()[p] : o;
        Index k = pos[(size_t)c]++;
        row_idx_[(size_t)k] = r;
        vals_[(size_t)k] = m.valuePtr()[p];
      }
    return *this;
  }
  const std::vector<Index>& col_ptr() const { return col_ptr_; }
  const std::vector<Index>& row_idx() const { return row_idx_; }
  const std::vector<Scalar>& vals() const { return vals_; }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<Index> col_ptr_, row_idx_;
  std::vector<Scalar> vals_;
};

template <>
class Map<const VectorXd> {
 public:
  Map(const double* p, Index n) : p_(p), n_(n) {}
  Index size() const { return n_; }
  double operator()(Index i) const { return p_[i]; }

 private:
  const double* p_;
  Index n_;
};

template <>
class Map<VectorXd> {
 public:
  Map(double* p, Index n) : p_(p), n_(n) {}
  Map& operator=(const VectorXd& v) {
    for (Index i = 0; i < n_; ++i) p_[i] = v(i);
    return *this;
  }

 private:
  double* p_;
  Index n_;
};

}  // namespace Eigen
