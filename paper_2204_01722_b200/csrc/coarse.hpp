// Assembled p = 1 coarse operator (coo_symbolic / coo_numeric,
// assembly.hpp:142-230) and its Cholesky solver (CholeskyCoarseSolver,
// coarse_solver.hpp:16-47), on device.
#pragma once

#include <memory>
#include <vector>

#include "operator.hpp"

namespace hxg {

struct CsrMatrix {
  int n = 0;
  std::vector<int> row_ptr_h, cols_h;  // host copy of the pattern
  DevBuf<int> row_ptr, cols, rows;     // rows: row index per slot
  DevBuf<double> vals;
  long long nnz() const { return (long long)cols_h.size(); }
};

// y = A x, one warp per row, fixed-order reduction.
void csr_matvec(const CsrMatrix& a, const double* x, double* y, cudaStream_t s);

class CoarseAssembly {
 public:
  // Symbolic phase (coo_symbolic): the CSR pattern of the box operator of
  // any order (every node pair sharing an element) with constrained
  // rows/columns reduced to the identity.  The p = 1 level is the coarse
  // operator; higher orders serve the "assembled" representation of the
  // performance study (study.hpp:191-232).
  explicit CoarseAssembly(const Operator& op);
  // Pattern only, for an order-box.p lattice and constraint mask (the
  // global coarse matrix of the partitioned solver).
  CoarseAssembly(const BoxDev& box, const std::vector<uint8_t>& mask);
  CsrMatrix& mutable_matrix() { return a_; }
  // Numeric phase (coo_numeric + fill_from_coo): element matrices, then a
  // per-slot sum over elements in increasing element order.
  void numeric(Operator& op);
  const CsrMatrix& matrix() const { return a_; }
  // y = A x (CsrMatrix::matvec), device vectors.
  void matvec(const double* x, double* y, cudaStream_t s) const;
  // Slot sums from caller-provided element matrices (same layout as the
  // ones numeric() computes: E x M x M, M = 3 (p + 1)^3, unmasked).
  void numeric_from_elements(const double* elem, cudaStream_t s);
  // The element matrices of the last numeric() (device).
  const double* element_matrices() const { return elem_.p; }
  const BoxDev& box() const { return box_; }

 private:
  CsrMatrix a_;
  DevBuf<double> elem_;
  DevBuf<uint8_t> mask_;
  BoxDev box_;
};

class CoarseSolverImpl;

// Coarse levels up to this many DoFs use the dense device factorization.
constexpr int kDenseCoarseMax = 6000;

class CoarseSolver {
 public:
  CoarseSolver();
  ~CoarseSolver();
  // analyzePattern (first call) + factorize; throws NOT_SPD on failure.
  // npd = nodes per dimension of the Q1 lattice (nested-dissection order).
  void factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s);
  void solve(const double* b, double* x, cudaStream_t s);
  bool ready() const;
  void set_mode(int m) { mode_ = m; }

 private:
  int mode_ = 0;
  int active_ = 0;  // backend used by the last factorize
  std::unique_ptr<CoarseSolverImpl> impl_;
  std::unique_ptr<class NdCholesky> nd_;
};

}  // namespace hxg
