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

class CoarseAssembly {
 public:
  // Symbolic phase (coo_symbolic): the CSR pattern of the box Q1 operator
  // with constrained rows/columns reduced to the identity.
  explicit CoarseAssembly(const Operator& op);
  // Numeric phase (coo_numeric + fill_from_coo): element matrices, then a
  // per-slot sum over elements in increasing element order.
  void numeric(Operator& op);
  const CsrMatrix& matrix() const { return a_; }

 private:
  CsrMatrix a_;
  DevBuf<double> elem_;
  DevBuf<uint8_t> mask_;
  BoxDev box_;
};

class CoarseSolverImpl;

class CoarseSolver {
 public:
  CoarseSolver();
  ~CoarseSolver();
  // analyzePattern (first call) + factorize; throws NOT_SPD on failure.
  void factorize(const CsrMatrix& a, const int cells[3], cudaStream_t s);
  void solve(const double* b, double* x, cudaStream_t s);
  bool ready() const;

 private:
  std::unique_ptr<CoarseSolverImpl> impl_;
};

}  // namespace hxg
