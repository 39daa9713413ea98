// On-device sparse Cholesky of the assembled p = 1 coarse operator
// (CholeskyCoarseSolver, coarse_solver.hpp:16-47, which uses Eigen's
// SimplicialLLT): geometric nested dissection of the Q1 node lattice and a
// multifrontal LL^T with dense fronts factored by cuSOLVER/cuBLAS FP64; the
// per-V-cycle triangular solves run level by level over the dissection tree.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <vector>

#include "coarse.hpp"

namespace hxg {

class NdCholesky {
 public:
  NdCholesky() = default;
  ~NdCholesky();
  NdCholesky(const NdCholesky&) = delete;
  NdCholesky& operator=(const NdCholesky&) = delete;

  // Symbolic analysis (first call) + numeric factorization of the CSR
  // matrix (both triangles stored) on the npd[0] x npd[1] x npd[2] lattice,
  // 3 DoFs per node.  Throws NOT_SPD if a pivot block is not SPD.
  void factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s);
  void solve(const double* b, double* x, cudaStream_t s);
  bool ready() const { return ready_; }
  double factor_bytes() const { return (double)lsize_ * sizeof(double); }

 private:
  struct Front {
    int parent = -1;
    int child[2] = {-1, -1};
    int level = 0;      // depth in the dissection tree (root = 0)
    int piv0 = 0;       // first pivot in the new numbering (pivots contiguous)
    int np = 0;         // pivots (DoFs)
    int ns = 0;         // shell (update) rows
    size_t loff = 0;    // offset of the (np + ns) x np panel in L
    size_t rows_off = 0;  // offset of the shell rows (new numbering) in shell_rows
    size_t map_off[2] = {0, 0};  // offsets of the child-update maps
  };
  void analyze(const CsrMatrix& a, const int npd[3]);

  bool analyzed_ = false, ready_ = false;
  int n_ = 0;
  std::vector<Front> fronts_;           // postorder
  std::vector<std::vector<int>> levels_;  // fronts per depth
  size_t lsize_ = 0, max_front_ = 0, max_update_ = 0;

  // device
  DevBuf<int> perm_;         // new -> old DoF
  DevBuf<int> shell_rows_;   // concatenated shell rows (new numbering)
  DevBuf<int> child_map_;    // concatenated child update -> parent front positions
  DevBuf<long long> asm_dst_;  // assembly: destination offset in the front workspace
  DevBuf<int> asm_src_;      // assembly: CSR slot
  DevBuf<double> L_;         // factor panels
  DevBuf<double> work_;      // current front (m x m)
  DevBuf<double> stack_;     // pending update matrices
  DevBuf<double> wvec_;      // solve work vector (new numbering)
  DevBuf<double> ubuf_;      // per-front update vectors (forward sweep)
  DevBuf<double> ybuf_;      // large-front vector
  DevBuf<int> info_;
  DevBuf<double> potrf_ws_;
  DevBuf<int> dfront_piv0_, dfront_np_, dfront_ns_, c0_, c1_;
  DevBuf<long long> dfront_loff_, dfront_rows_off_, map0_, map1_, uoff_;
  DevBuf<int> small_lists_;               // small fronts, grouped by level
  std::vector<size_t> small_off_;         // per level offsets into small_lists_
  std::vector<std::vector<int>> big_;     // large fronts per level
  std::vector<size_t> asm_begin_;  // per front range in the assembly lists
  cublasHandle_t cublas_ = nullptr;
  cusolverDnHandle_t cusolver_ = nullptr;
};

}  // namespace hxg
