// Inexact coarse mode (SURVEY.md §7.2 hard part 3): the p = 1 coarse level of
// the p-multigrid hierarchy is solved by ONE geometric h-multigrid V-cycle
// instead of the reference's exact SimplicialLLT solve (coarse_solver.hpp:
// 16-47, called from multigrid.hpp:167-170).  A documented deviation, opt-in
// (hxg_mg_set_coarse_mode(mg, 4)), reported beside the exact mode.
//
// Levels: the assembled Q1 matrix A_0 on the lattice of the fine cells, then
// Galerkin operators A_{l+1} = P~^T A_l P~ on lattices of ceil(c / 2) cells,
// P = trilinear interpolation (x I3), P~ = M_f P M_c with constrained rows
// (fine) and columns (coarse) removed.  A_{l+1} is formed element by element
// from the level's element matrices (children of a coarse element are its
// 2 x 2 x 2 fine cells; trilinear interpolation is continuous, so the sum of
// the element products is the exact triple product) and assembled with the
// coarse-assembly slot sums.  Smoothing: degree-2 Chebyshev-Jacobi on [0.1,
// 1.1] lambda_max (the reference's smoother, smoother.hpp:15-63) with
// lambda_max from 10 Lanczos steps on rough_seed (cg.hpp:138-184), one pre
// and one post sweep; bottom (<= kHmgBottomMax DoFs): dense Cholesky inverse
// applied by a fixed-order GEMV.  The cycle is a fixed symmetric linear
// operator, so the outer PCG stays valid.
//
// Partitioned: every h-level is distributed like the
// p-levels -- this rank's block of each lattice (the Galerkin element
// products are block-local while the block's cells stay even), level
// operator = local CSR product + interface sums (constrained rows identity),
// owned-entry dots, global rough_seed slices, restriction = x 1/2 on the
// shared fine planes, local, interface sum; prolongation local (consistent).
// Only the bottom (<= kHmgBottomMax DoFs globally, or where a block's cells
// turn odd) is replicated: its matrix summed over the blocks once per setup
// (one all-reduce), its right-hand side once per cycle.
#pragma once

#include <memory>
#include <vector>

#include "coarse.hpp"
#include "dist.hpp"
#include "solver.hpp"

namespace hxg {

// Coarsen while the level has more DoFs than this (the bottom's dense inverse
// costs O(n^3) per setup: 2187 DoF 6 ms, 375 DoF < 1 ms).
constexpr int kHmgBottomMax = 1000;
// Largest bottom accepted when the coarsening has to stop early (thin boxes,
// blocks whose cells turn odd): a 16000-DoF dense inverse is 2 GB.
constexpr int kHmgBottomLimit = 16000;

// Dense SPD inverse (dense_chol_inv + W^T W once per setup), applied with a
// hand-written fixed-order GEMV.
class DenseInverse {
 public:
  ~DenseInverse();
  void factorize(const CsrMatrix& a, cudaStream_t s);
  void solve(const double* b, double* x, cudaStream_t s) const;
  int n() const { return n_; }

 private:
  void* handle_ = nullptr;  // cublasHandle_t
  int n_ = 0;
  DevBuf<double> inv_, work_, wfac_, scratch_;
  DevBuf<int> info_;
};

class HmgCoarse {
 public:
  HmgCoarse();
  ~HmgCoarse();
  // a0: assembled Q1 matrix on box0 (order 1) with constraint mask0 (host,
  // empty = none); elem0: its element matrices (E x 24 x 24, unmasked, the
  // CoarseAssembly layout).  Symbolic work (lattices, masks, patterns) on the
  // first call, numeric work every call.
  // part: null for one process; else box0 / mask0 / a0 / elem0 are this
  // rank's block of the p = 1 level.
  void setup(const CsrMatrix& a0, const BoxDev& box0, const std::vector<uint8_t>& mask0,
             const double* elem0, cudaStream_t s, Partition* part = nullptr);
  // x = V(b): one h-multigrid V-cycle from x = 0.
  void solve(const double* b, double* x, cudaStream_t s);
  bool ready() const { return ready_; }
  int num_levels() const { return (int)levels_.size(); }
  long long level_size(int l) const;
  // Level l's assembled matrix (l = 0: the p = 1 level it was set up on).
  const CsrMatrix& level_matrix(int l) const;
  const std::vector<uint8_t>& level_mask(int l) const;

 private:
  struct HLevel;
  struct Replicated;
  void cycle(size_t l, const double* b, double* x, cudaStream_t s);
  void apply_level(HLevel& lv, const double* x, double* y, cudaStream_t s);
  std::vector<std::unique_ptr<HLevel>> levels_;
  DenseInverse bottom_;
  std::unique_ptr<Replicated> rep_;  // partitioned bottom
  Partition* part_ = nullptr;
  bool ready_ = false;
};

}  // namespace hxg
