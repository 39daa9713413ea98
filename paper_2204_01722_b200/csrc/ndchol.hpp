// On-device sparse Cholesky of the assembled p = 1 coarse operator
// (CholeskyCoarseSolver, coarse_solver.hpp:16-47, which uses Eigen's
// SimplicialLLT): geometric nested dissection of the Q1 node lattice and a
// multifrontal LL^T with dense fronts factored on FP64 tensor-core GEMMs.
// Each front keeps its panel as [L11^-1; L21], so the per-V-cycle triangular
// solves are bandwidth-bound GEMVs (two dependent ones per front and
// direction), batched over every front of a dissection-tree level.
#pragma once

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <memory>
#include <utility>
#include <vector>

#include "coarse.hpp"

namespace hxg {

class NdCholesky {
 public:
  // leaf_nodes: dissection stops at regions of at most this many lattice
  // nodes (0: the default); a leaf larger than the lattice gives one dense
  // front (the dense coarse mode).
  explicit NdCholesky(long long leaf_nodes = 0);
  ~NdCholesky();
  NdCholesky(const NdCholesky&) = delete;
  NdCholesky& operator=(const NdCholesky&) = delete;

  // Symbolic analysis (first call) + numeric factorization of the CSR
  // matrix (both triangles stored) on the npd[0] x npd[1] x npd[2] lattice,
  // 3 DoFs per node.  Throws NOT_SPD if a pivot block is not SPD.
  void factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s);
  // The ~120 dependent per-level launches of a solve are replayed from a
  // CUDA graph (captured on an internal stream once per factorization);
  // HXG_NO_GRAPH=1 launches them directly.
  void solve(const double* b, double* x, cudaStream_t s);
  bool ready() const { return ready_; }
  double factor_bytes() const { return (double)lsize_ * sizeof(double); }
  int num_levels() const { return (int)levels_.size(); }

 private:
  void solve_launch(cudaStream_t s);  // per-level core on wvec_
  void run_graph(cudaStream_t s);
  cudaStream_t gstream_ = nullptr;
  cudaEvent_t gev_in_ = nullptr, gev_out_ = nullptr;
  cudaGraphExec_t graph_ = nullptr;
  // the captured numeric factorisation (per pattern and value buffer)
  void factor_launch(const CsrMatrix& a, cudaStream_t s);
  cudaGraphExec_t fgraph_ = nullptr;
  const double* fgraph_vals_ = nullptr;
  bool fgraph_failed_ = false;
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

  long long leaf_nodes_;
  bool analyzed_ = false, ready_ = false;
  int n_ = 0;
  std::vector<Front> fronts_;           // postorder
  std::vector<std::vector<int>> levels_;  // fronts per depth
  size_t lsize_ = 0;

  // device
  DevBuf<int> perm_;         // new -> old DoF
  DevBuf<int> shell_rows_;   // concatenated shell rows (new numbering)
  DevBuf<int> child_map_;    // concatenated child update -> parent front positions
  DevBuf<long long> asm_dst_;  // assembly: destination offset in the front workspace
  DevBuf<int> asm_src_;      // assembly: CSR slot
  DevBuf<double> L_;         // factor panels
  struct Lane;
  void plan_lanes();
  void factor_front(int t, Lane& lane, const CsrMatrix& a,
                    std::vector<std::pair<size_t, int>>& stack);
  std::vector<std::unique_ptr<Lane>> lanes_;
  std::vector<int> lane_of_;
  std::vector<int> top_;  // fronts above the lane depth (postorder)
  std::vector<size_t> handoff_off_;  // subtree roots: offset of the handed-over update
  DevBuf<double> handoff_;
  DevBuf<double> wvec_;      // solve work vector (new numbering)
  DevBuf<double> ubuf_;      // per-front update vectors (forward sweep)
  DevBuf<double> yvec_;      // per-front front vectors
  DevBuf<double> part_f_, part_b_;  // GEMV tile partial sums
  DevBuf<int> info_;
  // Per-front solve metadata and the tile lists (see ndchol.cu).
  DevBuf<int> dfront_piv0_, dfront_np_, dfront_ns_, c0_, c1_;
  DevBuf<long long> dfront_loff_, dfront_rows_off_, yoff_, uoff_;
  DevBuf<int> src0_, src1_;  // front position -> child update index (or -1)
  // GEMV tiles per panel part (0 = W block, 1 = L21 block), row tiles per
  // part and for the whole front (2), column tiles.
  DevBuf<int> ftile0_[2], btile0_[2], ftile_front_[2], btile_front_[2];
  DevBuf<int> rtile_front_[3], rtile_rb_[3], ctile_front_, ctile_cb_;
  // Per level: [begin, end) into the tile lists.
  std::vector<int> lev_ft_[2], lev_bt_[2], lev_rt_[3], lev_ct_;
  std::vector<size_t> asm_begin_;  // per front range in the assembly lists
};

}  // namespace hxg
