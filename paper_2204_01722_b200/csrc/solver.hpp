// Host orchestration of the device p-multigrid solver: Chebyshev smoother,
// Lanczos lambda_max, PCG and the V-cycle (smoother.hpp, cg.hpp,
// multigrid.hpp).  All vectors are device pointers; control scalars (dots)
// come back to the host once per reduction, as in the reference.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>
#include <vector>

#include "coarse.hpp"
#include "dist.hpp"
#include "operator.hpp"
#include "transfer.hpp"
#include "vector.hpp"

namespace hxg {

// HXG_PROFILE=1: print the phases of setup_numeric (device-synchronised).
struct PhaseTimer {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTimer(cudaStream_t st) : on(std::getenv("HXG_PROFILE") != nullptr), s(st) {
    if (on) {
      cudaStreamSynchronize(s);
      t = std::chrono::steady_clock::now();
    }
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hxg] %-28s %9.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// LinearOperator (cg.hpp:16-19) over device vectors.
using DevOp = std::function<void(const double*, double*)>;
// dot (cg.hpp:34-38); partitioned: owned entries, all-reduced.
using DotFn = std::function<double(const double*, const double*)>;

struct CgResult {
  int iterations = 0;
  bool converged = false;
  std::vector<double> history;
  double eig_min = 0.0, eig_max = 0.0;
};

// Extremal Ritz values of the CG/Lanczos tridiagonal (cg.hpp:56-73).
void lanczos_eigs(const std::vector<double>& alphas, const std::vector<double>& betas,
                  double& eig_min, double& eig_max);
// rough_seed (cg.hpp:138-147): mt19937(0x9e3779b9) stream, constrained zeroed.
std::vector<double> rough_seed(long long n, const std::vector<uint8_t>& mask);

// cg_solve (cg.hpp:81-134).
CgResult cg_solve(long long n, const DevOp& a, const DevOp& m, const double* b, double* x,
                  double rtol, int max_iterations, cudaStream_t s, const DotFn* dotf = nullptr);
// estimate_lambda_max (cg.hpp:152-184).
double estimate_lambda_max(long long n, const DevOp& a, const double* inv_diag,
                           const double* seed, int iterations, cudaStream_t s,
                           const DotFn* dotf = nullptr);

// ChebyshevSmoother (smoother.hpp:15-63), degree 2 on [0.1, 1.1] lambda_max.
struct Chebyshev {
  int degree = 2;
  double lambda_max = 0.0, lo = 0.0, hi = 0.0;
  DevBuf<double> inv_diag, r, d;
  DevBuf<double> seed;  // rough_seed (cg.hpp:138-147), fixed per level
  bool ready = false;
  // A: the level operator; diag(out): its assembled diagonal; seed(): the
  // Lanczos start vector (first call only); dotf: null = local dots.
  void create(long long n, cudaStream_t s, int degree_, const DevOp& A,
              const std::function<void(double*)>& diag, const DotFn* dotf,
              const std::function<std::vector<double>()>& seed_fn);
  // One sweep; x_zero = x is known to be exactly zero (A x = 0 is skipped,
  // bitwise-identical: SURVEY.md Appendix A).
  void apply(const DevOp& A, long long n, cudaStream_t s, const double* b, double* x, bool x_zero);
};

struct Level {
  int order = 0;
  std::unique_ptr<Operator> owned;
  Operator* op = nullptr;
  std::unique_ptr<Transfer> from_coarser;  // levels > 0
  Chebyshev smoother;
  DevBuf<double> residual, correction, restricted;
  DevBuf<double> scaled;  // partitioned: interface-scaled copy for the restriction
};

class Hierarchy {
 public:
  // part: null for one process; else the fine operator is this rank's block
  // and fixed_face_mask names the GLOBAL Dirichlet faces.
  Hierarchy(Operator* fine, int fixed_face_mask, std::vector<int> schedule, int pre_smooth,
            int post_smooth, Partition* part = nullptr);
  ~Hierarchy();
  int num_levels() const { return (int)levels_.size(); }
  Level& level(int k) { return *levels_[(size_t)k]; }
  Partition* partition() const { return part_; }
  void setup_numeric();
  // coo_numeric only (assembly.hpp:178-230): the assembled coarse operator
  // without smoothers or factorization (this rank's block when partitioned).
  void assemble_coarse();
  void prolong(int coarse_level, const double* xc, double* xf);
  void restrict_to(int coarse_level, const double* xf, double* xc);
  void v_cycle(const double* b, double* x, bool x_zero = false);
  void coarse_solve(const double* b, double* x);
  // The level operator (local apply + interface sums when partitioned), its
  // dot, one smoother sweep.
  void level_apply(int k, const double* x, double* y);
  double level_dot(int k, const double* x, const double* y);
  void smooth(int k, const double* b, double* x);
  // The fine-level residual (operator.hpp:146-180) + interface sums; an
  // inverted element on any rank raises on every rank.
  void residual(const double* u, double* f);
  const CsrMatrix& coarse_matrix() const {
    if (!assembly_) throw Error(HXG_ERR_STATE_NOT_INITIALIZED, "coarse operator not assembled");
    return assembly_->matrix();
  }
  // 0 automatic (dense below kDenseCoarseMax DoFs), 1 dense, 2 sparse ND,
  // 3 csrchol, 4 inexact: one Galerkin h-multigrid V-cycle (hcoarse.hpp).
  void set_coarse_mode(int m) { coarse_mode_ = m; }
  int coarse_mode() const { return coarse_mode_; }
  const class HmgCoarse* hmg() const { return hmg_.get(); }
  cudaStream_t stream() const { return levels_.back()->op->stream(); }
  // The level operators follow the fine operator's stream: a caller may
  // hxg_op_set_stream the fine operator after the hierarchy is built, and
  // every entry point re-points the coarse levels before issuing work, so a
  // V-cycle never splits across two streams.
  void follow_stream() {
    cudaStream_t s = stream();
    for (auto& lv : levels_)
      if (lv->op->stream() != s) lv->op->set_stream(s);
  }

 private:
  void cycle(int k, const double* b, double* x, bool x_zero);
  std::vector<std::unique_ptr<Level>> levels_;
  std::unique_ptr<CoarseAssembly> assembly_;
  CoarseSolver coarse_;
  std::unique_ptr<class HmgCoarse> hmg_;
  int pre_ = 1, post_ = 1, degree_ = 2, coarse_mode_ = 0;
  Partition* part_ = nullptr;
  int global_faces_ = 0;
  cudaStream_t side_ = nullptr;  // partitioned: the overlapped interface exchange
  DotWorkspace ws_;
  // Partitioned coarse level (the replicated fallback of SURVEY.md §8(e)):
  // the global p = 1 matrix summed from the blocks' assembled matrices (one
  // all-reduce of its values per numeric setup), factorized on every rank;
  // each coarse solve all-reduces the owned right-hand side entries.
  struct DistCoarse;
  std::unique_ptr<DistCoarse> dc_;
  void dist_coarse_numeric();
  void dist_coarse_solve(const double* b, double* x);
};

// Nonlinear driver (nonlinear.hpp): Newton-CG with the critical-point line
// search and load continuation, on device vectors.
struct NewtonConfig {  // nonlinear.hpp:16-24
  int max_iterations = 50;
  double rtol = 1e-8, atol = 1e-10, linear_rtol = 1e-3;
  int linear_max_iterations = 500;
  bool use_line_search = true;
  int load_steps = 1;
  // Reproduce the reference's functor-copy defect:
  // after a line search the residual is read from the un-invoked original
  // evaluator, i.e. zero.  Off by default (the intended algorithm).
  bool reference_line_search_quirk = false;
  // ProblemConfig::solver (config.hpp:15, :60-64): 0 Newton-CG, 1 L-BFGS with
  // `lbfgs_memory` pairs and the V-cycle as H0, rebuilt every
  // `precond_refresh` iterations (0 = never).
  int solver = 0;
  int lbfgs_memory = 5;
  int precond_refresh = 10;
};
struct IterationRecord {  // nonlinear.hpp:26-36
  int load_step = 0;
  double time = 1.0;
  int iteration = 0;
  double fnorm = 0.0, fnorm_rel = 0.0;
  int cg_iterations = 0;
  bool cg_converged = true;
  double condition_estimate = 0.0, alpha = 1.0;
};
struct SolveReport {  // nonlinear.hpp:50-56
  bool converged = false;
  int iterations = 0, total_cg_iterations = 0;
  double final_fnorm = 0.0;
  std::vector<IterationRecord> records;
};
// NonlinearSystem (nonlinear.hpp) over device vectors: the operator's
// residual / Jacobian, dots and the V-cycle of its hierarchy -- the
// partitioned versions when the hierarchy has a Partition.
struct System {
  long long n = 0;
  cudaStream_t s = nullptr;
  std::function<void(const double*, double*)> residual;
  DevOp jacobian, precond;
  DotFn dot;
  std::function<void()> prepare;  // setup_numeric at the linearisation point
};
System make_system(Operator& op, Hierarchy& mg);
// newton_solve (nonlinear.hpp:162-216) on op's residual / Jacobian with the
// p-MG V-cycle rebuilt at every linearisation point.
SolveReport newton_solve(Operator& op, Hierarchy& mg, const NewtonConfig& cfg, double* u,
                         int load_step, double time);
// lbfgs_solve (nonlinear.hpp:226-308) with the V-cycle as the initial
// inverse Hessian of the two-loop recursion.
SolveReport lbfgs_solve(Operator& op, Hierarchy& mg, const NewtonConfig& cfg, double* u,
                        int load_step, double time);
// FemProblem::solve (problem.hpp:118-127): load_continuation
// (nonlinear.hpp:325-366) over t_k = k / load_steps with whole-face zero
// Dirichlet values; returns the per-step reports.
std::vector<SolveReport> solve_continuation(Operator& op, Hierarchy& mg, const NewtonConfig& cfg,
                                            double* u, int max_bisections,
                                            std::vector<double>* times);

}  // namespace hxg
