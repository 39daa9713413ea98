/*
 * hexmg_b200.h — C-ABI of the B200-native FP64 matrix-free p-multigrid path.
 *
 * Drop-in boundary for the reference header library `hexmg`
 * (/root/reference/proj/include/hexmg).  Every entry point names the
 * reference interface it replaces (file:line).  Plain pointers and sizes
 * only; device pointers unless the name ends in `_host`.  All calls return
 * 0 (HXG_OK) or an HXG_ERR_* code; details (including the first inverted
 * element/point and its Jacobian) come from hxg_last_error(), thread-local,
 * mirroring the reference's typed exceptions (errors.hpp:9-104).
 *
 * Vector layouts are the reference's: L-vectors interleave 3 components per
 * lattice node (`3*node + c`, mesh.hpp:24, :98); nodes are numbered x-fastest
 * on the (p*nx+1)(p*ny+1)(p*nz+1) Gauss-Lobatto lattice (mesh.hpp:14-33).
 * Constrained (Dirichlet) entries pass through Jacobian applies and are zero
 * in residuals (operator.hpp:177-179, :212-214).
 *
 * Threading: a handle is not reentrant (the reference operator has mutable
 * scratch, operator.hpp:369-372); calls on one handle are serialised on its
 * stream.  Results do not depend on launch configuration: every reduction
 * (scatter, dot) runs in a fixed order.
 */
#ifndef HEXMG_B200_H
#define HEXMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HXG_OK = 0,
  HXG_ERR_GENERIC = 1,
  HXG_ERR_INVERTED_ELEMENT = 2,   /* InvertedElementError      errors.hpp:9    */
  HXG_ERR_STATE_NOT_INITIALIZED = 3, /* StateNotInitializedError errors.hpp:46 */
  HXG_ERR_INDEFINITE = 4,         /* IndefiniteOperatorError   errors.hpp:55   */
  HXG_ERR_NOT_SPD = 5,            /* NotSpdError               errors.hpp:68   */
  HXG_ERR_INVALID_SMOOTHER = 6,   /* InvalidSmootherError      errors.hpp:62   */
  HXG_ERR_INVALID_ARGUMENT = 7,   /* std::invalid_argument (size mismatch etc.) */
  HXG_ERR_CUDA = 8,
  HXG_ERR_UNSUPPORTED = 9,
  HXG_ERR_STEP_REJECTED = 10      /* StepRejectedError         errors.hpp       */
};

typedef struct {
  int code;
  int element;     /* InvertedElementError::element(), -1 if n/a */
  int point;       /* InvertedElementError::point(),   -1 if n/a */
  double jacobian; /* InvertedElementError::jacobian(); the curvature
                      of an IndefiniteOperatorError                 */
  char message[512];
} hxg_error;

/* Last error of the calling thread. */
int hxg_last_error(hxg_error* out);
const char* hxg_version(void);

typedef struct hxg_state_s* hxg_state_t; /* QuadratureStateStore   operator.hpp:60-64 */
typedef struct hxg_op_s* hxg_op_t;       /* MatrixFreeOperator     operator.hpp:70    */
typedef struct hxg_mg_s* hxg_mg_t;       /* MultigridHierarchy     multigrid.hpp:88   */
typedef struct hxg_chol_s* hxg_chol_t;   /* CholeskyCoarseSolver   coarse_solver.hpp:16 */
typedef struct hxg_asm_s* hxg_asm_t;     /* CooAssembly            assembly.hpp:134   */
typedef struct hxg_comm_s* hxg_comm_t;   /* communicator of a partitioned hierarchy  */

/*
 * Operator descriptor = the arguments of the MatrixFreeOperator constructor
 * (operator.hpp:72-97) flattened to arrays: BoxMesh (counts/order,
 * mesh.hpp:19-33; restriction is analytic, mesh.hpp:119-138), Basis1D
 * (basis.hpp:117-130), GeometricFactors dxidX/weight (mesh.hpp:169-189,
 * reference layout (e, q, 9) and (e, q)), NeoHookean (material.hpp:15-18),
 * JacobianStorage (0 Current, 1 InitialNative, 2 InitialTuned, 3 InitialAD;
 * material.hpp:66-78), Constraints mask
 * (operator.hpp:29-35; NULL = unconstrained).  Host pointers, copied.
 */
typedef struct {
  int order;             /* p                                  */
  int qpts;              /* q, points per dimension            */
  int cells[3];          /* BoxMesh::counts                    */
  const double* interp;  /* q x (p+1) Basis1D::interp          */
  const double* deriv;   /* q x (p+1) Basis1D::deriv           */
  const double* colloc;  /* q x q     Basis1D::colloc_deriv    */
  const double* dxidX;   /* E*q^3*9   GeometricFactors::dxidX  */
  const double* weight;  /* E*q^3     GeometricFactors::weight */
  double mu, lambda;     /* NeoHookean                         */
  int storage;           /* JacobianStorage 0..3 (see above)   */
  const uint8_t* mask;   /* 3*num_nodes Constraints::mask or NULL */
  /* Device-side geometry: when dxidX/weight are NULL
   * and both of these are given, the geometric factors of the axis-aligned
   * box BoxMesh (build_box_mesh, mesh.hpp:35-60; affine elements) are
   * computed on the device: dxi/dX = diag(2 cells / extents), w detJ =
   * w_x w_y w_z prod(extents / (2 cells)) -- no E*q^3*10 host arrays. */
  const double* extents; /* 3, or NULL                          */
  const double* qweights;/* q Gauss-Legendre weights, or NULL   */
} hxg_op_desc;

/* QuadratureStateStore shared by all levels of a hierarchy
 * (multigrid.hpp:229-249); reference-counted. */
int hxg_state_create(hxg_state_t* out);
int hxg_state_release(hxg_state_t s);

/* MatrixFreeOperator ctor (operator.hpp:72-97).  `state` may be NULL (a new
 * store is created).  The handle keeps a reference on the state. */
int hxg_op_create(const hxg_op_desc* desc, hxg_state_t state, hxg_op_t* out);
int hxg_op_destroy(hxg_op_t op);
/* size() = 3 * num_nodes (operator.hpp:99). */
int hxg_op_size(hxg_op_t op, int64_t* n);
int hxg_op_num_elements(hxg_op_t op, int64_t* ne);
/* Stream for all work of this handle (cudaStream_t; NULL = legacy default). */
int hxg_op_set_stream(hxg_op_t op, void* stream);
/* set_external_load / set_load_scale (operator.hpp:112-122); host load, may be NULL. */
int hxg_op_set_external_load(hxg_op_t op, const double* load_host);
int hxg_op_set_load_scale(hxg_op_t op, double s);
/* set_jacobian_perturbation test hook (operator.hpp:124-126). */
int hxg_op_set_jacobian_perturbation(hxg_op_t op, double eps);
/* stored_bytes_per_dof (operator.hpp:137-141): the reference byte model. */
int hxg_op_stored_bytes_per_dof(hxg_op_t op, double* out);
/* residual / jacobian apply counters (operator.hpp:128-133). */
int hxg_op_counters(hxg_op_t op, int64_t* residual_applies, int64_t* jacobian_applies);

/* apply_residual (operator.hpp:146-180): writes the shared state; raises
 * HXG_ERR_INVERTED_ELEMENT with the lexicographically first (e, q). */
int hxg_op_apply_residual(hxg_op_t op, const double* u, double* f);
/* apply_jacobian (operator.hpp:184-215). */
int hxg_op_apply_jacobian(hxg_op_t op, const double* du, double* y);
/* Same, host buffers: H2D copy, apply, D2H copy (end-to-end path). */
int hxg_op_apply_jacobian_host(hxg_op_t op, const double* du_host, double* y_host);
int hxg_op_apply_residual_host(hxg_op_t op, const double* u_host, double* f_host);
/* extract_diagonal (operator.hpp:247-283): constrained entries are 1. */
int hxg_op_extract_diagonal(hxg_op_t op, double* d);
/* total_strain_energy (operator.hpp:287-315). */
int hxg_op_total_strain_energy(hxg_op_t op, const double* u, double* energy);
/* Quadrature state in the reference layout (e, q, 17), host. */
int hxg_op_export_state(hxg_op_t op, double* state_host);
/* Apply kernel variant: 0 = fused brick kernel (default), 1 = two-pass
 * (element kernel + node-ordered sum; reference summation order). */
int hxg_op_set_variant(hxg_op_t op, int variant);
/* Number of kernels one Jacobian apply launches with the current variant. */
int hxg_op_kernel_launches(hxg_op_t op, int* n);

/* ElementRestriction gather / scatter_add (mesh.hpp:88-116) on the
 * operator's lattice: E-vector layout (e, c, a), x-fastest a. */
int hxg_op_gather(hxg_op_t op, const double* l_vec, double* e_vec);
int hxg_op_scatter_add(hxg_op_t op, const double* e_vec, double* l_vec);

/*
 * Multigrid hierarchy (build_hierarchy, multigrid.hpp:212-268).  `fine` is
 * the finest operator; the library builds each coarser level p -> ceil(p/2)
 * -> .. -> 1 on the fine rule and shared state, with Dirichlet masks
 * re-derived from `fixed_face_mask` (bit f = Face f in -x,+x,-y,+y,-z,+z
 * order, all components; build_constraints, operator.hpp:36-55).
 * `schedule` may be NULL (default_schedule, multigrid.hpp:15-19).
 */
int hxg_mg_create(hxg_op_t fine, int fixed_face_mask, const int* schedule, int num_levels,
                  int pre_smooth, int post_smooth, hxg_mg_t* out);
int hxg_mg_destroy(hxg_mg_t mg);
int hxg_mg_num_levels(hxg_mg_t mg, int* n);
int hxg_mg_level_size(hxg_mg_t mg, int level, int64_t* n);
int hxg_mg_level_op(hxg_mg_t mg, int level, hxg_op_t* op); /* borrowed */
/* setup_numeric (multigrid.hpp:100-113): diagonals, Chebyshev lambda_max by
 * 10 Lanczos steps, coarse assembly (assembly.hpp:142-230) + Cholesky. */
int hxg_mg_setup_numeric(hxg_mg_t mg);
/* coo_numeric only (assembly.hpp:178-230): assemble the p = 1 operator on the
 * current state without building smoothers or factorizing (read it back with
 * hxg_mg_coarse_csr_host). */
int hxg_mg_assemble_coarse(hxg_mg_t mg);
/* Coarse Cholesky backend: 0 automatic (dense below a few thousand DoFs,
 * else nested-dissection multifrontal), 1 dense (one front), 2
 * nested-dissection multifrontal (3 is no longer accepted).  Takes effect
 * at the next setup_numeric.  4 = INEXACT coarse mode, a documented
 * deviation from the reference's exact SimplicialLLT (coarse_solver.hpp:
 * 16-47): the p = 1 level is solved by one Galerkin h-multigrid V-cycle
 * (Chebyshev-Jacobi smoothing, dense bottom); single-process hierarchies. */
int hxg_mg_set_coarse_mode(hxg_mg_t mg, int mode);
int hxg_mg_lambda_max(hxg_mg_t mg, int level, double* out);
/* prolong / restrict_to (multigrid.hpp:122-135). */
int hxg_mg_prolong(hxg_mg_t mg, int coarse_level, const double* xc, double* xf);
int hxg_mg_restrict(hxg_mg_t mg, int coarse_level, const double* xf, double* xc);
/* v_cycle (multigrid.hpp:137-144); preconditioner() zero-initialises x. */
int hxg_mg_vcycle(hxg_mg_t mg, const double* b, double* x);
/* ChebyshevSmoother::apply on level k (smoother.hpp:41-62). */
int hxg_mg_smooth(hxg_mg_t mg, int level, const double* b, double* x);
/* Assembled coarse operator (CSR, sorted columns) — copy to host. */
int hxg_mg_coarse_nnz(hxg_mg_t mg, int64_t* nnz);
/* Device copy of the assembled coarse values (CSR order of
 * hxg_mg_coarse_csr_host), no host round trip. */
int hxg_mg_coarse_vals_device(hxg_mg_t mg, double* vals_dev);
int hxg_mg_coarse_csr_host(hxg_mg_t mg, int* row_ptr, int* cols, double* vals);
/* Inexact coarse mode (4): number of h-multigrid levels after the last
 * setup_numeric (0 when the mode is not active), and level l's Galerkin
 * matrix (CSR, sorted columns; l = 0 is the p = 1 level) with its constraint
 * mask (n bytes) -- for inspection and tests. */
int hxg_mg_hmg_levels(hxg_mg_t mg, int* levels);
int hxg_mg_hmg_level_nnz(hxg_mg_t mg, int level, int64_t* n, int64_t* nnz);
int hxg_mg_hmg_level_csr_host(hxg_mg_t mg, int level, int* row_ptr, int* cols, double* vals,
                              uint8_t* mask);
/* Coarse Cholesky solve (coarse_solver.hpp:35-40). */
int hxg_mg_coarse_solve(hxg_mg_t mg, const double* b, double* x);

/* Standalone CholeskyCoarseSolver (coarse_solver.hpp:16-47) on a caller's
 * assembled Q1 lattice matrix (CSR, both triangles, sorted columns, host
 * arrays; npd = nodes per dimension, n = 3 * nodes).  analyzePattern on
 * create, factorize per numeric setup, solve per V-cycle (device vectors).
 * Used for the replicated coarse solve of the slab-partitioned p-MG. mode as
 * hxg_mg_set_coarse_mode. */
int hxg_chol_create(int n, const int* row_ptr, const int* cols, const int npd[3], int mode,
                    hxg_chol_t* out);
int hxg_chol_factorize(hxg_chol_t h, const double* vals_host);
/* Same with the values already on the device. */
int hxg_chol_factorize_device(hxg_chol_t h, const double* vals_dev);
int hxg_chol_solve(hxg_chol_t h, const double* b, double* x);
int hxg_chol_destroy(hxg_chol_t h);

/* Assembled representation of an operator of any order (CooAssembly:
 * coo_symbolic / coo_numeric / CsrMatrix::matvec, assembly.hpp:134-230):
 * CSR over all DoFs, constrained rows and columns reduced to the identity,
 * slot values summed over elements in increasing element order.  create =
 * symbolic; numeric needs the operator's state (StateNotInitialized
 * otherwise); matvec on device vectors.  The "assembled" rows of the
 * performance study (study.hpp:191-232).  The operator must outlive the
 * handle (it is re-read by numeric). */
int hxg_asm_create(hxg_op_t op, hxg_asm_t* out);
int hxg_asm_numeric(hxg_asm_t a);
int hxg_asm_nnz(hxg_asm_t a, int64_t* nnz);
int hxg_asm_matvec(hxg_asm_t a, const double* x, double* y);
int hxg_asm_csr_host(hxg_asm_t a, int* row_ptr, int* cols, double* vals);
int hxg_asm_destroy(hxg_asm_t a);

/*
 * Partitioned (multi-GPU) p-multigrid, SURVEY.md §8(e).  The reference is
 * single-process; the paper distributes the same operator with
 * sums of the shared nodes after every apply (A = P^T E^T B^T D B E P,
 * PAPER.md:224-228, :316).  The box of global_cells elements is cut into
 * dims[0] x dims[1] x dims[2] contiguous element blocks (rank = x fastest,
 * hxg_partition_block gives this rank's block); each rank creates its fine
 * operator on its block (hxg_op_create with the block's cells, geometry,
 * Dirichlet mask and load) and the partitioned hierarchy over it.  Then
 *   hxg_mg_apply / hxg_mg_residual   the operator / residual + interface sums,
 *   hxg_mg_dot                       owned-entry dot, all-reduced,
 *   hxg_mg_setup_numeric / _vcycle   smoothers on the summed diagonal,
 *                                    lambda_max from the GLOBAL rough_seed,
 *                                    transfers with the interface scaling,
 *                                    the coarse level summed into the global
 *                                    Q1 matrix and factorized on every rank,
 *   hxg_cg_solve(op, mg, ...)        PCG with owned-entry dots,
 *   hxg_newton_solve / hxg_solve_continuation   Newton-CG (L-BFGS: 1 rank).
 * Communicator: the built-in NCCL one (libnccl.so.2 resolved at run time;
 * the unique id from hxg_nccl_unique_id on one rank, broadcast by the caller)
 * or a caller-supplied table.  Entry points are stream-ordered on `stream`
 * (the operator's stream); return 0 on success.
 */
typedef struct {
  void* ctx;
  /* Grouped neighbour exchange: for each i < npeers send counts[i] doubles
   * from send[i] to peers[i] and receive as many into recv[i] (device
   * buffers). */
  int (*exchange)(void* ctx, int npeers, const int* peers, const double* const* send,
                  double* const* recv, const int64_t* counts, void* stream);
  /* In-place all-reduce of `count` device doubles; op 0 = sum, 1 = max. */
  int (*allreduce)(void* ctx, double* data, int64_t count, int op, void* stream);
} hxg_comm_ops;
int hxg_comm_create(int rank, int world, const hxg_comm_ops* ops, hxg_comm_t* out);
int hxg_nccl_unique_id(void* id128);
int hxg_comm_create_nccl(int rank, int world, const void* id128, hxg_comm_t* out);
int hxg_comm_destroy(hxg_comm_t comm);
/* This rank's block: local element counts and first global element. */
int hxg_partition_block(const int global_cells[3], const int dims[3], int rank, int cells[3],
                        int e0[3]);
/* build_hierarchy (multigrid.hpp:212-268) on this rank's block; the
 * Dirichlet faces are GLOBAL faces (bit f = -x,+x,-y,+y,-z,+z). */
int hxg_mg_create_partitioned(hxg_op_t fine, hxg_comm_t comm, const int global_cells[3],
                              const int dims[3], int global_fixed_face_mask, const int* schedule,
                              int num_levels, int pre_smooth, int post_smooth, hxg_mg_t* out);
/* Level operator (apply_jacobian + interface sums when partitioned). */
int hxg_mg_apply(hxg_mg_t mg, int level, const double* x, double* y);
/* Owned-entry dot on a level (all-reduced when partitioned). */
int hxg_mg_dot(hxg_mg_t mg, int level, const double* x, const double* y, double* out);
/* Fine residual (operator.hpp:146-180) + interface sums; an inverted
 * element on any rank raises HXG_ERR_INVERTED_ELEMENT on every rank. */
int hxg_mg_residual(hxg_mg_t mg, const double* u, double* f);
int hxg_stream_synchronize(void* stream);

/* CgReport (cg.hpp:42-50). */
typedef struct {
  int iterations;
  int converged;
  double eig_min, eig_max;
  double initial_natural_norm, final_natural_norm;
} hxg_cg_report;

/* cg_solve (cg.hpp:81-134) with A = op's Jacobian.  precond: 0 identity,
 * 1 Jacobi (1/extract_diagonal), 2 p-MG V-cycle (mg required). */
int hxg_cg_solve(hxg_op_t op, hxg_mg_t mg, int precond, const double* b, double* x, double rtol,
                 int max_iterations, hxg_cg_report* report, double* history_host,
                 int history_capacity);

/* Nonlinear driver (nonlinear.hpp): NewtonConfig (:16-24), IterationRecord
 * (:26-36), SolveReport (:50-56).  reference_line_search_quirk = 1 reproduces
 * the reference's functor-copy defect (residual read as zero after a line
 * search); 0 runs the intended algorithm. */
typedef struct {
  int max_iterations;
  double rtol, atol, linear_rtol;
  int linear_max_iterations;
  int use_line_search;
  int load_steps;
  int reference_line_search_quirk;
  int solver;          /* 0 Newton-CG, 1 L-BFGS (config.hpp:15)            */
  int lbfgs_memory;    /* L-BFGS pairs (config.hpp:62)                      */
  int precond_refresh; /* L-BFGS preconditioner rebuild interval, 0 = never */
} hxg_newton_config;
typedef struct {
  int load_step;
  double time;
  int iteration;
  double fnorm, fnorm_rel;
  int cg_iterations, cg_converged;
  double condition_estimate, alpha;
} hxg_iteration_record;
typedef struct {
  int converged;
  int load_steps_taken;
  int newton_iterations;
  int cg_iterations;
  double final_fnorm;
  int num_records; /* records written (<= capacity) */
} hxg_solve_report;
/* The reference defaults (config.hpp:55-61). */
int hxg_newton_config_default(hxg_newton_config* cfg);
/* newton_solve (nonlinear.hpp:162-216) from the device iterate u (updated in
 * place); the p-MG hierarchy is set up at every linearisation point. */
int hxg_newton_solve(hxg_op_t op, hxg_mg_t mg, const hxg_newton_config* cfg, double* u,
                     int load_step, double time, hxg_solve_report* report,
                     hxg_iteration_record* records, int capacity);
/* lbfgs_solve (nonlinear.hpp:226-308): V-cycle as H0 of the two-loop
 * recursion, critical-point line search. */
int hxg_lbfgs_solve(hxg_op_t op, hxg_mg_t mg, const hxg_newton_config* cfg, double* u,
                    int load_step, double time, hxg_solve_report* report,
                    hxg_iteration_record* records, int capacity);
/* FemProblem::solve (problem.hpp:118-127): load_continuation
 * (nonlinear.hpp:325-366) from u = 0 over cfg->load_steps, whole-face zero
 * Dirichlet values; u (device) receives the solution. */
int hxg_solve_continuation(hxg_op_t op, hxg_mg_t mg, const hxg_newton_config* cfg, double* u,
                           int max_bisections, hxg_solve_report* report,
                           hxg_iteration_record* records, int capacity);

/* estimate_lambda_max (cg.hpp:152-184) of D^-1 A on `op` with rough_seed. */
int hxg_lambda_max_jacobi(hxg_op_t op, int iterations, double* out);

/* Deterministic device dot product (owned entries in fixed order). */
int hxg_dot(const double* x, const double* y, int64_t n, void* stream, double* out);

/* Device memory helpers for callers without their own allocator. */
int hxg_malloc(void** p, size_t bytes);
int hxg_free(void* p);
/* 1 if p is device (or managed) memory, 0 for host memory. */
int hxg_pointer_is_device(const void* p, int* is_device);
int hxg_memcpy_h2d(void* dst, const void* src, size_t bytes);
int hxg_memcpy_d2h(void* dst, const void* src, size_t bytes);
int hxg_device_synchronize(void);

/*
 * Host setup restating the reference's problem construction (FemProblem,
 * problem.hpp:19-58): box mesh, basis on Gauss-Legendre q points, geometric
 * factors, Dirichlet faces, traction load.  Fills arrays for hxg_op_desc.
 */
int hxg_setup_basis(int p, int q, double* nodes, double* points, double* weights,
                    double* interp, double* deriv, double* pinv, double* colloc);
int hxg_setup_geometry(const double extents[3], const int cells[3], int p, int q,
                       double* dxidX, double* weight);
int hxg_setup_constraints(const int cells[3], int p, int fixed_face_mask, uint8_t* mask);
int hxg_setup_traction_load(const double extents[3], const int cells[3], int p, int q, int face,
                            const double traction[3], double* load);

/* Timing helper: `repeats` Jacobian applies of x into y on the op's stream,
 * bracketed by CUDA events after `warmup` applies; returns milliseconds. */
/* Per-kernel split of the fused apply (instrumentation for the roofline):
 * mean ms of the brick kernel (ms[0]) and of the boundary fix-up (ms[1]) over
 * `repeats` applies, events on the operator's stream. */
int hxg_op_time_jacobian_parts(hxg_op_t op, const double* x, double* y, int warmup, int repeats,
                               double ms[2]);
int hxg_op_time_jacobian(hxg_op_t op, const double* x, double* y, int warmup, int repeats,
                         double* ms);

#ifdef __cplusplus
}
#endif

#endif /* HEXMG_B200_H */
