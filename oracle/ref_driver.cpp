// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Thin extern "C" driver over the UNMODIFIED reference headers under
// /root/reference/proj/include (compiled in place by oracle/Makefile, with the
// Eigen-API shim in oracle/eigen_shim first on the include path).  Output goes
// to oracle/_ref/libhexmg_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's CPU-baseline leg load it, as the checker / CPU baseline — never
// the product path.
//
// Every entry point forwards to the reference call it is named after:
//   ref_apply_residual  -> MatrixFreeOperator::apply_residual   operator.hpp:146
//   ref_apply_jacobian  -> MatrixFreeOperator::apply_jacobian   operator.hpp:184
//   ref_extract_diagonal-> MatrixFreeOperator::extract_diagonal operator.hpp:247
//   ref_mg_setup        -> MultigridHierarchy::setup_numeric    multigrid.hpp:100
//   ref_prolong/restrict-> MultigridHierarchy::prolong/restrict_to multigrid.hpp:122-135
//   ref_vcycle          -> MultigridHierarchy::v_cycle          multigrid.hpp:137
//   ref_cg              -> cg_solve                             cg.hpp:81
//   ref_verify          -> run_verification                     verify.hpp:63
//   ref_parse_config    -> parse_problem_config                 config.hpp:164
//   ref_accuracy_study  -> run_accuracy_study                   study.hpp:114
//   ref_performance_study -> run_performance_study              study.hpp:170
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

// verify.hpp uses format_double from study.hpp without including it
// (reference quirk); include study.hpp first like the CLI does.
#include "hexmg/study.hpp"
#include "hexmg/verify.hpp"
#include "hexmg/problem.hpp"
#include "hexmg/multigrid.hpp"
#include "hexmg/nonlinear.hpp"
#include "hexmg/vtk.hpp"

using namespace hexmg;

namespace {

thread_local std::string g_err;
int g_storage = 0;  // JacobianStorage for the next ref_create (ProblemConfig::storage)

struct RefProblem {
  ProblemConfig cfg;
  std::unique_ptr<FemProblem> problem;
  bool mg_ready = false;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InvertedElementError& e) {
    g_err = e.what();
    return 2;
  } catch (const StateNotInitializedError& e) {
    g_err = e.what();
    return 3;
  } catch (const IndefiniteOperatorError& e) {
    g_err = e.what();
    return 4;
  } catch (const NotSpdError& e) {
    g_err = e.what();
    return 5;
  } catch (const InvalidSmootherError& e) {
    g_err = e.what();
    return 6;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

MatrixFreeOperator& level_op(RefProblem* h, int level) {
  auto& hier = h->problem->hierarchy();
  if (level < 0) return h->problem->op();
  return *hier.levels.at((size_t)level).op;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// fixed_mask: bit f set => face f (Face enum order -x,+x,-y,+y,-z,+z) fixed.
// traction_face: -1 none, else Face index.
void* ref_create(const double* extents, const int* cells, int order, int qpts, int fixed_mask,
                 int traction_face, const double* traction, double young, double poisson,
                 int threads) {
  auto* h = new RefProblem();
  int rc = guarded([&] {
    ProblemConfig& cfg = h->cfg;
    cfg.extents = {extents[0], extents[1], extents[2]};
    cfg.cells = {cells[0], cells[1], cells[2]};
    cfg.order = order;
    cfg.quadrature_points = qpts;
    cfg.fixed_faces.clear();
    for (int f = 0; f < 6; ++f)
      if (fixed_mask & (1 << f)) cfg.fixed_faces.push_back(static_cast<Face>(f));
    static const char* names[] = {"-x", "+x", "-y", "+y", "-z", "+z"};
    cfg.traction_face = traction_face < 0 ? "none" : names[traction_face];
    cfg.traction = {traction[0], traction[1], traction[2]};
    cfg.youngs_modulus = young;
    cfg.poisson_ratio = poisson;
    cfg.threads = threads;
    cfg.storage = static_cast<JacobianStorage>(g_storage);
    h->problem = std::make_unique<FemProblem>(cfg);
  });
  if (rc != 0) {
    delete h;
    return nullptr;
  }
  return h;
}

void ref_set_storage(int s) { g_storage = s; }
int ref_state_stride(void* p) {
  return quadrature_state_stride(static_cast<RefProblem*>(p)->problem->op().storage());
}

void ref_destroy(void* p) { delete static_cast<RefProblem*>(p); }

int ref_size(void* p) { return static_cast<RefProblem*>(p)->problem->size(); }
int ref_num_elements(void* p) { return static_cast<RefProblem*>(p)->problem->op().num_elements(); }
int ref_points_per_element(void* p) {
  return static_cast<RefProblem*>(p)->problem->op().points_per_element();
}
int ref_num_levels(void* p) {
  return static_cast<RefProblem*>(p)->problem->hierarchy().num_levels();
}
int ref_level_size(void* p, int k) { return level_op(static_cast<RefProblem*>(p), k).size(); }
int ref_level_order(void* p, int k) {
  return static_cast<RefProblem*>(p)->problem->hierarchy().levels.at((size_t)k).order;
}
void ref_set_threads(void* p, int t) {
  auto* h = static_cast<RefProblem*>(p);
  h->problem->op().set_threads(t);
  for (auto& l : h->problem->hierarchy().levels) l.op->set_threads(t);
}
void ref_set_time(void* p, double t) { static_cast<RefProblem*>(p)->problem->set_time(t); }
void ref_set_jacobian_perturbation(void* p, double eps) {
  static_cast<RefProblem*>(p)->problem->op().set_jacobian_perturbation(eps);
}

// ---- setup data ----------------------------------------------------------
int ref_basis(int p, int q, double* nodes, double* points, double* weights, double* interp,
              double* deriv, double* pinv, double* colloc) {
  return guarded([&] {
    Basis1D b = build_lagrange_basis(p, q);
    std::memcpy(nodes, b.nodes.data(), sizeof(double) * b.nodes.size());
    std::memcpy(points, b.rule.points.data(), sizeof(double) * q);
    std::memcpy(weights, b.rule.weights.data(), sizeof(double) * q);
    std::memcpy(interp, b.interp.data(), sizeof(double) * b.interp.size());
    std::memcpy(deriv, b.deriv.data(), sizeof(double) * b.deriv.size());
    std::memcpy(pinv, b.pinv_interp.data(), sizeof(double) * b.pinv_interp.size());
    std::memcpy(colloc, b.colloc_deriv.data(), sizeof(double) * b.colloc_deriv.size());
  });
}

void ref_mesh_coords(void* p, double* out) {
  const auto& m = static_cast<RefProblem*>(p)->problem->mesh();
  std::memcpy(out, m.coords.data(), sizeof(double) * m.coords.size());
}

void ref_restriction(void* p, int level, int32_t* idx, int32_t* mult) {
  const auto& r = level_op(static_cast<RefProblem*>(p), level).restriction();
  std::memcpy(idx, r.indices.data(), sizeof(int32_t) * r.indices.size());
  std::memcpy(mult, r.multiplicity.data(), sizeof(int32_t) * r.multiplicity.size());
}

void ref_geometry(void* p, double* dxidX, double* weight) {
  const auto& g = static_cast<RefProblem*>(p)->problem->op().geometry();
  std::memcpy(dxidX, g.dxidX.data(), sizeof(double) * g.dxidX.size());
  std::memcpy(weight, g.weight.data(), sizeof(double) * g.weight.size());
}

void ref_constraints(void* p, int level, uint8_t* mask, double* values) {
  const auto& c = *level_op(static_cast<RefProblem*>(p), level).constraints();
  std::memcpy(mask, c.mask.data(), c.mask.size());
  if (values) std::memcpy(values, c.values.data(), sizeof(double) * c.values.size());
}

void ref_external_load(void* p, double* out) {
  const auto& l = static_cast<RefProblem*>(p)->problem->op().external_load();
  std::memcpy(out, l.data(), sizeof(double) * l.size());
}

void ref_impose_dirichlet(void* p, double* u) {
  auto* h = static_cast<RefProblem*>(p);
  h->problem->impose_dirichlet(std::span<double>(u, (size_t)h->problem->size()));
}

// ---- operator ------------------------------------------------------------
int ref_apply_residual(void* p, const double* u, double* f) {
  auto* h = static_cast<RefProblem*>(p);
  size_t n = (size_t)h->problem->size();
  return guarded([&] {
    h->problem->op().apply_residual(std::span<const double>(u, n), std::span<double>(f, n));
  });
}

int ref_apply_jacobian(void* p, int level, const double* du, double* y) {
  auto* h = static_cast<RefProblem*>(p);
  auto& op = level_op(h, level);
  size_t n = (size_t)op.size();
  return guarded(
      [&] { op.apply_jacobian(std::span<const double>(du, n), std::span<double>(y, n)); });
}

int ref_extract_diagonal(void* p, int level, double* d) {
  auto* h = static_cast<RefProblem*>(p);
  auto& op = level_op(h, level);
  return guarded([&] { op.extract_diagonal(std::span<double>(d, (size_t)op.size())); });
}

int ref_state(void* p, double* out) {
  auto* h = static_cast<RefProblem*>(p);
  const auto& st = *h->problem->op().state();
  std::memcpy(out, st.data.data(), sizeof(double) * st.data.size());
  return st.valid ? 0 : 3;
}

int ref_energy(void* p, const double* u, double* out) {
  auto* h = static_cast<RefProblem*>(p);
  size_t n = (size_t)h->problem->size();
  return guarded(
      [&] { *out = h->problem->op().total_strain_energy(std::span<const double>(u, n)); });
}

double ref_stored_bytes_per_dof(void* p) {
  return static_cast<RefProblem*>(p)->problem->op().stored_bytes_per_dof();
}

// ---- multigrid -----------------------------------------------------------
int ref_mg_setup(void* p) {
  auto* h = static_cast<RefProblem*>(p);
  return guarded([&] {
    h->problem->hierarchy().setup_numeric();
    h->mg_ready = true;
  });
}

double ref_level_lambda_max(void* p, int k) {
  return static_cast<RefProblem*>(p)->problem->hierarchy().levels.at((size_t)k).smoother.lambda_max;
}

void ref_level_inv_diag(void* p, int k, double* out) {
  const auto& s = static_cast<RefProblem*>(p)->problem->hierarchy().levels.at((size_t)k).smoother;
  std::memcpy(out, s.inv_diag.data(), sizeof(double) * s.inv_diag.size());
}

int ref_prolong(void* p, int coarse_level, const double* xc, double* xf) {
  auto* h = static_cast<RefProblem*>(p);
  auto& hier = h->problem->hierarchy();
  size_t nc = (size_t)hier.levels[(size_t)coarse_level].op->size();
  size_t nf = (size_t)hier.levels[(size_t)coarse_level + 1].op->size();
  return guarded([&] {
    hier.prolong(coarse_level, std::span<const double>(xc, nc), std::span<double>(xf, nf));
  });
}

int ref_restrict(void* p, int coarse_level, const double* xf, double* xc) {
  auto* h = static_cast<RefProblem*>(p);
  auto& hier = h->problem->hierarchy();
  size_t nc = (size_t)hier.levels[(size_t)coarse_level].op->size();
  size_t nf = (size_t)hier.levels[(size_t)coarse_level + 1].op->size();
  return guarded([&] {
    hier.restrict_to(coarse_level, std::span<const double>(xf, nf), std::span<double>(xc, nc));
  });
}

int ref_smoother_apply(void* p, int k, const double* b, double* x) {
  auto* h = static_cast<RefProblem*>(p);
  auto& hier = h->problem->hierarchy();
  size_t n = (size_t)hier.levels[(size_t)k].op->size();
  return guarded([&] {
    hier.levels[(size_t)k].smoother.apply(hier.level_operator(k), std::span<const double>(b, n),
                                          std::span<double>(x, n));
  });
}

int ref_vcycle(void* p, const double* b, double* x) {
  auto* h = static_cast<RefProblem*>(p);
  size_t n = (size_t)h->problem->size();
  return guarded([&] {
    h->problem->hierarchy().v_cycle(std::span<const double>(b, n), std::span<double>(x, n));
  });
}

int ref_coarse_nnz(void* p) {
  return (int)static_cast<RefProblem*>(p)->problem->hierarchy().coarse_matrix().nnz();
}

void ref_coarse_csr(void* p, int* rowptr, int* cols, double* vals) {
  const auto& a = static_cast<RefProblem*>(p)->problem->hierarchy().coarse_matrix();
  std::memcpy(rowptr, a.row_offsets.data(), sizeof(int) * a.row_offsets.size());
  std::memcpy(cols, a.cols.data(), sizeof(int) * a.cols.size());
  std::memcpy(vals, a.vals.data(), sizeof(double) * a.vals.size());
}

// ---- solvers -------------------------------------------------------------
// precond: 0 identity, 1 Jacobi (1/extract_diagonal of the fine operator),
// 2 p-multigrid V-cycle (requires ref_mg_setup).
int ref_cg(void* p, int precond, const double* b, double* x, double rtol, int maxit, int* its,
           int* converged, double* eig_min, double* eig_max, double* history, int hist_cap) {
  auto* h = static_cast<RefProblem*>(p);
  auto& op = h->problem->op();
  int n = op.size();
  return guarded([&] {
    LinearOperator a{n, [&op](std::span<const double> xx, std::span<double> yy) {
                       op.apply_jacobian(xx, yy);
                     }};
    LinearOperator m;
    if (precond == 0) {
      m = identity_operator(n);
    } else if (precond == 1) {
      std::vector<double> d((size_t)n);
      op.extract_diagonal(d);
      for (auto& v : d) v = 1.0 / v;
      m = diagonal_operator(std::move(d));
    } else {
      m = h->problem->hierarchy().preconditioner();
    }
    CgReport rep = cg_solve(a, m, std::span<const double>(b, (size_t)n),
                            std::span<double>(x, (size_t)n), rtol, maxit);
    *its = rep.iterations;
    *converged = rep.converged ? 1 : 0;
    *eig_min = rep.eig_min;
    *eig_max = rep.eig_max;
    for (int i = 0; i < hist_cap && i < (int)rep.history.size(); ++i) history[i] = rep.history[i];
  });
}

// Lanczos lambda_max of D^-1 A on the fine level from the reference rough seed.
int ref_lambda_max_jacobi(void* p, int level, int iterations, double* out) {
  auto* h = static_cast<RefProblem*>(p);
  auto& op = level_op(h, level);
  int n = op.size();
  return guarded([&] {
    std::vector<double> d((size_t)n);
    op.extract_diagonal(d);
    for (auto& v : d) v = 1.0 / v;
    LinearOperator a{n, [&op](std::span<const double> xx, std::span<double> yy) {
                       op.apply_jacobian(xx, yy);
                     }};
    auto seed = rough_seed(n, op.constraints()->mask);
    *out = estimate_lambda_max(a, diagonal_operator(std::move(d)), seed, iterations);
  });
}

void ref_rough_seed(int n, const uint8_t* mask, double* out) {
  auto v = rough_seed(n, mask ? std::span<const uint8_t>(mask, (size_t)n)
                              : std::span<const uint8_t>());
  std::memcpy(out, v.data(), sizeof(double) * v.size());
}

// Reference perf harness timing (study.hpp:198-212): 3 warm-ups then
// `repeats` Jacobian applies of x; returns wall seconds for the repeats.
double ref_time_jacobian(void* p, const double* x, int warmup, int repeats) {
  auto* h = static_cast<RefProblem*>(p);
  auto& op = h->problem->op();
  size_t n = (size_t)op.size();
  std::vector<double> y(n);
  for (int w = 0; w < warmup; ++w) op.apply_jacobian(std::span<const double>(x, n), y);
  auto t0 = std::chrono::steady_clock::now();
  for (int k = 0; k < repeats; ++k) op.apply_jacobian(std::span<const double>(x, n), y);
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Newton solve with load continuation through FemProblem::solve
// (problem.hpp:118-127).  Returns totals; u receives the solution.
int ref_newton(void* p, int load_steps, int line_search, double linear_rtol, double* u,
               int* newton_its, int* cg_its, double* final_fnorm) {
  auto* h = static_cast<RefProblem*>(p);
  return guarded([&] {
    ProblemConfig cfg = h->cfg;
    cfg.load_steps = load_steps;
    cfg.line_search = line_search != 0;
    cfg.linear_rtol = linear_rtol;
    h->problem = std::make_unique<FemProblem>(cfg);
    h->cfg = cfg;
    ContinuationReport rep = h->problem->solve();
    int ni = 0, ci = 0;
    double fn = 0.0;
    for (const auto& s : rep.steps) {
      ni += s.iterations;
      ci += s.total_cg_iterations;
      fn = s.final_fnorm;
    }
    *newton_its = ni;
    *cg_its = ci;
    *final_fnorm = fn;
    const auto& sol = h->problem->solution();
    std::memcpy(u, sol.data(), sizeof(double) * sol.size());
  });
}

// Same through the configured nonlinear solver (config.hpp:15, :60-64):
// solver 0 Newton-CG, 1 L-BFGS with `memory` pairs, preconditioner refresh.
int ref_solve(void* p, int load_steps, int line_search, double linear_rtol, int solver,
              int memory, int refresh, double* u, int* iterations, int* cg_its,
              double* final_fnorm) {
  auto* h = static_cast<RefProblem*>(p);
  return guarded([&] {
    ProblemConfig cfg = h->cfg;
    cfg.load_steps = load_steps;
    cfg.line_search = line_search != 0;
    cfg.linear_rtol = linear_rtol;
    cfg.solver = solver == 1 ? SolverKind::Lbfgs : SolverKind::NewtonCg;
    cfg.lbfgs_memory = memory;
    cfg.precond_refresh = refresh;
    h->problem = std::make_unique<FemProblem>(cfg);
    h->cfg = cfg;
    ContinuationReport rep = h->problem->solve();
    int ni = 0, ci = 0;
    double fn = 0.0;
    for (const auto& st : rep.steps) {
      ni += st.iterations;
      ci += st.total_cg_iterations;
      fn = st.final_fnorm;
    }
    *iterations = ni;
    *cg_its = ci;
    *final_fnorm = fn;
    const auto& sol = h->problem->solution();
    std::memcpy(u, sol.data(), sizeof(double) * sol.size());
  });
}

// The reference invariant suite; writes "name:pass:detail\n" lines.
int ref_verify(int threads, double perturbation, char* out, int cap) {
  std::string s;
  int rc = guarded([&] {
    VerifyOptions o;
    o.threads = threads;
    o.jacobian_perturbation = perturbation;
    for (const auto& r : run_verification(o))
      s += r.name + ":" + (r.passed ? "1" : "0") + ":" + r.detail + "\n";
  });
  std::snprintf(out, (size_t)cap, "%s", s.c_str());
  return rc;
}

// Config parser (config.hpp:164-262): canonical "key=value" dump of the
// parsed ProblemConfig, or the ConfigError message via ref_last_error.
int ref_parse_config(const char* text, char* out, int cap) {
  std::string s;
  int rc = guarded([&] {
    std::istringstream in(text);
    ProblemConfig c = parse_problem_config(in);
    auto d = [](double v) { return format_double(v); };
    s += "case_id=" + c.case_id + "\n";
    s += "extents=" + d(c.extents[0]) + " " + d(c.extents[1]) + " " + d(c.extents[2]) + "\n";
    s += "cells=" + std::to_string(c.cells[0]) + " " + std::to_string(c.cells[1]) + " " +
         std::to_string(c.cells[2]) + "\n";
    s += "order=" + std::to_string(c.order) + "\n";
    s += "geometry_order=" + std::to_string(c.geometry_order) + "\n";
    s += "quadrature_points=" + std::to_string(c.quadrature_points) + "\n";
    NeoHookean m = c.material();
    s += "material=" + d(m.mu) + " " + d(m.lambda) + "\n";
    s += "storage=" + std::to_string((int)c.storage) + "\n";
    s += "fixed_faces=";
    for (Face f : c.fixed_faces) s += std::to_string((int)f) + " ";
    s += "\ntraction_face=" + c.traction_face + "\n";
    s += "traction=" + d(c.traction[0]) + " " + d(c.traction[1]) + " " + d(c.traction[2]) + "\n";
    s += "body_force=" + d(c.body_force[0]) + " " + d(c.body_force[1]) + " " + d(c.body_force[2]) + "\n";
    s += "solver=" + std::to_string((int)c.solver) + "\n";
    s += "newton=" + std::to_string(c.load_steps) + " " + d(c.newton_rtol) + " " + d(c.newton_atol) +
         " " + std::to_string(c.newton_max_iterations) + " " + d(c.linear_rtol) + " " +
         std::to_string(c.linear_max_iterations) + " " + std::to_string((int)c.line_search) + " " +
         std::to_string(c.lbfgs_memory) + " " + std::to_string(c.precond_refresh) + "\n";
    s += "mg=" + std::to_string(c.mg_pre_smooth) + " " + std::to_string(c.mg_post_smooth) + "\n";
    s += "flags=" + std::to_string((int)c.deterministic) + " " + std::to_string((int)c.write_vtk) + "\n";
    s += "study_cases=";
    for (const auto& k : c.study_cases) s += k.id() + " ";
    s += "\nstudy_reference=" + c.study_reference.id() + "\n";
    s += "perf_orders=";
    for (int o : c.perf_orders) s += std::to_string(o) + " ";
    s += "\nperf_target_dofs=";
    for (long t : c.perf_target_dofs) s += std::to_string(t) + " ";
    s += "\nperf_representations=";
    for (const auto& r : c.perf_representations) s += r + " ";
    s += "\nperf_repeats=" + std::to_string(c.perf_repeats) + "\n";
  });
  std::snprintf(out, (size_t)cap, "%s", s.c_str());
  return rc;
}

// Legacy VTK of a displacement field on the problem's mesh (vtk.hpp:15-55).
int ref_write_vtk(void* p, const double* u, char* out, int cap) {
  std::ostringstream os;
  int rc = guarded([&] {
    auto* h = static_cast<RefProblem*>(p);
    const BoxMesh& m = h->problem->mesh();
    write_vtk(os, m, std::span<const double>(u, (size_t)m.num_dofs()));
  });
  std::snprintf(out, (size_t)cap, "%s", os.str().c_str());
  return rc;
}

// Study harness (study.hpp:114-233) on a config text; CSV into out.
int ref_accuracy_study(const char* text, char* out, int cap) {
  std::ostringstream csv;
  int rc = guarded([&] {
    std::istringstream in(text);
    run_accuracy_study(parse_problem_config(in), csv);
  });
  std::snprintf(out, (size_t)cap, "%s", csv.str().c_str());
  return rc;
}
int ref_performance_study(const char* text, char* out, int cap) {
  std::ostringstream csv;
  int rc = guarded([&] {
    std::istringstream in(text);
    run_performance_study(parse_problem_config(in), csv);
  });
  std::snprintf(out, (size_t)cap, "%s", csv.str().c_str());
  return rc;
}

}  // extern "C"
