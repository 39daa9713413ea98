// TEST INFRASTRUCTURE.  A reference-side caller switched to the B200 drop-in:
// the UNMODIFIED reference headers (/root/reference/proj/include, compiled in
// place by oracle/Makefile with the Eigen-API shim) build the problem --
// BoxMesh, Basis1D, GeometricFactors, Constraints, traction load -- exactly
// as FemProblem does (problem.hpp:19-58); hexmg::b200::MatrixFreeOperator is
// constructed from those same objects with the reference constructor
// signature (operator.hpp:72-97) and compared against
// hexmg::MatrixFreeOperator; then hexmg::b200::build_hierarchy + cg_solve
// against the reference's build_hierarchy + cg_solve (multigrid.hpp:212,
// cg.hpp:81); then the reference exception types through the drop-in.
//
// usage: test_dropin order n [threads]   -> one JSON line, exit 0 iff all pass
#include <hexmg/problem.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>

#include "hexmg_b200.hpp"

namespace {

double rel(const std::vector<double>& a, const std::vector<double>& b) {
  double d = 0.0, n = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    d += (a[i] - b[i]) * (a[i] - b[i]);
    n += b[i] * b[i];
  }
  return std::sqrt(d / (n > 0 ? n : 1e-300));
}

template <class T>
std::shared_ptr<const T> borrow(const T& x) {  // non-owning alias
  return std::shared_ptr<const T>(std::shared_ptr<const T>(), &x);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s order n [threads]\n", argv[0]);
    return 2;
  }
  const int p = std::atoi(argv[1]), n = std::atoi(argv[2]);
  const int threads = argc > 3 ? std::atoi(argv[3]) : (int)std::thread::hardware_concurrency();
  hexmg::ProblemConfig cfg;
  cfg.order = p;
  cfg.cells = {n, n, n};
  cfg.traction_face = "+x";
  cfg.traction = {0.0, 0.0, -0.02};
  cfg.threads = threads;
  hexmg::FemProblem ref(cfg);
  hexmg::MatrixFreeOperator& rop = ref.op();
  const int N = rop.size();

  // The drop-in, from the reference's own objects.
  auto op = std::make_shared<hexmg::b200::MatrixFreeOperator>(
      borrow(rop.mesh()), rop.basis(), borrow(rop.geometry()), rop.material(), rop.storage(),
      rop.constraints());
  op->set_external_load(rop.external_load());
  bool ok = op->size() == N;

  // Reference exception type before any residual (operator.hpp:187).
  bool state_err = false;
  {
    std::vector<double> x(N, 0.0), y(N);
    try {
      op->apply_jacobian(x, y);
    } catch (const hexmg::StateNotInitializedError&) {
      state_err = true;
    }
  }
  ok = ok && state_err;

  // Smooth tau != 0 state, constrained entries zero.
  const auto& X = rop.mesh().coords;
  const auto& mask = rop.constraints()->mask;
  std::vector<double> u(N);
  for (int i = 0; i < N / 3; ++i) {
    const double x = X[3 * i], y = X[3 * i + 1], z = X[3 * i + 2];
    const double s = std::sin(M_PI * x / 2) * std::sin(M_PI * y) * std::sin(M_PI * z);
    const double v[3] = {-0.05 * x + 0.02 * s, 0.03 * s, 0.01 * x * x};
    for (int c = 0; c < 3; ++c) u[3 * i + c] = mask[3 * i + c] ? 0.0 : 0.2 * v[c];
  }
  std::vector<double> f_ref(N), f(N), y_ref(N), y(N), d_ref(N), d(N), dx(N);
  for (int i = 0; i < N; ++i) dx[i] = 1e-3 * std::sin(0.7 * i);
  rop.apply_residual(u, f_ref);
  op->apply_residual(u, f);
  rop.apply_jacobian(dx, y_ref);
  op->apply_jacobian(dx, y);
  rop.extract_diagonal(d_ref);
  op->extract_diagonal(d);
  const double e_ref = rop.total_strain_energy(u), e = op->total_strain_energy(u);
  const double r_res = rel(f, f_ref), r_jac = rel(y, y_ref), r_diag = rel(d, d_ref);
  const double r_energy = std::abs(e - e_ref) / std::abs(e_ref);
  ok = ok && r_res < 1e-11 && r_jac < 1e-12 && r_diag < 1e-12 && r_energy < 1e-12;
  ok = ok && op->stored_bytes_per_dof() == rop.stored_bytes_per_dof();

  // p-MG PCG at u = 0, b = -F(0) (the SURVEY.md §8(c) goldens' setting).
  std::vector<double> zero(N, 0.0), b(N);
  rop.apply_residual(zero, b);
  for (double& v : b) v = -v;
  op->apply_residual(zero, f);
  ref.hierarchy().setup_numeric();
  std::vector<double> x_ref(N, 0.0), x(N, 0.0);
  const int fine = ref.hierarchy().num_levels() - 1;
  auto rep_ref = hexmg::cg_solve(ref.hierarchy().level_operator(fine),
                                 ref.hierarchy().preconditioner(), b, x_ref, 1e-8, 500);
  hexmg::b200::MultigridHierarchy mg = hexmg::b200::build_hierarchy(op, ref.dirichlet());
  mg.setup_numeric();
  auto rep = hexmg::b200::cg_solve(*op, &mg, b, x, 1e-8, 500);
  const int dits = rep.iterations - rep_ref.iterations;
  const double r_x = rel(x, x_ref);
  ok = ok && rep.converged && rep_ref.converged && std::abs(dits) <= 1 && r_x < 1e-7 &&
       mg.num_levels() == ref.hierarchy().num_levels();

  // InvertedElementError with the reference's (element, point) (material.hpp:132,
  // operator.hpp:166-168): a state that inverts elements.
  std::vector<double> ubad(N);
  for (int i = 0; i < N / 3; ++i) {
    const double x0 = X[3 * i];
    ubad[3 * i] = mask[3 * i] ? 0.0 : -1.5 * x0;  // compresses x by 2.5x -> J < 0
  }
  int re = -2, rq = -2, be = -1, bq = -1;
  try {
    rop.apply_residual(ubad, f_ref);
  } catch (const hexmg::InvertedElementError& ex) {
    re = ex.element();
    rq = ex.point();
  }
  try {
    op->apply_residual(ubad, f);
  } catch (const hexmg::InvertedElementError& ex) {
    be = ex.element();
    bq = ex.point();
  }
  ok = ok && re == be && rq == bq && re >= 0;

  std::printf(
      "{\"order\": %d, \"cells\": %d, \"dofs\": %d, \"state_not_initialized\": %s, "
      "\"residual_rel\": %.3e, \"jacobian_rel\": %.3e, \"diagonal_rel\": %.3e, "
      "\"energy_rel\": %.3e, \"pcg_iterations\": %d, \"pcg_iterations_ref\": %d, "
      "\"solution_rel\": %.3e, \"inverted_ref\": [%d, %d], \"inverted\": [%d, %d], "
      "\"levels\": %d, \"ok\": %s}\n",
      p, n, N, state_err ? "true" : "false", r_res, r_jac, r_diag, r_energy, rep.iterations,
      rep_ref.iterations, r_x, re, rq, be, bq, mg.num_levels(), ok ? "true" : "false");
  return ok ? 0 : 1;
}
