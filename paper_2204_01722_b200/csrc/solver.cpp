#include "solver.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <limits>
#include <random>
#include <string>

namespace hxg {

namespace {

// IndefiniteOperatorError (errors.hpp:55-60); the curvature travels in the
// error's value slot so the C++ drop-in can rethrow the reference type.
Error indefinite(double curvature) {
  Error e(HXG_ERR_INDEFINITE,
          "operator is not positive definite (p^T A p = " + std::to_string(curvature) + ")");
  e.jacobian = curvature;
  return e;
}

// Krylov work vectors and the dot workspace (pinned result slots), kept
// across calls: cudaMalloc / cudaMallocHost / cudaFree per solve would
// synchronise the device and cost more than a V-cycle.  One set per vector
// length; handles are not reentrant (like the reference's operators), so a
// process-wide pool is enough.
struct KrylovWork {
  DevBuf<double> v[5];
  DotWorkspace ws;
  explicit KrylovWork(size_t n) {
    for (auto& b : v) b.alloc(n);
  }
};
KrylovWork& krylov_work(size_t n) {
  static std::mutex mu;
  static std::vector<std::pair<size_t, KrylovWork*>>* pool =
      new std::vector<std::pair<size_t, KrylovWork*>>();  // leaked: outlives the CUDA context
  std::lock_guard<std::mutex> g(mu);
  for (auto& e : *pool)
    if (e.first == n) return *e.second;
  pool->emplace_back(n, new KrylovWork(n));
  return *pool->back().second;
}

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

int sturm_count(const std::vector<double>& d, const std::vector<double>& e, double x) {
  int count = 0;
  double q = 1.0;
  for (size_t i = 0; i < d.size(); ++i) {
    q = d[i] - x - (i ? (e[i - 1] * e[i - 1]) / q : 0.0);
    if (q == 0.0) q = -1e-300;
    if (q < 0.0) ++count;
  }
  return count;
}

// k-th smallest eigenvalue of the symmetric tridiagonal (d, e) by bisection.
double tridiag_eig(const std::vector<double>& d, const std::vector<double>& e, int k) {
  int n = (int)d.size();
  double lo = d[0], hi = d[0];
  for (int i = 0; i < n; ++i) {
    double r = (i > 0 ? std::abs(e[i - 1]) : 0.0) + (i + 1 < n ? std::abs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
  }
  double sc = std::max(std::abs(lo), std::abs(hi));
  lo -= 1e-14 * sc + 1e-300;
  hi += 1e-14 * sc + 1e-300;
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(d, e, mid) > k)
      hi = mid;
    else
      lo = mid;
  }
  return 0.5 * (lo + hi);
}

}  // namespace

void lanczos_eigs(const std::vector<double>& alphas, const std::vector<double>& betas,
                  double& eig_min, double& eig_max) {
  int k = (int)alphas.size();
  if (k == 0) {
    eig_min = eig_max = 0.0;
    return;
  }
  std::vector<double> d(k), e(std::max(k - 1, 0));
  d[0] = 1.0 / alphas[0];
  for (int i = 1; i < k; ++i) {
    d[i] = 1.0 / alphas[i] + betas[i - 1] / alphas[i - 1];
    e[i - 1] = std::sqrt(betas[i - 1]) / alphas[i - 1];
  }
  eig_min = tridiag_eig(d, e, 0);
  eig_max = tridiag_eig(d, e, k - 1);
}

std::vector<double> rough_seed(long long n, const std::vector<uint8_t>& mask) {
  std::mt19937 rng(0x9e3779b9u);
  std::vector<double> v((size_t)n);
  for (long long i = 0; i < n; ++i) v[(size_t)i] = 2.0 * (rng() * (1.0 / 4294967296.0)) - 1.0;
  if (!mask.empty())
    for (long long i = 0; i < n; ++i)
      if (mask[(size_t)i]) v[(size_t)i] = 0.0;
  return v;
}

CgResult cg_solve(long long n, const DevOp& a, const DevOp& m, const double* b, double* x,
                  double rtol, int max_iterations, cudaStream_t s) {
  KrylovWork& w = krylov_work((size_t)n);
  DevBuf<double>&r = w.v[0], &z = w.v[1], &p = w.v[2], &ap = w.v[3];
  DotWorkspace& ws = w.ws;
  a(x, r.p);
  vsub_from(r.p, b, n, s);
  m(r.p, z.p);
  double rz = dot(r.p, z.p, n, ws, s);
  if (rz < 0.0) throw indefinite(rz);
  CgResult rep;
  double nat0 = std::sqrt(rz);
  if (nat0 == 0.0) {
    rep.converged = true;
    return rep;
  }
  rep.history.push_back(nat0);
  vcopy(p.p, z.p, n, s);
  std::vector<double> alphas, betas;
  for (int it = 0; it < max_iterations; ++it) {
    a(p.p, ap.p);
    double pap = dot(p.p, ap.p, n, ws, s);
    if (pap <= 0.0)
      throw indefinite(pap);
    double alpha = rz / pap;
    alphas.push_back(alpha);
    cg_update_xr(x, r.p, p.p, ap.p, alpha, n, s);
    m(r.p, z.p);
    double rz_new = dot(r.p, z.p, n, ws, s);
    ++rep.iterations;
    double nat = std::sqrt(std::max(rz_new, 0.0));
    if (nat > 0.0) rep.history.push_back(nat);
    if (nat <= rtol * nat0) {
      rep.converged = true;
      break;
    }
    if (rz_new <= 0.0) {
      rep.converged = rz_new == 0.0;
      break;
    }
    double beta = rz_new / rz;
    betas.push_back(beta);
    cg_update_p(p.p, z.p, beta, n, s);
    rz = rz_new;
  }
  if (betas.size() >= alphas.size() && !alphas.empty()) betas.resize(alphas.size() - 1);
  lanczos_eigs(alphas, betas, rep.eig_min, rep.eig_max);
  return rep;
}

double estimate_lambda_max(long long n, const DevOp& a, const double* inv_diag,
                           const double* seed, int iterations, cudaStream_t s) {
  KrylovWork& w = krylov_work((size_t)n);
  DevBuf<double>&x = w.v[0], &r = w.v[1], &z = w.v[2], &p = w.v[3], &ap = w.v[4];
  DotWorkspace& ws = w.ws;
  vzero(x.p, n, s);
  vcopy(r.p, seed, n, s);
  vscale_mul(z.p, inv_diag, r.p, n, s);
  double rz = dot(r.p, z.p, n, ws, s);
  std::vector<double> alphas, betas;
  double eig_min = 0.0, eig_max = 1.0;
  if (rz <= 0.0) return eig_max;
  vcopy(p.p, z.p, n, s);
  for (int it = 0; it < iterations; ++it) {
    a(p.p, ap.p);
    double pap = dot(p.p, ap.p, n, ws, s);
    if (pap <= 0.0) break;
    double alpha = rz / pap;
    alphas.push_back(alpha);
    cg_update_xr(x.p, r.p, p.p, ap.p, alpha, n, s);
    vscale_mul(z.p, inv_diag, r.p, n, s);
    double rz_new = dot(r.p, z.p, n, ws, s);
    if (rz_new <= 0.0) break;
    if (it + 1 < iterations) betas.push_back(rz_new / rz);
    cg_update_p(p.p, z.p, rz_new / rz, n, s);
    rz = rz_new;
  }
  if (!alphas.empty()) {
    betas.resize(alphas.size() - 1);
    lanczos_eigs(alphas, betas, eig_min, eig_max);
  }
  return eig_max;
}

void Chebyshev::create(Operator& op, int degree_) {
  degree = degree_;
  long long n = op.size();
  cudaStream_t s = op.stream();
  if (inv_diag.n != (size_t)n) {  // first setup: buffers and the (constant) seed
    inv_diag.alloc((size_t)n);
    r.alloc((size_t)n);
    d.alloc((size_t)n);
    seed.upload(rough_seed(n, op.mask_host()));
  }
  op.extract_diagonal(d.p);  // d doubles as the diagonal scratch here
  if (!vreciprocal(inv_diag.p, d.p, n, s))
    throw Error(HXG_ERR_INVALID_SMOOTHER, "invalid smoother: zero diagonal entry");
  lambda_max = estimate_lambda_max(
      n, [&op](const double* x, double* y) { op.apply_jacobian(x, y); }, inv_diag.p, seed.p, 10, s);
  lo = 0.1 * lambda_max;
  hi = 1.1 * lambda_max;
  ready = true;
}

void Chebyshev::apply(Operator& op, const double* b, double* x, bool x_zero) {
  long long n = op.size();
  cudaStream_t s = op.stream();
  double theta = 0.5 * (hi + lo);
  double delta = 0.5 * (hi - lo);
  double sigma = theta / delta;
  double rho = 1.0 / sigma;
  if (x_zero) {
    cheb_first_zero(x, d.p, b, inv_diag.p, theta, n, s);
  } else {
    op.apply_jacobian(x, r.p);
    cheb_first(x, r.p, d.p, b, inv_diag.p, theta, n, s);
  }
  for (int k = 2; k <= degree; ++k) {
    op.apply_jacobian(x, r.p);
    double rho_new = 1.0 / (2.0 * sigma - rho);
    cheb_step(x, r.p, d.p, b, inv_diag.p, rho_new * rho, 2.0 * rho_new / delta, n, s);
    rho = rho_new;
  }
}

Hierarchy::Hierarchy(Operator* fine, int fixed_face_mask, std::vector<int> schedule,
                     int pre_smooth, int post_smooth)
    : pre_(pre_smooth), post_(post_smooth) {
  int p = fine->p();
  if (schedule.empty()) {
    schedule.push_back(p);
    while (schedule.back() > 1) schedule.push_back((schedule.back() + 1) / 2);
  }
  if (schedule.front() != p)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "schedule must start at the fine order");
  for (size_t i = 1; i < schedule.size(); ++i)
    if (schedule[i] >= schedule[i - 1])
      throw Error(HXG_ERR_INVALID_ARGUMENT, "schedule orders must strictly decrease");
  if (schedule.back() != 1) throw Error(HXG_ERR_INVALID_ARGUMENT, "schedule must end at order 1");
  Rule rule = gauss_legendre(fine->q());
  levels_.resize(schedule.size());
  for (size_t s = 0; s < schedule.size(); ++s) {
    size_t idx = schedule.size() - 1 - s;
    levels_[idx] = std::make_unique<Level>();
    Level& lv = *levels_[idx];
    lv.order = schedule[s];
    if (s == 0) {
      lv.op = fine;
      continue;
    }
    Basis b = build_basis(schedule[s], rule);
    std::vector<uint8_t> mask;
    face_mask(fine->cells(), schedule[s], fixed_face_mask, mask);
    lv.owned = std::make_unique<Operator>(schedule[s], fine->q(), fine->cells(), b.interp, b.deriv,
                                          b.colloc, fine->mu(), fine->lambda(), mask.data(),
                                          fine->state(), fine->geometry(), fine->storage());
    lv.owned->set_stream(fine->stream());
    lv.op = lv.owned.get();
  }
  for (size_t k = 1; k < levels_.size(); ++k)
    levels_[k]->from_coarser =
        std::make_unique<Transfer>(fine->cells(), levels_[k]->order, levels_[k - 1]->order);
  for (auto& lv : levels_) {
    size_t n = (size_t)lv->op->size();
    lv->residual.alloc(n);
    lv->correction.alloc(n);
    lv->restricted.alloc(n);
  }
}

void Hierarchy::setup_numeric() {
  follow_stream();
  PhaseTimer pt(stream());
  for (int k = 1; k < num_levels(); ++k) {
    level(k).smoother.create(*level(k).op, degree_);
    pt.mark("smoother (diag + lambda_max)");
  }
  if (!assembly_) assembly_ = std::make_unique<CoarseAssembly>(*level(0).op);
  assembly_->numeric(*level(0).op);
  pt.mark("coarse assembly");
  coarse_.set_mode(coarse_mode_);
  coarse_.factorize(assembly_->matrix(), level(0).op->box().npd, stream());
  pt.mark("coarse factorization");
}

void Hierarchy::assemble_coarse() {
  follow_stream();
  if (!assembly_) assembly_ = std::make_unique<CoarseAssembly>(*level(0).op);
  assembly_->numeric(*level(0).op);
}

void Hierarchy::prolong(int coarse_level, const double* xc, double* xf) {
  follow_stream();
  level(coarse_level + 1).from_coarser->prolong(xc, xf, stream());
}

void Hierarchy::restrict_to(int coarse_level, const double* xf, double* xc) {
  follow_stream();
  level(coarse_level + 1).from_coarser->restrict_to(xf, xc, stream());
}

void Hierarchy::coarse_solve(const double* b, double* x) {
  follow_stream();
  coarse_.solve(b, x, stream());
}

void Hierarchy::v_cycle(const double* b, double* x, bool x_zero) {
  follow_stream();
  cycle(num_levels() - 1, b, x, x_zero);
  Operator* op = levels_.back()->op;
  vmask_copy(x, b, op->mask(), op->size(), stream());
}

void Hierarchy::cycle(int k, const double* b, double* x, bool x_zero) {
  cudaStream_t s = stream();
  if (k == 0) {
    coarse_.solve(b, x, s);
    return;
  }
  Level& lv = level(k);
  Operator& op = *lv.op;
  long long n = op.size();
  for (int i = 0; i < pre_; ++i) {
    lv.smoother.apply(op, b, x, x_zero && i == 0);
  }
  bool still_zero = x_zero && pre_ == 0;
  double* r = lv.residual.p;
  if (still_zero) {
    vcopy(r, b, n, s);
  } else {
    op.apply_jacobian(x, r);
    vsub_from(r, b, n, s);
  }
  Level& cl = level(k - 1);
  double* rc = cl.restricted.p;
  restrict_to(k - 1, r, rc);
  vmask_zero(rc, cl.op->mask(), cl.op->size(), s);
  double* ec = cl.correction.p;
  vzero(ec, cl.op->size(), s);
  cycle(k - 1, rc, ec, true);
  prolong(k - 1, ec, r);
  vmask_zero(r, op.mask(), n, s);
  if (still_zero)
    vcopy(x, r, n, s);
  else
    vadd(x, r, n, s);
  for (int i = 0; i < post_; ++i) lv.smoother.apply(op, b, x, false);
}

}  // namespace hxg

namespace hxg {

namespace {

// critical_point_line_search (nonlinear.hpp:77-129): one secant step on
// g(a) = F(u + a du)^T du from g(0), g(1), clamped to [0.1, 2]; non-finite
// samples halve the trial point up to five times.
struct LineSearch {
  double alpha = 1.0;
};
LineSearch critical_point_line_search(const std::function<double(double)>& g_eval, double g0) {
  constexpr int kMaxHalvings = 5;
  double trial = 1.0;
  double g1 = g_eval(trial);
  int halvings = 0;
  while (!std::isfinite(g1) && halvings < kMaxHalvings) {
    trial *= 0.5;
    g1 = g_eval(trial);
    ++halvings;
  }
  if (!std::isfinite(g1))
    throw Error(HXG_ERR_STEP_REJECTED, "residual not evaluable along the search direction");
  double alpha;
  if (g0 >= 0.0) {
    alpha = trial;  // ascent warning
  } else if (g1 == g0) {
    alpha = trial;  // degenerate secant
  } else {
    alpha = trial * g0 / (g0 - g1);
    alpha = std::clamp(alpha, 0.1, 2.0);
    if (halvings > 0) alpha = std::min(alpha, trial);
  }
  LineSearch res;
  if (alpha == trial) {
    res.alpha = alpha;
    return res;
  }
  double ga = g_eval(alpha);
  while (!std::isfinite(ga) && halvings < kMaxHalvings) {
    alpha *= 0.5;
    ga = g_eval(alpha);
    ++halvings;
  }
  if (!std::isfinite(ga))
    throw Error(HXG_ERR_STEP_REJECTED, "residual not evaluable at the line search result");
  res.alpha = alpha;
  return res;
}

}  // namespace

SolveReport newton_solve(Operator& op, Hierarchy& mg, const NewtonConfig& cfg, double* u,
                         int load_step, double time) {
  const long long n = op.size();
  cudaStream_t s = op.stream();
  DevBuf<double> f((size_t)n), rhs((size_t)n), du((size_t)n), ut((size_t)n), ft((size_t)n);
  DotWorkspace ws;
  auto norm2 = [&](const double* v) { return std::sqrt(dot(v, v, n, ws, s)); };
  op.apply_residual(u, f.p);
  const double fnorm0 = norm2(f.p);
  SolveReport report;
  if (fnorm0 <= cfg.atol) {
    report.converged = true;
    report.final_fnorm = fnorm0;
    return report;
  }
  DevOp jac = [&op](const double* x, double* y) { op.apply_jacobian(x, y); };
  DevOp pre = [&mg, n, s](const double* r, double* z) {
    vzero(z, n, s);
    mg.v_cycle(r, z, true);
  };
  // g(a) = F(u + a du)^T du; F of the last evaluation stays in ft (and the
  // quadrature state at u + a du).  Inverted elements read as NaN.
  auto g_eval = [&](double a) {
    vwaxpy(ut.p, u, a, du.p, n, s);
    try {
      op.apply_residual(ut.p, ft.p);
    } catch (const Error& e) {
      if (e.code != HXG_ERR_INVERTED_ELEMENT) throw;
      return std::numeric_limits<double>::quiet_NaN();
    }
    const double g = dot(ft.p, du.p, n, ws, s);
    return std::isfinite(g) ? g : std::numeric_limits<double>::quiet_NaN();
  };
  double fnorm = fnorm0;
  for (int it = 1; it <= cfg.max_iterations; ++it) {
    mg.setup_numeric();
    vneg(rhs.p, f.p, n, s);
    vzero(du.p, n, s);
    CgResult cg = cg_solve(n, jac, pre, rhs.p, du.p, cfg.linear_rtol, cfg.linear_max_iterations, s);
    IterationRecord rec;
    rec.load_step = load_step;
    rec.time = time;
    rec.iteration = it;
    rec.cg_iterations = cg.iterations;
    rec.cg_converged = cg.converged;
    rec.condition_estimate = cg.eig_min > 0.0 ? cg.eig_max / cg.eig_min : 0.0;
    report.total_cg_iterations += cg.iterations;
    if (cfg.use_line_search) {
      rec.alpha = critical_point_line_search(g_eval, dot(f.p, du.p, n, ws, s)).alpha;
    } else {
      if (!std::isfinite(g_eval(1.0)))
        throw Error(HXG_ERR_STEP_REJECTED, "residual not evaluable at the full Newton step");
      rec.alpha = 1.0;
    }
    vwaxpy(u, u, rec.alpha, du.p, n, s);
    // The search's last evaluation was at the accepted point.
    if (cfg.use_line_search && cfg.reference_line_search_quirk)
      vzero(f.p, n, s);
    else
      vcopy(f.p, ft.p, n, s);
    fnorm = norm2(f.p);
    rec.fnorm = fnorm;
    rec.fnorm_rel = fnorm / fnorm0;
    report.records.push_back(rec);
    report.iterations = it;
    if (fnorm <= std::max(cfg.rtol * fnorm0, cfg.atol)) {
      report.converged = true;
      break;
    }
  }
  // Leave the quadrature state at the accepted iterate.
  op.apply_residual(u, f.p);
  report.final_fnorm = norm2(f.p);
  return report;
}

SolveReport lbfgs_solve(Operator& op, Hierarchy& mg, const NewtonConfig& cfg, double* u,
                        int load_step, double time) {
  const long long n = op.size();
  cudaStream_t s = op.stream();
  const int mem = std::max(cfg.lbfgs_memory, 0);
  DevBuf<double> f((size_t)n), q((size_t)n), d((size_t)n), ut((size_t)n), ft((size_t)n);
  DevBuf<double> ts((size_t)n), ty((size_t)n);
  std::vector<DevBuf<double>> S(mem), Y(mem);
  for (int i = 0; i < mem; ++i) {
    S[i].alloc((size_t)n);
    Y[i].alloc((size_t)n);
  }
  DotWorkspace ws;
  auto dotp = [&](const double* a, const double* b) { return dot(a, b, n, ws, s); };
  auto norm2 = [&](const double* v) { return std::sqrt(dotp(v, v)); };
  op.apply_residual(u, f.p);
  const double fnorm0 = norm2(f.p);
  SolveReport report;
  if (fnorm0 <= cfg.atol) {
    report.converged = true;
    report.final_fnorm = fnorm0;
    return report;
  }
  mg.setup_numeric();
  auto g_eval = [&](double a) {
    vwaxpy(ut.p, u, a, d.p, n, s);
    try {
      op.apply_residual(ut.p, ft.p);
    } catch (const Error& e) {
      if (e.code != HXG_ERR_INVERTED_ELEMENT) throw;
      return std::numeric_limits<double>::quiet_NaN();
    }
    const double g = dotp(ft.p, d.p);
    return std::isfinite(g) ? g : std::numeric_limits<double>::quiet_NaN();
  };
  // history ring: slot of pair i (oldest first) = (head + i) % mem
  int head = 0, h = 0;
  std::vector<double> rho(mem > 0 ? mem : 1), acoef(mem > 0 ? mem : 1);
  for (int it = 1; it <= cfg.max_iterations; ++it) {
    // two-loop recursion: d = -H f, H0 = the V-cycle
    vcopy(q.p, f.p, n, s);
    for (int i = h - 1; i >= 0; --i) {
      const int k = (head + i) % mem;
      acoef[(size_t)i] = rho[(size_t)k] * dotp(S[k].p, q.p);
      vwaxpy(q.p, q.p, -acoef[(size_t)i], Y[k].p, n, s);
    }
    vzero(d.p, n, s);
    mg.v_cycle(q.p, d.p, true);
    for (int i = 0; i < h; ++i) {
      const int k = (head + i) % mem;
      const double beta = rho[(size_t)k] * dotp(Y[k].p, d.p);
      vwaxpy(d.p, d.p, acoef[(size_t)i] - beta, S[k].p, n, s);
    }
    vneg(d.p, d.p, n, s);
    IterationRecord rec;
    rec.load_step = load_step;
    rec.time = time;
    rec.iteration = it;
    rec.alpha = critical_point_line_search(g_eval, dotp(f.p, d.p)).alpha;
    // s = alpha d, u += s, y = F_new - F (the quirk reads F_new as zero)
    const bool quirk = cfg.reference_line_search_quirk;
    vzero(ts.p, n, s);
    vwaxpy(ts.p, ts.p, rec.alpha, d.p, n, s);
    vwaxpy(u, u, 1.0, ts.p, n, s);
    if (quirk) {
      vneg(ty.p, f.p, n, s);
      vzero(f.p, n, s);
    } else {
      vwaxpy(ty.p, ft.p, -1.0, f.p, n, s);
      vcopy(f.p, ft.p, n, s);
    }
    const double sy = dotp(ts.p, ty.p);
    if (mem > 0 && sy > 0.0) {  // push back; drop the oldest beyond `memory`
      const int slot = h < mem ? (head + h) % mem : head;
      vcopy(S[slot].p, ts.p, n, s);
      vcopy(Y[slot].p, ty.p, n, s);
      rho[(size_t)slot] = 1.0 / sy;
      if (h < mem)
        ++h;
      else
        head = (head + 1) % mem;
    }
    const double fnorm = norm2(f.p);
    rec.fnorm = fnorm;
    rec.fnorm_rel = fnorm / fnorm0;
    report.records.push_back(rec);
    report.iterations = it;
    if (fnorm <= std::max(cfg.rtol * fnorm0, cfg.atol)) {
      report.converged = true;
      break;
    }
    if (cfg.precond_refresh > 0 && it % cfg.precond_refresh == 0) {
      op.apply_residual(u, f.p);  // pin the state to the current iterate
      mg.setup_numeric();
    }
  }
  op.apply_residual(u, f.p);
  report.final_fnorm = norm2(f.p);
  return report;
}

std::vector<SolveReport> solve_continuation(Operator& op, Hierarchy& mg, const NewtonConfig& cfg,
                                            double* u, int max_bisections,
                                            std::vector<double>* times) {
  if (cfg.load_steps < 1 || cfg.max_iterations < 1 || cfg.rtol <= 0 || cfg.atol <= 0 ||
      cfg.linear_rtol <= 0)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "solver tolerances must be positive and counts >= 1");
  const long long n = op.size();
  cudaStream_t s = op.stream();
  DevBuf<double> saved((size_t)n);
  vzero(u, n, s);  // FemProblem::solve starts from zero (problem.hpp:119)
  vcopy(saved.p, u, n, s);
  std::vector<SolveReport> steps;
  double t_done = 0.0;
  for (int step = 1; step <= cfg.load_steps; ++step) {
    const double target = (double)step / cfg.load_steps;
    int bisections = 0;
    double t_try = target;
    while (true) {
      op.set_load_scale(t_try);  // set_time (problem.hpp:70-73)
      vcopy(u, saved.p, n, s);
      // impose_dirichlet: whole-face zero values (u = t * 0 on the mask)
      vmask_zero(u, op.mask(), n, s);
      bool ok = false;
      try {
        SolveReport r = cfg.solver == 1 ? lbfgs_solve(op, mg, cfg, u, step, t_try)
                                        : newton_solve(op, mg, cfg, u, step, t_try);
        ok = r.converged;
        if (ok) {
          steps.push_back(std::move(r));
          if (times) times->push_back(t_try);
        }
      } catch (const Error& e) {
        if (e.code != HXG_ERR_STEP_REJECTED && e.code != HXG_ERR_INVERTED_ELEMENT) throw;
        ok = false;
      }
      if (ok) {
        t_done = t_try;
        vcopy(saved.p, u, n, s);
        if (t_try == target) break;
        t_try = target;
      } else {
        if (++bisections > max_bisections)
          throw Error(HXG_ERR_STEP_REJECTED,
                      "load step failed after " + std::to_string(max_bisections) + " bisections");
        t_try = 0.5 * (t_done + t_try);
      }
    }
  }
  return steps;
}

}  // namespace hxg
