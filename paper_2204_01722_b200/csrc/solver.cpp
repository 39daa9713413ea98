#include "solver.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <random>

namespace hxg {

namespace {

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
  if (rz < 0.0) throw Error(HXG_ERR_INDEFINITE, "operator is not positive definite (p^T A p = " +
                                                    std::to_string(rz) + ")");
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
      throw Error(HXG_ERR_INDEFINITE,
                  "operator is not positive definite (p^T A p = " + std::to_string(pap) + ")");
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
                                          fine->state(), fine->geometry());
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
  if (!assembly_) assembly_ = std::make_unique<CoarseAssembly>(*level(0).op);
  assembly_->numeric(*level(0).op);
}

void Hierarchy::prolong(int coarse_level, const double* xc, double* xf) {
  level(coarse_level + 1).from_coarser->prolong(xc, xf, stream());
}

void Hierarchy::restrict_to(int coarse_level, const double* xf, double* xc) {
  level(coarse_level + 1).from_coarser->restrict_to(xf, xc, stream());
}

void Hierarchy::coarse_solve(const double* b, double* x) { coarse_.solve(b, x, stream()); }

void Hierarchy::v_cycle(const double* b, double* x, bool x_zero) {
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
