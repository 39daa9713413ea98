#include "solver.hpp"

#include "hcoarse.hpp"

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
  DevBuf<double> sc;  // device scalars of the Lanczos recurrence
  DotWorkspace ws;
  explicit KrylovWork(size_t n) {
    for (auto& b : v) b.alloc(n);
    sc.alloc(128);
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
                  double rtol, int max_iterations, cudaStream_t s, const DotFn* dotf) {
  KrylovWork& w = krylov_work((size_t)n);
  DevBuf<double>&r = w.v[0], &z = w.v[1], &p = w.v[2], &ap = w.v[3];
  DotWorkspace& ws = w.ws;
  auto dot = [&](const double* u, const double* v, long long nn, DotWorkspace& wsp,
                 cudaStream_t st) { return dotf ? (*dotf)(u, v) : ::hxg::dot(u, v, nn, wsp, st); };
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
                           const double* seed, int iterations, cudaStream_t s, const DotFn* dotf) {
  KrylovWork& w = krylov_work((size_t)n);
  DevBuf<double>&x = w.v[0], &r = w.v[1], &z = w.v[2], &p = w.v[3], &ap = w.v[4];
  DotWorkspace& ws = w.ws;
  auto dot = [&](const double* u, const double* v, long long nn, DotWorkspace& wsp,
                 cudaStream_t st) { return dotf ? (*dotf)(u, v) : ::hxg::dot(u, v, nn, wsp, st); };
  vzero(x.p, n, s);
  vcopy(r.p, seed, n, s);
  vscale_mul(z.p, inv_diag, r.p, n, s);
  std::vector<double> alphas, betas;
  double eig_min = 0.0, eig_max = 1.0;
  if (!dotf && 2 * iterations + 1 <= (int)w.sc.n) {
    // One process: the recurrence runs on device scalars (rz_k = sc[2k],
    // p^T A p = sc[2k + 1]) and the host reads them once at the end,
    // replaying the same breaks -- the same operations, no per-step syncs.
    double* sc = w.sc.p;
    dot_to(r.p, z.p, n, ws, sc, s);
    vcopy(p.p, z.p, n, s);
    for (int it = 0; it < iterations; ++it) {
      a(p.p, ap.p);
      dot_to(p.p, ap.p, n, ws, sc + 2 * it + 1, s);
      cg_update_xr_dev(x.p, r.p, p.p, ap.p, sc + 2 * it, sc + 2 * it + 1, n, s);
      vscale_mul(z.p, inv_diag, r.p, n, s);
      dot_to(r.p, z.p, n, ws, sc + 2 * it + 2, s);
      cg_update_p_dev(p.p, z.p, sc + 2 * it + 2, sc + 2 * it, n, s);
    }
    std::vector<double> h((size_t)(2 * iterations + 1));
    HXG_CUDA(cudaMemcpyAsync(h.data(), sc, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
    HXG_CUDA(cudaStreamSynchronize(s));
    double rz = h[0];
    if (rz <= 0.0) return eig_max;
    for (int it = 0; it < iterations; ++it) {
      const double pap = h[(size_t)(2 * it + 1)];
      if (pap <= 0.0) break;
      alphas.push_back(rz / pap);
      const double rz_new = h[(size_t)(2 * it + 2)];
      if (rz_new <= 0.0) break;
      if (it + 1 < iterations) betas.push_back(rz_new / rz);
      rz = rz_new;
    }
    if (!alphas.empty()) {
      betas.resize(alphas.size() - 1);
      lanczos_eigs(alphas, betas, eig_min, eig_max);
    }
    return eig_max;
  }
  double rz = dot(r.p, z.p, n, ws, s);
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

void Chebyshev::create(long long n, cudaStream_t s, int degree_, const DevOp& A,
                       const std::function<void(double*)>& diag, const DotFn* dotf,
                       const std::function<std::vector<double>()>& seed_fn) {
  degree = degree_;
  if (inv_diag.n != (size_t)n) {  // first setup: buffers and the (constant) seed
    inv_diag.alloc((size_t)n);
    r.alloc((size_t)n);
    d.alloc((size_t)n);
    seed.upload(seed_fn());
  }
  PhaseTimer pt(s);
  diag(d.p);  // d doubles as the diagonal scratch here
  if (!vreciprocal(inv_diag.p, d.p, n, s))
    throw Error(HXG_ERR_INVALID_SMOOTHER, "invalid smoother: zero diagonal entry");
  pt.mark("  smoother diagonal");
  lambda_max = estimate_lambda_max(n, A, inv_diag.p, seed.p, 10, s, dotf);
  pt.mark("  smoother lambda_max");
  lo = 0.1 * lambda_max;
  hi = 1.1 * lambda_max;
  ready = true;
}

void Chebyshev::apply(const DevOp& A, long long n, cudaStream_t s, const double* b, double* x,
                      bool x_zero) {
  double theta = 0.5 * (hi + lo);
  double delta = 0.5 * (hi - lo);
  double sigma = theta / delta;
  double rho = 1.0 / sigma;
  if (x_zero) {
    cheb_first_zero(x, d.p, b, inv_diag.p, theta, n, s);
  } else {
    A(x, r.p);
    cheb_first(x, r.p, d.p, b, inv_diag.p, theta, n, s);
  }
  for (int k = 2; k <= degree; ++k) {
    A(x, r.p);
    double rho_new = 1.0 / (2.0 * sigma - rho);
    cheb_step(x, r.p, d.p, b, inv_diag.p, rho_new * rho, 2.0 * rho_new / delta, n, s);
    rho = rho_new;
  }
}

// Partitioned coarse level: global p = 1 pattern (global mask), local ->
// global slot and DoF maps.
struct Hierarchy::DistCoarse {
  std::unique_ptr<CoarseAssembly> global;  // pattern + summed values
  int gnpd[3];
  DevBuf<long long> slot_map;   // local slot -> global slot (-1: not summed)
  DevBuf<long long> diag_slots;  // global constrained rows' diagonal slot
  DevBuf<long long> dof_map;    // local DoF -> global DoF
  DevBuf<double> gvec, gsol;
};

namespace {

__global__ void scatter_slots(const double* __restrict__ lv, const long long* __restrict__ map,
                              long long n, double* __restrict__ gv) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (map[i] >= 0) gv[map[i]] = lv[i];
}
__global__ void set_ones(double* __restrict__ v, const long long* __restrict__ idx, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[idx[i]] = 1.0;
}
__global__ void scatter_owned(const double* __restrict__ b, const uint8_t* __restrict__ owned,
                              const long long* __restrict__ map, long long n, double* __restrict__ g) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (owned[i]) g[map[i]] = b[i];
}
__global__ void gather_dofs(const double* __restrict__ g, const long long* __restrict__ map,
                            long long n, double* __restrict__ x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = g[map[i]];
}
inline int grid_n(long long n) {
  long long g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

Hierarchy::Hierarchy(Operator* fine, int fixed_face_mask, std::vector<int> schedule,
                     int pre_smooth, int post_smooth, Partition* part)
    : pre_(pre_smooth), post_(post_smooth), part_(part), global_faces_(fixed_face_mask) {
  int p = fine->p();
  if (part_) {
    for (int d = 0; d < 3; ++d)
      if (fine->cells()[d] != part_->cells()[d])
        throw Error(HXG_ERR_INVALID_ARGUMENT, "fine operator cells != this rank's block");
    fixed_face_mask = part_->local_faces(fixed_face_mask);
  }
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
    if (part_) lv->scaled.alloc(n);
  }
}

Hierarchy::~Hierarchy() {
  if (side_) cudaStreamDestroy(side_);
}

void Hierarchy::level_apply(int k, const double* x, double* y) {
  Level& lv = level(k);
  // constrained rows are the identity on every block holding them, not
  // summed (operator.hpp:212-214): the interface sum keeps x there (only
  // shared-plane entries were summed; one rank: nothing to exchange)
  static const bool overlap = [] {
    const char* e = std::getenv("HXG_OVERLAP");
    return !e || std::atoi(e) != 0;
  }();
  if (part_ && overlap && part_->comm().world() > 1 && lv.op->fused()) {
    // the interface layer first, its exchange on a side stream while the
    // interior bricks run
    if (!side_) HXG_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
    const int order = lv.order;
    const uint8_t* m = lv.op->mask();
    lv.op->apply_jacobian_split(x, y, part_->interface_faces(), side_,
                                [&]() { part_->exchange(order, y, side_, x, m); });
    return;
  }
  lv.op->apply_jacobian(x, y);
  if (part_) part_->exchange(lv.order, y, stream(), x, lv.op->mask());
}

double Hierarchy::level_dot(int k, const double* x, const double* y) {
  if (part_) return part_->dot(level(k).order, x, y, stream());
  return dot(x, y, level(k).op->size(), ws_, stream());
}

void Hierarchy::smooth(int k, const double* b, double* x) {
  follow_stream();
  Level& lv = level(k);
  if (!lv.smoother.ready) throw Error(HXG_ERR_GENERIC, "smoother not set up");
  lv.smoother.apply([this, k](const double* xx, double* yy) { level_apply(k, xx, yy); },
                    lv.op->size(), stream(), b, x, false);
}

void Hierarchy::residual(const double* u, double* f) {
  follow_stream();
  Operator& op = *levels_.back()->op;
  if (!part_) {
    op.apply_residual(u, f);
    return;
  }
  // every rank learns of an inverted element anywhere (max all-reduce of
  // the failure flag), then the residual's interface sums
  bool bad = false;
  Error saved(HXG_ERR_INVERTED_ELEMENT, "");
  try {
    op.apply_residual(u, f);
  } catch (const Error& e) {
    if (e.code != HXG_ERR_INVERTED_ELEMENT) throw;
    bad = true;
    saved = e;
  }
  if (part_->allreduce_max(bad ? 1.0 : 0.0, stream()) > 0.0) {
    if (bad) throw saved;
    throw Error(HXG_ERR_INVERTED_ELEMENT, "non-positive deformation jacobian on another rank");
  }
  part_->exchange(levels_.back()->order, f, stream());
}

void Hierarchy::setup_numeric() {
  follow_stream();
  PhaseTimer pt(stream());
  cudaStream_t s = stream();
  for (int k = 1; k < num_levels(); ++k) {
    Level& lv = level(k);
    Operator* op = lv.op;
    const int order = lv.order;
    DotFn dotf = [this, k](const double* x, const double* y) { return level_dot(k, x, y); };
    lv.smoother.create(
        op->size(), s, degree_, [this, k](const double* x, double* y) { level_apply(k, x, y); },
        [this, op, order, s](double* d) {
          op->extract_diagonal(d);
          if (part_) {  // summed over the blocks; constrained entries stay 1
            part_->exchange(order, d, s);
            vmask_fill(d, 1.0, op->mask(), op->size(), s);
          }
        },
        part_ ? &dotf : nullptr,
        [this, op, order]() {
          return part_ ? part_->global_seed_slice(order, op->mask_host())
                       : rough_seed(op->size(), op->mask_host());
        });
    pt.mark("smoother (diag + lambda_max)");
  }
  if (!assembly_) assembly_ = std::make_unique<CoarseAssembly>(*level(0).op);
  assembly_->numeric(*level(0).op);
  pt.mark("coarse assembly");
  if (coarse_mode_ == 4) {  // inexact: h-multigrid (distributed with the hierarchy)
    if (!hmg_) hmg_ = std::make_unique<HmgCoarse>();
    hmg_->setup(assembly_->matrix(), level(0).op->box(), level(0).op->mask_host(),
                assembly_->element_matrices(), s, part_);
  } else if (part_) {
    dist_coarse_numeric();
  } else {
    coarse_.set_mode(coarse_mode_);
    coarse_.factorize(assembly_->matrix(), level(0).op->box().npd, s);
  }
  pt.mark("coarse factorization");
}

void Hierarchy::dist_coarse_numeric() {
  cudaStream_t s = stream();
  const CsrMatrix& la = assembly_->matrix();
  if (!dc_) {  // symbolic: global pattern and the maps, once
    dc_ = std::make_unique<DistCoarse>();
    int gc[3];
    for (int d = 0; d < 3; ++d) gc[d] = part_->gcells()[d];
    BoxDev gbox = make_box(gc, 1);
    std::vector<uint8_t> gmask;
    face_mask(gc, 1, global_faces_, gmask);
    dc_->global = std::make_unique<CoarseAssembly>(gbox, gmask);
    for (int d = 0; d < 3; ++d) dc_->gnpd[d] = gbox.npd[d];
    const CsrMatrix& ga = dc_->global->matrix();
    int ln[3];
    part_->npd(1, ln);
    const int* e0 = part_->e0();
    auto to_global = [&](long long dof) {
      const long long node = dof / 3;
      const int c = (int)(dof % 3);
      const long long ix = node % ln[0], iy = (node / ln[0]) % ln[1], iz = node / ((long long)ln[0] * ln[1]);
      return 3 * ((ix + e0[0]) + (long long)gbox.npd[0] * ((iy + e0[1]) + (long long)gbox.npd[1] * (iz + e0[2]))) + c;
    };
    std::vector<long long> smap(la.cols_h.size(), -1), dmap((size_t)la.n);
    for (int r = 0; r < la.n; ++r) {
      const long long gr = to_global(r);
      dmap[(size_t)r] = gr;
      if (gmask[(size_t)gr]) continue;  // constrained rows: identity re-imposed globally
      const int* gb = ga.cols_h.data() + ga.row_ptr_h[(size_t)gr];
      const int* ge = ga.cols_h.data() + ga.row_ptr_h[(size_t)gr + 1];
      for (int sl = la.row_ptr_h[(size_t)r]; sl < la.row_ptr_h[(size_t)r + 1]; ++sl) {
        const long long gcol = to_global(la.cols_h[(size_t)sl]);
        if (gmask[(size_t)gcol]) continue;
        const int* it = std::lower_bound(gb, ge, (int)gcol);
        if (it == ge || *it != (int)gcol)
          throw Error(HXG_ERR_GENERIC, "partitioned coarse pattern: slot outside the global pattern");
        smap[(size_t)sl] = ga.row_ptr_h[(size_t)gr] + (it - gb);
      }
    }
    std::vector<long long> diag;
    for (int r = 0; r < ga.n; ++r)
      if (gmask[(size_t)r]) diag.push_back(ga.row_ptr_h[(size_t)r]);  // the row's only slot
    dc_->slot_map.upload(smap);
    dc_->dof_map.upload(dmap);
    if (!diag.empty()) dc_->diag_slots.upload(diag);
    dc_->gvec.alloc((size_t)ga.n);
    dc_->gsol.alloc((size_t)ga.n);
  }
  CsrMatrix& ga = dc_->global->mutable_matrix();
  const long long gnnz = ga.nnz(), lnnz = la.nnz();
  HXG_CUDA(cudaMemsetAsync(ga.vals.p, 0, sizeof(double) * gnnz, s));
  scatter_slots<<<grid_n(lnnz), 256, 0, s>>>(la.vals.p, dc_->slot_map.p, lnnz, ga.vals.p);
  HXG_CUDA(cudaGetLastError());
  part_->comm().allreduce(ga.vals.p, gnnz, 0, s);
  if (dc_->diag_slots.n)
    set_ones<<<grid_n((long long)dc_->diag_slots.n), 256, 0, s>>>(ga.vals.p, dc_->diag_slots.p,
                                                                 (long long)dc_->diag_slots.n);
  HXG_CUDA(cudaGetLastError());
  coarse_.set_mode(coarse_mode_);
  coarse_.factorize(ga, dc_->gnpd, s);
}

void Hierarchy::dist_coarse_solve(const double* b, double* x) {
  cudaStream_t s = stream();
  const long long n = level(0).op->size(), gn = (long long)dc_->gvec.n;
  HXG_CUDA(cudaMemsetAsync(dc_->gvec.p, 0, sizeof(double) * gn, s));
  scatter_owned<<<grid_n(n), 256, 0, s>>>(b, part_->owned(1), dc_->dof_map.p, n, dc_->gvec.p);
  HXG_CUDA(cudaGetLastError());
  part_->comm().allreduce(dc_->gvec.p, gn, 0, s);
  coarse_.solve(dc_->gvec.p, dc_->gsol.p, s);
  gather_dofs<<<grid_n(n), 256, 0, s>>>(dc_->gsol.p, dc_->dof_map.p, n, x);
  HXG_CUDA(cudaGetLastError());
}

void Hierarchy::assemble_coarse() {
  follow_stream();
  if (!assembly_) assembly_ = std::make_unique<CoarseAssembly>(*level(0).op);
  assembly_->numeric(*level(0).op);
}

// Partitioned transfers: a shared fine node gets the same prolongated value
// from every block (its elements agree there), so the interface sum counts
// it once per sharing block: x 1/2 per shared direction.  The restriction is
// the exact transpose: x 1/2 on the shared fine planes, local, interface sum.
void Hierarchy::prolong(int coarse_level, const double* xc, double* xf) {
  follow_stream();
  level(coarse_level + 1).from_coarser->prolong(xc, xf, stream());
  if (part_) {
    const int pf = level(coarse_level + 1).order;
    part_->exchange(pf, xf, stream());
    part_->scale_interfaces(pf, xf, 0.5, stream());
  }
}

void Hierarchy::restrict_to(int coarse_level, const double* xf, double* xc) {
  follow_stream();
  Level& fl = level(coarse_level + 1);
  if (!part_) {
    fl.from_coarser->restrict_to(xf, xc, stream());
    return;
  }
  vcopy(fl.scaled.p, xf, fl.op->size(), stream());
  part_->scale_interfaces(fl.order, fl.scaled.p, 0.5, stream());
  fl.from_coarser->restrict_to(fl.scaled.p, xc, stream());
  part_->exchange(level(coarse_level).order, xc, stream());
}

void Hierarchy::coarse_solve(const double* b, double* x) {
  follow_stream();
  if (coarse_mode_ == 4 && hmg_ && hmg_->ready())
    hmg_->solve(b, x, stream());
  else if (part_)
    dist_coarse_solve(b, x);
  else
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
    coarse_solve(b, x);
    return;
  }
  Level& lv = level(k);
  Operator& op = *lv.op;
  long long n = op.size();
  DevOp A = [this, k](const double* xx, double* yy) { level_apply(k, xx, yy); };
  for (int i = 0; i < pre_; ++i) {
    lv.smoother.apply(A, n, s, b, x, x_zero && i == 0);
  }
  bool still_zero = x_zero && pre_ == 0;
  double* r = lv.residual.p;
  if (still_zero) {
    vcopy(r, b, n, s);
  } else {
    level_apply(k, x, r);
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
  for (int i = 0; i < post_; ++i) lv.smoother.apply(A, n, s, b, x, false);
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

System make_system(Operator& op, Hierarchy& mg) {
  System sys;
  sys.n = op.size();
  sys.s = op.stream();
  const int fine = mg.num_levels() - 1;
  Hierarchy* h = &mg;
  const long long n = sys.n;
  cudaStream_t s = sys.s;
  sys.residual = [h](const double* u, double* f) { h->residual(u, f); };
  sys.jacobian = [h, fine](const double* x, double* y) { h->level_apply(fine, x, y); };
  sys.dot = [h, fine](const double* x, const double* y) { return h->level_dot(fine, x, y); };
  sys.prepare = [h] { h->setup_numeric(); };
  sys.precond = [h, n, s](const double* r, double* z) {
    vzero(z, n, s);
    h->v_cycle(r, z, true);
  };
  return sys;
}

namespace {

SolveReport newton_solve_sys(const System& sys, const NewtonConfig& cfg, double* u, int load_step,
                             double time) {
  const long long n = sys.n;
  cudaStream_t s = sys.s;
  DevBuf<double> f((size_t)n), rhs((size_t)n), du((size_t)n), ut((size_t)n), ft((size_t)n);
  auto dot = [&sys](const double* x, const double* y, long long, DotWorkspace&, cudaStream_t) {
    return sys.dot(x, y);
  };
  DotWorkspace ws;
  auto norm2 = [&](const double* v) { return std::sqrt(dot(v, v, n, ws, s)); };
  sys.residual(u, f.p);
  const double fnorm0 = norm2(f.p);
  SolveReport report;
  if (fnorm0 <= cfg.atol) {
    report.converged = true;
    report.final_fnorm = fnorm0;
    return report;
  }
  const DevOp& jac = sys.jacobian;
  const DevOp& pre = sys.precond;
  // g(a) = F(u + a du)^T du; F of the last evaluation stays in ft (and the
  // quadrature state at u + a du).  Inverted elements read as NaN.
  auto g_eval = [&](double a) {
    vwaxpy(ut.p, u, a, du.p, n, s);
    try {
      sys.residual(ut.p, ft.p);
    } catch (const Error& e) {
      if (e.code != HXG_ERR_INVERTED_ELEMENT) throw;
      return std::numeric_limits<double>::quiet_NaN();
    }
    const double g = dot(ft.p, du.p, n, ws, s);
    return std::isfinite(g) ? g : std::numeric_limits<double>::quiet_NaN();
  };
  double fnorm = fnorm0;
  for (int it = 1; it <= cfg.max_iterations; ++it) {
    sys.prepare();
    vneg(rhs.p, f.p, n, s);
    vzero(du.p, n, s);
    CgResult cg =
        cg_solve(n, jac, pre, rhs.p, du.p, cfg.linear_rtol, cfg.linear_max_iterations, s, &sys.dot);
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
  sys.residual(u, f.p);
  report.final_fnorm = norm2(f.p);
  return report;
}

}  // namespace

SolveReport newton_solve(Operator& op, Hierarchy& mg, const NewtonConfig& cfg, double* u,
                         int load_step, double time) {
  return newton_solve_sys(make_system(op, mg), cfg, u, load_step, time);
}

SolveReport lbfgs_solve(Operator& op, Hierarchy& mg, const NewtonConfig& cfg, double* u,
                        int load_step, double time) {
  if (mg.partition())
    throw Error(HXG_ERR_UNSUPPORTED, "L-BFGS runs on one process (Newton-CG is partitioned)");
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
