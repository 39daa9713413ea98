/*
 * hexmg_b200.hpp — C++ drop-in for the reference's matrix-free p-multigrid
 * path (hexmg, /root/reference/proj/include/hexmg), over the C-ABI of
 * hexmg_b200.h.
 *
 * The classes keep the reference's names, constructor arguments and member
 * signatures, and take the reference's own value types (BoxMesh, Basis1D,
 * GeometricFactors, NeoHookean, JacobianStorage, Constraints,
 * QuadratureStateStore, DirichletBC), so a caller switches with
 *
 *     #include <hexmg_b200.hpp>
 *     using hexmg::b200::MatrixFreeOperator;      // was hexmg::MatrixFreeOperator
 *     using hexmg::b200::build_hierarchy;         // was hexmg::build_hierarchy
 *
 * Errors are rethrown as the reference's exception types (errors.hpp:9-79):
 * InvertedElementError(J, element, point), StateNotInitializedError,
 * IndefiniteOperatorError, InvalidSmootherError, NotSpdError,
 * StepRejectedError, std::invalid_argument.
 *
 * Spans may be host or device memory (checked per call): device spans run
 * in place on the operator's stream; host spans are copied (the reference's
 * host-vector calling convention, used by the parity tests).  The quadrature
 * state lives on the device; QuadratureStateStore objects passed in only
 * identify which operators share it (multigrid.hpp:229-249), their `data`
 * is not mirrored (export_state() copies it out in the reference layout).
 *
 * Needs the reference headers on the include path (the caller already has
 * them: they define the argument types) and links libhexmg_b200.so.
 */
#ifndef HEXMG_B200_HPP
#define HEXMG_B200_HPP

#include <hexmg/basis.hpp>
#include <hexmg/errors.hpp>
#include <hexmg/material.hpp>
#include <hexmg/mesh.hpp>
#include <hexmg/operator.hpp>  // Constraints, QuadratureStateStore, DirichletBC

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hexmg_b200.h"

namespace hexmg::b200 {

/// Rethrows the calling thread's last C-ABI error as the reference type.
[[noreturn]] inline void rethrow_last_error(int code) {
  hxg_error e{};
  hxg_last_error(&e);
  const std::string msg = e.message;
  auto strip = [&](const char* prefix) {  // the reference types add their own prefix
    const std::string p(prefix);
    return msg.compare(0, p.size(), p) == 0 ? msg.substr(p.size()) : msg;
  };
  switch (code) {
    case HXG_ERR_INVERTED_ELEMENT: throw InvertedElementError(e.jacobian, e.element, e.point);
    case HXG_ERR_STATE_NOT_INITIALIZED: throw StateNotInitializedError();
    case HXG_ERR_INDEFINITE: throw IndefiniteOperatorError(e.jacobian);
    case HXG_ERR_INVALID_SMOOTHER: throw InvalidSmootherError(strip("invalid smoother: "));
    case HXG_ERR_NOT_SPD: throw NotSpdError(strip("factorization failed, matrix not SPD: "));
    case HXG_ERR_STEP_REJECTED: throw StepRejectedError(strip("nonlinear step rejected: "));
    case HXG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw std::runtime_error("hexmg_b200: " + msg);
  }
}

inline void check(int rc) {
  if (rc != HXG_OK) rethrow_last_error(rc);
}

namespace detail {

/// Device scratch for host-span calls (grown on demand, freed with the owner).
struct DeviceBuffer {
  double* p = nullptr;
  size_t n = 0;
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (p) hxg_free(p);
  }
  double* get(size_t need) {
    if (need > n) {
      if (p) hxg_free(p);
      p = nullptr;
      check(hxg_malloc(reinterpret_cast<void**>(&p), need * sizeof(double)));
      n = need;
    }
    return p;
  }
};

inline bool on_device(const void* p) {
  int dev = 0;
  check(hxg_pointer_is_device(p, &dev));
  return dev != 0;
}

/// Input span -> device pointer (copied through `buf` when on the host).
inline const double* device_in(std::span<const double> x, DeviceBuffer& buf) {
  if (x.empty() || on_device(x.data())) return x.data();
  double* d = buf.get(x.size());
  check(hxg_memcpy_h2d(d, x.data(), x.size() * sizeof(double)));
  return d;
}

/// Device handle of a QuadratureStateStore: operators constructed on the
/// same store share one device state (the reference shares the store
/// between all levels of a hierarchy, multigrid.hpp:229-249).
inline hxg_state_t shared_state(const std::shared_ptr<QuadratureStateStore>& store) {
  struct Entry {
    std::weak_ptr<QuadratureStateStore> key;
    hxg_state_t state;
  };
  static std::mutex mu;
  static std::map<const QuadratureStateStore*, Entry> table;
  std::lock_guard<std::mutex> lock(mu);
  for (auto it = table.begin(); it != table.end();) {  // drop stores that died
    if (it->second.key.expired()) {
      hxg_state_release(it->second.state);
      it = table.erase(it);
    } else {
      ++it;
    }
  }
  auto it = table.find(store.get());
  if (it != table.end()) return it->second.state;
  hxg_state_t s = nullptr;
  check(hxg_state_create(&s));
  table[store.get()] = Entry{store, s};
  return s;
}

}  // namespace detail

/// MatrixFreeOperator (operator.hpp:70-373) on the B200: the constructor,
/// residual / Jacobian / diagonal / energy members and counters of the
/// reference, backed by the fused sm_100a kernels.
class MatrixFreeOperator {
 public:
  // operator.hpp:72-97
  MatrixFreeOperator(std::shared_ptr<const BoxMesh> mesh, Basis1D basis,
                     std::shared_ptr<const GeometricFactors> geometry, NeoHookean material,
                     JacobianStorage storage,
                     std::shared_ptr<const Constraints> constraints = nullptr,
                     std::shared_ptr<QuadratureStateStore> state = nullptr)
      : mesh_(std::move(mesh)),
        basis_(std::move(basis)),
        geometry_(std::move(geometry)),
        material_(material),
        storage_(storage),
        constraints_(std::move(constraints)),
        state_(std::move(state)) {
    if (geometry_->num_elements != mesh_->num_elements() ||
        geometry_->points_per_element != basis_.num_points_3d())
      throw std::invalid_argument("geometric factors do not match basis quadrature");
    if (constraints_ && !constraints_->mask.empty() &&
        constraints_->mask.size() != (size_t)mesh_->num_dofs())
      throw std::invalid_argument("constraint mask size mismatch");
    if (!state_) state_ = std::make_shared<QuadratureStateStore>();
    state_->stride = quadrature_state_stride(storage_);
    hxg_op_desc d{};
    d.order = basis_.order;
    d.qpts = basis_.num_points_1d();
    for (int k = 0; k < 3; ++k) d.cells[k] = mesh_->counts[k];
    d.interp = basis_.interp.data();
    d.deriv = basis_.deriv.data();
    d.colloc = basis_.colloc_deriv.data();
    d.dxidX = geometry_->dxidX.data();
    d.weight = geometry_->weight.data();
    d.mu = material_.mu;
    d.lambda = material_.lambda;
    d.storage = static_cast<int>(storage_);
    d.mask = constraints_ && !constraints_->mask.empty() ? constraints_->mask.data() : nullptr;
    check(hxg_op_create(&d, detail::shared_state(state_), &h_));
  }
  MatrixFreeOperator(const MatrixFreeOperator&) = delete;
  MatrixFreeOperator& operator=(const MatrixFreeOperator&) = delete;
  ~MatrixFreeOperator() {
    if (h_) hxg_op_destroy(h_);
  }

  int size() const { return mesh_->num_dofs(); }  // operator.hpp:99
  int num_elements() const { return mesh_->num_elements(); }
  int points_per_element() const { return basis_.num_points_3d(); }
  const BoxMesh& mesh() const { return *mesh_; }
  const Basis1D& basis() const { return basis_; }
  const GeometricFactors& geometry() const { return *geometry_; }
  const NeoHookean& material() const { return material_; }
  JacobianStorage storage() const { return storage_; }
  const std::shared_ptr<QuadratureStateStore>& state() const { return state_; }
  const std::shared_ptr<const Constraints>& constraints() const { return constraints_; }

  /// Host threads have no meaning on the device (kept for source compatibility).
  void set_threads(int n) { threads_ = n < 1 ? 1 : n; }
  int threads() const { return threads_; }

  // operator.hpp:112-122
  void set_external_load(std::vector<double> load) {
    if (!load.empty() && load.size() != (size_t)size())
      throw std::invalid_argument("external load size mismatch");
    external_load_ = std::move(load);
    check(hxg_op_set_external_load(h_, external_load_.empty() ? nullptr : external_load_.data()));
  }
  const std::vector<double>& external_load() const { return external_load_; }
  void set_load_scale(double s) {
    load_scale_ = s;
    check(hxg_op_set_load_scale(h_, s));
  }
  double load_scale() const { return load_scale_; }
  void set_jacobian_perturbation(double eps) { check(hxg_op_set_jacobian_perturbation(h_, eps)); }

  // operator.hpp:128-133
  size_t residual_apply_count() const { return counters().first - base_.first; }
  size_t jacobian_apply_count() const { return counters().second - base_.second; }
  void reset_counters() { base_ = counters(); }

  // operator.hpp:137-141
  double stored_bytes_per_dof() const {
    double v = 0.0;
    check(hxg_op_stored_bytes_per_dof(h_, &v));
    return v;
  }

  /// apply_residual (operator.hpp:146-180): writes the shared state.
  void apply_residual(std::span<const double> u, std::span<double> out) {
    check_sizes(u.size(), out.size());
    if (on_device(out)) {
      check(hxg_op_apply_residual(h_, detail::device_in(u, in_), out.data()));
    } else {
      double* y = out_.get(out.size());
      check(hxg_op_apply_residual(h_, detail::device_in(u, in_), y));
      check(hxg_memcpy_d2h(out.data(), y, out.size() * sizeof(double)));
    }
  }

  /// apply_jacobian (operator.hpp:184-215).
  void apply_jacobian(std::span<const double> du, std::span<double> out) const {
    check_sizes(du.size(), out.size());
    if (on_device(out)) {
      check(hxg_op_apply_jacobian(h_, detail::device_in(du, in_), out.data()));
    } else if (!du.empty() && !detail::on_device(du.data())) {
      // host -> host: the pipelined end-to-end path (copies overlap the apply)
      check(hxg_op_apply_jacobian_host(h_, du.data(), out.data()));
    } else {
      double* y = out_.get(out.size());
      check(hxg_op_apply_jacobian(h_, du.data(), y));
      check(hxg_memcpy_d2h(out.data(), y, out.size() * sizeof(double)));
    }
  }

  /// extract_diagonal (operator.hpp:247-283).
  void extract_diagonal(std::span<double> out) const {
    check_sizes(out.size(), out.size());
    if (on_device(out)) {
      check(hxg_op_extract_diagonal(h_, out.data()));
    } else {
      double* d = out_.get(out.size());
      check(hxg_op_extract_diagonal(h_, d));
      check(hxg_memcpy_d2h(out.data(), d, out.size() * sizeof(double)));
    }
  }

  /// total_strain_energy (operator.hpp:287-315).
  double total_strain_energy(std::span<const double> u) const {
    check_sizes(u.size(), u.size());
    double e = 0.0;
    check(hxg_op_total_strain_energy(h_, detail::device_in(u, in_), &e));
    return e;
  }

  /// The device state in the reference layout (e, q, stride) -> state()->data.
  void export_state() const {
    state_->data.resize((size_t)num_elements() * points_per_element() * state_->stride);
    check(hxg_op_export_state(h_, state_->data.data()));
    state_->valid = true;
  }

  hxg_op_t handle() const { return h_; }

 private:
  void check_sizes(size_t a, size_t b) const {
    if (a != (size_t)size() || b != (size_t)size())
      throw std::invalid_argument("operator apply size mismatch");
  }
  static bool on_device(std::span<double> s) { return !s.empty() && detail::on_device(s.data()); }
  std::pair<size_t, size_t> counters() const {
    int64_t r = 0, j = 0;
    check(hxg_op_counters(h_, &r, &j));
    return {(size_t)r, (size_t)j};
  }

  std::shared_ptr<const BoxMesh> mesh_;
  Basis1D basis_;
  std::shared_ptr<const GeometricFactors> geometry_;
  NeoHookean material_;
  JacobianStorage storage_;
  std::shared_ptr<const Constraints> constraints_;
  std::shared_ptr<QuadratureStateStore> state_;
  std::vector<double> external_load_;
  double load_scale_ = 1.0;
  int threads_ = 1;
  std::pair<size_t, size_t> base_{0, 0};
  hxg_op_t h_ = nullptr;
  mutable detail::DeviceBuffer in_, out_;
};

/// CgReport (cg.hpp:42-50).
struct CgReport {
  int iterations = 0;
  bool converged = false;
  std::vector<double> history;  // natural norm sqrt(r^T M r) per iteration
  double eig_min = 0.0;
  double eig_max = 0.0;
  double condition() const { return eig_min > 0.0 ? eig_max / eig_min : 1.0; }
};

/// MultigridHierarchy (multigrid.hpp:88-194): levels p -> ceil(p/2) -> .. -> 1
/// on the fine rule and shared state, Chebyshev(2)-Jacobi smoothing, exact
/// coarse Cholesky on the device.
class MultigridHierarchy {
 public:
  MultigridHierarchy() = default;
  MultigridHierarchy(MultigridHierarchy&& o) noexcept { *this = std::move(o); }
  MultigridHierarchy& operator=(MultigridHierarchy&& o) noexcept {
    std::swap(h_, o.h_);
    std::swap(fine_, o.fine_);
    pre_smooth = o.pre_smooth;
    post_smooth = o.post_smooth;
    return *this;
  }
  ~MultigridHierarchy() {
    if (h_) hxg_mg_destroy(h_);
  }

  int pre_smooth = 1;
  int post_smooth = 1;

  int num_levels() const {
    int n = 0;
    check(hxg_mg_num_levels(h_, &n));
    return n;
  }
  int level_size(int k) const {
    int64_t n = 0;
    check(hxg_mg_level_size(h_, k, &n));
    return (int)n;
  }
  const MatrixFreeOperator& finest() const { return *fine_; }

  /// setup_numeric (multigrid.hpp:100-113).
  void setup_numeric() { check(hxg_mg_setup_numeric(h_)); }

  /// prolong / restrict_to (multigrid.hpp:122-135).
  void prolong(int coarse_level, std::span<const double> xc, std::span<double> xf) const {
    transfer(coarse_level, xc, xf, true);
  }
  void restrict_to(int coarse_level, std::span<const double> xf, std::span<double> xc) const {
    transfer(coarse_level, xf, xc, false);
  }

  /// v_cycle (multigrid.hpp:137-144): x is the initial guess and the result.
  void v_cycle(std::span<const double> b, std::span<double> x) const {
    const size_t n = (size_t)fine_->size();
    if (b.size() != n || x.size() != n) throw std::invalid_argument("v_cycle size mismatch");
    if (!x.empty() && detail::on_device(x.data())) {
      check(hxg_mg_vcycle(h_, detail::device_in(b, in_), x.data()));
      return;
    }
    double* xd = out_.get(n);
    check(hxg_memcpy_h2d(xd, x.data(), n * sizeof(double)));
    check(hxg_mg_vcycle(h_, detail::device_in(b, in_), xd));
    check(hxg_memcpy_d2h(x.data(), xd, n * sizeof(double)));
  }

  hxg_mg_t handle() const { return h_; }

 private:
  friend MultigridHierarchy build_hierarchy(std::shared_ptr<MatrixFreeOperator>,
                                            const std::vector<DirichletBC>&, std::vector<int>,
                                            int, int);
  void transfer(int k, std::span<const double> in, std::span<double> out, bool up) const {
    const size_t nc = (size_t)level_size(k), nf = (size_t)level_size(k + 1);
    if (in.size() != (up ? nc : nf) || out.size() != (up ? nf : nc))
      throw std::invalid_argument("transfer size mismatch");
    const double* src = detail::device_in(in, in_);
    const bool dev = !out.empty() && detail::on_device(out.data());
    double* dst = dev ? out.data() : out_.get(out.size());
    check(up ? hxg_mg_prolong(h_, k, src, dst) : hxg_mg_restrict(h_, k, src, dst));
    if (!dev) check(hxg_memcpy_d2h(out.data(), dst, out.size() * sizeof(double)));
  }

  hxg_mg_t h_ = nullptr;
  std::shared_ptr<MatrixFreeOperator> fine_;
  mutable detail::DeviceBuffer in_, out_;
};

/// build_hierarchy (multigrid.hpp:212-268).  Coarse Dirichlet sets are
/// re-derived from the same faces; faces must constrain all components
/// with zero values (the BCs of every reference problem, problem.hpp:19-58).
inline MultigridHierarchy build_hierarchy(std::shared_ptr<MatrixFreeOperator> fine,
                                          const std::vector<DirichletBC>& bcs,
                                          std::vector<int> schedule = {}, int pre_smooth = 1,
                                          int post_smooth = 1) {
  const int p = fine->basis().order;
  if (!schedule.empty()) {
    if (schedule.front() != p) throw std::invalid_argument("schedule must start at the fine order");
    for (size_t i = 1; i < schedule.size(); ++i)
      if (schedule[i] >= schedule[i - 1])
        throw std::invalid_argument("schedule orders must strictly decrease");
    if (schedule.back() != 1) throw std::invalid_argument("schedule must end at order 1");
  }
  int faces = 0;
  for (const auto& bc : bcs) {
    if (!(bc.components[0] && bc.components[1] && bc.components[2]) || bc.value[0] != 0.0 ||
        bc.value[1] != 0.0 || bc.value[2] != 0.0)
      throw std::invalid_argument(
          "hexmg_b200 hierarchy: Dirichlet faces must constrain all components to zero");
    faces |= 1 << static_cast<int>(bc.face);
  }
  MultigridHierarchy h;
  h.pre_smooth = pre_smooth;
  h.post_smooth = post_smooth;
  h.fine_ = fine;
  check(hxg_mg_create(fine->handle(), faces, schedule.empty() ? nullptr : schedule.data(),
                      (int)schedule.size(), pre_smooth, post_smooth, &h.h_));
  return h;
}

/// cg_solve (cg.hpp:81-134) with A = op's Jacobian and the hierarchy's
/// V-cycle as preconditioner (mg may be null: identity).  b and x are host or
/// device; x is the initial guess and the result.
inline CgReport cg_solve(const MatrixFreeOperator& op, const MultigridHierarchy* mg,
                         std::span<const double> b, std::span<double> x, double rtol,
                         int max_iterations) {
  const size_t n = (size_t)op.size();
  if (b.size() != n || x.size() != n) throw std::invalid_argument("cg_solve size mismatch");
  detail::DeviceBuffer bb, xb;
  const double* bd = detail::device_in(b, bb);
  const bool xdev = !x.empty() && detail::on_device(x.data());
  double* xd = xdev ? x.data() : xb.get(n);
  if (!xdev) check(hxg_memcpy_h2d(xd, x.data(), n * sizeof(double)));
  hxg_cg_report r{};
  std::vector<double> hist((size_t)max_iterations + 1);
  check(hxg_cg_solve(op.handle(), mg ? mg->handle() : nullptr, mg ? 2 : 0, bd, xd, rtol,
                     max_iterations, &r, hist.data(), (int)hist.size()));
  if (!xdev) check(hxg_memcpy_d2h(x.data(), xd, n * sizeof(double)));
  CgReport rep;
  rep.iterations = r.iterations;
  rep.converged = r.converged != 0;
  rep.eig_min = r.eig_min;
  rep.eig_max = r.eig_max;
  hist.resize((size_t)(r.iterations + 1 < (int)hist.size() ? r.iterations + 1 : hist.size()));
  rep.history = std::move(hist);
  return rep;
}

}  // namespace hexmg::b200

#endif  // HEXMG_B200_HPP
