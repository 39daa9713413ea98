// MatrixFreeOperator on device (operator.hpp:70-373).
#include "operator.hpp"

#include <cmath>

#include <algorithm>
#include <cstring>
#include <string>

#include "apply_kernels.cuh"
#include "diag_kernels.cuh"
#include "dispatch.hpp"
#include "fused_apply.cuh"
#include "node_kernels.cuh"

namespace hxg {

namespace {

// Permutes reference-layout per-point data (e, q, S) into the blocked layout.
void to_blocked(const QLayout& lay, long long E, int nq, int S, const double* src,
                std::vector<double>& dst, const double* src_w = nullptr) {
  dst.assign((size_t)lay.total_points() * S, 0.0);
  for (long long e = 0; e < E; ++e)
    for (int qp = 0; qp < nq; ++qp) {
      long long brick;
      int qz, t;
      lay.locate(e, qp, brick, qz, t);
      size_t base = (size_t)(((brick * lay.Q + qz) * S) * lay.T + t);
      int sv = src_w ? S - 1 : S;
      for (int s = 0; s < sv; ++s)
        dst[base + (size_t)s * lay.T] = src[((size_t)e * nq + qp) * sv + s];
      if (src_w) dst[base + (size_t)(S - 1) * lay.T] = src_w[(size_t)e * nq + qp];
    }
}

}  // namespace

std::shared_ptr<Geometry> Operator::make_geometry(const int cells[3], int q, const double* dxidX,
                                                  const double* weight) {
  auto g = std::make_shared<Geometry>();
  g->lay = QLayout::make(cells, q);
  long long E = (long long)cells[0] * cells[1] * cells[2];
  std::vector<double> blocked;
  to_blocked(g->lay, E, q * q * q, kGeoStride, dxidX, blocked, weight);
  g->data.upload(blocked);
  return g;
}

namespace {
// Box geometry in the blocked layout ((brick, qz, s, t), 10 scalars): every
// element of build_box_mesh is the same affine map, so dxi/dX = diag(2/h)
// and w detJ = w_qx w_qy w_qz h_x h_y h_z / 8 at every point.
__global__ void box_geometry_kernel(QLayout lay, double gx, double gy, double gz, double jac,
                                    const double* __restrict__ qw, double* __restrict__ geo) {
  const long long total = lay.total_points();
  const int Q = lay.Q, NE = lay.B[0] * lay.B[1] * lay.B[2];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / lay.T;  // brick * Q + qz
    const int t = (int)(i - row * lay.T), qz = (int)(row % Q);
    const int col = t / NE, qx = col % Q, qy = col / Q;
    double* g = geo + row * kGeoStride * lay.T + t;
    for (int s = 0; s < 9; ++s) g[(long long)s * lay.T] = 0.0;
    g[0] = gx;
    g[4LL * lay.T] = gy;
    g[8LL * lay.T] = gz;
    g[9LL * lay.T] = qw[qx] * qw[qy] * qw[qz] * jac;
  }
}
}  // namespace

std::shared_ptr<Geometry> Operator::make_box_geometry(const int cells[3], int q,
                                                      const double extents[3],
                                                      const double* qweights) {
  auto g = std::make_shared<Geometry>();
  g->lay = QLayout::make(cells, q);
  g->data.alloc((size_t)g->lay.total_points() * kGeoStride);
  DevBuf<double> qw;
  qw.upload(qweights, (size_t)q);
  double h[3];
  for (int d = 0; d < 3; ++d) {
    if (!(extents[d] > 0.0)) throw Error(HXG_ERR_INVALID_ARGUMENT, "box extents must be positive");
    h[d] = extents[d] / cells[d];
  }
  g->box = true;
  for (int d = 0; d < 3; ++d) g->g[d] = 2.0 / h[d];
  g->jac = 0.125 * h[0] * h[1] * h[2];
  for (int i = 0; i < q && i < kMaxQ; ++i) g->qw[i] = qweights[i];
  box_geometry_kernel<<<grid_for(g->lay.total_points(), 256), 256>>>(
      g->lay, g->g[0], g->g[1], g->g[2], g->jac, qw.p, g->data.p);
  HXG_CUDA(cudaGetLastError());
  HXG_CUDA(cudaDeviceSynchronize());  // qw is released on return
  return g;
}

Operator::Operator(int p, int q, const int cells[3], const std::vector<double>& interp,
                   const std::vector<double>& deriv, const std::vector<double>& colloc, double mu,
                   double lambda, const uint8_t* mask_host, std::shared_ptr<State> state,
                   std::shared_ptr<Geometry> geometry, int storage)
    : p_(p), q_(q), mu_(mu), lambda_(lambda), storage_(storage), interp_(interp), deriv_(deriv),
      colloc_(colloc), state_(std::move(state)), geometry_(std::move(geometry)) {
  if (storage < kStorageCurrent || storage > kStorageInitialAD)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "unknown JacobianStorage " + std::to_string(storage));
  dispatch_pq(p, q, [](auto, auto) {});  // validates the pair
  for (int d = 0; d < 3; ++d) {
    if (cells[d] < 1) throw Error(HXG_ERR_INVALID_ARGUMENT, "element counts must be >= 1");
    cells_[d] = cells[d];
  }
  int n = p + 1;
  if ((int)interp.size() != q * n || (int)deriv.size() != q * n || (int)colloc.size() != q * q)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "basis tabulation sizes do not match (p, q)");
  box_ = make_box(cells, p);
  lay_ = QLayout::make(cells, q);
  std::vector<double> tab(interp);
  tab.insert(tab.end(), colloc.begin(), colloc.end());
  tab_.upload(tab);
  interp_d_.upload(interp);
  deriv_d_.upload(deriv);
  if (mask_host) {
    mask_host_.assign(mask_host, mask_host + size());
    mask_.upload(mask_host_);
    // Whole-face detection: faces whose every DoF is constrained; the mask
    // is analytic when it equals the union of those faces.
    int bits = 0;
    for (int f = 0; f < 6; ++f) {
      std::vector<uint8_t> fm;
      face_mask(cells, p, 1 << f, fm);
      bool all = true;
      for (size_t i = 0; i < fm.size() && all; ++i)
        if (fm[i] && !mask_host_[i]) all = false;
      if (all) bits |= 1 << f;
    }
    std::vector<uint8_t> gen;
    face_mask(cells, p, bits, gen);
    face_bits_ = gen == mask_host_ ? bits : -1;
  }
  if (!state_) state_ = std::make_shared<State>();
  if (state_->storage >= 0 && state_->storage != storage_)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "quadrature state shared between different JacobianStorage");
  size_t need = (size_t)lay_.total_points() * state_row(device_state_stride(storage_), q_);
  if (state_->data.n != need) {
    state_->data.alloc(need);
    HXG_CUDA(cudaMemset(state_->data.p, 0, need * sizeof(double)));
    state_->lay = lay_;
    state_->valid = false;
  }
  state_->storage = storage_;
  if (geometry_ && (geometry_->lay.Q != q || geometry_->lay.cells[0] != cells[0] ||
                    geometry_->lay.cells[1] != cells[1] || geometry_->lay.cells[2] != cells[2]))
    throw Error(HXG_ERR_INVALID_ARGUMENT, "geometric factors do not match basis quadrature");
  fail_.alloc(1);
}

void Operator::set_external_load(const double* host) {
  if (!host) {
    load_.release();
    return;
  }
  load_.upload(host, (size_t)size());
}

double Operator::stored_bytes_per_dof() const {
  // operator.hpp:137-141 — the reference's byte model (state in its own
  // layout: E * q^3 * 17 doubles, plus input and output vectors).
  double state_bytes =
      (double)num_elements() * q_ * q_ * q_ * ref_state_stride(storage_) * sizeof(double);
  double vec_bytes = 2.0 * (double)size() * sizeof(double);
  return (state_bytes + vec_bytes) / (double)size();
}

void Operator::launch_element(int mode, const double* x, bool mask_input) {
  ElemParams prm{};
  prm.box = box_;
  prm.lay = lay_;
  prm.x = x;
  prm.mask = mask_input ? mask() : nullptr;
  prm.tab = tab_.p;
  prm.state = state_->data.p;
  prm.state_out = state_->data.p;
  prm.geo = geometry_ ? geometry_->data.p : nullptr;
  prm.mu = mu_;
  prm.lambda = lambda_;
  prm.perturb = perturb_;
  prm.storage = storage_;
  if (perturb_ != 0.0 && !prm.geo)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "the perturbation hook needs geometric factors");
  prm.fail = fail_.p;
  size_t ev_need = (size_t)num_elements() * 3 * (p_ + 1) * (p_ + 1) * (p_ + 1);
  if (evec_.n != ev_need) evec_.alloc(ev_need);
  prm.evec = evec_.p;
  dispatch_pq(p_, q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = Dims<P, Q>;
    size_t smem = sizeof(double) * (D::TAB + D::NE * D::ELEM_SMEM);
    int grid = (int)lay_.num_bricks();
    auto launch = [&](auto k) {
      HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k<<<grid, D::T, smem, stream_>>>(prm);
    };
    auto by_storage = [&](auto Mc) {
      constexpr int M = decltype(Mc)::value;
      switch (storage_) {
        case kStorageInitialNative: launch(element_apply_kernel<P, Q, M, kStorageInitialNative>); break;
        case kStorageInitialTuned: launch(element_apply_kernel<P, Q, M, kStorageInitialTuned>); break;
        case kStorageInitialAD: launch(element_apply_kernel<P, Q, M, kStorageInitialAD>); break;
        default: launch(element_apply_kernel<P, Q, M, kStorageCurrent>);
      }
    };
    if (mode == kJacobian)
      by_storage(std::integral_constant<int, kJacobian>{});
    else
      by_storage(std::integral_constant<int, kResidual>{});
  });
  HXG_CUDA(cudaGetLastError());
}

void Operator::launch_node_sum(const double* evec, double* out, const double* x, int epilogue) {
  NodeParams np{};
  np.box = box_;
  np.evec = evec;
  np.out = out;
  np.x = x;
  np.mask = mask();
  np.load = load_.n ? load_.p : nullptr;
  np.load_scale = load_scale_;
  np.epilogue = epilogue;
  dispatch_p(p_, [&](auto Pc) {
    constexpr int P = decltype(Pc)::value;
    node_sum_kernel<P><<<grid_for(box_.num_nodes(), 256), 256, 0, stream_>>>(np);
  });
  HXG_CUDA(cudaGetLastError());
}

void Operator::apply_residual(const double* u, double* f) {
  if (!geometry_) throw Error(HXG_ERR_INVALID_ARGUMENT, "residual needs geometric factors");
  ++residual_applies_;
  const unsigned long long none = ~0ull;
  HXG_CUDA(cudaMemcpyAsync(fail_.p, &none, sizeof(none), cudaMemcpyHostToDevice, stream_));
  // one brick pass (state + f) where the fused kernel covers the operator
  const bool fz = variant_ == 0 && storage_ == kStorageCurrent && fused_supported(p_, q_);
  if (fz)
    fused_residual(*this, u, f);
  else
    launch_element(kResidual, u, false);
  unsigned long long fail = none;
  HXG_CUDA(cudaMemcpyAsync(&fail, fail_.p, sizeof(fail), cudaMemcpyDeviceToHost, stream_));
  HXG_CUDA(cudaStreamSynchronize(stream_));
  if (fail != none) {
    int nq = q_ * q_ * q_;
    long long e = (long long)(fail / nq);
    int qp = (int)(fail % nq);
    long long brick;
    int qz, t;
    lay_.locate(e, qp, brick, qz, t);
    double J = 0.0;
    size_t off = (size_t)(((brick * lay_.Q + qz) * state_row(device_state_stride(storage_), q_)) *
                              lay_.T + state_lane(t, q_));
    HXG_CUDA(cudaMemcpy(&J, state_->data.p + off, sizeof(double), cudaMemcpyDeviceToHost));
    Error err(HXG_ERR_INVERTED_ELEMENT, "non-positive deformation jacobian " + std::to_string(J) +
                                            " in element " + std::to_string(e) +
                                            " at quadrature point " + std::to_string(qp));
    err.element = (int)e;
    err.point = qp;
    err.jacobian = J;
    throw err;
  }
  state_->valid = true;
  if (!fz) launch_node_sum(evec_.p, f, nullptr, kEpiResidual);
}

void Operator::apply_jacobian_host(const double* xh, double* yh) {
  if (!state_->valid) throw Error(HXG_ERR_STATE_NOT_INITIALIZED,
                                  "quadrature state not initialized: evaluate the residual at the "
                                  "linearization point first");
  if (fused()) {
    ++jacobian_applies_;
    fused_jacobian_host(*this, xh, yh);
    return;
  }
  if (!pipe_) pipe_ = std::make_unique<HostPipe>();
  size_t n = (size_t)size();
  if (pipe_->x.n != n) {
    pipe_->x.alloc(n);
    pipe_->y.alloc(n);
  }
  HXG_CUDA(cudaMemcpyAsync(pipe_->x.p, xh, n * sizeof(double), cudaMemcpyHostToDevice, stream_));
  apply_jacobian(pipe_->x.p, pipe_->y.p);
  HXG_CUDA(cudaMemcpyAsync(yh, pipe_->y.p, n * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  HXG_CUDA(cudaStreamSynchronize(stream_));
}

bool Operator::fused() const {
  return variant_ == 0 && fused_supported(p_, q_) && (storage_ == kStorageCurrent || q_ == p_ + 1);
}

int Operator::kernel_launches() const { return fused() ? fused_launches(p_, q_) : 2; }

void Operator::apply_jacobian(const double* du, double* y) {
  if (!state_->valid) throw Error(HXG_ERR_STATE_NOT_INITIALIZED,
                                  "quadrature state not initialized: evaluate the residual at the "
                                  "linearization point first");
  ++jacobian_applies_;
  if (fused()) {
    fused_jacobian(*this, du, y);
    return;
  }
  launch_element(kJacobian, du, true);
  launch_node_sum(evec_.p, y, du, kEpiJacobian);
}

void Operator::apply_jacobian_split(const double* du, double* y, int iface, cudaStream_t side,
                                    const std::function<void()>& exchange) {
  if (!state_->valid) throw Error(HXG_ERR_STATE_NOT_INITIALIZED,
                                  "quadrature state not initialized: evaluate the residual at the "
                                  "linearization point first");
  if (!fused()) throw Error(HXG_ERR_UNSUPPORTED, "split apply needs the fused path");
  ++jacobian_applies_;
  fused_jacobian_split(*this, du, y, iface, side, exchange);
}

void Operator::extract_diagonal(double* d) {
  if (!state_->valid) throw Error(HXG_ERR_STATE_NOT_INITIALIZED,
                                  "quadrature state not initialized: evaluate the residual at the "
                                  "linearization point first");
  size_t ev_need = (size_t)num_elements() * 3 * (p_ + 1) * (p_ + 1) * (p_ + 1);
  if (evec_.n != ev_need) evec_.alloc(ev_need);
  DiagParams prm{};
  prm.box = box_;
  prm.lay = lay_;
  prm.interp = interp_d_.p;
  prm.deriv = deriv_d_.p;
  prm.state = state_->data.p;
  prm.geo = geometry_ ? geometry_->data.p : nullptr;
  prm.mu = mu_;
  prm.lambda = lambda_;
  prm.perturb = perturb_;
  prm.storage = storage_;
  if (perturb_ != 0.0 && !prm.geo)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "the perturbation hook needs geometric factors");
  prm.out = evec_.p;
  dispatch_pq(p_, q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    size_t smem = sizeof(double) * (2 * Q * (P + 1) + Q * Q * Q * 27);
    auto k = diag_element_kernel<P, Q>;
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)num_elements(), 128, smem, stream_>>>(prm);
  });
  HXG_CUDA(cudaGetLastError());
  launch_node_sum(evec_.p, d, nullptr, kEpiDiagonal);
}

void Operator::element_matrices(double* out) {
  if (!state_->valid) throw Error(HXG_ERR_STATE_NOT_INITIALIZED,
                                  "quadrature state not initialized: evaluate the residual at the "
                                  "linearization point first");
  DiagParams prm{};
  prm.box = box_;
  prm.lay = lay_;
  prm.interp = interp_d_.p;
  prm.deriv = deriv_d_.p;
  prm.state = state_->data.p;
  prm.geo = geometry_ ? geometry_->data.p : nullptr;
  prm.mu = mu_;
  prm.lambda = lambda_;
  prm.perturb = perturb_;
  prm.storage = storage_;
  if (perturb_ != 0.0 && !prm.geo)
    throw Error(HXG_ERR_INVALID_ARGUMENT, "the perturbation hook needs geometric factors");
  prm.out = out;
  if (p_ == 1) {  // the coarse level: two-stage contraction
    dispatch_q(q_, [&](auto Qc) {
      constexpr int Q = decltype(Qc)::value;
      // D (and the 4 x 72 x 8 group reduction) + node gradients
      constexpr size_t smem = sizeof(double) * (kQ1AsmChunk * 81 + kQ1AsmChunk * 24);
      static_assert(kQ1AsmChunk * (81 + 24) >= 4 * 72 * 8, "reduction fits the D + G buffers");
      auto launch = [&](auto k) {
        HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared));
        k<<<(unsigned)num_elements(), kQ1AsmThreads, smem, stream_>>>(prm);
      };
      switch (storage_) {
        case kStorageInitialNative: launch(assemble_element_q1_kernel<Q, kStorageInitialNative>); break;
        case kStorageInitialTuned: launch(assemble_element_q1_kernel<Q, kStorageInitialTuned>); break;
        case kStorageInitialAD: launch(assemble_element_q1_kernel<Q, kStorageInitialAD>); break;
        default: launch(assemble_element_q1_kernel<Q, kStorageCurrent>);
      }
    });
    HXG_CUDA(cudaGetLastError());
    return;
  }
  dispatch_pq(p_, q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    size_t smem = sizeof(double) * (2 * Q * (P + 1) + Q * Q * Q * 81);
    auto k = assemble_element_kernel<P, Q>;
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)num_elements(), 256, smem, stream_>>>(prm);
  });
  HXG_CUDA(cudaGetLastError());
}

double Operator::total_strain_energy(const double* u) {
  if (!geometry_) throw Error(HXG_ERR_INVALID_ARGUMENT, "energy needs geometric factors");
  DevBuf<double> part((size_t)num_elements());
  const unsigned long long none = ~0ull;
  HXG_CUDA(cudaMemcpyAsync(fail_.p, &none, sizeof(none), cudaMemcpyHostToDevice, stream_));
  ElemParams prm{};
  prm.box = box_;
  prm.lay = lay_;
  prm.x = u;
  prm.tab = tab_.p;
  prm.geo = geometry_->data.p;
  prm.mu = mu_;
  prm.lambda = lambda_;
  prm.fail = fail_.p;
  prm.energy_part = part.p;
  dispatch_pq(p_, q_, [&](auto Pc, auto Qc) {
    constexpr int P = decltype(Pc)::value, Q = decltype(Qc)::value;
    using D = Dims<P, Q>;
    size_t smem = sizeof(double) * (D::TAB + D::NE * D::ELEM_SMEM + D::T);
    auto k = element_energy_kernel<P, Q>;
    HXG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)lay_.num_bricks(), D::T, smem, stream_>>>(prm);
  });
  HXG_CUDA(cudaGetLastError());
  std::vector<double> host((size_t)num_elements());
  unsigned long long fail = none;
  HXG_CUDA(cudaMemcpyAsync(&fail, fail_.p, sizeof(fail), cudaMemcpyDeviceToHost, stream_));
  HXG_CUDA(cudaMemcpyAsync(host.data(), part.p, host.size() * sizeof(double),
                           cudaMemcpyDeviceToHost, stream_));
  HXG_CUDA(cudaStreamSynchronize(stream_));
  if (fail != none) {
    int nq = q_ * q_ * q_;
    Error err(HXG_ERR_INVERTED_ELEMENT,
              "non-positive deformation jacobian in element " + std::to_string(fail / nq) +
                  " at quadrature point " + std::to_string(fail % nq));
    err.element = (int)(fail / nq);
    err.point = (int)(fail % nq);
    throw err;
  }
  double total = 0.0;
  for (double v : host) total += v;  // element order (operator.hpp:312-314)
  return total;
}

void Operator::export_state(double* host) const {
  // Stored [sqrt(w detJ) xi (9), tau (6), mu - lambda log J] back to the
  // reference's (e, q, 17) Current layout; w detJ from the geometry.
  if (storage_ != kStorageCurrent) {  // stored in the reference layout already
    const int S = device_state_stride(storage_), SP = state_row(S, q_);
    std::vector<double> blocked((size_t)lay_.total_points() * SP);
    HXG_CUDA(cudaMemcpy(blocked.data(), state_->data.p, blocked.size() * sizeof(double),
                        cudaMemcpyDeviceToHost));
    const int nq = q_ * q_ * q_;
    for (long long e = 0; e < num_elements(); ++e)
      for (int qp = 0; qp < nq; ++qp) {
        long long brick;
        int qz, t;
        lay_.locate(e, qp, brick, qz, t);
        const size_t base = (size_t)(brick * lay_.Q + qz) * SP * lay_.T + state_lane(t, q_);
        double* out = host + ((size_t)e * nq + qp) * S;
        for (int k = 0; k < S; ++k) out[k] = blocked[base + state_pair_off(k, lay_.T, q_)];
      }
    return;
  }
  if (!geometry_) throw Error(HXG_ERR_INVALID_ARGUMENT, "state export needs geometric factors");
  size_t tot = (size_t)lay_.total_points() * kStateStride;
  std::vector<double> blocked(tot), geo((size_t)lay_.total_points() * kGeoStride);
  HXG_CUDA(cudaMemcpy(blocked.data(), state_->data.p, tot * sizeof(double), cudaMemcpyDeviceToHost));
  HXG_CUDA(cudaMemcpy(geo.data(), geometry_->data.p, geo.size() * sizeof(double),
                      cudaMemcpyDeviceToHost));
  int nq = q_ * q_ * q_;
  for (long long e = 0; e < num_elements(); ++e)
    for (int qp = 0; qp < nq; ++qp) {
      long long brick;
      int qz, t;
      lay_.locate(e, qp, brick, qz, t);
      const size_t row = (size_t)(brick * lay_.Q + qz);
      const size_t base = row * kStateStride * lay_.T + state_lane(t, q_);
      const double wdet = geo[(row * kGeoStride + 9) * lay_.T + t];
      const double isw = 1.0 / std::sqrt(wdet);
      double* out = host + ((size_t)e * nq + qp) * kRefStateScalars;
      out[0] = wdet;
      for (int k = 0; k < 9; ++k) out[1 + k] = blocked[base + state_pair_off(k, lay_.T, q_)] * isw;
      for (int k = 0; k < 6; ++k) out[10 + k] = blocked[base + state_pair_off(9 + k, lay_.T, q_)];
      out[16] = mu_ - blocked[base + state_pair_off(15, lay_.T, q_)];
    }
}

namespace {

template <int P>
__global__ void gather_kernel(BoxDev box, const double* x, double* ev) {
  constexpr int N = P + 1, N3 = N * N * N;
  long long total = box.num_elements() * 3 * N3;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < total;
       r += (long long)gridDim.x * blockDim.x) {
    long long e = r / (3 * N3);
    int rem = (int)(r % (3 * N3));
    int c = rem / N3, a = rem % N3;
    int i = a % N, j = (a / N) % N, k = a / (N * N);
    long long ex = e % box.cells[0], ey = (e / box.cells[0]) % box.cells[1],
              ez = e / ((long long)box.cells[0] * box.cells[1]);
    long long node = (P * ex + i) + box.npd[0] * ((P * ey + j) + (long long)box.npd[1] * (P * ez + k));
    ev[r] = x[3 * node + c];
  }
}

}  // namespace

void Operator::gather(const double* l, double* e) {
  dispatch_p(p_, [&](auto Pc) {
    constexpr int P = decltype(Pc)::value;
    gather_kernel<P><<<grid_for(num_elements() * 3 * (P + 1) * (P + 1) * (P + 1), 256), 256, 0,
                       stream_>>>(box_, l, e);
  });
  HXG_CUDA(cudaGetLastError());
}

void Operator::scatter_add(const double* e, double* l) {
  // scatter_add accumulates into l in element order (mesh.hpp:105-116).
  NodeParams np{};
  np.box = box_;
  np.evec = e;
  np.out = l;
  np.epilogue = kEpiNone;
  np.accumulate = 1;
  dispatch_p(p_, [&](auto Pc) {
    constexpr int P = decltype(Pc)::value;
    node_sum_kernel<P><<<grid_for(box_.num_nodes(), 256), 256, 0, stream_>>>(np);
  });
  HXG_CUDA(cudaGetLastError());
}

}  // namespace hxg
