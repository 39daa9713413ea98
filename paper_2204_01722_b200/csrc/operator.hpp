// Device-resident matrix-free operator (MatrixFreeOperator, operator.hpp:70-373).
#pragma once

#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <vector>

#include "common.hpp"
#include "setup.hpp"

namespace hxg {

// Owning device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) HXG_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void upload(const T* host, size_t count) {
    if (count != n) alloc(count);
    if (count) HXG_CUDA(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
  }
  void upload(const std::vector<T>& v) { upload(v.data(), v.size()); }
};

// QuadratureStateStore (operator.hpp:60-64): blocked device layout.
struct State {
  DevBuf<double> data;
  QLayout lay;
  bool valid = false;
  int storage = -1;  // JacobianStorage the data is laid out for (-1: unallocated)
};

// Geometry shared between levels (multigrid.hpp:229-230): blocked layout,
// kGeoStride doubles per point.
struct Geometry {
  DevBuf<double> data;
  QLayout lay;
  // Box meshes (build_box_mesh: every element the same affine map): the
  // factors are dxi/dX = diag(g), w detJ = w_qx w_qy w_qz jac, so kernels
  // that only read them (the fused residual) can form them in registers.
  bool box = false;
  double g[3] = {0.0, 0.0, 0.0};
  double jac = 0.0;
  double qw[kMaxQ] = {0.0, 0.0, 0.0, 0.0, 0.0};
};

// Streams, events and device staging for the pipelined host-buffer apply
// (H2D of z-chunks / compute / D2H overlapped).
struct HostPipe {
  static constexpr int kMaxChunks = 64;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t in_ready[kMaxChunks], out_ready[kMaxChunks], done_evt = nullptr;
  DevBuf<double> x, y;
  HostPipe() {
    HXG_CUDA(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
    HXG_CUDA(cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking));
    HXG_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    for (int i = 0; i < kMaxChunks; ++i) {
      HXG_CUDA(cudaEventCreateWithFlags(&in_ready[i], cudaEventDisableTiming));
      HXG_CUDA(cudaEventCreateWithFlags(&out_ready[i], cudaEventDisableTiming));
    }
    HXG_CUDA(cudaEventCreateWithFlags(&done_evt, cudaEventDisableTiming));
  }
  ~HostPipe() {
    for (int i = 0; i < kMaxChunks; ++i) {
      cudaEventDestroy(in_ready[i]);
      cudaEventDestroy(out_ready[i]);
    }
    cudaEventDestroy(done_evt);
    cudaStreamDestroy(h2d);
    cudaStreamDestroy(comp);
    cudaStreamDestroy(d2h);
  }
};

class Operator {
 public:
  // desc fields as hxg_op_desc; geometry may come from desc (host arrays) or
  // be shared from another operator.
  Operator(int p, int q, const int cells[3], const std::vector<double>& interp,
           const std::vector<double>& deriv, const std::vector<double>& colloc, double mu,
           double lambda, const uint8_t* mask_host, std::shared_ptr<State> state,
           std::shared_ptr<Geometry> geometry, int storage = kStorageCurrent);

  // Builds a Geometry from reference-layout host arrays (e, q, 9) / (e, q).
  // Affine box geometry computed on the device (no host arrays).
  static std::shared_ptr<Geometry> make_box_geometry(const int cells[3], int q,
                                                     const double extents[3],
                                                     const double* qweights);
  static std::shared_ptr<Geometry> make_geometry(const int cells[3], int q, const double* dxidX,
                                                 const double* weight);

  int p() const { return p_; }
  int q() const { return q_; }
  int storage() const { return storage_; }
  // The fused brick kernel serves Current storage; the initial-configuration
  // variants run the two-pass element path.
  bool fused() const;
  long long size() const { return 3 * box_.num_nodes(); }
  long long num_elements() const { return box_.num_elements(); }
  const BoxDev& box() const { return box_; }
  const QLayout& layout() const { return lay_; }
  const int* cells() const { return cells_; }
  const uint8_t* mask() const { return mask_.n ? mask_.p : nullptr; }
  // >= 0 when the constraint mask is exactly a union of whole faces (all
  // components) — bit f = Face f — so kernels can test it analytically;
  // -1 for general masks.
  int face_bits() const { return face_bits_; }
  const std::vector<uint8_t>& mask_host() const { return mask_host_; }
  const std::shared_ptr<State>& state() const { return state_; }
  const std::shared_ptr<Geometry>& geometry() const { return geometry_; }
  double mu() const { return mu_; }
  double lambda() const { return lambda_; }
  const std::vector<double>& interp_host() const { return interp_; }
  const std::vector<double>& deriv_host() const { return deriv_; }
  const std::vector<double>& colloc_host() const { return colloc_; }

  cudaStream_t stream() const { return stream_; }
  void set_stream(cudaStream_t s) { stream_ = s; }
  void set_external_load(const double* host);
  void set_load_scale(double s) { load_scale_ = s; }
  void set_jacobian_perturbation(double eps) { perturb_ = eps; }
  void set_variant(int v) { variant_ = v; }
  int variant() const { return variant_; }
  int kernel_launches() const;

  double stored_bytes_per_dof() const;
  long long residual_applies() const { return residual_applies_; }
  long long jacobian_applies() const { return jacobian_applies_; }

  void apply_residual(const double* u, double* f);
  void apply_jacobian(const double* du, double* y);
  void extract_diagonal(double* d);
  double total_strain_energy(const double* u);
  void export_state(double* host) const;
  void gather(const double* l, double* e);
  void scatter_add(const double* e, double* l);
  // Element matrices (e, 3N^3, 3N^3) of the assembled operator.
  void element_matrices(double* out);

  // Host buffers in, host buffers out: pipelined over z-chunks when the fused
  // path applies (H2D / compute / D2H overlap), else stage + apply + copy.
  void apply_jacobian_host(const double* xh, double* yh);

  friend void fused_jacobian(Operator& op, const double* du, double* y);
  friend void fused_jacobian_split(Operator& op, const double* du, double* y, int iface,
                                   cudaStream_t side, const std::function<void()>& exchange);
  // Partitioned apply with the exchange overlapped (fused path only):
  // see fused_jacobian_split.
  void apply_jacobian_split(const double* du, double* y, int iface, cudaStream_t side,
                            const std::function<void()>& exchange);
  // Instrumentation: when set, the next fused apply records this event on
  // the stream between the brick kernel and the fix-up kernel (then clears it).
  void set_split_event(cudaEvent_t e) { split_evt_ = e; }
  friend void fused_residual(Operator& op, const double* u, double* f);
  friend void fused_jacobian_host(Operator& op, const double* xh, double* yh);

 private:
  void launch_element(int mode, const double* x, bool mask_input);
  void launch_node_sum(const double* evec, double* out, const double* x, int epilogue);

  int p_, q_;
  int cells_[3];
  BoxDev box_;
  QLayout lay_;
  double mu_, lambda_;
  double load_scale_ = 1.0, perturb_ = 0.0;
  int variant_ = 0;
  int storage_ = kStorageCurrent;
  int face_bits_ = 0;
  std::vector<double> interp_, deriv_, colloc_;
  std::vector<uint8_t> mask_host_;
  DevBuf<double> tab_;     // B (Q x N) then Dc (Q x Q)
  DevBuf<double> interp_d_, deriv_d_;
  DevBuf<uint8_t> mask_;
  DevBuf<double> load_;
  DevBuf<double> evec_;    // E-vector scratch for the two-pass path
  DevBuf<double> partial_; // brick-boundary partial sums for the fused path
  cudaEvent_t split_evt_ = nullptr;
  // partitioned apply: bricks touching the interface faces first, then the rest
  DevBuf<int> blist_;
  int blist_iface_ = -1, blist_na_ = 0;
  cudaEvent_t ev_a_ = nullptr, ev_x_ = nullptr;
  std::unique_ptr<HostPipe> pipe_;
  DevBuf<unsigned long long> fail_;
  std::shared_ptr<State> state_;
  std::shared_ptr<Geometry> geometry_;
  cudaStream_t stream_ = nullptr;
  long long residual_applies_ = 0, jacobian_applies_ = 0;
};

}  // namespace hxg
