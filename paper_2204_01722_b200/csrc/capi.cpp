// extern "C" boundary (include/hexmg_b200.h).  Every entry point catches
// and maps exceptions to codes + thread-local detail.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "coarse.hpp"
#include "common.hpp"
#include "operator.hpp"
#include "setup.hpp"
#include "solver.hpp"
#include "hcoarse.hpp"
#include "vector.hpp"

struct hxg_state_s {
  std::shared_ptr<hxg::State> s;
};
struct hxg_op_s {
  std::unique_ptr<hxg::Operator> owned;
  hxg::Operator* op = nullptr;
};
struct hxg_comm_s {
  std::unique_ptr<hxg::Comm> c;
};
struct hxg_mg_s {
  std::unique_ptr<hxg::Partition> part;  // partitioned hierarchies
  std::unique_ptr<hxg::Hierarchy> h;
  std::vector<hxg_op_s> level_handles;
};
struct hxg_chol_s {
  hxg::CsrMatrix a;
  hxg::CoarseSolver solver;
  int npd[3] = {0, 0, 0};
  cudaStream_t stream = nullptr;
};

namespace {

thread_local hxg_error g_err{0, -1, -1, 0.0, {0}};

void set_error(int code, const char* msg, int element = -1, int point = -1, double j = 0.0) {
  g_err.code = code;
  g_err.element = element;
  g_err.point = point;
  g_err.jacobian = j;
  std::snprintf(g_err.message, sizeof(g_err.message), "%s", msg);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return HXG_OK;
  } catch (const hxg::Error& e) {
    set_error(e.code, e.what(), e.element, e.point, e.jacobian);
    return e.code;
  } catch (const std::bad_alloc&) {
    set_error(HXG_ERR_GENERIC, "out of host memory");
    return HXG_ERR_GENERIC;
  } catch (const std::exception& e) {
    set_error(HXG_ERR_GENERIC, e.what());
    return HXG_ERR_GENERIC;
  }
}

hxg::Operator& OP(hxg_op_t h) {
  if (!h || !h->op) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "null operator handle");
  return *h->op;
}

hxg::Hierarchy& MG(hxg_mg_t h) {
  if (!h || !h->h) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "null hierarchy handle");
  return *h->h;
}

}  // namespace

extern "C" {

int hxg_last_error(hxg_error* out) {
  if (out) *out = g_err;
  return g_err.code;
}

const char* hxg_version(void) { return "hexmg-b200 0.1 (sm_100a, FP64)"; }

int hxg_state_create(hxg_state_t* out) {
  return guarded([&] {
    auto* s = new hxg_state_s();
    s->s = std::make_shared<hxg::State>();
    *out = s;
  });
}

int hxg_state_release(hxg_state_t s) {
  delete s;
  return HXG_OK;
}

int hxg_op_create(const hxg_op_desc* d, hxg_state_t state, hxg_op_t* out) {
  return guarded([&] {
    if (!d) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "null descriptor");
    int n = d->order + 1, q = d->qpts;
    std::vector<double> interp(d->interp, d->interp + q * n);
    std::vector<double> deriv(d->deriv, d->deriv + q * n);
    std::vector<double> colloc(d->colloc, d->colloc + q * q);
    std::shared_ptr<hxg::Geometry> geo;
    if (d->dxidX && d->weight)
      geo = hxg::Operator::make_geometry(d->cells, q, d->dxidX, d->weight);
    else if (d->extents && d->qweights)
      geo = hxg::Operator::make_box_geometry(d->cells, q, d->extents, d->qweights);
    auto* h = new hxg_op_s();
    h->owned = std::make_unique<hxg::Operator>(d->order, q, d->cells, interp, deriv, colloc, d->mu,
                                               d->lambda, d->mask, state ? state->s : nullptr, geo,
                                               d->storage);
    h->op = h->owned.get();
    *out = h;
  });
}

int hxg_op_destroy(hxg_op_t op) {
  delete op;
  return HXG_OK;
}

int hxg_op_size(hxg_op_t op, int64_t* n) { return guarded([&] { *n = OP(op).size(); }); }
int hxg_op_num_elements(hxg_op_t op, int64_t* ne) {
  return guarded([&] { *ne = OP(op).num_elements(); });
}
int hxg_op_set_stream(hxg_op_t op, void* stream) {
  return guarded([&] { OP(op).set_stream((cudaStream_t)stream); });
}
int hxg_op_set_external_load(hxg_op_t op, const double* load) {
  return guarded([&] { OP(op).set_external_load(load); });
}
int hxg_op_set_load_scale(hxg_op_t op, double s) {
  return guarded([&] { OP(op).set_load_scale(s); });
}
int hxg_op_set_jacobian_perturbation(hxg_op_t op, double eps) {
  return guarded([&] { OP(op).set_jacobian_perturbation(eps); });
}
int hxg_op_stored_bytes_per_dof(hxg_op_t op, double* out) {
  return guarded([&] { *out = OP(op).stored_bytes_per_dof(); });
}
int hxg_op_counters(hxg_op_t op, int64_t* r, int64_t* j) {
  return guarded([&] {
    *r = OP(op).residual_applies();
    *j = OP(op).jacobian_applies();
  });
}
int hxg_op_set_variant(hxg_op_t op, int v) { return guarded([&] { OP(op).set_variant(v); }); }
int hxg_op_kernel_launches(hxg_op_t op, int* n) {
  return guarded([&] { *n = OP(op).kernel_launches(); });
}

int hxg_op_apply_residual(hxg_op_t op, const double* u, double* f) {
  return guarded([&] { OP(op).apply_residual(u, f); });
}
int hxg_op_apply_jacobian(hxg_op_t op, const double* du, double* y) {
  return guarded([&] { OP(op).apply_jacobian(du, y); });
}

namespace {
struct Pinned {
  double* p = nullptr;
  size_t n = 0;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};
}  // namespace

int hxg_op_apply_jacobian_host(hxg_op_t op, const double* du_host, double* y_host) {
  return guarded([&] { OP(op).apply_jacobian_host(du_host, y_host); });
}

int hxg_op_apply_residual_host(hxg_op_t op, const double* u_host, double* f_host) {
  return guarded([&] {
    auto& o = OP(op);
    size_t n = (size_t)o.size();
    hxg::DevBuf<double> x(n), y(n);
    cudaStream_t s = o.stream();
    HXG_CUDA(cudaMemcpyAsync(x.p, u_host, n * sizeof(double), cudaMemcpyHostToDevice, s));
    o.apply_residual(x.p, y.p);
    HXG_CUDA(cudaMemcpyAsync(f_host, y.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    HXG_CUDA(cudaStreamSynchronize(s));
  });
}

int hxg_op_extract_diagonal(hxg_op_t op, double* d) {
  return guarded([&] { OP(op).extract_diagonal(d); });
}
int hxg_op_total_strain_energy(hxg_op_t op, const double* u, double* energy) {
  return guarded([&] { *energy = OP(op).total_strain_energy(u); });
}
int hxg_op_export_state(hxg_op_t op, double* host) {
  return guarded([&] {
    if (!OP(op).state()->valid)
      throw hxg::Error(HXG_ERR_STATE_NOT_INITIALIZED, "quadrature state not initialized");
    OP(op).export_state(host);
  });
}
int hxg_op_gather(hxg_op_t op, const double* l, double* e) {
  return guarded([&] { OP(op).gather(l, e); });
}
int hxg_op_scatter_add(hxg_op_t op, const double* e, double* l) {
  return guarded([&] { OP(op).scatter_add(e, l); });
}

int hxg_op_time_jacobian_parts(hxg_op_t op, const double* x, double* y, int warmup, int repeats,
                               double ms[2]) {
  return guarded([&] {
    auto& o = OP(op);
    if (!o.fused()) throw hxg::Error(HXG_ERR_UNSUPPORTED, "per-kernel timing needs the fused path");
    if (repeats < 1 || repeats > 1000) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "repeats in 1..1000");
    cudaStream_t s = o.stream();
    for (int w = 0; w < warmup; ++w) o.apply_jacobian(x, y);
    std::vector<cudaEvent_t> ev(3 * (size_t)repeats);
    for (auto& e : ev) HXG_CUDA(cudaEventCreate(&e));
    HXG_CUDA(cudaStreamSynchronize(s));
    for (int r = 0; r < repeats; ++r) {
      HXG_CUDA(cudaEventRecord(ev[3 * r], s));
      o.set_split_event(ev[3 * r + 1]);
      o.apply_jacobian(x, y);
      HXG_CUDA(cudaEventRecord(ev[3 * r + 2], s));
    }
    HXG_CUDA(cudaEventSynchronize(ev.back()));
    double a = 0.0, b = 0.0;
    for (int r = 0; r < repeats; ++r) {
      float f = 0.f, g = 0.f;
      HXG_CUDA(cudaEventElapsedTime(&f, ev[3 * r], ev[3 * r + 1]));
      HXG_CUDA(cudaEventElapsedTime(&g, ev[3 * r + 1], ev[3 * r + 2]));
      a += f;
      b += g;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    ms[0] = a / repeats;
    ms[1] = b / repeats;
  });
}
int hxg_op_time_jacobian(hxg_op_t op, const double* x, double* y, int warmup, int repeats,
                         double* ms) {
  return guarded([&] {
    auto& o = OP(op);
    cudaStream_t s = o.stream();
    for (int w = 0; w < warmup; ++w) o.apply_jacobian(x, y);
    cudaEvent_t a, b;
    HXG_CUDA(cudaEventCreate(&a));
    HXG_CUDA(cudaEventCreate(&b));
    HXG_CUDA(cudaStreamSynchronize(s));
    HXG_CUDA(cudaEventRecord(a, s));
    for (int r = 0; r < repeats; ++r) o.apply_jacobian(x, y);
    HXG_CUDA(cudaEventRecord(b, s));
    HXG_CUDA(cudaEventSynchronize(b));
    float f = 0.f;
    HXG_CUDA(cudaEventElapsedTime(&f, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *ms = f;
  });
}

// ---- multigrid -------------------------------------------------------------

int hxg_mg_create(hxg_op_t fine, int fixed_face_mask, const int* schedule, int num_levels,
                  int pre_smooth, int post_smooth, hxg_mg_t* out) {
  return guarded([&] {
    std::vector<int> sched;
    if (schedule) sched.assign(schedule, schedule + num_levels);
    auto* h = new hxg_mg_s();
    h->h = std::make_unique<hxg::Hierarchy>(&OP(fine), fixed_face_mask, sched, pre_smooth,
                                            post_smooth);
    h->level_handles.resize((size_t)h->h->num_levels());
    for (int k = 0; k < h->h->num_levels(); ++k) h->level_handles[(size_t)k].op = h->h->level(k).op;
    *out = h;
  });
}

int hxg_mg_create_partitioned(hxg_op_t fine, hxg_comm_t comm, const int global_cells[3],
                              const int dims[3], int global_fixed_face_mask, const int* schedule,
                              int num_levels, int pre_smooth, int post_smooth, hxg_mg_t* out) {
  return guarded([&] {
    if (!comm || !comm->c) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "null communicator");
    std::vector<int> sched;
    if (schedule) sched.assign(schedule, schedule + num_levels);
    auto h = std::make_unique<hxg_mg_s>();
    h->part = std::make_unique<hxg::Partition>(comm->c.get(), global_cells, dims);
    h->h = std::make_unique<hxg::Hierarchy>(&OP(fine), global_fixed_face_mask, sched, pre_smooth,
                                            post_smooth, h->part.get());
    h->level_handles.resize((size_t)h->h->num_levels());
    for (int k = 0; k < h->h->num_levels(); ++k) h->level_handles[(size_t)k].op = h->h->level(k).op;
    *out = h.release();
  });
}

int hxg_mg_apply(hxg_mg_t mg, int level, const double* x, double* y) {
  return guarded([&] {
    MG(mg).follow_stream();
    MG(mg).level_apply(level, x, y);
  });
}
int hxg_mg_dot(hxg_mg_t mg, int level, const double* x, const double* y, double* out) {
  return guarded([&] {
    MG(mg).follow_stream();
    *out = MG(mg).level_dot(level, x, y);
  });
}
int hxg_mg_residual(hxg_mg_t mg, const double* u, double* f) {
  return guarded([&] { MG(mg).residual(u, f); });
}

int hxg_mg_destroy(hxg_mg_t mg) {
  delete mg;
  return HXG_OK;
}
int hxg_mg_num_levels(hxg_mg_t mg, int* n) { return guarded([&] { *n = MG(mg).num_levels(); }); }
int hxg_mg_level_size(hxg_mg_t mg, int level, int64_t* n) {
  return guarded([&] { *n = MG(mg).level(level).op->size(); });
}
int hxg_mg_level_op(hxg_mg_t mg, int level, hxg_op_t* op) {
  return guarded([&] {
    if (level < 0 || level >= MG(mg).num_levels())
      throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "level out of range");
    *op = &mg->level_handles[(size_t)level];
  });
}
int hxg_mg_setup_numeric(hxg_mg_t mg) { return guarded([&] { MG(mg).setup_numeric(); }); }
int hxg_mg_assemble_coarse(hxg_mg_t mg) { return guarded([&] { MG(mg).assemble_coarse(); }); }
int hxg_mg_set_coarse_mode(hxg_mg_t mg, int mode) {
  return guarded([&] {
    if (mode < 0 || mode > 4 || mode == 3)
      throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "coarse mode must be 0, 1, 2 or 4");
    MG(mg).set_coarse_mode(mode);
  });
}
int hxg_mg_lambda_max(hxg_mg_t mg, int level, double* out) {
  return guarded([&] { *out = MG(mg).level(level).smoother.lambda_max; });
}
int hxg_mg_prolong(hxg_mg_t mg, int coarse_level, const double* xc, double* xf) {
  return guarded([&] { MG(mg).prolong(coarse_level, xc, xf); });
}
int hxg_mg_restrict(hxg_mg_t mg, int coarse_level, const double* xf, double* xc) {
  return guarded([&] { MG(mg).restrict_to(coarse_level, xf, xc); });
}
int hxg_mg_vcycle(hxg_mg_t mg, const double* b, double* x) {
  return guarded([&] { MG(mg).v_cycle(b, x, false); });
}
int hxg_mg_smooth(hxg_mg_t mg, int level, const double* b, double* x) {
  return guarded([&] {
    MG(mg).smooth(level, b, x);
  });
}
int hxg_mg_coarse_vals_device(hxg_mg_t mg, double* vals_dev) {
  return guarded([&] {
    // ordered after the assembly kernels on the hierarchy's stream
    const auto& a = MG(mg).coarse_matrix();
    cudaStream_t s = MG(mg).stream();
    HXG_CUDA(cudaMemcpyAsync(vals_dev, a.vals.p, sizeof(double) * a.cols_h.size(),
                             cudaMemcpyDeviceToDevice, s));
    HXG_CUDA(cudaStreamSynchronize(s));
  });
}
int hxg_mg_coarse_nnz(hxg_mg_t mg, int64_t* nnz) {
  return guarded([&] { *nnz = MG(mg).coarse_matrix().nnz(); });
}
int hxg_mg_coarse_csr_host(hxg_mg_t mg, int* row_ptr, int* cols, double* vals) {
  return guarded([&] {
    const auto& a = MG(mg).coarse_matrix();
    std::memcpy(row_ptr, a.row_ptr_h.data(), sizeof(int) * a.row_ptr_h.size());
    std::memcpy(cols, a.cols_h.data(), sizeof(int) * a.cols_h.size());
    cudaStream_t s = MG(mg).stream();
    HXG_CUDA(cudaMemcpyAsync(vals, a.vals.p, sizeof(double) * a.cols_h.size(),
                             cudaMemcpyDeviceToHost, s));
    HXG_CUDA(cudaStreamSynchronize(s));
  });
}
int hxg_mg_hmg_levels(hxg_mg_t mg, int* levels) {
  return guarded([&] {
    const hxg::HmgCoarse* h = MG(mg).hmg();
    *levels = h && h->ready() ? h->num_levels() : 0;
  });
}
int hxg_mg_hmg_level_nnz(hxg_mg_t mg, int level, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    const hxg::HmgCoarse* h = MG(mg).hmg();
    if (!h || !h->ready() || level < 0 || level >= h->num_levels())
      throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "no such h-multigrid level");
    *n = h->level_matrix(level).n;
    *nnz = h->level_matrix(level).nnz();
  });
}
int hxg_mg_hmg_level_csr_host(hxg_mg_t mg, int level, int* row_ptr, int* cols, double* vals,
                              uint8_t* mask) {
  return guarded([&] {
    const hxg::HmgCoarse* h = MG(mg).hmg();
    if (!h || !h->ready() || level < 0 || level >= h->num_levels())
      throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "no such h-multigrid level");
    const auto& a = h->level_matrix(level);
    std::memcpy(row_ptr, a.row_ptr_h.data(), sizeof(int) * a.row_ptr_h.size());
    std::memcpy(cols, a.cols_h.data(), sizeof(int) * a.cols_h.size());
    std::memcpy(mask, h->level_mask(level).data(), h->level_mask(level).size());
    cudaStream_t s = MG(mg).stream();
    HXG_CUDA(cudaMemcpyAsync(vals, a.vals.p, sizeof(double) * a.cols_h.size(),
                             cudaMemcpyDeviceToHost, s));
    HXG_CUDA(cudaStreamSynchronize(s));
  });
}
int hxg_mg_coarse_solve(hxg_mg_t mg, const double* b, double* x) {
  return guarded([&] { MG(mg).coarse_solve(b, x); });
}

int hxg_cg_solve(hxg_op_t op, hxg_mg_t mg, int precond, const double* b, double* x, double rtol,
                 int max_iterations, hxg_cg_report* report, double* history, int cap) {
  return guarded([&] {
    auto& o = OP(op);
    long long n = o.size();
    cudaStream_t s = o.stream();
    hxg::DevOp a = [&o](const double* xx, double* yy) { o.apply_jacobian(xx, yy); };
    // a partitioned hierarchy: its fine level operator and owned-entry dots
    hxg::Hierarchy* ph = mg && mg->h && mg->h->partition() ? mg->h.get() : nullptr;
    hxg::DotFn dotf;
    if (ph) {
      if (ph->level(ph->num_levels() - 1).op != &o)
        throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "op is not the partitioned hierarchy's fine level");
      const int fine = ph->num_levels() - 1;
      ph->follow_stream();
      a = [ph, fine](const double* xx, double* yy) { ph->level_apply(fine, xx, yy); };
      dotf = [ph, fine](const double* xx, const double* yy) { return ph->level_dot(fine, xx, yy); };
    }
    hxg::DevOp m;
    hxg::DevBuf<double> inv;
    if (precond == 0) {
      m = [n, s](const double* r, double* z) { hxg::vcopy(z, r, n, s); };
    } else if (precond == 1) {
      hxg::DevBuf<double> d((size_t)n);
      o.extract_diagonal(d.p);
      inv.alloc((size_t)n);
      hxg::vreciprocal(inv.p, d.p, n, s);
      const double* ip = inv.p;
      m = [n, s, ip](const double* r, double* z) { hxg::vscale_mul(z, ip, r, n, s); };
    } else {
      auto& h = MG(mg);
      m = [&h, n, s](const double* r, double* z) {
        hxg::vzero(z, n, s);
        h.v_cycle(r, z, true);
      };
    }
    if (ph && precond == 1) {  // the Jacobi diagonal needs the interface sums too
      hxg::DevBuf<double> d((size_t)n);
      o.extract_diagonal(d.p);
      ph->partition()->exchange(o.p(), d.p, s);
      hxg::vmask_fill(d.p, 1.0, o.mask(), n, s);
      hxg::vreciprocal(inv.p, d.p, n, s);
    }
    hxg::CgResult res = hxg::cg_solve(n, a, m, b, x, rtol, max_iterations, s, ph ? &dotf : nullptr);
    if (report) {
      report->iterations = res.iterations;
      report->converged = res.converged ? 1 : 0;
      report->eig_min = res.eig_min;
      report->eig_max = res.eig_max;
      report->initial_natural_norm = res.history.empty() ? 0.0 : res.history.front();
      report->final_natural_norm = res.history.empty() ? 0.0 : res.history.back();
    }
    if (history)
      for (int i = 0; i < cap && i < (int)res.history.size(); ++i) history[i] = res.history[(size_t)i];
  });
}

int hxg_lambda_max_jacobi(hxg_op_t op, int iterations, double* out) {
  return guarded([&] {
    auto& o = OP(op);
    long long n = o.size();
    cudaStream_t s = o.stream();
    hxg::DevBuf<double> d((size_t)n), inv((size_t)n);
    o.extract_diagonal(d.p);
    hxg::vreciprocal(inv.p, d.p, n, s);
    auto seed_h = hxg::rough_seed(n, o.mask_host());
    hxg::DevBuf<double> seed;
    seed.upload(seed_h);
    *out = hxg::estimate_lambda_max(
        n, [&o](const double* x, double* y) { o.apply_jacobian(x, y); }, inv.p, seed.p, iterations,
        s);
  });
}

int hxg_dot(const double* x, const double* y, int64_t n, void* stream, double* out) {
  return guarded([&] {
    hxg::DotWorkspace ws;
    *out = hxg::dot(x, y, n, ws, (cudaStream_t)stream);
  });
}

// ---- communicators ---------------------------------------------------------
int hxg_comm_create(int rank, int world, const hxg_comm_ops* ops, hxg_comm_t* out) {
  return guarded([&] {
    if (!ops || rank < 0 || rank >= world)
      throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "bad communicator arguments");
    auto* c = new hxg_comm_s();
    c->c = std::make_unique<hxg::Comm>(rank, world, *ops);
    *out = c;
  });
}
int hxg_nccl_unique_id(void* id128) { return guarded([&] { hxg::nccl_unique_id(id128); }); }
int hxg_comm_create_nccl(int rank, int world, const void* id128, hxg_comm_t* out) {
  return guarded([&] {
    auto* c = new hxg_comm_s();
    c->c = hxg::make_nccl_comm(rank, world, id128);
    *out = c;
  });
}
int hxg_comm_destroy(hxg_comm_t c) {
  delete c;
  return HXG_OK;
}
int hxg_partition_block(const int global_cells[3], const int dims[3], int rank, int cells[3],
                        int e0[3]) {
  return guarded([&] {
    const int world = dims[0] * dims[1] * dims[2];
    if (rank < 0 || rank >= world) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "rank outside the partition");
    const int coords[3] = {rank % dims[0], (rank / dims[0]) % dims[1], rank / (dims[0] * dims[1])};
    for (int d = 0; d < 3; ++d) {
      const int base = global_cells[d] / dims[d], extra = global_cells[d] % dims[d];
      if (base < 1) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "more blocks than element layers");
      cells[d] = base + (coords[d] < extra ? 1 : 0);
      e0[d] = coords[d] * base + (coords[d] < extra ? coords[d] : extra);
    }
  });
}
int hxg_stream_synchronize(void* stream) {
  return guarded([&] { HXG_CUDA(cudaStreamSynchronize((cudaStream_t)stream)); });
}

int hxg_malloc(void** p, size_t bytes) { return guarded([&] { HXG_CUDA(cudaMalloc(p, bytes)); }); }
int hxg_free(void* p) { return guarded([&] { HXG_CUDA(cudaFree(p)); }); }
int hxg_pointer_is_device(const void* p, int* is_device) {
  return guarded([&] {
    cudaPointerAttributes a{};
    HXG_CUDA(cudaPointerGetAttributes(&a, p));
    *is_device = a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
  });
}
// Host-staged copies (caller communicators, the C++ wrapper's host spans):
// ordered after earlier work like cudaMemcpy on the legacy default stream,
// and complete on return -- a pageable H2D cudaMemcpy may return before its
// DMA lands, and the library's side stream (overlapped exchange) is
// non-blocking, so the H2D also waits for the legacy stream.
int hxg_memcpy_h2d(void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    HXG_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    HXG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
  });
}
int hxg_memcpy_d2h(void* dst, const void* src, size_t bytes) {
  return guarded([&] { HXG_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)); });
}
int hxg_device_synchronize(void) { return guarded([&] { HXG_CUDA(cudaDeviceSynchronize()); }); }

// ---- host setup ------------------------------------------------------------

int hxg_setup_basis(int p, int q, double* nodes, double* points, double* weights, double* interp,
                    double* deriv, double* pinv, double* colloc) {
  return guarded([&] {
    hxg::Basis b = hxg::build_basis(p, q);
    auto cp = [](double* dst, const std::vector<double>& v) {
      if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(nodes, b.nodes);
    cp(points, b.rule.points);
    cp(weights, b.rule.weights);
    cp(interp, b.interp);
    cp(deriv, b.deriv);
    cp(pinv, b.pinv);
    cp(colloc, b.colloc);
  });
}

int hxg_setup_geometry(const double extents[3], const int cells[3], int p, int q, double* dxidX,
                       double* weight) {
  return guarded([&] {
    hxg::Basis b = hxg::build_basis(p, q);
    std::vector<double> dx, w;
    hxg::geometry(extents, cells, p, b, dx, w);
    std::memcpy(dxidX, dx.data(), dx.size() * sizeof(double));
    std::memcpy(weight, w.data(), w.size() * sizeof(double));
  });
}

int hxg_setup_constraints(const int cells[3], int p, int fixed_face_mask, uint8_t* mask) {
  return guarded([&] {
    std::vector<uint8_t> m;
    hxg::face_mask(cells, p, fixed_face_mask, m);
    std::memcpy(mask, m.data(), m.size());
  });
}

int hxg_setup_traction_load(const double extents[3], const int cells[3], int p, int q, int face,
                            const double traction[3], double* load) {
  return guarded([&] {
    hxg::Basis b = hxg::build_basis(p, q);
    std::vector<double> l;
    hxg::traction_load(extents, cells, p, b, face, traction, l);
    std::memcpy(load, l.data(), l.size() * sizeof(double));
  });
}

}  // extern "C"

/* Standalone coarse Cholesky on a Q1 lattice matrix (the replicated coarse
 * solve of the distributed p-MG). */
int hxg_chol_create(int n, const int* row_ptr, const int* cols, const int npd[3], int mode,
                    hxg_chol_t* out) {
  return guarded([&] {
    if (!out || n <= 0 || !row_ptr || !cols || !npd)
      throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "hxg_chol_create: bad arguments");
    if ((long long)npd[0] * npd[1] * npd[2] * 3 != n)
      throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "hxg_chol_create: n != 3 * nodes(npd)");
    auto h = std::make_unique<hxg_chol_s>();
    h->a.n = n;
    h->a.row_ptr_h.assign(row_ptr, row_ptr + n + 1);
    h->a.cols_h.assign(cols, cols + row_ptr[n]);
    std::vector<int> rows((size_t)row_ptr[n]);
    for (int i = 0; i < n; ++i)
      for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) rows[(size_t)k] = i;
    h->a.row_ptr.upload(h->a.row_ptr_h);
    h->a.cols.upload(h->a.cols_h);
    h->a.rows.upload(rows);
    h->a.vals.alloc((size_t)row_ptr[n]);
    for (int d = 0; d < 3; ++d) h->npd[d] = npd[d];
    if (mode < 0 || mode > 2)
      throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "coarse Cholesky mode must be 0, 1 or 2");
    h->solver.set_mode(mode);
    *out = h.release();
  });
}
int hxg_chol_factorize(hxg_chol_t h, const double* vals_host) {
  return guarded([&] {
    if (!h) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "null Cholesky handle");
    HXG_CUDA(cudaMemcpy(h->a.vals.p, vals_host, sizeof(double) * h->a.cols_h.size(),
                        cudaMemcpyHostToDevice));
    // a pageable H2D copy may return before its DMA lands; the handle's
    // stream may be non-blocking
    HXG_CUDA(cudaDeviceSynchronize());
    h->solver.factorize(h->a, h->npd, h->stream);
  });
}
int hxg_chol_factorize_device(hxg_chol_t h, const double* vals_dev) {
  return guarded([&] {
    if (!h) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "null Cholesky handle");
    // The producer of vals_dev may be on any stream: wait for the device
    // (a setup-time call), then copy on the handle's stream.
    HXG_CUDA(cudaDeviceSynchronize());
    HXG_CUDA(cudaMemcpyAsync(h->a.vals.p, vals_dev, sizeof(double) * h->a.cols_h.size(),
                             cudaMemcpyDeviceToDevice, h->stream));
    h->solver.factorize(h->a, h->npd, h->stream);
  });
}
int hxg_chol_solve(hxg_chol_t h, const double* b, double* x) {
  return guarded([&] {
    if (!h) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "null Cholesky handle");
    h->solver.solve(b, x, h->stream);
  });
}
int hxg_chol_destroy(hxg_chol_t h) {
  return guarded([&] { delete h; });
}

struct hxg_asm_s {
  hxg::Operator* op;
  std::unique_ptr<hxg::CoarseAssembly> a;
};

int hxg_asm_create(hxg_op_t op, hxg_asm_t* out) {
  return guarded([&] {
    auto* h = new hxg_asm_s();
    h->op = &OP(op);
    h->a = std::make_unique<hxg::CoarseAssembly>(OP(op));
    *out = h;
  });
}
int hxg_asm_numeric(hxg_asm_t a) {
  return guarded([&] {
    a->a->numeric(*a->op);
    HXG_CUDA(cudaStreamSynchronize(a->op->stream()));
  });
}
int hxg_asm_nnz(hxg_asm_t a, int64_t* nnz) {
  return guarded([&] { *nnz = a->a->matrix().nnz(); });
}
int hxg_asm_matvec(hxg_asm_t a, const double* x, double* y) {
  return guarded([&] { a->a->matvec(x, y, a->op->stream()); });
}
int hxg_asm_csr_host(hxg_asm_t a, int* row_ptr, int* cols, double* vals) {
  return guarded([&] {
    const auto& m = a->a->matrix();
    if (row_ptr) std::memcpy(row_ptr, m.row_ptr_h.data(), sizeof(int) * m.row_ptr_h.size());
    if (cols) std::memcpy(cols, m.cols_h.data(), sizeof(int) * m.cols_h.size());
    if (vals) {
      HXG_CUDA(cudaStreamSynchronize(a->op->stream()));
      HXG_CUDA(cudaMemcpy(vals, m.vals.p, sizeof(double) * m.cols_h.size(), cudaMemcpyDeviceToHost));
    }
  });
}
int hxg_asm_destroy(hxg_asm_t a) {
  return guarded([&] { delete a; });
}

namespace {
hxg::NewtonConfig to_config(const hxg_newton_config* c) {
  hxg::NewtonConfig nc;
  if (c) {
    nc.max_iterations = c->max_iterations;
    nc.rtol = c->rtol;
    nc.atol = c->atol;
    nc.linear_rtol = c->linear_rtol;
    nc.linear_max_iterations = c->linear_max_iterations;
    nc.use_line_search = c->use_line_search != 0;
    nc.load_steps = c->load_steps;
    nc.reference_line_search_quirk = c->reference_line_search_quirk != 0;
    nc.solver = c->solver;
    nc.lbfgs_memory = c->lbfgs_memory;
    nc.precond_refresh = c->precond_refresh;
  }
  return nc;
}
void fill_report(const std::vector<hxg::SolveReport>& steps, bool converged,
                 hxg_solve_report* rep, hxg_iteration_record* recs, int cap) {
  if (!rep) return;
  *rep = hxg_solve_report{};
  rep->converged = converged ? 1 : 0;
  rep->load_steps_taken = (int)steps.size();
  int k = 0;
  for (const auto& s : steps) {
    rep->newton_iterations += s.iterations;
    rep->cg_iterations += s.total_cg_iterations;
    rep->final_fnorm = s.final_fnorm;
    for (const auto& r : s.records) {
      if (recs && k < cap)
        recs[k++] = hxg_iteration_record{r.load_step, r.time, r.iteration, r.fnorm, r.fnorm_rel,
                                         r.cg_iterations, r.cg_converged ? 1 : 0,
                                         r.condition_estimate, r.alpha};
    }
  }
  rep->num_records = k;
}
}  // namespace

int hxg_newton_config_default(hxg_newton_config* cfg) {
  return guarded([&] {
    if (!cfg) throw hxg::Error(HXG_ERR_INVALID_ARGUMENT, "null config");
    hxg::NewtonConfig d;
    *cfg = hxg_newton_config{d.max_iterations, d.rtol, d.atol, d.linear_rtol,
                             d.linear_max_iterations, d.use_line_search ? 1 : 0, d.load_steps,
                             d.reference_line_search_quirk ? 1 : 0, d.solver, d.lbfgs_memory,
                             d.precond_refresh};
  });
}

int hxg_newton_solve(hxg_op_t op, hxg_mg_t mg, const hxg_newton_config* cfg, double* u,
                     int load_step, double time, hxg_solve_report* report,
                     hxg_iteration_record* records, int capacity) {
  return guarded([&] {
    auto r = hxg::newton_solve(OP(op), MG(mg), to_config(cfg), u, load_step, time);
    const bool conv = r.converged;
    fill_report({r}, conv, report, records, capacity);
  });
}

int hxg_lbfgs_solve(hxg_op_t op, hxg_mg_t mg, const hxg_newton_config* cfg, double* u,
                    int load_step, double time, hxg_solve_report* report,
                    hxg_iteration_record* records, int capacity) {
  return guarded([&] {
    auto r = hxg::lbfgs_solve(OP(op), MG(mg), to_config(cfg), u, load_step, time);
    const bool conv = r.converged;
    fill_report({r}, conv, report, records, capacity);
  });
}

int hxg_solve_continuation(hxg_op_t op, hxg_mg_t mg, const hxg_newton_config* cfg, double* u,
                           int max_bisections, hxg_solve_report* report,
                           hxg_iteration_record* records, int capacity) {
  return guarded([&] {
    auto steps = hxg::solve_continuation(OP(op), MG(mg), to_config(cfg), u, max_bisections, nullptr);
    fill_report(steps, true, report, records, capacity);
  });
}
