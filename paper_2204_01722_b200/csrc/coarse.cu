#include "coarse.hpp"

#include <cusolverDn.h>

#include <algorithm>

#include "dispatch.hpp"

namespace hxg {

namespace {

// Per-slot value: sum over the elements shared by the row and column nodes,
// ascending element index (the reference COO entry order, assembly.hpp:121-130).
__global__ void fill_csr_kernel(BoxDev box, const int* __restrict__ rows,
                                const int* __restrict__ cols, const uint8_t* __restrict__ mask,
                                const double* __restrict__ elem, long long nnz, double* vals) {
  constexpr int N = 2, N3 = 8, M = 24;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nnz;
       s += (long long)gridDim.x * blockDim.x) {
    int r = rows[s], c = cols[s];
    if (mask[r] || mask[c]) {
      vals[s] = (r == c) ? 1.0 : 0.0;  // identity tail for constrained DoFs
      continue;
    }
    long long nr = r / 3, nc = c / 3;
    int ca = r % 3, cb = c % 3;
    int g[3] = {(int)(nr % box.npd[0]), (int)((nr / box.npd[0]) % box.npd[1]),
                (int)(nr / ((long long)box.npd[0] * box.npd[1]))};
    int h[3] = {(int)(nc % box.npd[0]), (int)((nc / box.npd[0]) % box.npd[1]),
                (int)(nc / ((long long)box.npd[0] * box.npd[1]))};
    int lo[3], hi[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = max(max(g[d], h[d]) - 1, 0);
      hi[d] = min(min(g[d], h[d]), box.cells[d] - 1);
    }
    double acc = 0.0;
    for (int ez = lo[2]; ez <= hi[2]; ++ez)
      for (int ey = lo[1]; ey <= hi[1]; ++ey)
        for (int ex = lo[0]; ex <= hi[0]; ++ex) {
          long long e = ex + box.cells[0] * (ey + (long long)box.cells[1] * ez);
          int a = (g[0] - ex) + N * ((g[1] - ey) + N * (g[2] - ez));
          int b = (h[0] - ex) + N * ((h[1] - ey) + N * (h[2] - ez));
          acc += elem[e * (M * M) + (a * 3 + ca) * M + b * 3 + cb];
        }
    (void)N3;
    vals[s] = acc;
  }
}

__global__ void csr_to_dense_kernel(const int* rows, const int* cols, const double* vals,
                                    long long nnz, int n, double* dense) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nnz;
       s += (long long)gridDim.x * blockDim.x)
    dense[(size_t)cols[s] * n + rows[s]] = vals[s];
}

}  // namespace

CoarseAssembly::CoarseAssembly(const Operator& op) {
  if (op.p() != 1) throw Error(HXG_ERR_UNSUPPORTED, "coarse assembly expects the p = 1 level");
  box_ = op.box();
  const auto& mask = op.mask_host();
  long long nn = box_.num_nodes();
  int n = (int)(3 * nn);
  a_.n = n;
  auto fixed = [&](long long dof) { return !mask.empty() && mask[(size_t)dof] != 0; };
  a_.row_ptr_h.assign((size_t)n + 1, 0);
  a_.cols_h.clear();
  a_.cols_h.reserve((size_t)n * 81);
  std::vector<int> rows;
  rows.reserve((size_t)n * 81);
  for (long long node = 0; node < nn; ++node) {
    int g[3] = {(int)(node % box_.npd[0]), (int)((node / box_.npd[0]) % box_.npd[1]),
                (int)(node / ((long long)box_.npd[0] * box_.npd[1]))};
    for (int ca = 0; ca < 3; ++ca) {
      long long r = 3 * node + ca;
      if (fixed(r)) {
        a_.cols_h.push_back((int)r);
        rows.push_back((int)r);
      } else {
        for (int dz = -1; dz <= 1; ++dz)
          for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
              int h[3] = {g[0] + dx, g[1] + dy, g[2] + dz};
              bool ok = true;
              for (int d = 0; d < 3; ++d) ok = ok && h[d] >= 0 && h[d] < box_.npd[d];
              if (!ok) continue;
              long long nb = h[0] + box_.npd[0] * (h[1] + (long long)box_.npd[1] * h[2]);
              for (int cb = 0; cb < 3; ++cb) {
                long long c = 3 * nb + cb;
                if (fixed(c)) continue;
                a_.cols_h.push_back((int)c);
                rows.push_back((int)r);
              }
            }
      }
      a_.row_ptr_h[(size_t)r + 1] = (int)a_.cols_h.size();
    }
  }
  a_.row_ptr.upload(a_.row_ptr_h);
  a_.cols.upload(a_.cols_h);
  a_.rows.upload(rows);
  a_.vals.alloc(a_.cols_h.size());
  if (!mask.empty()) {
    mask_.upload(mask);
  } else {
    std::vector<uint8_t> z((size_t)n, 0);
    mask_.upload(z);
  }
}

void CoarseAssembly::numeric(Operator& op) {
  size_t need = (size_t)op.num_elements() * 24 * 24;
  if (elem_.n != need) elem_.alloc(need);
  op.element_matrices(elem_.p);
  long long nnz = a_.nnz();
  fill_csr_kernel<<<grid_for(nnz, 256), 256, 0, op.stream()>>>(box_, a_.rows.p, a_.cols.p, mask_.p,
                                                                 elem_.p, nnz, a_.vals.p);
  HXG_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Dense device Cholesky for coarse levels that fit (cuSOLVER potrf/potrs).

class CoarseSolverImpl {
 public:
  ~CoarseSolverImpl() {
    if (handle_) cusolverDnDestroy(handle_);
  }
  void factorize(const CsrMatrix& a, cudaStream_t s) {
    n_ = a.n;
    size_t bytes = (size_t)n_ * n_ * sizeof(double);
    if (bytes > (size_t)48 << 30)
      throw Error(HXG_ERR_UNSUPPORTED, "coarse problem too large for the dense factorization");
    if (!handle_) {
      if (cusolverDnCreate(&handle_) != CUSOLVER_STATUS_SUCCESS)
        throw Error(HXG_ERR_CUDA, "cusolverDnCreate failed");
    }
    cusolverDnSetStream(handle_, s);
    if (dense_.n != (size_t)n_ * n_) dense_.alloc((size_t)n_ * n_);
    HXG_CUDA(cudaMemsetAsync(dense_.p, 0, bytes, s));
    csr_to_dense_kernel<<<grid_for(a.nnz(), 256), 256, 0, s>>>(a.rows.p, a.cols.p, a.vals.p,
                                                              a.nnz(), n_, dense_.p);
    HXG_CUDA(cudaGetLastError());
    int lwork = 0;
    if (cusolverDnDpotrf_bufferSize(handle_, CUBLAS_FILL_MODE_LOWER, n_, dense_.p, n_, &lwork) !=
        CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "potrf_bufferSize failed");
    if (work_.n < (size_t)lwork) work_.alloc((size_t)lwork);
    if (info_.n == 0) info_.alloc(1);
    if (cusolverDnDpotrf(handle_, CUBLAS_FILL_MODE_LOWER, n_, dense_.p, n_, work_.p, lwork,
                         info_.p) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "potrf failed");
    int info = 0;
    HXG_CUDA(cudaMemcpyAsync(&info, info_.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    HXG_CUDA(cudaStreamSynchronize(s));
    if (info != 0) {
      ready_ = false;
      throw Error(HXG_ERR_NOT_SPD, "factorization failed, matrix not SPD: coarse Cholesky "
                                   "factorization failed at level 0");
    }
    ready_ = true;
  }
  void solve(const double* b, double* x, cudaStream_t s) {
    if (!ready_) throw Error(HXG_ERR_GENERIC, "coarse solver not factorized");
    if (x != b) HXG_CUDA(cudaMemcpyAsync(x, b, sizeof(double) * n_, cudaMemcpyDeviceToDevice, s));
    cusolverDnSetStream(handle_, s);
    if (cusolverDnDpotrs(handle_, CUBLAS_FILL_MODE_LOWER, n_, 1, dense_.p, n_, x, n_, info_.p) !=
        CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "potrs failed");
  }
  bool ready() const { return ready_; }

 private:
  cusolverDnHandle_t handle_ = nullptr;
  int n_ = 0;
  bool ready_ = false;
  DevBuf<double> dense_, work_;
  DevBuf<int> info_;
};

CoarseSolver::CoarseSolver() : impl_(new CoarseSolverImpl()) {}
CoarseSolver::~CoarseSolver() = default;
void CoarseSolver::factorize(const CsrMatrix& a, const int[3], cudaStream_t s) {
  impl_->factorize(a, s);
}
void CoarseSolver::solve(const double* b, double* x, cudaStream_t s) { impl_->solve(b, x, s); }
bool CoarseSolver::ready() const { return impl_->ready(); }

}  // namespace hxg
