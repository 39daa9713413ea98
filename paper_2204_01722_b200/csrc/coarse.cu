#include "coarse.hpp"

#include <cusolverDn.h>
#include <cusolverSp.h>
#include <cusolverSp_LOWLEVEL_PREVIEW.h>
#include <cusparse.h>

#include <algorithm>

#include "dispatch.hpp"
#include "ndchol.hpp"
#include "solver.hpp"

namespace hxg {

namespace {

// Elements containing node coordinate g along one axis (order P, c cells).
__host__ __device__ inline void node_elems(int g, int P, int c, int& lo, int& hi) {
  lo = g > 0 ? (g - 1) / P : 0;
  hi = g / P < c - 1 ? g / P : c - 1;
}

// Per-slot value: sum over the elements shared by the row and column nodes,
// ascending element index (the reference COO entry order, assembly.hpp:121-130).
template <int P>
__global__ void fill_csr_kernel(BoxDev box, const int* __restrict__ rows,
                                const int* __restrict__ cols, const uint8_t* __restrict__ mask,
                                const double* __restrict__ elem, long long nnz, double* vals) {
  constexpr int N = P + 1, M = 3 * N * N * N;
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
      int l1, h1, l2, h2;
      node_elems(g[d], P, box.cells[d], l1, h1);
      node_elems(h[d], P, box.cells[d], l2, h2);
      lo[d] = max(l1, l2);
      hi[d] = min(h1, h2);
    }
    double acc = 0.0;
    for (int ez = lo[2]; ez <= hi[2]; ++ez)
      for (int ey = lo[1]; ey <= hi[1]; ++ey)
        for (int ex = lo[0]; ex <= hi[0]; ++ex) {
          long long e = ex + box.cells[0] * (ey + (long long)box.cells[1] * ez);
          int a = (g[0] - P * ex) + N * ((g[1] - P * ey) + N * (g[2] - P * ez));
          int b = (h[0] - P * ex) + N * ((h[1] - P * ey) + N * (h[2] - P * ez));
          acc += elem[e * (M * M) + (a * 3 + ca) * M + b * 3 + cb];
        }
    vals[s] = acc;
  }
}

// CsrMatrix::matvec (assembly.hpp): one warp per row, lanes over the row's
// slots, fixed-order shuffle reduction.
__global__ void csr_matvec_kernel(int n, const int* __restrict__ row_ptr,
                                  const int* __restrict__ cols, const double* __restrict__ vals,
                                  const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    double acc = 0.0;
    for (int s = row_ptr[r] + lane; s < row_ptr[r + 1]; s += 32) acc += vals[s] * __ldg(x + cols[s]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) y[r] = acc;
  }
}

__global__ void csr_to_dense_kernel(const int* rows, const int* cols, const double* vals,
                                    long long nnz, int n, double* dense) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nnz;
       s += (long long)gridDim.x * blockDim.x)
    dense[(size_t)cols[s] * n + rows[s]] = vals[s];
}

}  // namespace

CoarseAssembly::CoarseAssembly(const Operator& op) : CoarseAssembly(op.box(), op.mask_host()) {}

CoarseAssembly::CoarseAssembly(const BoxDev& box, const std::vector<uint8_t>& mask) {
  box_ = box;
  const int P = box.p;
  long long nn = box_.num_nodes();
  if (3 * nn > 0x7fffffffLL) throw Error(HXG_ERR_UNSUPPORTED, "assembled operator exceeds int32 rows");
  int n = (int)(3 * nn);
  a_.n = n;
  auto fixed = [&](long long dof) { return !mask.empty() && mask[(size_t)dof] != 0; };
  // Unconstrained pattern size, separable over the axes: 9 prod_d sum_g
  // (nodes coupled to g along d); refuse int32 overflow before allocating.
  double bound = 9.0;
  for (int d = 0; d < 3; ++d) {
    double sum = 0.0;
    for (int g = 0; g < box_.npd[d]; ++g) {
      int el, eh;
      node_elems(g, P, box_.cells[d], el, eh);
      sum += P * (eh + 1) - P * el + 1;
    }
    bound *= sum;
  }
  // (constraints only remove entries: past twice the limit no mask brings it back)
  if (bound > (mask.empty() ? 1.0 : 2.0) * 2147483647.0)
    throw Error(HXG_ERR_UNSUPPORTED, "assembled operator exceeds int32 nonzeros");
  const long long per_row = 3LL * (2 * P + 1) * (2 * P + 1) * (2 * P + 1);
  a_.row_ptr_h.assign((size_t)n + 1, 0);
  a_.cols_h.clear();
  a_.cols_h.reserve((size_t)std::min<long long>((long long)n * per_row, 1LL << 31));
  std::vector<int> rows;
  rows.reserve(a_.cols_h.capacity());
  for (long long node = 0; node < nn; ++node) {
    int g[3] = {(int)(node % box_.npd[0]), (int)((node / box_.npd[0]) % box_.npd[1]),
                (int)(node / ((long long)box_.npd[0] * box_.npd[1]))};
    int lo[3], hi[3];  // node range of the elements containing the node
    for (int d = 0; d < 3; ++d) {
      int el, eh;
      node_elems(g[d], P, box_.cells[d], el, eh);
      lo[d] = P * el;
      hi[d] = P * (eh + 1);
    }
    for (int ca = 0; ca < 3; ++ca) {
      long long r = 3 * node + ca;
      if (fixed(r)) {
        a_.cols_h.push_back((int)r);
        rows.push_back((int)r);
      } else {
        for (int hz = lo[2]; hz <= hi[2]; ++hz)
          for (int hy = lo[1]; hy <= hi[1]; ++hy)
            for (int hx = lo[0]; hx <= hi[0]; ++hx) {
              long long nb = hx + box_.npd[0] * (hy + (long long)box_.npd[1] * hz);
              for (int cb = 0; cb < 3; ++cb) {
                long long c = 3 * nb + cb;
                if (fixed(c)) continue;
                a_.cols_h.push_back((int)c);
                rows.push_back((int)r);
              }
            }
      }
      if (a_.cols_h.size() > 0x7fffffffULL)
        throw Error(HXG_ERR_UNSUPPORTED, "assembled operator exceeds int32 nonzeros");
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
  dispatch_p(op.p(), [&](auto Pc) {
    constexpr int P = decltype(Pc)::value, M = 3 * (P + 1) * (P + 1) * (P + 1);
    size_t need = (size_t)op.num_elements() * M * M;
    if (elem_.n != need) elem_.alloc(need);
    PhaseTimer pt(op.stream());
    op.element_matrices(elem_.p);
    pt.mark("  element matrices");
    long long nnz = a_.nnz();
    fill_csr_kernel<P><<<grid_for(nnz, 256), 256, 0, op.stream()>>>(box_, a_.rows.p, a_.cols.p,
                                                                     mask_.p, elem_.p, nnz, a_.vals.p);
    pt.mark("  slot sums (fill csr)");
  });
  HXG_CUDA(cudaGetLastError());
}

void CoarseAssembly::numeric_from_elements(const double* elem, cudaStream_t s) {
  dispatch_p(box_.p, [&](auto Pc) {
    constexpr int P = decltype(Pc)::value;
    long long nnz = a_.nnz();
    fill_csr_kernel<P><<<grid_for(nnz, 256), 256, 0, s>>>(box_, a_.rows.p, a_.cols.p, mask_.p, elem,
                                                          nnz, a_.vals.p);
  });
  HXG_CUDA(cudaGetLastError());
}

void csr_matvec(const CsrMatrix& a, const double* x, double* y, cudaStream_t s) {
  csr_matvec_kernel<<<grid_for((long long)a.n * 32, 256), 256, 0, s>>>(a.n, a.row_ptr.p, a.cols.p,
                                                                       a.vals.p, x, y);
  HXG_CUDA(cudaGetLastError());
}

void CoarseAssembly::matvec(const double* x, double* y, cudaStream_t s) const { csr_matvec(a_, x, y, s); }

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

// ---------------------------------------------------------------------------
// Sparse device Cholesky for larger coarse levels: geometric nested dissection
// of the Q1 node lattice (host, once per pattern), the permuted CSR refilled
// on device by a gather, and cuSOLVER's device csrchol (symbolic once,
// numeric per setup, triangular solves per V-cycle).

namespace {

// Nested-dissection order (new -> old) of the nx x ny x nz node lattice:
// split the longest axis at its middle plane; order left, right, separator.
void nd_nodes(const int npd[3], int lo0, int hi0, int lo1, int hi1, int lo2, int hi2,
              std::vector<int>& order) {
  const int n[3] = {hi0 - lo0, hi1 - lo1, hi2 - lo2};
  if (n[0] <= 0 || n[1] <= 0 || n[2] <= 0) return;
  const long long cnt = (long long)n[0] * n[1] * n[2];
  int ax = 0;
  if (n[1] > n[ax]) ax = 1;
  if (n[2] > n[ax]) ax = 2;
  if (cnt <= 64 || n[ax] < 3) {
    for (int z = lo2; z < hi2; ++z)
      for (int y = lo1; y < hi1; ++y)
        for (int x = lo0; x < hi0; ++x) order.push_back(x + npd[0] * (y + npd[1] * z));
    return;
  }
  int lo[3] = {lo0, lo1, lo2}, hi[3] = {hi0, hi1, hi2};
  const int mid = lo[ax] + n[ax] / 2;
  int a_hi[3] = {hi[0], hi[1], hi[2]}, b_lo[3] = {lo[0], lo[1], lo[2]};
  a_hi[ax] = mid;
  b_lo[ax] = mid + 1;
  nd_nodes(npd, lo[0], a_hi[0], lo[1], a_hi[1], lo[2], a_hi[2], order);
  nd_nodes(npd, b_lo[0], hi[0], b_lo[1], hi[1], b_lo[2], hi[2], order);
  int s_lo[3] = {lo[0], lo[1], lo[2]}, s_hi[3] = {hi[0], hi[1], hi[2]};
  s_lo[ax] = mid;
  s_hi[ax] = mid + 1;
  for (int z = s_lo[2]; z < s_hi[2]; ++z)
    for (int y = s_lo[1]; y < s_hi[1]; ++y)
      for (int x = s_lo[0]; x < s_hi[0]; ++x) order.push_back(x + npd[0] * (y + npd[1] * z));
}

__global__ void gather_kernel(const double* __restrict__ src, const int* __restrict__ idx,
                              long long n, double* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}

__global__ void scatter_kernel(const double* __restrict__ src, const int* __restrict__ idx,
                               long long n, double* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[idx[i]] = src[i];
}

}  // namespace

class SparseCholeskyImpl {
 public:
  ~SparseCholeskyImpl() {
    if (info_) cusolverSpDestroyCsrcholInfo(info_);
    if (descr_) cusparseDestroyMatDescr(descr_);
    if (handle_) cusolverSpDestroy(handle_);
  }
  void factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s) {
    if (!handle_) {
      if (cusolverSpCreate(&handle_) != CUSOLVER_STATUS_SUCCESS)
        throw Error(HXG_ERR_CUDA, "cusolverSpCreate failed");
      cusparseCreateMatDescr(&descr_);
      cusparseSetMatType(descr_, CUSPARSE_MATRIX_TYPE_GENERAL);
      cusparseSetMatIndexBase(descr_, CUSPARSE_INDEX_BASE_ZERO);
    }
    cusolverSpSetStream(handle_, s);
    if (!analyzed_) analyze(a, npd);
    const long long nnz = a.nnz();
    gather_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(a.vals.p, slot_.p, nnz, pvals_.p);
    HXG_CUDA(cudaGetLastError());
    if (cusolverSpDcsrcholFactor(handle_, n_, (int)nnz, descr_, pvals_.p, prow_.p, pcol_.p,
                                 info_, buffer_.p) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "csrcholFactor failed");
    int pos = -1;
    if (cusolverSpDcsrcholZeroPivot(handle_, info_, 0.0, &pos) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "csrcholZeroPivot failed");
    if (pos >= 0) {
      ready_ = false;
      throw Error(HXG_ERR_NOT_SPD, "factorization failed, matrix not SPD: coarse Cholesky "
                                   "factorization failed at level 0");
    }
    ready_ = true;
  }
  void solve(const double* b, double* x, cudaStream_t s) {
    if (!ready_) throw Error(HXG_ERR_GENERIC, "coarse solver not factorized");
    cusolverSpSetStream(handle_, s);
    gather_kernel<<<grid_for(n_, 256), 256, 0, s>>>(b, perm_.p, n_, pb_.p);
    if (cusolverSpDcsrcholSolve(handle_, n_, pb_.p, px_.p, info_, buffer_.p) !=
        CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "csrcholSolve failed");
    scatter_kernel<<<grid_for(n_, 256), 256, 0, s>>>(px_.p, perm_.p, n_, x);
    HXG_CUDA(cudaGetLastError());
  }
  bool ready() const { return ready_; }

 private:
  void analyze(const CsrMatrix& a, const int npd[3]) {
    n_ = a.n;
    std::vector<int> nodes;
    nodes.reserve((size_t)n_ / 3);
    nd_nodes(npd, 0, npd[0], 0, npd[1], 0, npd[2], nodes);
    if ((long long)nodes.size() * 3 != n_) throw Error(HXG_ERR_GENERIC, "ND ordering incomplete");
    std::vector<int> perm((size_t)n_), inv((size_t)n_);
    for (size_t k = 0; k < nodes.size(); ++k)
      for (int c = 0; c < 3; ++c) perm[3 * k + c] = 3 * nodes[k] + c;
    for (int i = 0; i < n_; ++i) inv[(size_t)perm[(size_t)i]] = i;
    // Permuted CSR: new row i = old row perm[i], columns mapped by inv, sorted.
    std::vector<int> prow((size_t)n_ + 1, 0), pcol, slot;
    pcol.reserve(a.cols_h.size());
    slot.reserve(a.cols_h.size());
    std::vector<std::pair<int, int>> tmp;
    for (int i = 0; i < n_; ++i) {
      int r = perm[(size_t)i];
      tmp.clear();
      for (int k = a.row_ptr_h[(size_t)r]; k < a.row_ptr_h[(size_t)r + 1]; ++k)
        tmp.emplace_back(inv[(size_t)a.cols_h[(size_t)k]], k);
      std::sort(tmp.begin(), tmp.end());
      for (auto& t : tmp) {
        pcol.push_back(t.first);
        slot.push_back(t.second);
      }
      prow[(size_t)i + 1] = (int)pcol.size();
    }
    perm_.upload(perm);
    prow_.upload(prow);
    pcol_.upload(pcol);
    slot_.upload(slot);
    pvals_.alloc(pcol.size());
    pb_.alloc((size_t)n_);
    px_.alloc((size_t)n_);
    if (cusolverSpCreateCsrcholInfo(&info_) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "csrcholInfo create failed");
    if (cusolverSpXcsrcholAnalysis(handle_, n_, (int)pcol.size(), descr_, prow_.p, pcol_.p,
                                   info_) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "csrcholAnalysis failed");
    size_t internal = 0, work = 0;
    // BufferInfo needs values; a gather of the current ones gives valid data.
    gather_kernel<<<grid_for((long long)pcol.size(), 256), 256>>>(a.vals.p, slot_.p,
                                                                (long long)pcol.size(), pvals_.p);
    if (cusolverSpDcsrcholBufferInfo(handle_, n_, (int)pcol.size(), descr_, pvals_.p, prow_.p,
                                     pcol_.p, info_, &internal, &work) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "csrcholBufferInfo failed");
    buffer_.alloc(work / sizeof(double) + 1);
    analyzed_ = true;
  }

  cusolverSpHandle_t handle_ = nullptr;
  cusparseMatDescr_t descr_ = nullptr;
  csrcholInfo_t info_ = nullptr;
  bool analyzed_ = false, ready_ = false;
  int n_ = 0;
  DevBuf<int> perm_, prow_, pcol_, slot_;
  DevBuf<double> pvals_, pb_, px_, buffer_;
};

CoarseSolver::CoarseSolver() : impl_(new CoarseSolverImpl()) {}
CoarseSolver::~CoarseSolver() = default;
// Backends: 1 dense potrf, 2 nested-dissection multifrontal (ndchol.cu),
// 3 cuSOLVER csrchol on the ND-permuted matrix.  Mode 0 picks dense for
// small coarse levels and the multifrontal solver otherwise.
void CoarseSolver::factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s) {
  active_ = mode_ != 0 ? mode_ : (a.n <= kDenseCoarseMax ? 1 : 2);
  if (active_ == 1) {
    impl_->factorize(a, s);
  } else if (active_ == 2) {
    if (!nd_) nd_ = std::make_unique<NdCholesky>();
    nd_->factorize(a, npd, s);
  } else {
    if (!sparse_) sparse_ = std::make_unique<SparseCholeskyImpl>();
    sparse_->factorize(a, npd, s);
  }
}
void CoarseSolver::solve(const double* b, double* x, cudaStream_t s) {
  if (active_ == 2)
    nd_->solve(b, x, s);
  else if (active_ == 3)
    sparse_->solve(b, x, s);
  else
    impl_->solve(b, x, s);
}
bool CoarseSolver::ready() const {
  if (active_ == 2) return nd_ && nd_->ready();
  if (active_ == 3) return sparse_ && sparse_->ready();
  return impl_->ready();
}

}  // namespace hxg
