#include "coarse.hpp"


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
// Dense coarse mode: the multifrontal solver with one front holding the whole
// lattice (dense_chol_inv factor + inverse, GEMV solves; ndchol.cu).

class CoarseSolverImpl {
 public:
  void factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s) {
    if ((size_t)a.n * a.n * sizeof(double) > (size_t)48 << 30)
      throw Error(HXG_ERR_UNSUPPORTED, "coarse problem too large for the dense factorization");
    if (!nd_ || n_ != a.n) nd_ = std::make_unique<NdCholesky>((long long)npd[0] * npd[1] * npd[2] + 1);
    n_ = a.n;
    nd_->factorize(a, npd, s);
  }
  void solve(const double* b, double* x, cudaStream_t s) {
    if (!ready()) throw Error(HXG_ERR_GENERIC, "coarse solver not factorized");
    nd_->solve(b, x, s);
  }
  bool ready() const { return nd_ && nd_->ready(); }

 private:
  int n_ = 0;
  std::unique_ptr<NdCholesky> nd_;
};

CoarseSolver::CoarseSolver() : impl_(new CoarseSolverImpl()) {}
CoarseSolver::~CoarseSolver() = default;
// Backends: 1 dense (one front), 2 nested-dissection multifrontal
// (ndchol.cu).  Mode 0 picks dense for small coarse levels and the
// multifrontal solver otherwise.
void CoarseSolver::factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s) {
  active_ = mode_ != 0 ? mode_ : (a.n <= kDenseCoarseMax ? 1 : 2);
  if (active_ == 1) {
    impl_->factorize(a, npd, s);
  } else if (active_ == 2) {
    if (!nd_) nd_ = std::make_unique<NdCholesky>();
    nd_->factorize(a, npd, s);
  } else {
    throw Error(HXG_ERR_INVALID_ARGUMENT, "coarse solver mode must be 0, 1 or 2");
  }
}
void CoarseSolver::solve(const double* b, double* x, cudaStream_t s) {
  if (active_ == 2)
    nd_->solve(b, x, s);
  else
    impl_->solve(b, x, s);
}
bool CoarseSolver::ready() const {
  if (active_ == 2) return nd_ && nd_->ready();
  return impl_->ready();
}

}  // namespace hxg
