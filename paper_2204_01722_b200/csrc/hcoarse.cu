// Inexact coarse mode: one Galerkin h-multigrid V-cycle on the assembled Q1
// level (see hcoarse.hpp).  Every kernel is gather-based with fixed-order
// sums, so the cycle is bitwise reproducible run to run.
#include "hcoarse.hpp"

#include <cusolverDn.h>

#include <algorithm>

#include "dispatch.hpp"

namespace hxg {

namespace {

constexpr int M1 = 24;  // DoFs of a Q1 element (8 nodes x 3)

// Trilinear weight of coarse-local node B (0/1 along each axis) at the fine
// node of child offset ch and fine-local offset a: t = (ch + a) / 2.
__host__ __device__ inline double w1(int t2, int B) {  // t2 = 2 t in {0, 1, 2}
  return B ? 0.5 * t2 : 1.0 - 0.5 * t2;
}

// Coarse element matrices E_c = sum_children W^T (M A_f M) W (x I3), children
// in increasing (z, y, x) order.  One CTA per coarse element.
__global__ void __launch_bounds__(288) galerkin_kernel(BoxDev fbox, BoxDev cbox,
                                                       const uint8_t* __restrict__ fmask,
                                                       const double* __restrict__ felem,
                                                       double* __restrict__ celem) {
  __shared__ double Af[M1 * M1];
  __shared__ double T[M1 * M1];
  __shared__ double W[8][8];
  const long long ce = blockIdx.x;
  const int cx = (int)(ce % cbox.cells[0]), cy = (int)((ce / cbox.cells[0]) % cbox.cells[1]),
            cz = (int)(ce / ((long long)cbox.cells[0] * cbox.cells[1]));
  const int tid = threadIdx.x;
  double acc[2] = {0.0, 0.0};
  for (int ch = 0; ch < 8; ++ch) {
    const int i = ch & 1, j = (ch >> 1) & 1, k = ch >> 2;
    const int fx = 2 * cx + i, fy = 2 * cy + j, fz = 2 * cz + k;
    if (fx >= fbox.cells[0] || fy >= fbox.cells[1] || fz >= fbox.cells[2]) continue;
    const long long fe = fx + (long long)fbox.cells[0] * (fy + (long long)fbox.cells[1] * fz);
    const double* A = felem + fe * (M1 * M1);
    // masked fine element matrix: constrained fine rows / columns are zero
    for (int idx = tid; idx < M1 * M1; idx += blockDim.x) {
      const int r = idx / M1, c = idx % M1;
      auto dof = [&](int m) {
        const int a = m / 3, comp = m % 3;
        const long long node = (fx + (a & 1)) +
                               (long long)fbox.npd[0] * ((fy + ((a >> 1) & 1)) +
                                                         (long long)fbox.npd[1] * (fz + (a >> 2)));
        return 3 * node + comp;
      };
      const bool m = fmask && (fmask[dof(r)] || fmask[dof(c)]);
      Af[idx] = m ? 0.0 : A[idx];
    }
    if (tid < 64) {
      const int a = tid >> 3, B = tid & 7;
      W[a][B] = w1(i + (a & 1), B & 1) * w1(j + ((a >> 1) & 1), (B >> 1) & 1) *
                w1(k + (a >> 2), B >> 2);
    }
    __syncthreads();
    // T[r][B c] = sum_a Af[r][a c] W[a][B]
    for (int idx = tid; idx < M1 * M1; idx += blockDim.x) {
      const int r = idx / M1, Bc = idx % M1, B = Bc / 3, c = Bc % 3;
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < 8; ++a) s += Af[r * M1 + a * 3 + c] * W[a][B];
      T[idx] = s;
    }
    __syncthreads();
    // E[A c'][B c] += sum_a' W[a'][A] T[a' c'][B c]
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = tid + q * 288;
      const int Ac = idx / M1, Bc = idx % M1, Aa = Ac / 3, cp = Ac % 3;
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < 8; ++a) s += W[a][Aa] * T[(a * 3 + cp) * M1 + Bc];
      acc[q] += s;
    }
    __syncthreads();
  }
  double* E = celem + ce * (M1 * M1);
  E[tid] = acc[0];
  E[tid + 288] = acc[1];
}

// x_f += P~ x_c: fine node g takes coarse g / 2 (even) or the mean of
// (g -+ 1) / 2 (odd) along each axis; constrained fine rows and coarse
// columns are dropped.
__global__ void prolong_add_kernel(BoxDev fbox, BoxDev cbox, const uint8_t* __restrict__ fmask,
                                   const uint8_t* __restrict__ cmask, const double* __restrict__ xc,
                                   double* __restrict__ xf) {
  const long long n = 3 * fbox.num_nodes();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (fmask && fmask[i]) continue;
    const long long node = i / 3;
    const int comp = (int)(i % 3);
    const int g[3] = {(int)(node % fbox.npd[0]), (int)((node / fbox.npd[0]) % fbox.npd[1]),
                      (int)(node / ((long long)fbox.npd[0] * fbox.npd[1]))};
    int lo[3], cnt[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      lo[d] = g[d] >> 1;
      cnt[d] = (g[d] & 1) ? 2 : 1;
    }
    double s = 0.0;
    for (int z = 0; z < cnt[2]; ++z)
      for (int y = 0; y < cnt[1]; ++y)
        for (int x = 0; x < cnt[0]; ++x) {
          const long long cd =
              3 * ((lo[0] + x) + (long long)cbox.npd[0] * ((lo[1] + y) + (long long)cbox.npd[1] * (lo[2] + z))) +
              comp;
          if (cmask && cmask[cd]) continue;
          const double w = (cnt[0] == 2 ? 0.5 : 1.0) * (cnt[1] == 2 ? 0.5 : 1.0) * (cnt[2] == 2 ? 0.5 : 1.0);
          s += w * xc[cd];
        }
    xf[i] += s;
  }
}

// r_c = P~^T r_f: coarse node G gathers fine 2G (weight 1) and 2G -+ 1
// (weight 1/2) along each axis, increasing fine index.
__global__ void restrict_kernel(BoxDev fbox, BoxDev cbox, const uint8_t* __restrict__ fmask,
                                const uint8_t* __restrict__ cmask, const double* __restrict__ rf,
                                double* __restrict__ rc) {
  const long long n = 3 * cbox.num_nodes();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (cmask && cmask[i]) {
      rc[i] = 0.0;
      continue;
    }
    const long long node = i / 3;
    const int comp = (int)(i % 3);
    const int G[3] = {(int)(node % cbox.npd[0]), (int)((node / cbox.npd[0]) % cbox.npd[1]),
                      (int)(node / ((long long)cbox.npd[0] * cbox.npd[1]))};
    double s = 0.0;
    for (int dz = -1; dz <= 1; ++dz) {
      const int gz = 2 * G[2] + dz;
      if (gz < 0 || gz >= fbox.npd[2]) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int gy = 2 * G[1] + dy;
        if (gy < 0 || gy >= fbox.npd[1]) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          const int gx = 2 * G[0] + dx;
          if (gx < 0 || gx >= fbox.npd[0]) continue;
          const long long fd =
              3 * (gx + (long long)fbox.npd[0] * (gy + (long long)fbox.npd[1] * gz)) + comp;
          if (fmask && fmask[fd]) continue;
          const double w = (dx ? 0.5 : 1.0) * (dy ? 0.5 : 1.0) * (dz ? 0.5 : 1.0);
          s += w * rf[fd];
        }
      }
    }
    rc[i] = s;
  }
}

__global__ void csr_diag_kernel(int n, const int* __restrict__ row_ptr, const int* __restrict__ cols,
                                const double* __restrict__ vals, double* __restrict__ d) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int s = row_ptr[r]; s < row_ptr[r + 1]; ++s)
      if (cols[s] == r) v = vals[s];
    d[r] = v;
  }
}

__global__ void to_dense_kernel(const int* rows, const int* cols, const double* vals, long long nnz,
                                int n, double* dense) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nnz;
       s += (long long)gridDim.x * blockDim.x)
    dense[(size_t)cols[s] * n + rows[s]] = vals[s];
}

// potri leaves the lower triangle: mirror it so every row is contiguous.
__global__ void symmetrize_kernel(int n, double* a) {
  const long long total = (long long)n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(t / n), r = (int)(t % n);  // column-major (r, c)
    if (r < c) a[t] = a[(size_t)r * n + c];       // upper (r, c) = lower (c, r)
  }
}

// y = A^{-1} b with the symmetric dense inverse: warp per row (row r =
// column r, contiguous), fixed-order lane sums + shuffle tree.
__global__ void dense_symv_kernel(int n, const double* __restrict__ a, const double* __restrict__ b,
                                  double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const double* row = a + (size_t)r * n;
    double s = 0.0;
    for (int c = lane; c < n; c += 32) s += row[c] * b[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[r] = s;
  }
}

}  // namespace

// ---------------------------------------------------------------------------

DenseInverse::~DenseInverse() {
  if (handle_) cusolverDnDestroy((cusolverDnHandle_t)handle_);
}

void DenseInverse::factorize(const CsrMatrix& a, cudaStream_t s) {
  n_ = a.n;
  auto h = (cusolverDnHandle_t)handle_;
  if (!h) {
    if (cusolverDnCreate(&h) != CUSOLVER_STATUS_SUCCESS) throw Error(HXG_ERR_CUDA, "cusolverDnCreate failed");
    handle_ = h;
  }
  cusolverDnSetStream(h, s);
  const size_t nn = (size_t)n_ * n_;
  if (inv_.n != nn) inv_.alloc(nn);
  HXG_CUDA(cudaMemsetAsync(inv_.p, 0, nn * sizeof(double), s));
  to_dense_kernel<<<grid_for(a.nnz(), 256), 256, 0, s>>>(a.rows.p, a.cols.p, a.vals.p, a.nnz(), n_,
                                                         inv_.p);
  HXG_CUDA(cudaGetLastError());
  int l1 = 0, l2 = 0;
  if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n_, inv_.p, n_, &l1) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnDpotri_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n_, inv_.p, n_, &l2) != CUSOLVER_STATUS_SUCCESS)
    throw Error(HXG_ERR_CUDA, "potrf/potri bufferSize failed");
  const size_t lw = (size_t)std::max(l1, l2);
  if (work_.n < lw) work_.alloc(lw);
  if (!info_.n) info_.alloc(1);
  int info = 0;
  if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, n_, inv_.p, n_, work_.p, (int)work_.n, info_.p) !=
      CUSOLVER_STATUS_SUCCESS)
    throw Error(HXG_ERR_CUDA, "potrf failed");
  HXG_CUDA(cudaMemcpyAsync(&info, info_.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  HXG_CUDA(cudaStreamSynchronize(s));
  if (info != 0)
    throw Error(HXG_ERR_NOT_SPD, "factorization failed, matrix not SPD: h-multigrid bottom level");
  if (cusolverDnDpotri(h, CUBLAS_FILL_MODE_LOWER, n_, inv_.p, n_, work_.p, (int)work_.n, info_.p) !=
      CUSOLVER_STATUS_SUCCESS)
    throw Error(HXG_ERR_CUDA, "potri failed");
  symmetrize_kernel<<<grid_for((long long)nn, 256), 256, 0, s>>>(n_, inv_.p);
  HXG_CUDA(cudaGetLastError());
}

void DenseInverse::solve(const double* b, double* x, cudaStream_t s) const {
  dense_symv_kernel<<<grid_for((long long)n_ * 32, 256), 256, 0, s>>>(n_, inv_.p, b, x);
  HXG_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------

struct HmgCoarse::HLevel {
  BoxDev box;
  std::vector<uint8_t> mask_h;
  DevBuf<uint8_t> mask;
  const CsrMatrix* A = nullptr;
  std::unique_ptr<CoarseAssembly> asmb;  // levels >= 1
  DevBuf<double> elem;                   // levels >= 1: Galerkin element matrices
  DevBuf<double> b, x, r;
  Chebyshev smoother;
  long long n() const { return 3 * box.num_nodes(); }
  const uint8_t* m() const { return mask.n ? mask.p : nullptr; }
};

HmgCoarse::HmgCoarse() = default;
HmgCoarse::~HmgCoarse() = default;

long long HmgCoarse::level_size(int l) const { return levels_[(size_t)l]->n(); }

void HmgCoarse::setup(const CsrMatrix& a0, const BoxDev& box0, const std::vector<uint8_t>& mask0,
                      const double* elem0, cudaStream_t s) {
  if (box0.p != 1) throw Error(HXG_ERR_UNSUPPORTED, "h-multigrid coarse mode needs the p = 1 level");
  if (levels_.empty() || levels_[0]->A != &a0) {  // symbolic: lattices, masks, patterns
    levels_.clear();
    auto l0 = std::make_unique<HLevel>();
    l0->box = box0;
    l0->mask_h = mask0.empty() ? std::vector<uint8_t>((size_t)(3 * box0.num_nodes()), 0) : mask0;
    l0->mask.upload(l0->mask_h);
    l0->A = &a0;
    levels_.push_back(std::move(l0));
    for (;;) {
      HLevel& f = *levels_.back();
      const bool can = f.box.cells[0] >= 2 && f.box.cells[1] >= 2 && f.box.cells[2] >= 2;
      if (f.n() <= kHmgBottomMax || !can) break;
      auto c = std::make_unique<HLevel>();
      int cc[3];
      for (int d = 0; d < 3; ++d) cc[d] = (f.box.cells[d] + 1) / 2;
      c->box = make_box(cc, 1);
      // a coarse DoF is constrained iff every fine DoF it interpolates to is
      // (its column of P~ is zero)
      c->mask_h.assign((size_t)c->n(), 1);
      for (long long node = 0; node < c->box.num_nodes(); ++node) {
        const int G[3] = {(int)(node % c->box.npd[0]), (int)((node / c->box.npd[0]) % c->box.npd[1]),
                          (int)(node / ((long long)c->box.npd[0] * c->box.npd[1]))};
        for (int comp = 0; comp < 3; ++comp) {
          bool all = true;
          for (int dz = -1; dz <= 1 && all; ++dz)
            for (int dy = -1; dy <= 1 && all; ++dy)
              for (int dx = -1; dx <= 1 && all; ++dx) {
                const int g[3] = {2 * G[0] + dx, 2 * G[1] + dy, 2 * G[2] + dz};
                bool in = true;
                for (int d = 0; d < 3; ++d) in = in && g[d] >= 0 && g[d] < f.box.npd[d];
                if (!in) continue;
                const long long fd =
                    3 * (g[0] + (long long)f.box.npd[0] * (g[1] + (long long)f.box.npd[1] * g[2])) + comp;
                all = f.mask_h[(size_t)fd] != 0;
              }
          c->mask_h[(size_t)(3 * node + comp)] = all ? 1 : 0;
        }
      }
      c->mask.upload(c->mask_h);
      c->asmb = std::make_unique<CoarseAssembly>(c->box, c->mask_h);
      c->A = &c->asmb->matrix();
      c->elem.alloc((size_t)c->box.num_elements() * M1 * M1);
      c->b.alloc((size_t)c->n());
      c->x.alloc((size_t)c->n());
      levels_.push_back(std::move(c));
    }
    if (levels_.back()->n() > 4 * kHmgBottomMax)
      throw Error(HXG_ERR_UNSUPPORTED, "h-multigrid coarse mode: bottom level too large (thin box)");
    for (size_t l = 0; l + 1 < levels_.size(); ++l) levels_[l]->r.alloc((size_t)levels_[l]->n());
  }
  // numeric: Galerkin element matrices + slot sums, level by level
  for (size_t l = 0; l + 1 < levels_.size(); ++l) {
    HLevel& f = *levels_[l];
    HLevel& c = *levels_[l + 1];
    const double* fe = l == 0 ? elem0 : f.elem.p;
    galerkin_kernel<<<(unsigned)c.box.num_elements(), 288, 0, s>>>(f.box, c.box, f.m(), fe, c.elem.p);
    HXG_CUDA(cudaGetLastError());
    c.asmb->numeric_from_elements(c.elem.p, s);
  }
  // smoothers on every level above the bottom
  for (size_t l = 0; l + 1 < levels_.size(); ++l) {
    HLevel& lv = *levels_[l];
    const CsrMatrix* A = lv.A;
    const long long n = lv.n();
    lv.smoother.create(
        n, s, 2, [A, s](const double* x, double* y) { csr_matvec(*A, x, y, s); },
        [A, n, s](double* d) {
          csr_diag_kernel<<<grid_for(n, 256), 256, 0, s>>>((int)n, A->row_ptr.p, A->cols.p, A->vals.p, d);
          HXG_CUDA(cudaGetLastError());
        },
        nullptr, [&lv, n]() { return rough_seed(n, lv.mask_h); });
  }
  bottom_.factorize(*levels_.back()->A, s);
  ready_ = true;
}

void HmgCoarse::cycle(size_t l, const double* b, double* x, cudaStream_t s) {
  HLevel& lv = *levels_[l];
  if (l + 1 == levels_.size()) {
    bottom_.solve(b, x, s);
    return;
  }
  const CsrMatrix* A = lv.A;
  const long long n = lv.n();
  DevOp op = [A, s](const double* xx, double* yy) { csr_matvec(*A, xx, yy, s); };
  lv.smoother.apply(op, n, s, b, x, true);
  csr_matvec(*A, x, lv.r.p, s);
  vsub_from(lv.r.p, b, n, s);
  HLevel& c = *levels_[l + 1];
  restrict_kernel<<<grid_for(c.n(), 256), 256, 0, s>>>(lv.box, c.box, lv.m(), c.m(), lv.r.p, c.b.p);
  HXG_CUDA(cudaGetLastError());
  cycle(l + 1, c.b.p, c.x.p, s);
  prolong_add_kernel<<<grid_for(n, 256), 256, 0, s>>>(lv.box, c.box, lv.m(), c.m(), c.x.p, x);
  HXG_CUDA(cudaGetLastError());
  lv.smoother.apply(op, n, s, b, x, false);
}

void HmgCoarse::solve(const double* b, double* x, cudaStream_t s) {
  if (!ready_) throw Error(HXG_ERR_GENERIC, "h-multigrid coarse solver not set up");
  cycle(0, b, x, s);
}

}  // namespace hxg
