// Inexact coarse mode: one Galerkin h-multigrid V-cycle on the assembled Q1
// level (see hcoarse.hpp).  Every kernel is gather-based with fixed-order
// sums, so the cycle is bitwise reproducible run to run.
#include "hcoarse.hpp"
#include "densechol.hpp"

#include <cublas_v2.h>

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

// Lattice-stencil form of a level matrix: slot k = (s, cb), s = the
// neighbour offset (dx, dy, dz) in {-1, 0, 1}^3 (x fastest), stored as
// st[k n + r] (structure of arrays: every slot plane is read coalesced), no
// column indices; absent couplings (box edges, constrained columns) are 0.
__global__ void csr_to_stencil_kernel(BoxDev box, const int* __restrict__ rows,
                                      const int* __restrict__ cols, const double* __restrict__ vals,
                                      long long nnz, long long n, double* __restrict__ st) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nnz;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = rows[i], c = cols[i];
    const long long a = r / 3, b = c / 3;
    const int ax = (int)(a % box.npd[0]), ay = (int)((a / box.npd[0]) % box.npd[1]),
              az = (int)(a / ((long long)box.npd[0] * box.npd[1]));
    const int bx = (int)(b % box.npd[0]), by = (int)((b / box.npd[0]) % box.npd[1]),
              bz = (int)(b / ((long long)box.npd[0] * box.npd[1]));
    const int sl = ((bz - az + 1) * 3 + (by - ay + 1)) * 3 + (bx - ax + 1);
    st[(long long)(sl * 3 + (int)(c % 3)) * n + r] = vals[i];
  }
}

// y = A x on the stencil form: thread per row, the 81 couplings in fixed
// (slot, component) order.
__global__ void __launch_bounds__(256) stencil_matvec_kernel(BoxDev box, long long n,
                                                             const double* __restrict__ st,
                                                             const double* __restrict__ x,
                                                             double* __restrict__ y) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    const long long a = r / 3;
    const int ax = (int)(a % box.npd[0]), ay = (int)((a / box.npd[0]) % box.npd[1]),
              az = (int)(a / ((long long)box.npd[0] * box.npd[1]));
    double sum = 0.0;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
      const bool okz = az + dz >= 0 && az + dz < box.npd[2];
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy) {
        const bool oky = okz && ay + dy >= 0 && ay + dy < box.npd[1];
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
          const bool ok = oky && ax + dx >= 0 && ax + dx < box.npd[0];
          const int sl = ((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1);
          // out-of-box neighbours have zero couplings: read the row's own node
          const long long nb = ok ? a + dx + (long long)box.npd[0] * (dy + (long long)box.npd[1] * dz) : a;
#pragma unroll
          for (int cb = 0; cb < 3; ++cb)
            sum += __ldg(st + (long long)(sl * 3 + cb) * n + r) * __ldg(x + 3 * nb + cb);
        }
      }
    }
    y[r] = sum;
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

// The SYRK leaves the lower triangle: mirror it so every row is contiguous.
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

__global__ void slots_to_global(const double* __restrict__ lv, const long long* __restrict__ map,
                                long long n, double* __restrict__ gv) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (map[i] >= 0) gv[map[i]] = lv[i];
}
__global__ void ones_at(double* __restrict__ v, const long long* __restrict__ idx, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[idx[i]] = 1.0;
}
__global__ void owned_to_global(const double* __restrict__ b, const uint8_t* __restrict__ owned,
                                const long long* __restrict__ map, long long n, double* __restrict__ g) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    if (!owned || owned[i]) g[map[i]] = b[i];
}
__global__ void from_global(const double* __restrict__ g, const long long* __restrict__ map,
                            long long n, double* __restrict__ x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = g[map[i]];
}

}  // namespace

// ---------------------------------------------------------------------------

DenseInverse::~DenseInverse() {
  if (handle_) cublasDestroy((cublasHandle_t)handle_);
}

// A = L L^T and W = L^-1 by dense_chol_inv (densechol.cu), then
// A^-1 = W^T W (DSYRK, lower) mirrored to a full symmetric matrix.
void DenseInverse::factorize(const CsrMatrix& a, cudaStream_t s) {
  n_ = a.n;
  auto h = (cublasHandle_t)handle_;
  if (!h) {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) throw Error(HXG_ERR_CUDA, "cublasCreate failed");
    handle_ = h;
  }
  cublasSetStream(h, s);
  const size_t nn = (size_t)n_ * n_;
  if (inv_.n != nn) {
    inv_.alloc(nn);
    work_.alloc(nn);
    wfac_.alloc(nn);
  }
  const size_t ns = dense_chol_inv_scratch(n_);
  if (scratch_.n < ns) scratch_.alloc(ns);
  HXG_CUDA(cudaMemsetAsync(work_.p, 0, nn * sizeof(double), s));
  HXG_CUDA(cudaMemsetAsync(wfac_.p, 0, nn * sizeof(double), s));
  to_dense_kernel<<<grid_for(a.nnz(), 256), 256, 0, s>>>(a.rows.p, a.cols.p, a.vals.p, a.nnz(), n_,
                                                         work_.p);
  HXG_CUDA(cudaGetLastError());
  if (!info_.n) info_.alloc(1);
  HXG_CUDA(cudaMemsetAsync(info_.p, 0, sizeof(int), s));
  dense_chol_inv(h, s, work_.p, n_, wfac_.p, n_, n_, info_.p, scratch_.p);
  int info = 0;
  HXG_CUDA(cudaMemcpyAsync(&info, info_.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  HXG_CUDA(cudaStreamSynchronize(s));
  if (info != 0)
    throw Error(HXG_ERR_NOT_SPD, "factorization failed, matrix not SPD: h-multigrid bottom level");
  const double one = 1.0, zero = 0.0;
  if (cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, n_, n_, &one, wfac_.p, n_, &zero, inv_.p, n_) !=
      CUBLAS_STATUS_SUCCESS)
    throw Error(HXG_ERR_CUDA, "syrk (W^T W) failed");
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
  Lattice lat;  // partitioned: this block of the level's global lattice
  std::vector<uint8_t> mask_h;
  DevBuf<uint8_t> mask;
  const CsrMatrix* A = nullptr;
  std::unique_ptr<CoarseAssembly> asmb;  // levels >= 1
  DevBuf<double> elem;                   // levels >= 1: Galerkin element matrices
  DevBuf<double> st;                     // the level matrix in lattice-stencil form (81 n)
  DevBuf<double> b, x, r;
  DevBuf<double> scaled;  // partitioned: interface-scaled residual for the restriction
  Chebyshev smoother;
  long long n() const { return 3 * box.num_nodes(); }
  const uint8_t* m() const { return mask.n ? mask.p : nullptr; }
};

// The partitioned bottom: global lattice pattern + local -> global slot and
// DoF maps (built once), summed values (one all-reduce per setup), dense
// inverse on every rank.
struct HmgCoarse::Replicated {
  std::unique_ptr<CoarseAssembly> global;
  DevBuf<long long> slot_map, dof_map, diag_slots;
  DevBuf<double> gvec, gsol;
  DenseInverse inv;

  void symbolic(Partition& part, const Lattice& L, const CsrMatrix& la,
                const std::vector<uint8_t>& lmask, cudaStream_t s) {
    int gc[3] = {L.g[0] - 1, L.g[1] - 1, L.g[2] - 1};
    BoxDev gbox = make_box(gc, 1);
    const long long gn = 3 * gbox.num_nodes();
    auto to_global = [&](long long dof) {
      const long long node = dof / 3;
      const int c = (int)(dof % 3);
      const long long ix = node % L.n[0], iy = (node / L.n[0]) % L.n[1],
                      iz = node / ((long long)L.n[0] * L.n[1]);
      return 3 * ((ix + L.off[0]) + (long long)L.g[0] * ((iy + L.off[1]) + (long long)L.g[1] * (iz + L.off[2]))) + c;
    };
    // global mask: the blocks' masks agree on shared nodes; max-reduce them
    std::vector<double> gm((size_t)gn, 0.0);
    for (long long d = 0; d < la.n; ++d) gm[(size_t)to_global(d)] = lmask[(size_t)d];
    DevBuf<double> gmd;
    gmd.upload(gm);
    part.comm().allreduce(gmd.p, gn, 1, s);
    HXG_CUDA(cudaMemcpyAsync(gm.data(), gmd.p, sizeof(double) * gn, cudaMemcpyDeviceToHost, s));
    HXG_CUDA(cudaStreamSynchronize(s));
    std::vector<uint8_t> gmask((size_t)gn);
    for (long long d = 0; d < gn; ++d) gmask[(size_t)d] = gm[(size_t)d] > 0.5 ? 1 : 0;
    global = std::make_unique<CoarseAssembly>(gbox, gmask);
    const CsrMatrix& ga = global->matrix();
    std::vector<long long> smap(la.cols_h.size(), -1), dmap((size_t)la.n);
    for (int r = 0; r < la.n; ++r) {
      const long long gr = to_global(r);
      dmap[(size_t)r] = gr;
      if (gmask[(size_t)gr]) continue;  // identity re-imposed globally
      const int* gb = ga.cols_h.data() + ga.row_ptr_h[(size_t)gr];
      const int* ge = ga.cols_h.data() + ga.row_ptr_h[(size_t)gr + 1];
      for (int sl = la.row_ptr_h[(size_t)r]; sl < la.row_ptr_h[(size_t)r + 1]; ++sl) {
        const long long gcol = to_global(la.cols_h[(size_t)sl]);
        if (gmask[(size_t)gcol]) continue;
        const int* it = std::lower_bound(gb, ge, (int)gcol);
        if (it == ge || *it != (int)gcol)
          throw Error(HXG_ERR_GENERIC, "h-multigrid bottom: slot outside the global pattern");
        smap[(size_t)sl] = ga.row_ptr_h[(size_t)gr] + (it - gb);
      }
    }
    std::vector<long long> diag;
    for (int r = 0; r < ga.n; ++r)
      if (gmask[(size_t)r]) diag.push_back(ga.row_ptr_h[(size_t)r]);
    slot_map.upload(smap);
    dof_map.upload(dmap);
    if (!diag.empty()) diag_slots.upload(diag);
    gvec.alloc((size_t)ga.n);
    gsol.alloc((size_t)ga.n);
  }

  void numeric(Partition& part, const CsrMatrix& la, cudaStream_t s) {
    CsrMatrix& ga = global->mutable_matrix();
    const long long gnnz = ga.nnz(), lnnz = la.nnz();
    HXG_CUDA(cudaMemsetAsync(ga.vals.p, 0, sizeof(double) * gnnz, s));
    slots_to_global<<<grid_for(lnnz, 256), 256, 0, s>>>(la.vals.p, slot_map.p, lnnz, ga.vals.p);
    HXG_CUDA(cudaGetLastError());
    part.comm().allreduce(ga.vals.p, gnnz, 0, s);
    if (diag_slots.n)
      ones_at<<<grid_for((long long)diag_slots.n, 256), 256, 0, s>>>(ga.vals.p, diag_slots.p,
                                                                    (long long)diag_slots.n);
    HXG_CUDA(cudaGetLastError());
    inv.factorize(ga, s);
  }

  void solve(Partition& part, const Lattice& L, const double* b, double* x, cudaStream_t s) {
    const long long n = L.size(), gn = (long long)gvec.n;
    HXG_CUDA(cudaMemsetAsync(gvec.p, 0, sizeof(double) * gn, s));
    const uint8_t* own = part.comm().world() > 1 ? part.owned(L) : nullptr;
    owned_to_global<<<grid_for(n, 256), 256, 0, s>>>(b, own, dof_map.p, n, gvec.p);
    HXG_CUDA(cudaGetLastError());
    part.comm().allreduce(gvec.p, gn, 0, s);
    inv.solve(gvec.p, gsol.p, s);
    from_global<<<grid_for(n, 256), 256, 0, s>>>(gsol.p, dof_map.p, n, x);
    HXG_CUDA(cudaGetLastError());
  }
};

HmgCoarse::HmgCoarse() = default;
HmgCoarse::~HmgCoarse() = default;

long long HmgCoarse::level_size(int l) const { return levels_[(size_t)l]->n(); }
const CsrMatrix& HmgCoarse::level_matrix(int l) const { return *levels_[(size_t)l]->A; }
const std::vector<uint8_t>& HmgCoarse::level_mask(int l) const { return levels_[(size_t)l]->mask_h; }

void HmgCoarse::setup(const CsrMatrix& a0, const BoxDev& box0, const std::vector<uint8_t>& mask0,
                      const double* elem0, cudaStream_t s, Partition* part) {
  if (box0.p != 1) throw Error(HXG_ERR_UNSUPPORTED, "h-multigrid coarse mode needs the p = 1 level");
  if (levels_.empty() || levels_[0]->A != &a0 || part_ != part) {  // symbolic
    levels_.clear();
    rep_.reset();
    part_ = part;
    auto l0 = std::make_unique<HLevel>();
    l0->box = box0;
    l0->mask_h = mask0.empty() ? std::vector<uint8_t>((size_t)(3 * box0.num_nodes()), 0) : mask0;
    l0->mask.upload(l0->mask_h);
    l0->A = &a0;
    if (part_) l0->lat = part_->h_lattice(0);
    levels_.push_back(std::move(l0));
    for (;;) {
      HLevel& f = *levels_.back();
      bool can = f.box.cells[0] >= 2 && f.box.cells[1] >= 2 && f.box.cells[2] >= 2;
      long long global_n = f.n();
      if (part_) {  // coarsen while every block stays aligned; all ranks agree
        global_n = 3LL * f.lat.g[0] * f.lat.g[1] * f.lat.g[2];
        for (int d = 0; d < 3; ++d) can = can && f.box.cells[d] % 2 == 0 && f.lat.off[d] % 2 == 0;
        can = part_->allreduce_max(can ? 0.0 : 1.0, s) == 0.0;
      }
      if (global_n <= kHmgBottomMax || !can) break;
      auto c = std::make_unique<HLevel>();
      int cc[3];
      for (int d = 0; d < 3; ++d) cc[d] = (f.box.cells[d] + 1) / 2;
      c->box = make_box(cc, 1);
      if (part_) c->lat = part_->h_lattice((int)levels_.size());
      // a coarse DoF is constrained iff every fine DoF it interpolates to is
      // (its column of P~ is zero); with whole-face constraints the block's
      // view of the support decides like the global one
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
    for (size_t l = 0; l + 1 < levels_.size(); ++l) {
      levels_[l]->r.alloc((size_t)levels_[l]->n());
      if (part_) levels_[l]->scaled.alloc((size_t)levels_[l]->n());
    }
    if (part_) {
      HLevel& bl = *levels_.back();
      rep_ = std::make_unique<Replicated>();
      rep_->symbolic(*part_, bl.lat, *bl.A, bl.mask_h, s);
      if (rep_->global->matrix().n > kHmgBottomLimit)
        throw Error(HXG_ERR_UNSUPPORTED, "h-multigrid coarse mode: bottom level too large (block "
                                         "cells odd early: use even block sizes)");
    } else if (levels_.back()->n() > kHmgBottomLimit) {
      throw Error(HXG_ERR_UNSUPPORTED, "h-multigrid coarse mode: bottom level too large (thin box)");
    }
  }
  PhaseTimer pt(s);
  // numeric: Galerkin element matrices + slot sums, level by level
  for (size_t l = 0; l + 1 < levels_.size(); ++l) {
    HLevel& f = *levels_[l];
    HLevel& c = *levels_[l + 1];
    const double* fe = l == 0 ? elem0 : f.elem.p;
    galerkin_kernel<<<(unsigned)c.box.num_elements(), 288, 0, s>>>(f.box, c.box, f.m(), fe, c.elem.p);
    HXG_CUDA(cudaGetLastError());
    c.asmb->numeric_from_elements(c.elem.p, s);
  }
  pt.mark("  hmg galerkin + assembly");
  // stencil forms of the smoothed levels (their SpMV has no column indices)
  for (size_t l = 0; l + 1 < levels_.size(); ++l) {
    HLevel& lv = *levels_[l];
    const long long n = lv.n(), nnz = lv.A->nnz();
    if (lv.st.n != (size_t)(81 * n)) lv.st.alloc((size_t)(81 * n));
    HXG_CUDA(cudaMemsetAsync(lv.st.p, 0, sizeof(double) * 81 * n, s));
    csr_to_stencil_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(lv.box, lv.A->rows.p, lv.A->cols.p,
                                                              lv.A->vals.p, nnz, n, lv.st.p);
    HXG_CUDA(cudaGetLastError());
  }
  pt.mark("  hmg stencils");
  // smoothers on every level above the bottom
  for (size_t l = 0; l + 1 < levels_.size(); ++l) {
    HLevel& lv = *levels_[l];
    const CsrMatrix* A = lv.A;
    const long long n = lv.n();
    Partition* part_l = part_;
    DotFn dotf = [part_l, &lv, s](const double* x, const double* y) { return part_l->dot(lv.lat, x, y, s); };
    lv.smoother.create(
        n, s, 2, [this, &lv, s](const double* x, double* y) { apply_level(lv, x, y, s); },
        [this, A, n, s, &lv](double* d) {
          csr_diag_kernel<<<grid_for(n, 256), 256, 0, s>>>((int)n, A->row_ptr.p, A->cols.p, A->vals.p, d);
          HXG_CUDA(cudaGetLastError());
          if (part_) {  // summed over the blocks; constrained entries stay 1
            part_->exchange(lv.lat, d, s);
            vmask_fill(d, 1.0, lv.m(), n, s);
          }
        },
        part_ ? &dotf : nullptr,
        [this, &lv, n]() {
          return part_ ? part_->global_seed_slice(lv.lat, lv.mask_h) : rough_seed(n, lv.mask_h);
        });
  }
  pt.mark("  hmg smoothers");
  if (part_)
    rep_->numeric(*part_, *levels_.back()->A, s);
  else
    bottom_.factorize(*levels_.back()->A, s);
  pt.mark("  hmg bottom inverse");
  ready_ = true;
}

void HmgCoarse::apply_level(HLevel& lv, const double* x, double* y, cudaStream_t s) {
  const long long n = lv.n();
  stencil_matvec_kernel<<<grid_for(n, 256), 256, 0, s>>>(lv.box, n, lv.st.p, x, y);
  HXG_CUDA(cudaGetLastError());
  if (part_) part_->exchange(lv.lat, y, s, x, lv.m());  // constrained rows: identity
}

void HmgCoarse::cycle(size_t l, const double* b, double* x, cudaStream_t s) {
  HLevel& lv = *levels_[l];
  if (l + 1 == levels_.size()) {
    if (part_)
      rep_->solve(*part_, lv.lat, b, x, s);
    else
      bottom_.solve(b, x, s);
    return;
  }
  const long long n = lv.n();
  DevOp op = [this, &lv, s](const double* xx, double* yy) { apply_level(lv, xx, yy, s); };
  lv.smoother.apply(op, n, s, b, x, true);
  apply_level(lv, x, lv.r.p, s);
  vsub_from(lv.r.p, b, n, s);
  HLevel& c = *levels_[l + 1];
  const double* rf = lv.r.p;
  if (part_) {  // shared fine entries are counted once per block: x 1/2 per shared direction
    vcopy(lv.scaled.p, lv.r.p, n, s);
    part_->scale_interfaces(lv.lat, lv.scaled.p, 0.5, s);
    rf = lv.scaled.p;
  }
  restrict_kernel<<<grid_for(c.n(), 256), 256, 0, s>>>(lv.box, c.box, lv.m(), c.m(), rf, c.b.p);
  HXG_CUDA(cudaGetLastError());
  if (part_) part_->exchange(c.lat, c.b.p, s);
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
