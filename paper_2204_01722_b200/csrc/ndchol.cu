// Nested-dissection multifrontal Cholesky on device (see ndchol.hpp).
//
// Symbolic phase (host, once per pattern): recursive bisection of the node
// box along its longest axis by a one-node-thick separator plane (the
// 27-point Q1 coupling cannot cross it); leaves of <= kLeafNodes nodes.
// Each tree node is a front: its pivots (separator or leaf DoFs, contiguous
// in the new numbering) plus its shell = lattice nodes adjacent to its
// region, all of which are ancestor pivots.  Numeric phase (device, per
// setup): postorder over fronts, assemble original entries + children's
// update matrices (extend-add, fixed order), potrf / trsm / syrk on the
// dense front, keep the (np + ns) x np panel.  Solve (per V-cycle): forward
// sweep leaves -> root passing update vectors up the tree, backward sweep
// root -> leaves reading ancestor values; fronts of one tree level run in
// one launch (one CTA per small front), large fronts use cuBLAS.
#include "ndchol.hpp"

#include <algorithm>
#include <functional>

#include "dispatch.hpp"

namespace hxg {

namespace {

constexpr int kLeafNodes = 128;
constexpr int kSmallM = 2048;   // small fronts: one CTA, front vector in smem
constexpr int kSolveThreads = 256;

__global__ void assemble_kernel(const long long* __restrict__ dst, const int* __restrict__ src,
                                long long n, const double* __restrict__ vals, double* front) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    front[dst[i]] = vals[src[i]];
}

// work[map[r] + map[c] * m] += U[r + c * ns] for r >= c (lower triangles).
__global__ void extend_add_kernel(const double* __restrict__ U, int ns,
                                  const int* __restrict__ map, double* work, int m) {
  const long long total = (long long)ns * ns;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / ns), r = (int)(e % ns);
    if (r < c) continue;
    work[map[r] + (long long)map[c] * m] += U[e];
  }
}

__global__ void permute_gather(const double* __restrict__ b, const int* __restrict__ perm, int n,
                               double* __restrict__ w) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    w[i] = b[perm[i]];
}

__global__ void permute_scatter(const double* __restrict__ w, const int* __restrict__ perm, int n,
                                double* __restrict__ x) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[perm[i]] = w[i];
}

struct SolveArgs {
  const int* fronts;  // front ids of this level
  const int* piv0;
  const int* np;
  const int* ns;
  const long long* loff;
  const long long* rows_off;
  const int* child0;
  const int* child1;
  const long long* map0;  // child-update map offsets
  const long long* map1;
  const int* maps;
  const int* shell;
  const long long* uoff;  // update-vector offsets
  const double* L;
  double* w;
  double* ubuf;
};

// y = [w(piv); 0] + extend(u_c0) + extend(u_c1)  (front vector, size m)
__device__ void build_front_vector(const SolveArgs& a, int t, int np, int m, double* y) {
  for (int k = threadIdx.x; k < m; k += blockDim.x) y[k] = k < np ? a.w[a.piv0[t] + k] : 0.0;
  __syncthreads();
  const int ch[2] = {a.child0[t], a.child1[t]};
  const long long mo[2] = {a.map0[t], a.map1[t]};
  for (int q = 0; q < 2; ++q) {
    const int c = ch[q];
    if (c < 0) continue;
    const int nsc = a.ns[c];
    const double* u = a.ubuf + a.uoff[c];
    const int* mp = a.maps + mo[q];
    for (int k = threadIdx.x; k < nsc; k += blockDim.x) y[mp[k]] += u[k];
    __syncthreads();
  }
}

// Forward sweep on small fronts: one CTA per front, column-oriented
// substitution through the whole (np + ns) x np panel.
__global__ void __launch_bounds__(kSolveThreads) fwd_small_kernel(SolveArgs a) {
  __shared__ double y[kSmallM];
  __shared__ double zj;
  const int t = a.fronts[blockIdx.x];
  const int np = a.np[t], ns = a.ns[t], m = np + ns;
  build_front_vector(a, t, np, m, y);
  const double* L = a.L + a.loff[t];
  for (int j = 0; j < np; ++j) {
    if (threadIdx.x == 0) {
      zj = y[j] / L[j + (long long)j * m];
      y[j] = zj;
    }
    __syncthreads();
    const double z = zj;
    const double* col = L + (long long)j * m;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) y[i] -= col[i] * z;
    __syncthreads();
  }
  for (int k = threadIdx.x; k < m; k += blockDim.x) {
    if (k < np)
      a.w[a.piv0[t] + k] = y[k];
    else
      a.ubuf[a.uoff[t] + (k - np)] = y[k];
  }
}

// Backward sweep on small fronts: x_j = (x_j - sum_{i > j} L_ij x_i) / L_jj.
__global__ void __launch_bounds__(kSolveThreads) bwd_small_kernel(SolveArgs a) {
  __shared__ double x[kSmallM];
  __shared__ double red[kSolveThreads / 32];
  const int t = a.fronts[blockIdx.x];
  const int np = a.np[t], ns = a.ns[t], m = np + ns;
  const int* sh = a.shell + a.rows_off[t];
  for (int k = threadIdx.x; k < m; k += blockDim.x)
    x[k] = k < np ? a.w[a.piv0[t] + k] : a.w[sh[k - np]];
  __syncthreads();
  const double* L = a.L + a.loff[t];
  for (int j = np - 1; j >= 0; --j) {
    const double* col = L + (long long)j * m;
    double s = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) s += col[i] * x[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += red[q];
      x[j] = (x[j] - tot) / col[j];
    }
    __syncthreads();
  }
  for (int k = threadIdx.x; k < np; k += blockDim.x) a.w[a.piv0[t] + k] = x[k];
}

// Large fronts: the front vector lives in global scratch (ybuf), cuBLAS does
// the dense triangular solve and the panel product.
__global__ void big_build_kernel(SolveArgs a, int t, double* ybuf) {
  const int np = a.np[t], ns = a.ns[t], m = np + ns;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x)
    ybuf[k] = k < np ? a.w[a.piv0[t] + k] : 0.0;
}
__global__ void big_extend_kernel(SolveArgs a, int t, int q, double* ybuf) {
  const int c = q == 0 ? a.child0[t] : a.child1[t];
  if (c < 0) return;
  const int nsc = a.ns[c];
  const double* u = a.ubuf + a.uoff[c];
  const int* mp = a.maps + (q == 0 ? a.map0[t] : a.map1[t]);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nsc; k += gridDim.x * blockDim.x)
    ybuf[mp[k]] += u[k];
}
__global__ void big_fwd_store_kernel(SolveArgs a, int t, const double* ybuf) {
  const int np = a.np[t], ns = a.ns[t], m = np + ns;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x) {
    if (k < np)
      a.w[a.piv0[t] + k] = ybuf[k];
    else
      a.ubuf[a.uoff[t] + (k - np)] = ybuf[k];
  }
}
__global__ void big_bwd_load_kernel(SolveArgs a, int t, double* ybuf) {
  const int np = a.np[t], ns = a.ns[t], m = np + ns;
  const int* sh = a.shell + a.rows_off[t];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x)
    ybuf[k] = k < np ? a.w[a.piv0[t] + k] : a.w[sh[k - np]];
}
__global__ void big_bwd_store_kernel(SolveArgs a, int t, const double* ybuf) {
  const int np = a.np[t];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < np; k += gridDim.x * blockDim.x)
    a.w[a.piv0[t] + k] = ybuf[k];
}

void cublas_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) throw Error(HXG_ERR_CUDA, std::string(what) + " failed");
}

}  // namespace

NdCholesky::~NdCholesky() {
  if (cublas_) cublasDestroy(cublas_);
  if (cusolver_) cusolverDnDestroy(cusolver_);
}

void NdCholesky::analyze(const CsrMatrix& a, const int npd[3]) {
  n_ = a.n;
  const long long nn = (long long)npd[0] * npd[1] * npd[2];
  if (nn * 3 != n_) throw Error(HXG_ERR_INVALID_ARGUMENT, "coarse matrix does not match lattice");
  struct Box {
    int lo[3], hi[3];
  };
  std::vector<Box> region, pivot;
  fronts_.clear();
  std::function<int(Box, int)> build = [&](Box r, int level) -> int {
    int n[3] = {r.hi[0] - r.lo[0], r.hi[1] - r.lo[1], r.hi[2] - r.lo[2]};
    long long cnt = (long long)n[0] * n[1] * n[2];
    int ax = 0;
    if (n[1] > n[ax]) ax = 1;
    if (n[2] > n[ax]) ax = 2;
    Front f;
    f.level = level;
    Box piv = r;
    if (cnt > kLeafNodes && n[ax] >= 3) {
      int mid = r.lo[ax] + n[ax] / 2;
      Box left = r, right = r;
      left.hi[ax] = mid;
      right.lo[ax] = mid + 1;
      f.child[0] = build(left, level + 1);
      f.child[1] = build(right, level + 1);
      piv.lo[ax] = mid;
      piv.hi[ax] = mid + 1;
    }
    int id = (int)fronts_.size();
    fronts_.push_back(f);
    region.push_back(r);
    pivot.push_back(piv);
    for (int c : f.child)
      if (c >= 0) fronts_[(size_t)c].parent = id;
    return id;
  };
  Box all{{0, 0, 0}, {npd[0], npd[1], npd[2]}};
  build(all, 0);
  const int nf = (int)fronts_.size();

  // New numbering: pivots of each front contiguous, fronts in postorder.
  std::vector<int> newidx((size_t)n_, -1), perm((size_t)n_);
  int counter = 0;
  for (int t = 0; t < nf; ++t) {
    const Box& p = pivot[(size_t)t];
    fronts_[(size_t)t].piv0 = counter;
    for (int z = p.lo[2]; z < p.hi[2]; ++z)
      for (int y = p.lo[1]; y < p.hi[1]; ++y)
        for (int x = p.lo[0]; x < p.hi[0]; ++x) {
          int node = x + npd[0] * (y + npd[1] * z);
          for (int c = 0; c < 3; ++c) {
            newidx[(size_t)(3 * node + c)] = counter;
            perm[(size_t)counter] = 3 * node + c;
            ++counter;
          }
        }
    fronts_[(size_t)t].np = counter - fronts_[(size_t)t].piv0;
  }
  if (counter != n_) throw Error(HXG_ERR_GENERIC, "nested dissection numbering incomplete");

  // Shells (sorted new indices), child maps, panel offsets, stack bound.
  std::vector<int> shell_rows;
  std::vector<std::vector<int>> shell((size_t)nf);
  lsize_ = 0;
  max_front_ = 0;
  for (int t = 0; t < nf; ++t) {
    const Box& r = region[(size_t)t];
    int lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::max(r.lo[d] - 1, 0);
      hi[d] = std::min(r.hi[d] + 1, npd[d]);
    }
    auto& sh = shell[(size_t)t];
    for (int z = lo[2]; z < hi[2]; ++z)
      for (int y = lo[1]; y < hi[1]; ++y)
        for (int x = lo[0]; x < hi[0]; ++x) {
          bool inside = x >= r.lo[0] && x < r.hi[0] && y >= r.lo[1] && y < r.hi[1] &&
                        z >= r.lo[2] && z < r.hi[2];
          if (inside) continue;
          int node = x + npd[0] * (y + npd[1] * z);
          for (int c = 0; c < 3; ++c) sh.push_back(newidx[(size_t)(3 * node + c)]);
        }
    std::sort(sh.begin(), sh.end());
    Front& f = fronts_[(size_t)t];
    f.ns = (int)sh.size();
    if (!sh.empty() && sh.front() < f.piv0 + f.np)
      throw Error(HXG_ERR_GENERIC, "nested dissection shell is not ancestral");
    f.rows_off = shell_rows.size();
    shell_rows.insert(shell_rows.end(), sh.begin(), sh.end());
    f.loff = lsize_;
    const size_t m = (size_t)f.np + f.ns;
    lsize_ += m * (size_t)f.np;
    max_front_ = std::max(max_front_, m * m);
  }
  // Position of a new index within front t's rows (pivots then shell).
  auto pos_in = [&](int t, int ni) -> int {
    const Front& f = fronts_[(size_t)t];
    if (ni >= f.piv0 && ni < f.piv0 + f.np) return ni - f.piv0;
    const auto& sh = shell[(size_t)t];
    auto it = std::lower_bound(sh.begin(), sh.end(), ni);
    if (it == sh.end() || *it != ni) return -1;
    return f.np + (int)(it - sh.begin());
  };
  std::vector<int> maps;
  for (int t = 0; t < nf; ++t) {
    Front& f = fronts_[(size_t)t];
    for (int q = 0; q < 2; ++q) {
      int c = f.child[q];
      f.map_off[q] = maps.size();
      if (c < 0) continue;
      for (int ni : shell[(size_t)c]) {
        int p = pos_in(t, ni);
        if (p < 0) throw Error(HXG_ERR_GENERIC, "child update row missing from parent front");
        maps.push_back(p);
      }
    }
  }
  // Update-stack bound: simulate the postorder push/pop.
  {
    std::vector<size_t> stack;
    size_t cur = 0, peak = 0;
    for (int t = 0; t < nf; ++t) {
      const Front& f = fronts_[(size_t)t];
      int nch = (f.child[0] >= 0) + (f.child[1] >= 0);
      for (int k = 0; k < nch; ++k) {
        cur -= stack.back();
        stack.pop_back();
      }
      size_t u = (size_t)f.ns * f.ns;
      stack.push_back(u);
      cur += u;
      peak = std::max(peak, cur);
    }
    max_update_ = peak;
  }
  // Assembly lists: lower-triangle original entries with a pivot column.
  std::vector<long long> adst;
  std::vector<int> asrc, afront;
  asm_begin_.assign((size_t)nf + 1, 0);
  for (int t = 0; t < nf; ++t) {
    const Front& f = fronts_[(size_t)t];
    const int m = f.np + f.ns;
    asm_begin_[(size_t)t] = adst.size();
    for (int pj = 0; pj < f.np; ++pj) {
      int jold = perm[(size_t)(f.piv0 + pj)];
      for (int k = a.row_ptr_h[(size_t)jold]; k < a.row_ptr_h[(size_t)jold + 1]; ++k) {
        int ni = newidx[(size_t)a.cols_h[(size_t)k]];
        if (ni < f.piv0) continue;  // eliminated in a descendant front
        int pi = pos_in(t, ni);
        if (pi < 0) throw Error(HXG_ERR_GENERIC, "matrix entry outside its front");
        if (pi < pj) continue;      // upper triangle
        adst.push_back((long long)pi + (long long)pj * m);
        asrc.push_back(k);
        afront.push_back(t);
      }
    }
  }
  asm_begin_[(size_t)nf] = adst.size();

  // Levels for the batched solves: small fronts (one CTA each) and large
  // fronts (cuBLAS) per tree depth.
  int maxlev = 0;
  for (const auto& f : fronts_) maxlev = std::max(maxlev, f.level);
  levels_.assign((size_t)maxlev + 1, {});
  for (int t = 0; t < nf; ++t) levels_[(size_t)fronts_[(size_t)t].level].push_back(t);
  std::vector<int> sl;
  small_off_.assign(levels_.size() + 1, 0);
  big_.assign(levels_.size(), {});
  for (size_t l = 0; l < levels_.size(); ++l) {
    small_off_[l] = sl.size();
    for (int t : levels_[l]) {
      const Front& f = fronts_[(size_t)t];
      if (f.np + f.ns <= kSmallM)
        sl.push_back(t);
      else
        big_[l].push_back(t);
    }
  }
  small_off_[levels_.size()] = sl.size();

  // Device copies.
  perm_.upload(perm);
  shell_rows_.upload(shell_rows.empty() ? std::vector<int>{0} : shell_rows);
  child_map_.upload(maps.empty() ? std::vector<int>{0} : maps);
  asm_dst_.upload(adst);
  asm_src_.upload(asrc);
  small_lists_.upload(sl.empty() ? std::vector<int>{0} : sl);
  (void)afront;
  std::vector<int> piv0(nf), np(nf), ns(nf), c0(nf), c1(nf);
  std::vector<long long> loff(nf), roff(nf), m0(nf), m1(nf), uoff(nf);
  long long ucount = 0;
  for (int t = 0; t < nf; ++t) {
    const Front& f = fronts_[(size_t)t];
    piv0[t] = f.piv0;
    np[t] = f.np;
    ns[t] = f.ns;
    c0[t] = f.child[0];
    c1[t] = f.child[1];
    loff[t] = (long long)f.loff;
    roff[t] = (long long)f.rows_off;
    m0[t] = (long long)f.map_off[0];
    m1[t] = (long long)f.map_off[1];
    uoff[t] = ucount;
    ucount += f.ns;
  }
  dfront_piv0_.upload(piv0);
  dfront_np_.upload(np);
  dfront_ns_.upload(ns);
  dfront_loff_.upload(loff);
  dfront_rows_off_.upload(roff);
  c0_.upload(c0);
  c1_.upload(c1);
  map0_.upload(m0);
  map1_.upload(m1);
  uoff_.upload(uoff);
  ubuf_.alloc((size_t)std::max<long long>(ucount, 1));
  L_.alloc(lsize_);
  work_.alloc(max_front_);
  stack_.alloc(std::max<size_t>(max_update_, 1));
  wvec_.alloc((size_t)n_);
  size_t maxm = 0;
  for (const auto& f : fronts_) maxm = std::max(maxm, (size_t)(f.np + f.ns));
  ybuf_.alloc(maxm);
  info_.alloc((size_t)nf);
  analyzed_ = true;
}

void NdCholesky::factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s) {
  if (!cublas_) {
    cublas_check(cublasCreate(&cublas_), "cublasCreate");
    if (cusolverDnCreate(&cusolver_) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "cusolverDnCreate failed");
  }
  cublasSetStream(cublas_, s);
  cusolverDnSetStream(cusolver_, s);
  if (!analyzed_) analyze(a, npd);
  ready_ = false;
  HXG_CUDA(cudaMemsetAsync(info_.p, 0, sizeof(int) * fronts_.size(), s));
  std::vector<std::pair<size_t, int>> stack;  // (offset, ns)
  size_t top = 0;
  const double one = 1.0, minus_one = -1.0;
  for (int t = 0; t < (int)fronts_.size(); ++t) {
    const Front& f = fronts_[(size_t)t];
    const int m = f.np + f.ns;
    double* W = work_.p;
    HXG_CUDA(cudaMemsetAsync(W, 0, sizeof(double) * (size_t)m * m, s));
    const long long na = (long long)(asm_begin_[(size_t)t + 1] - asm_begin_[(size_t)t]);
    if (na > 0)
      assemble_kernel<<<grid_for(na, 256), 256, 0, s>>>(asm_dst_.p + asm_begin_[(size_t)t],
                                                        asm_src_.p + asm_begin_[(size_t)t], na,
                                                        a.vals.p, W);
    // Children's updates sit on top of the stack: child[1] above child[0].
    int nch = (f.child[0] >= 0) + (f.child[1] >= 0);
    std::vector<std::pair<size_t, int>> ups(stack.end() - nch, stack.end());
    for (int q = 0; q < nch; ++q) {
      const int c = f.child[q];
      const Front& fc = fronts_[(size_t)c];
      const auto& up = ups[(size_t)q];
      if (fc.ns > 0)
        extend_add_kernel<<<grid_for((long long)fc.ns * fc.ns, 256), 256, 0, s>>>(
            stack_.p + up.first, fc.ns, child_map_.p + f.map_off[q], W, m);
    }
    for (int q = 0; q < nch; ++q) stack.pop_back();
    top = stack.empty() ? 0 : stack.back().first + (size_t)stack.back().second * stack.back().second;
    HXG_CUDA(cudaGetLastError());
    // Dense partial factorization.
    int lwork = 0;
    if (cusolverDnDpotrf_bufferSize(cusolver_, CUBLAS_FILL_MODE_LOWER, f.np, W, m, &lwork) !=
        CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "potrf_bufferSize failed");
    if (potrf_ws_.n < (size_t)lwork) potrf_ws_.alloc((size_t)lwork * 2);
    if (cusolverDnDpotrf(cusolver_, CUBLAS_FILL_MODE_LOWER, f.np, W, m, potrf_ws_.p, lwork,
                         info_.p + t) != CUSOLVER_STATUS_SUCCESS)
      throw Error(HXG_ERR_CUDA, "potrf failed");
    if (f.ns > 0) {
      cublas_check(cublasDtrsm(cublas_, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T,
                               CUBLAS_DIAG_NON_UNIT, f.ns, f.np, &one, W, m, W + f.np, m),
                   "trsm");
      cublas_check(cublasDsyrk(cublas_, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, f.ns, f.np,
                               &minus_one, W + f.np, m, &one, W + f.np + (size_t)f.np * m, m),
                   "syrk");
    }
    HXG_CUDA(cudaMemcpyAsync(L_.p + f.loff, W, sizeof(double) * (size_t)m * f.np,
                             cudaMemcpyDeviceToDevice, s));
    if (f.ns > 0) {
      HXG_CUDA(cudaMemcpy2DAsync(stack_.p + top, sizeof(double) * f.ns,
                                 W + f.np + (size_t)f.np * m, sizeof(double) * m,
                                 sizeof(double) * f.ns, f.ns, cudaMemcpyDeviceToDevice, s));
    }
    stack.emplace_back(top, f.ns);
    top += (size_t)f.ns * f.ns;
  }
  std::vector<int> info(fronts_.size());
  HXG_CUDA(cudaMemcpyAsync(info.data(), info_.p, sizeof(int) * info.size(),
                           cudaMemcpyDeviceToHost, s));
  HXG_CUDA(cudaStreamSynchronize(s));
  for (int v : info)
    if (v != 0)
      throw Error(HXG_ERR_NOT_SPD, "factorization failed, matrix not SPD: coarse Cholesky "
                                   "factorization failed at level 0");
  ready_ = true;
}

void NdCholesky::solve(const double* b, double* x, cudaStream_t s) {
  if (!ready_) throw Error(HXG_ERR_GENERIC, "coarse solver not factorized");
  cublasSetStream(cublas_, s);
  SolveArgs a;
  a.piv0 = dfront_piv0_.p;
  a.np = dfront_np_.p;
  a.ns = dfront_ns_.p;
  a.loff = dfront_loff_.p;
  a.rows_off = dfront_rows_off_.p;
  a.child0 = c0_.p;
  a.child1 = c1_.p;
  a.map0 = map0_.p;
  a.map1 = map1_.p;
  a.maps = child_map_.p;
  a.shell = shell_rows_.p;
  a.uoff = uoff_.p;
  a.L = L_.p;
  a.w = wvec_.p;
  a.ubuf = ubuf_.p;
  permute_gather<<<grid_for(n_, 256), 256, 0, s>>>(b, perm_.p, n_, wvec_.p);
  const double one = 1.0, minus_one = -1.0;
  // Forward: deepest level first.
  for (int l = (int)levels_.size() - 1; l >= 0; --l) {
    const size_t ns0 = small_off_[(size_t)l], ns1 = small_off_[(size_t)l + 1];
    if (ns1 > ns0) {
      a.fronts = small_lists_.p + ns0;
      fwd_small_kernel<<<(unsigned)(ns1 - ns0), kSolveThreads, 0, s>>>(a);
    }
    for (int t : big_[(size_t)l]) {
      const Front& f = fronts_[(size_t)t];
      const int m = f.np + f.ns;
      big_build_kernel<<<grid_for(m, 256), 256, 0, s>>>(a, t, ybuf_.p);
      big_extend_kernel<<<grid_for(f.ns > 0 ? m : 1, 256), 256, 0, s>>>(a, t, 0, ybuf_.p);
      big_extend_kernel<<<grid_for(f.ns > 0 ? m : 1, 256), 256, 0, s>>>(a, t, 1, ybuf_.p);
      const double* L = L_.p + f.loff;
      cublas_check(cublasDtrsv(cublas_, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                               f.np, L, m, ybuf_.p, 1),
                   "trsv");
      if (f.ns > 0)
        cublas_check(cublasDgemv(cublas_, CUBLAS_OP_N, f.ns, f.np, &minus_one, L + f.np, m,
                                 ybuf_.p, 1, &one, ybuf_.p + f.np, 1),
                     "gemv");
      big_fwd_store_kernel<<<grid_for(m, 256), 256, 0, s>>>(a, t, ybuf_.p);
    }
    HXG_CUDA(cudaGetLastError());
  }
  // Backward: root first.
  for (size_t l = 0; l < levels_.size(); ++l) {
    for (int t : big_[l]) {
      const Front& f = fronts_[(size_t)t];
      const int m = f.np + f.ns;
      big_bwd_load_kernel<<<grid_for(m, 256), 256, 0, s>>>(a, t, ybuf_.p);
      const double* L = L_.p + f.loff;
      if (f.ns > 0)
        cublas_check(cublasDgemv(cublas_, CUBLAS_OP_T, f.ns, f.np, &minus_one, L + f.np, m,
                                 ybuf_.p + f.np, 1, &one, ybuf_.p, 1),
                     "gemv^T");
      cublas_check(cublasDtrsv(cublas_, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT,
                               f.np, L, m, ybuf_.p, 1),
                   "trsv^T");
      big_bwd_store_kernel<<<grid_for(f.np, 256), 256, 0, s>>>(a, t, ybuf_.p);
    }
    const size_t ns0 = small_off_[l], ns1 = small_off_[l + 1];
    if (ns1 > ns0) {
      a.fronts = small_lists_.p + ns0;
      bwd_small_kernel<<<(unsigned)(ns1 - ns0), kSolveThreads, 0, s>>>(a);
    }
    HXG_CUDA(cudaGetLastError());
  }
  permute_scatter<<<grid_for(n_, 256), 256, 0, s>>>(wvec_.p, perm_.p, n_, x);
  HXG_CUDA(cudaGetLastError());
}

}  // namespace hxg
