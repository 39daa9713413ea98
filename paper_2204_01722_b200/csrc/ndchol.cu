// Nested-dissection multifrontal Cholesky on device (see ndchol.hpp).
//
// Symbolic phase (host, once per pattern): recursive bisection of the node
// box along its longest axis by a one-node-thick separator plane (the
// 27-point Q1 coupling cannot cross it); leaves of <= kLeafNodes nodes.
// Each tree node is a front: its pivots (separator or leaf DoFs, contiguous
// in the new numbering) plus its shell = lattice nodes adjacent to its
// region, all of which are ancestor pivots.  Numeric phase (device, per
// setup): postorder over fronts, assemble original entries + children's
// update matrices (extend-add, fixed order), then the
// dense front in inverse form: (L11, W = L11^-1) by dense_chol_inv (densechol.cu),
// L21 = A21 W^T and M = [W; L21 W] by GEMM, S = A22 - L21 L21^T by syrk.  Solve (per V-cycle): forward
// sweep leaves -> root, z1 = L11^-1 y1 and u = y2 - L21 L11^-1 y1 in ONE
// GEMV with M, update vectors passed up the tree; backward sweep root ->
// leaves, x1 = M^T [z1; -x2] in one transposed GEMV.  Every front of a tree
// level runs in the same launches: the GEMVs are cut into fixed tiles
// (row block x column chunk) whose partial sums are reduced in a fixed
// order, so the solve is bandwidth-bound and deterministic.
#include "ndchol.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>

#include "densechol.hpp"
#include "dispatch.hpp"

namespace hxg {

namespace {

#ifndef HXG_ND_LEAF
#define HXG_ND_LEAF 256
#endif
constexpr int kLeafNodes = HXG_ND_LEAF;
#ifndef HXG_ND_LANE_DEPTH
#define HXG_ND_LANE_DEPTH 4
#endif
constexpr int kLaneDepth = HXG_ND_LANE_DEPTH;

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

__global__ void accumulate_info(int* dst, const int* src) {
  if (*src != 0 && *dst == 0) *dst = *src;
}
__global__ void zero_strict_upper(double* W, int ldw, int n) {
  const long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e / n), r = (int)(e % n);
    if (r < c) W[r + (size_t)c * ldw] = 0.0;
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

#ifndef HXG_ND_FC
#define HXG_ND_FC 128
#endif
#ifndef HXG_ND_BR
#define HXG_ND_BR 512
#endif
constexpr int kFR = 256;        // forward GEMV tile: rows (threads)
constexpr int kFC = HXG_ND_FC;  //                    columns (vector chunk in smem)
constexpr int kBC = 64;         // backward GEMV tile: columns (8 warps x 8)
constexpr int kBR = HXG_ND_BR;  //                     rows (vector chunk in smem)

// The panel of a front is [W; L21] (W = L11^-1): part 0 = the np x np top
// block (lower triangular), part 1 = the ns x np bottom block.
struct NdSolve {
  const int *piv0, *np, *ns, *child0, *child1;
  const long long *loff, *rows_off, *yoff, *uoff;
  const int *src0, *src1, *shell;
  const int* ftile0[2];       // per front: first forward tile of each part
  const int* btile0[2];       // per front: first backward tile of each part
  const int* ftile_front[2];  // forward tile -> front
  const int* btile_front[2];  // backward tile -> front
  const int* rtile_front[3];  // row tiles (front, rb): 0 top, 1 bottom, 2 whole front
  const int* rtile_rb[3];
  const int *ctile_front, *ctile_cb;  // column tiles (front, cb)
  const double* M;
  double *w, *u, *y, *part_f, *part_b;
};

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }
__device__ __forceinline__ int part_rows(int part, int np, int ns) { return part ? ns : np; }

// Forward front vector y = [w(piv); 0] + extend(u_child0) + extend(u_child1)
// (the children's update rows gathered through the inverse extend maps).
__global__ void __launch_bounds__(kFR) nd_fwd_assemble(NdSolve a, int rt0) {
  const int rt = rt0 + blockIdx.x, t = a.rtile_front[2][rt];
  const int np = a.np[t], m = np + a.ns[t];
  const int r = a.rtile_rb[2][rt] * kFR + threadIdx.x;
  if (r >= m) return;
  const long long yo = a.yoff[t];
  double v = r < np ? a.w[a.piv0[t] + r] : 0.0;
  const int s0 = a.src0[yo + r], s1 = a.src1[yo + r];
  if (s0 >= 0) v += a.u[a.uoff[a.child0[t]] + s0];
  if (s1 >= 0) v += a.u[a.uoff[a.child1[t]] + s1];
  a.y[yo + r] = v;
}

// Tile (row block rb of the part, column chunk cc) of part x y[0:np]: one
// row per thread.  Part 0: z1 = W y1; part 1: L21 z1 (z1 written back into
// y[0:np] by the part-0 finish).
__global__ void __launch_bounds__(kFR) nd_fwd_gemv(NdSolve a, int part, int ft0) {
  __shared__ double ys[kFC];
  const int tile = ft0 + blockIdx.x, t = a.ftile_front[part][tile];
  const int np = a.np[t], ns = a.ns[t], m = np + ns, nr = part_rows(part, np, ns);
  const int ncc = ceil_div(np, kFC), local = tile - a.ftile0[part][t];
  const int rb = local / ncc, cc = local - rb * ncc;
  const int row0 = rb * kFR, col0 = cc * kFC, ncols = min(kFC, np - col0);
  const int rend = min(row0 + kFR, nr);
  double* out = a.part_f + (size_t)tile * kFR;
  if (part == 0 && rend - 1 < col0) {  // strictly above the diagonal of W: zeros
    out[threadIdx.x] = 0.0;
    return;
  }
  const long long yo = a.yoff[t];
  for (int k = threadIdx.x; k < ncols; k += kFR) ys[k] = a.y[yo + col0 + k];
  __syncthreads();
  const int r = row0 + threadIdx.x;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (r < nr) {
    const double* col = a.M + a.loff[t] + (size_t)col0 * m + (part ? np : 0) + r;
    int k = 0;
    for (; k + 16 <= ncols; k += 16) {  // 16 loads in flight per thread
      double mv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) mv[q] = __ldg(col + (size_t)(k + q) * m);
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q & 3] = fma(mv[q], ys[k + q], acc[q & 3]);
    }
    for (; k < ncols; ++k) acc[k & 3] = fma(__ldg(col + (size_t)k * m), ys[k], acc[k & 3]);
  }
  out[threadIdx.x] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// Part 0: z1 -> w(piv) and y[0:np]; part 1: u = y2 - L21 z1 -> update vector.
__global__ void __launch_bounds__(kFR) nd_fwd_finish(NdSolve a, int part, int rt0) {
  const int rt = rt0 + blockIdx.x, t = a.rtile_front[part][rt];
  const int np = a.np[t], ns = a.ns[t], nr = part_rows(part, np, ns);
  const int rb = a.rtile_rb[part][rt], r = rb * kFR + threadIdx.x;
  if (r >= nr) return;
  const int ncc = ceil_div(np, kFC);
  const double* p = a.part_f + ((size_t)a.ftile0[part][t] + (size_t)rb * ncc) * kFR + threadIdx.x;
  double s = 0.0;
  for (int cc = 0; cc < ncc; ++cc) s += p[(size_t)cc * kFR];
  const long long yo = a.yoff[t];
  if (part == 0) {
    a.w[a.piv0[t] + r] = s;
    a.y[yo + r] = s;
  } else {
    a.u[a.uoff[t] + r] = a.y[yo + np + r] - s;
  }
}

// Backward front vector [z1; x2] (x2 = ancestor solution values).
__global__ void __launch_bounds__(kFR) nd_bwd_assemble(NdSolve a, int rt0) {
  const int rt = rt0 + blockIdx.x, t = a.rtile_front[2][rt];
  const int np = a.np[t], m = np + a.ns[t];
  const int r = a.rtile_rb[2][rt] * kFR + threadIdx.x;
  if (r >= m) return;
  a.y[a.yoff[t] + r] = r < np ? a.w[a.piv0[t] + r] : a.w[a.shell[a.rows_off[t] + (r - np)]];
}

// Tile (column block cb, row chunk rc of the part) of part^T v: 8 warps x 8
// columns, lanes stride the (contiguous) column, fixed-order warp reduction.
// Part 1: L21^T x2; part 0: W^T t.
__global__ void __launch_bounds__(256) nd_bwd_gemv(NdSolve a, int part, int bt0) {
  __shared__ double vs[kBR];
  const int tile = bt0 + blockIdx.x, t = a.btile_front[part][tile];
  const int np = a.np[t], ns = a.ns[t], m = np + ns, nr = part_rows(part, np, ns);
  const int nrc = ceil_div(nr, kBR), local = tile - a.btile0[part][t];
  const int cb = local / nrc, rc = local - cb * nrc;
  const int col0 = cb * kBC, row0 = rc * kBR, nrows = min(kBR, nr - row0);
  double* out = a.part_b + (size_t)tile * kBC;
  if (part == 0 && row0 + nrows <= col0) {  // rows above the diagonal of every column: zeros
    if (threadIdx.x < kBC) out[threadIdx.x] = 0.0;
    return;
  }
  const long long yo = a.yoff[t] + (part ? np : 0);
  for (int k = threadIdx.x; k < nrows; k += 256) vs[k] = a.y[yo + row0 + k];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* base = a.M + a.loff[t] + (part ? np : 0) + row0;
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  const int j0 = col0 + warp * 8;
  const int nq = min(8, np - j0);  // columns of this warp (warp-uniform)
  // 4 row strides per step: 32 loads in flight per lane
  int k = lane;
  if (nq == 8) {
    for (; k + 96 < nrows; k += 128) {
      double mv[4][8];
#pragma unroll
      for (int h = 0; h < 4; ++h)
#pragma unroll
        for (int q = 0; q < 8; ++q) mv[h][q] = __ldg(base + (size_t)(j0 + q) * m + k + 32 * h);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double vk = vs[k + 32 * h];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fma(mv[h][q], vk, acc[q]);
      }
    }
  }
  for (; k < nrows; k += 32) {
    const double vk = vs[k];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < nq) acc[q] = fma(__ldg(base + (size_t)(j0 + q) * m + k), vk, acc[q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
  }
  if (lane < 8) {
    double v = acc[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) v = lane == q ? acc[q] : v;
    out[warp * 8 + lane] = v;
  }
}

// Part 1: t = z1 - L21^T x2 -> y[0:np]; part 0: x1 = W^T t -> w(piv).
__global__ void __launch_bounds__(kBC) nd_bwd_finish(NdSolve a, int part, int ct0) {
  const int ct = ct0 + blockIdx.x, t = a.ctile_front[ct];
  const int np = a.np[t], ns = a.ns[t], nr = part_rows(part, np, ns);
  const int cb = a.ctile_cb[ct], j = cb * kBC + threadIdx.x;
  if (j >= np) return;
  const int nrc = ceil_div(nr, kBR);
  const double* p = a.part_b + ((size_t)a.btile0[part][t] + (size_t)cb * nrc) * kBC + threadIdx.x;
  double s = 0.0;
  for (int rc = 0; rc < nrc; ++rc) s += p[(size_t)rc * kBC];
  if (part == 1)
    a.y[a.yoff[t] + j] -= s;
  else
    a.w[a.piv0[t] + j] = s;
}

void cublas_check(cublasStatus_t s, const char* what) {
  if (s != CUBLAS_STATUS_SUCCESS) throw Error(HXG_ERR_CUDA, std::string(what) + " failed");
}

}  // namespace

NdCholesky::NdCholesky(long long leaf_nodes) : leaf_nodes_(leaf_nodes > 0 ? leaf_nodes : kLeafNodes) {}
NdCholesky::~NdCholesky() {
  if (graph_) cudaGraphExecDestroy(graph_);
  if (fgraph_) cudaGraphExecDestroy(fgraph_);
  if (gev_in_) cudaEventDestroy(gev_in_);
  if (gev_out_) cudaEventDestroy(gev_out_);
  if (gstream_) cudaStreamDestroy(gstream_);
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
    if (cnt > leaf_nodes_ && n[ax] >= 3) {
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
  }
  std::vector<int> maps;
  std::vector<int> spos((size_t)n_, -1);  // dense front-row lookup (filled per front)
  for (int t = 0; t < nf; ++t) {
    Front& f = fronts_[(size_t)t];
    const auto& sh = shell[(size_t)t];
    for (size_t i = 0; i < sh.size(); ++i) spos[(size_t)sh[i]] = f.np + (int)i;
    for (int q = 0; q < 2; ++q) {
      int c = f.child[q];
      f.map_off[q] = maps.size();
      if (c < 0) continue;
      for (int ni : shell[(size_t)c]) {
        const int p = ni >= f.piv0 && ni < f.piv0 + f.np ? ni - f.piv0 : spos[(size_t)ni];
        if (p < 0) throw Error(HXG_ERR_GENERIC, "child update row missing from parent front");
        maps.push_back(p);
      }
    }
    for (int r : sh) spos[(size_t)r] = -1;
  }
  // Assembly lists: lower-triangle original entries with a pivot column.
  std::vector<long long> adst;
  std::vector<int> asrc, afront;
  asm_begin_.assign((size_t)nf + 1, 0);
  // front-local row of a new index: a dense scratch map filled with the
  // front's shell rows (pivots are a contiguous range), O(1) lookups
  std::vector<int> shell_pos((size_t)n_, -1);
  for (int t = 0; t < nf; ++t) {
    const Front& f = fronts_[(size_t)t];
    const int m = f.np + f.ns;
    asm_begin_[(size_t)t] = adst.size();
    const auto& sh = shell[(size_t)t];
    for (size_t i = 0; i < sh.size(); ++i) shell_pos[(size_t)sh[i]] = f.np + (int)i;
    for (int pj = 0; pj < f.np; ++pj) {
      int jold = perm[(size_t)(f.piv0 + pj)];
      for (int k = a.row_ptr_h[(size_t)jold]; k < a.row_ptr_h[(size_t)jold + 1]; ++k) {
        int ni = newidx[(size_t)a.cols_h[(size_t)k]];
        if (ni < f.piv0) continue;  // eliminated in a descendant front
        const int pi = ni < f.piv0 + f.np ? ni - f.piv0 : shell_pos[(size_t)ni];
        if (pi < 0) throw Error(HXG_ERR_GENERIC, "matrix entry outside its front");
        if (pi < pj) continue;      // upper triangle
        adst.push_back((long long)pi + (long long)pj * m);
        asrc.push_back(k);
        afront.push_back(t);
      }
    }
    for (int r : sh) shell_pos[(size_t)r] = -1;
  }
  asm_begin_[(size_t)nf] = adst.size();

  // Levels for the batched solves and their GEMV tile lists.
  int maxlev = 0;
  for (const auto& f : fronts_) maxlev = std::max(maxlev, f.level);
  levels_.assign((size_t)maxlev + 1, {});
  for (int t = 0; t < nf; ++t) levels_[(size_t)fronts_[(size_t)t].level].push_back(t);
  auto cdiv = [](long long x, long long y) { return (int)((x + y - 1) / y); };
  std::vector<int> piv0(nf), np(nf), ns(nf), c0(nf), c1(nf);
  std::vector<int> ft0[2] = {std::vector<int>(nf), std::vector<int>(nf)};
  std::vector<int> bt0[2] = {std::vector<int>(nf), std::vector<int>(nf)};
  std::vector<long long> loff(nf), roff(nf), yoff(nf), uoff(nf);
  std::vector<int> ftf[2], btf[2], rtf[3], rtb[3], ctf, ctb;
  for (int q = 0; q < 2; ++q) {
    lev_ft_[q].assign(levels_.size() + 1, 0);
    lev_bt_[q].assign(levels_.size() + 1, 0);
  }
  for (int q = 0; q < 3; ++q) lev_rt_[q].assign(levels_.size() + 1, 0);
  lev_ct_.assign(levels_.size() + 1, 0);
  long long ucount = 0, ycount = 0;
  for (size_t l = 0; l <= levels_.size(); ++l) {
    for (int q = 0; q < 2; ++q) {
      lev_ft_[q][l] = (int)ftf[q].size();
      lev_bt_[q][l] = (int)btf[q].size();
    }
    for (int q = 0; q < 3; ++q) lev_rt_[q][l] = (int)rtf[q].size();
    lev_ct_[l] = (int)ctf.size();
    if (l == levels_.size()) break;
    for (int t : levels_[l]) {
      const Front& f = fronts_[(size_t)t];
      const int rows[3] = {f.np, f.ns, f.np + f.ns};
      for (int q = 0; q < 2; ++q) {
        ft0[q][t] = (int)ftf[q].size();
        for (int k = 0, n = cdiv(rows[q], kFR) * cdiv(f.np, kFC); k < n; ++k) ftf[q].push_back(t);
        bt0[q][t] = (int)btf[q].size();
        for (int k = 0, n = cdiv(f.np, kBC) * cdiv(rows[q], kBR); k < n; ++k) btf[q].push_back(t);
      }
      for (int q = 0; q < 3; ++q)
        for (int rb = 0; rb < cdiv(rows[q], kFR); ++rb) rtf[q].push_back(t), rtb[q].push_back(rb);
      for (int cb = 0; cb < cdiv(f.np, kBC); ++cb) ctf.push_back(t), ctb.push_back(cb);
    }
  }
  for (int t = 0; t < nf; ++t) {
    const Front& f = fronts_[(size_t)t];
    piv0[t] = f.piv0;
    np[t] = f.np;
    ns[t] = f.ns;
    c0[t] = f.child[0];
    c1[t] = f.child[1];
    loff[t] = (long long)f.loff;
    roff[t] = (long long)f.rows_off;
    uoff[t] = ucount;
    ucount += f.ns;
    yoff[t] = ycount;
    ycount += f.np + f.ns;
  }
  // Inverse extend maps: front position -> index in child q's update vector.
  std::vector<int> src0((size_t)ycount, -1), src1((size_t)ycount, -1);
  for (int t = 0; t < nf; ++t) {
    const Front& f = fronts_[(size_t)t];
    for (int q = 0; q < 2; ++q) {
      const int c = f.child[q];
      if (c < 0) continue;
      auto& src = q == 0 ? src0 : src1;
      const int nsc = fronts_[(size_t)c].ns;
      for (int k = 0; k < nsc; ++k) src[(size_t)yoff[t] + maps[f.map_off[q] + (size_t)k]] = k;
    }
  }

  // Device copies.
  auto up = [](DevBuf<int>& d, const std::vector<int>& v) {
    d.upload(v.empty() ? std::vector<int>{0} : v);
  };
  perm_.upload(perm);
  up(shell_rows_, shell_rows);
  up(child_map_, maps);
  asm_dst_.upload(adst);
  asm_src_.upload(asrc);
  (void)afront;
  up(dfront_piv0_, piv0);
  up(dfront_np_, np);
  up(dfront_ns_, ns);
  up(c0_, c0);
  up(c1_, c1);
  for (int q = 0; q < 2; ++q) {
    up(ftile0_[q], ft0[q]);
    up(btile0_[q], bt0[q]);
    up(ftile_front_[q], ftf[q]);
    up(btile_front_[q], btf[q]);
  }
  for (int q = 0; q < 3; ++q) {
    up(rtile_front_[q], rtf[q]);
    up(rtile_rb_[q], rtb[q]);
  }
  dfront_loff_.upload(loff);
  dfront_rows_off_.upload(roff);
  yoff_.upload(yoff);
  uoff_.upload(uoff);
  up(src0_, src0);
  up(src1_, src1);
  up(ctile_front_, ctf);
  up(ctile_cb_, ctb);
  ubuf_.alloc((size_t)std::max<long long>(ucount, 1));
  yvec_.alloc((size_t)std::max<long long>(ycount, 1));
  part_f_.alloc(std::max<size_t>(std::max(ftf[0].size(), ftf[1].size()), 1) * kFR);
  part_b_.alloc(std::max<size_t>(std::max(btf[0].size(), btf[1].size()), 1) * kBC);
  L_.alloc(lsize_);
  size_t maxnp = 1;
  for (const auto& f : fronts_) maxnp = std::max(maxnp, (size_t)f.np);
  wvec_.alloc((size_t)n_);
  info_.alloc(2 * (size_t)nf);  // first failed pivot per front
  analyzed_ = true;
}

// Lane = one stream + handles + workspaces.  The dissection tree is cut at
// depth kLaneDepth: each subtree there is factored on its own lane (its
// fronts are contiguous in postorder, with a private update stack), so the
// many small fronts of different subtrees run concurrently; the subtree
// roots hand their update matrices over in dedicated buffers, and the top
// fronts run on the caller's stream once every lane has finished.
struct NdCholesky::Lane {
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  cublasHandle_t cublas = nullptr;
  DevBuf<double> W, inv, tmp, stack, rscr, cublas_ws;
  std::vector<int> fronts;  // postorder
  bool own_stream = false;
  ~Lane() {
    if (cublas) cublasDestroy(cublas);
    if (done) cudaEventDestroy(done);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

void NdCholesky::plan_lanes() {
  const int nf = (int)fronts_.size();
  int maxlev = 0;
  for (const auto& f : fronts_) maxlev = std::max(maxlev, f.level);
  const int depth = std::min(kLaneDepth, maxlev);
  // subtree of each front: the ancestor at `depth` (or -1 for top fronts)
  std::vector<int> sub((size_t)nf, -1);
  std::vector<int> roots;
  for (int t = nf - 1; t >= 0; --t) {  // parents after children in postorder
    const Front& f = fronts_[(size_t)t];
    if (f.level == depth && depth > 0) {
      sub[(size_t)t] = (int)roots.size();
      roots.push_back(t);
    } else if (f.level > depth) {
      sub[(size_t)t] = sub[(size_t)f.parent];
    }
  }
  lanes_.clear();
  lanes_.resize(roots.size() + 1);  // lane 0 = the caller's stream
  for (auto& l : lanes_) l = std::make_unique<Lane>();
  lane_of_.assign((size_t)nf, 0);
  top_.clear();
  for (int t = 0; t < nf; ++t) {  // postorder: children before parents
    const Front& f = fronts_[(size_t)t];
    if (sub[(size_t)t] >= 0) {
      lane_of_[(size_t)t] = sub[(size_t)t] + 1;
      lanes_[(size_t)lane_of_[(size_t)t]]->fronts.push_back(t);
    } else {
      // a front above the lane depth runs on its first child's lane, after
      // the other child's lane has finished that child
      lane_of_[(size_t)t] = depth > 0 && f.child[0] >= 0 ? lane_of_[(size_t)f.child[0]] : 0;
      if (depth > 0)
        top_.push_back(t);
      else
        lanes_[0]->fronts.push_back(t);
    }
  }
  handoff_off_.assign((size_t)nf, (size_t)-1);
  size_t hsize = 0;
  for (int t = 0; t < nf; ++t) {
    if (depth == 0 || fronts_[(size_t)t].level > depth) continue;
    handoff_off_[(size_t)t] = hsize;  // subtree roots and the fronts above them
    hsize += (size_t)fronts_[(size_t)t].ns * fronts_[(size_t)t].ns;
  }
  handoff_.alloc(std::max<size_t>(hsize, 1));
  for (size_t li = 0; li < lanes_.size(); ++li) {
    Lane& L = *lanes_[li];
    if (li > 0) {
      HXG_CUDA(cudaStreamCreateWithFlags(&L.stream, cudaStreamNonBlocking));
      L.own_stream = true;
    }
    HXG_CUDA(cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming));
    cublas_check(cublasCreate(&L.cublas), "cublasCreate");
    L.cublas_ws.alloc((size_t)4 << 20);  // 32 MiB: no lazy allocation inside a capture
    cublas_check(cublasSetWorkspace(L.cublas, L.cublas_ws.p, L.cublas_ws.n * sizeof(double)),
                 "cublasSetWorkspace");
    cublasSetStream(L.cublas, L.stream);
    dense_chol_inv_warmup(L.cublas, L.stream);  // module loads / attributes outside any capture
    size_t mw = 1, mi = 1, mt = 1, ms = 1, cur = 0, peak = 1;
    std::vector<size_t> st;
    std::vector<int> mine = L.fronts;
    for (int t : top_)
      if (lane_of_[(size_t)t] == (int)li) mine.push_back(t);
    for (int t : mine) {
      const Front& f = fronts_[(size_t)t];
      const size_t m = (size_t)f.np + f.ns;
      mw = std::max(mw, m * m);
      mi = std::max(mi, (size_t)f.np * f.np);
      mt = std::max(mt, (size_t)f.np * f.ns);
      ms = std::max(ms, dense_chol_inv_scratch(f.np));
      // private stack: children in this lane are popped, the front pushed
      // (unless its update is handed over)
      for (int q = 0; q < 2; ++q) {
        const int c = f.child[q];
        if (c >= 0 && lane_of_[(size_t)c] == (int)li && handoff_off_[(size_t)c] == (size_t)-1) {
          cur -= st.back();
          st.pop_back();
        }
      }
      if (handoff_off_[(size_t)t] == (size_t)-1) {
        st.push_back((size_t)f.ns * f.ns);
        cur += st.back();
        peak = std::max(peak, cur);
      }
    }
    L.W.alloc(mw);
    L.inv.alloc(mi);
    L.tmp.alloc(mt);
    L.stack.alloc(peak);
    L.rscr.alloc(ms);  // dense_chol_inv's n2 x n1 scratch
  }
}

void NdCholesky::factor_front(int t, Lane& L, const CsrMatrix& a,
                              std::vector<std::pair<size_t, int>>& stack) {
  const Front& f = fronts_[(size_t)t];
  const int m = f.np + f.ns;
  cudaStream_t s = L.stream;
  const double one = 1.0, minus_one = -1.0, zero = 0.0;
  double* W = L.W.p;
  HXG_CUDA(cudaMemsetAsync(W, 0, sizeof(double) * (size_t)m * m, s));
  const long long na = (long long)(asm_begin_[(size_t)t + 1] - asm_begin_[(size_t)t]);
  if (na > 0)
    assemble_kernel<<<grid_for(na, 256), 256, 0, s>>>(asm_dst_.p + asm_begin_[(size_t)t],
                                                      asm_src_.p + asm_begin_[(size_t)t], na,
                                                      a.vals.p, W);
  // Children's updates: handed-over buffers, else this lane's stack (child[1]
  // above child[0]); extend-add in child order.
  const double* up[2] = {nullptr, nullptr};
  for (int q = 1; q >= 0; --q) {
    const int c = f.child[q];
    if (c < 0) continue;
    if (handoff_off_[(size_t)c] != (size_t)-1) {
      up[q] = handoff_.p + handoff_off_[(size_t)c];
    } else {
      up[q] = L.stack.p + stack.back().first;
      stack.pop_back();
    }
  }
  for (int q = 0; q < 2; ++q) {
    const int c = f.child[q];
    if (c < 0 || fronts_[(size_t)c].ns == 0) continue;
    const int nsc = fronts_[(size_t)c].ns;
    extend_add_kernel<<<grid_for((long long)nsc * nsc, 256), 256, 0, s>>>(
        up[q], nsc, child_map_.p + f.map_off[q], W, m);
  }
  HXG_CUDA(cudaGetLastError());
  // Dense partial factorization in inverse form, all level-3 work on FP64
  // tensor-core GEMMs (the cuBLAS trsm kernels are not): L11 = potrf(A11);
  // W = L11^-1 (trtri; the front's upper half is zero, so W's is too);
  // L21 = A21 W^T; S = A22 - L21 L21^T (syrk); M = [W; L21 W] written
  // straight into the factor.
  HXG_CUDA(cudaMemsetAsync(L.inv.p, 0, sizeof(double) * (size_t)f.np * f.np, s));
  dense_chol_inv(L.cublas, s, W, m, L.inv.p, f.np, f.np, info_.p + t, L.rscr.p);
  double* Lp = L_.p + f.loff;
  if (f.ns > 0) {
    // L21 = A21 W^T straight into the factor panel, then S = A22 - L21 L21^T
    cublas_check(cublasDgemm(L.cublas, CUBLAS_OP_N, CUBLAS_OP_T, f.ns, f.np, f.np, &one, W + f.np,
                             m, L.inv.p, f.np, &zero, Lp + f.np, m),
                 "gemm (L21)");
    cublas_check(cublasDsyrk(L.cublas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, f.ns, f.np, &minus_one,
                             Lp + f.np, m, &one, W + f.np + (size_t)f.np * m, m),
                 "syrk");
  }
  HXG_CUDA(cudaMemcpy2DAsync(Lp, sizeof(double) * m, L.inv.p, sizeof(double) * f.np,
                             sizeof(double) * f.np, f.np, cudaMemcpyDeviceToDevice, s));
  if (f.ns > 0) {
    double* dst;
    if (handoff_off_[(size_t)t] != (size_t)-1) {
      dst = handoff_.p + handoff_off_[(size_t)t];
    } else {
      const size_t top = stack.empty() ? 0
                                       : stack.back().first + (size_t)stack.back().second *
                                                                  stack.back().second;
      dst = L.stack.p + top;
      stack.emplace_back(top, f.ns);
    }
    HXG_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * f.ns, W + f.np + (size_t)f.np * m,
                               sizeof(double) * m, sizeof(double) * f.ns, f.ns,
                               cudaMemcpyDeviceToDevice, s));
  } else if (handoff_off_[(size_t)t] == (size_t)-1) {
    const size_t top = stack.empty() ? 0
                                     : stack.back().first + (size_t)stack.back().second *
                                                                stack.back().second;
    stack.emplace_back(top, 0);
  }
}

void NdCholesky::factorize(const CsrMatrix& a, const int npd[3], cudaStream_t s) {
  if (graph_) {  // the captured solve holds the previous buffers' launch parameters
    cudaGraphExecDestroy(graph_);
    graph_ = nullptr;
  }
  if (!analyzed_) {
    static const bool prof0 = std::getenv("HXG_PROFILE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    analyze(a, npd);
    auto t1 = std::chrono::steady_clock::now();
    plan_lanes();
    auto t2 = std::chrono::steady_clock::now();
    if (prof0)
      std::fprintf(stderr, "[hxg]   symbolic: analyze %.1f ms, lanes %.1f ms\n",
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(t2 - t1).count());
  }
  ready_ = false;
  // The numeric factorisation is ~40 k launches over 16 streams, fixed per
  // pattern: it is captured once into a graph (first call) and replayed,
  // which removes the host launch cost (HXG_NO_GRAPH=1 or HXG_PROFILE keep
  // it eager; a failed capture falls back to eager launches).
  static const bool no_fgraph = std::getenv("HXG_NO_GRAPH") != nullptr || std::getenv("HXG_PROFILE") != nullptr;
  if (!no_fgraph && !fgraph_failed_) {
    if (fgraph_ && fgraph_vals_ != a.vals.p) {
      cudaGraphExecDestroy(fgraph_);
      fgraph_ = nullptr;
    }
    if (!gstream_) {
      HXG_CUDA(cudaStreamCreateWithFlags(&gstream_, cudaStreamNonBlocking));
      HXG_CUDA(cudaEventCreateWithFlags(&gev_in_, cudaEventDisableTiming));
      HXG_CUDA(cudaEventCreateWithFlags(&gev_out_, cudaEventDisableTiming));
    }
    if (!fgraph_) {
      cudaGraph_t g = nullptr;
      try {
        HXG_CUDA(cudaStreamBeginCapture(gstream_, cudaStreamCaptureModeThreadLocal));
        factor_launch(a, gstream_);
        HXG_CUDA(cudaStreamEndCapture(gstream_, &g));
        HXG_CUDA(cudaGraphInstantiate(&fgraph_, g, 0));
        cudaGraphDestroy(g);
        fgraph_vals_ = a.vals.p;
      } catch (const Error&) {
        cudaGraph_t junk = nullptr;
        cudaStreamEndCapture(gstream_, &junk);
        if (junk) cudaGraphDestroy(junk);
        if (g) cudaGraphDestroy(g);
        fgraph_ = nullptr;
        cudaGetLastError();
        fgraph_failed_ = true;
      }
    }
    if (fgraph_) {
      HXG_CUDA(cudaEventRecord(gev_in_, s));
      HXG_CUDA(cudaStreamWaitEvent(gstream_, gev_in_, 0));
      HXG_CUDA(cudaGraphLaunch(fgraph_, gstream_));
      HXG_CUDA(cudaEventRecord(gev_out_, gstream_));
      HXG_CUDA(cudaStreamWaitEvent(s, gev_out_, 0));
    } else {
      factor_launch(a, s);
    }
  } else {
    factor_launch(a, s);
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

// Every launch of one numeric factorisation, ordered after earlier work on s
// and joined back into s.
void NdCholesky::factor_launch(const CsrMatrix& a, cudaStream_t s) {
  Lane& top = *lanes_[0];
  top.stream = s;
  for (auto& l : lanes_) {
    cublasSetStream(l->cublas, l->stream);
  }
  HXG_CUDA(cudaMemsetAsync(info_.p, 0, 2 * sizeof(int) * fronts_.size(), s));
  // The subtree lanes start after earlier work on the caller's stream.
  HXG_CUDA(cudaEventRecord(top.done, s));
  for (size_t li = 1; li < lanes_.size(); ++li)
    HXG_CUDA(cudaStreamWaitEvent(lanes_[li]->stream, top.done, 0));
  // Round-robin issue over the subtree lanes keeps every stream fed.
  std::vector<std::vector<std::pair<size_t, int>>> stacks(lanes_.size());
  std::vector<size_t> next(lanes_.size(), 0);
  for (bool more = true; more;) {
    more = false;
    for (size_t li = 1; li < lanes_.size(); ++li) {
      Lane& L = *lanes_[li];
      if (next[li] < L.fronts.size()) {
        factor_front(L.fronts[next[li]++], L, a, stacks[li]);
        more = more || next[li] < L.fronts.size();
      }
    }
  }
  static const bool prof = std::getenv("HXG_PROFILE") != nullptr;
  std::chrono::steady_clock::time_point t0;
  if (prof) {
    for (auto& l : lanes_) HXG_CUDA(cudaStreamSynchronize(l->stream));
    t0 = std::chrono::steady_clock::now();
  }
  // Fronts above the lane depth, in postorder, each on its first child's
  // lane once the other child's lane has finished (up to 2^level fronts of a
  // level run concurrently).
  for (int t : top_) {
    Lane& L = *lanes_[(size_t)lane_of_[(size_t)t]];
    for (int c : fronts_[(size_t)t].child) {
      if (c < 0 || lane_of_[(size_t)c] == lane_of_[(size_t)t]) continue;
      Lane& C = *lanes_[(size_t)lane_of_[(size_t)c]];
      HXG_CUDA(cudaEventRecord(C.done, C.stream));
      HXG_CUDA(cudaStreamWaitEvent(L.stream, C.done, 0));
    }
    factor_front(t, L, a, stacks[(size_t)lane_of_[(size_t)t]]);
  }
  for (int t : top.fronts) factor_front(t, top, a, stacks[0]);  // depth-0 trees
  for (size_t li = 1; li < lanes_.size(); ++li) {
    HXG_CUDA(cudaEventRecord(lanes_[li]->done, lanes_[li]->stream));
    HXG_CUDA(cudaStreamWaitEvent(s, lanes_[li]->done, 0));
  }
  if (prof) {
    HXG_CUDA(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[hxg]   fronts above the lanes (%zu) %.2f ms\n", top_.size(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                     .count());
  }
}

void NdCholesky::solve(const double* b, double* x, cudaStream_t s) {
  if (!ready_) throw Error(HXG_ERR_GENERIC, "coarse solver not factorized");
  static const bool direct = std::getenv("HXG_NO_GRAPH") != nullptr;
  // The permutations touch the caller's vectors and run on the caller's
  // stream; the per-level core (internal buffers only) is the graph, so it
  // does not depend on b / x and is captured once per factorization.
  permute_gather<<<grid_for(n_, 256), 256, 0, s>>>(b, perm_.p, n_, wvec_.p);
  HXG_CUDA(cudaGetLastError());
  if (direct) {
    solve_launch(s);
  } else {
    run_graph(s);
  }
  permute_scatter<<<grid_for(n_, 256), 256, 0, s>>>(wvec_.p, perm_.p, n_, x);
  HXG_CUDA(cudaGetLastError());
}

void NdCholesky::run_graph(cudaStream_t s) {
  if (!gstream_) {
    HXG_CUDA(cudaStreamCreateWithFlags(&gstream_, cudaStreamNonBlocking));
    HXG_CUDA(cudaEventCreateWithFlags(&gev_in_, cudaEventDisableTiming));
    HXG_CUDA(cudaEventCreateWithFlags(&gev_out_, cudaEventDisableTiming));
  }
  if (!graph_) {
    cudaGraph_t g = nullptr;
    HXG_CUDA(cudaStreamBeginCapture(gstream_, cudaStreamCaptureModeThreadLocal));
    solve_launch(gstream_);
    HXG_CUDA(cudaStreamEndCapture(gstream_, &g));
    HXG_CUDA(cudaGraphInstantiate(&graph_, g, 0));
    cudaGraphDestroy(g);
  }
  HXG_CUDA(cudaEventRecord(gev_in_, s));
  HXG_CUDA(cudaStreamWaitEvent(gstream_, gev_in_, 0));
  HXG_CUDA(cudaGraphLaunch(graph_, gstream_));
  HXG_CUDA(cudaEventRecord(gev_out_, gstream_));
  HXG_CUDA(cudaStreamWaitEvent(s, gev_out_, 0));
}

void NdCholesky::solve_launch(cudaStream_t s) {
  NdSolve a;
  a.piv0 = dfront_piv0_.p;
  a.np = dfront_np_.p;
  a.ns = dfront_ns_.p;
  a.child0 = c0_.p;
  a.child1 = c1_.p;
  a.loff = dfront_loff_.p;
  a.rows_off = dfront_rows_off_.p;
  a.yoff = yoff_.p;
  a.uoff = uoff_.p;
  a.src0 = src0_.p;
  a.src1 = src1_.p;
  a.shell = shell_rows_.p;
  for (int q = 0; q < 2; ++q) {
    a.ftile0[q] = ftile0_[q].p;
    a.btile0[q] = btile0_[q].p;
    a.ftile_front[q] = ftile_front_[q].p;
    a.btile_front[q] = btile_front_[q].p;
  }
  for (int q = 0; q < 3; ++q) {
    a.rtile_front[q] = rtile_front_[q].p;
    a.rtile_rb[q] = rtile_rb_[q].p;
  }
  a.ctile_front = ctile_front_.p;
  a.ctile_cb = ctile_cb_.p;
  a.M = L_.p;
  a.w = wvec_.p;
  a.u = ubuf_.p;
  a.y = yvec_.p;
  a.part_f = part_f_.p;
  a.part_b = part_b_.p;
  auto n_of = [](const std::vector<int>& lev, size_t l) { return lev[l + 1] - lev[l]; };
  // Forward, deepest level first: y = [y1; y2] assembled; z1 = W y1;
  // u = y2 - L21 z1 passed up.
  for (int l = (int)levels_.size() - 1; l >= 0; --l) {
    const size_t L = (size_t)l;
    if (!n_of(lev_rt_[2], L)) continue;
    nd_fwd_assemble<<<n_of(lev_rt_[2], L), kFR, 0, s>>>(a, lev_rt_[2][L]);
    for (int part = 0; part < 2; ++part) {
      if (n_of(lev_ft_[part], L))
        nd_fwd_gemv<<<n_of(lev_ft_[part], L), kFR, 0, s>>>(a, part, lev_ft_[part][L]);
      if (n_of(lev_rt_[part], L))
        nd_fwd_finish<<<n_of(lev_rt_[part], L), kFR, 0, s>>>(a, part, lev_rt_[part][L]);
    }
  }
  // Backward, root first: t = z1 - L21^T x2; x1 = W^T t.
  for (size_t l = 0; l < levels_.size(); ++l) {
    if (!n_of(lev_rt_[2], l)) continue;
    nd_bwd_assemble<<<n_of(lev_rt_[2], l), kFR, 0, s>>>(a, lev_rt_[2][l]);
    for (int part = 1; part >= 0; --part) {
      if (n_of(lev_bt_[part], l))
        nd_bwd_gemv<<<n_of(lev_bt_[part], l), 256, 0, s>>>(a, part, lev_bt_[part][l]);
      if (part == 0 || n_of(lev_bt_[part], l))
        nd_bwd_finish<<<n_of(lev_ct_, l), kBC, 0, s>>>(a, part, lev_ct_[l]);
    }
  }
  HXG_CUDA(cudaGetLastError());
}

}  // namespace hxg
