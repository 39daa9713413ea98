// Jacobi diagonal (extract_diagonal, operator.hpp:247-283) and element
// matrices for the assembled coarse operator (coo_numeric,
// assembly.hpp:188-230): pointwise 9x9 tensors by probing the linear
// Jacobian q-function (pointwise_jacobian_tensor, operator.hpp:233-243),
// contracted with the dense tabulation (dense_tabulation, basis.hpp:424-451).
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"
#include "element.cuh"
#include "qfunction.cuh"
#include "qfunction_initial.cuh"

namespace hxg {

struct DiagParams {
  BoxDev box;
  QLayout lay;
  const double* interp;  // Q x N
  const double* deriv;   // Q x N
  const double* state;
  const double* geo;  // geometric factors (w detJ for the perturbation hook)
  double mu, lambda, perturb;
  int storage;  // JacobianStorage of the state
  double* out;  // diag: E-vector (e, c, a); assembly: (e, 3N^3, 3N^3)
};

__device__ __forceinline__ long long state_offset(const QLayout& lay, long long e, int qpt, int S) {
  long long ex = e % lay.cells[0], ey = (e / lay.cells[0]) % lay.cells[1],
            ez = e / ((long long)lay.cells[0] * lay.cells[1]);
  long long bx = ex / lay.B[0], by = ey / lay.B[1], bz = ez / lay.B[2];
  int lx = (int)(ex - bx * lay.B[0]), ly = (int)(ey - by * lay.B[1]), lz = (int)(ez - bz * lay.B[2]);
  long long brick = bx + lay.nb[0] * (by + (long long)lay.nb[1] * bz);
  int le = lx + lay.B[0] * (ly + lay.B[1] * lz);
  int Q = lay.Q;
  int qx = qpt % Q, qy = (qpt / Q) % Q, qz = qpt / (Q * Q);
  int t = (qy * Q + qx) * (lay.B[0] * lay.B[1] * lay.B[2]) + le;
  return ((brick * Q + qz) * state_row(S, Q)) * (long long)lay.T + state_lane(t, Q);
}

// D[(c1,d1),(c2,d2)] at one point: 9 probes of the Jacobian q-function.
__device__ __forceinline__ void point_tensor(const DiagParams& prm, long long e, int qpt,
                                             double* d81) {
  const int S = device_state_stride(prm.storage);
  long long off = state_offset(prm.lay, e, qpt, S);
  double st[kMaxStateStride];
  for (int s = 0; s < S; ++s) st[s] = prm.state[off + state_pair_off(s, prm.lay.T, prm.lay.Q)];
  for (int u = 0; u < 9; ++u) {
    double G[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, H[9];
    G[u] = 1.0;
    switch (prm.storage) {
      case kStorageInitialNative: jacobian_qf_initial<kStorageInitialNative>(prm.mu, prm.lambda, G, st, H); break;
      case kStorageInitialTuned: jacobian_qf_initial<kStorageInitialTuned>(prm.mu, prm.lambda, G, st, H); break;
      case kStorageInitialAD: jacobian_qf_initial<kStorageInitialAD>(prm.mu, prm.lambda, G, st, H); break;
      default: jacobian_qf(prm.mu, prm.lambda, G, st, H);
    }
    if (prm.perturb != 0.0) {  // + eps w detJ G (w detJ = geometry scalar 9, same point)
      const long long T = prm.lay.T, row = off / T / state_row(S, prm.lay.Q);
      const long long t = state_paired(prm.lay.Q) ? (off % (2 * T)) / 2 : off % T;
      H[u] += prm.perturb * prm.geo[(row * kGeoStride + 9) * T + t];
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) d81[k * 9 + u] = H[k];
  }
}

// Dense-tabulation gradient of node a at point q (basis.hpp:439-447).
template <int N, int Q>
__device__ __forceinline__ void tab_grad(const double* sI, const double* sDv, int a, int qpt,
                                         double ga[3]) {
  int i = a % N, j = (a / N) % N, k = a / (N * N);
  int qa = qpt % Q, qb = (qpt / Q) % Q, qc = qpt / (Q * Q);
  double bi = sI[qa * N + i], bj = sI[qb * N + j], bk = sI[qc * N + k];
  double di = sDv[qa * N + i], dj = sDv[qb * N + j], dk = sDv[qc * N + k];
  ga[0] = di * bj * bk;
  ga[1] = bi * dj * bk;
  ga[2] = bi * bj * dk;
}

// One CTA per element.  Shared: interp, deriv, then per point the 27 entries
// D[(c,d1),(c,d2)].
template <int P, int Q>
__global__ void diag_element_kernel(DiagParams prm) {
  constexpr int N = P + 1, N3 = N * N * N, Q3 = Q * Q * Q;
  extern __shared__ double smem[];
  double* sI = smem;
  double* sDv = smem + Q * N;
  double* sT = smem + 2 * Q * N;  // Q3 * 27
  long long e = blockIdx.x;
  for (int r = threadIdx.x; r < Q * N; r += blockDim.x) {
    sI[r] = prm.interp[r];
    sDv[r] = prm.deriv[r];
  }
  // one q-function probe per thread (point, column u = (c, d2)): the
  // diagonal blocks need D[(c, d1), (c, d2)], i.e. rows c of every column
  const int S = device_state_stride(prm.storage);
  for (int w = threadIdx.x; w < Q3 * 9; w += blockDim.x) {
    const int qpt = w / 9, u = w - 9 * qpt, c = u / 3, d2 = u - 3 * c;
    const long long off = state_offset(prm.lay, e, qpt, S);
    double st[kMaxStateStride];
    for (int s = 0; s < S; ++s) st[s] = prm.state[off + state_pair_off(s, prm.lay.T, prm.lay.Q)];
    double G[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, H[9];
    G[u] = 1.0;
    switch (prm.storage) {
      case kStorageInitialNative: jacobian_qf_initial<kStorageInitialNative>(prm.mu, prm.lambda, G, st, H); break;
      case kStorageInitialTuned: jacobian_qf_initial<kStorageInitialTuned>(prm.mu, prm.lambda, G, st, H); break;
      case kStorageInitialAD: jacobian_qf_initial<kStorageInitialAD>(prm.mu, prm.lambda, G, st, H); break;
      default: jacobian_qf(prm.mu, prm.lambda, G, st, H);
    }
    if (prm.perturb != 0.0) {  // + eps w detJ G (as point_tensor)
      const long long T = prm.lay.T, row = off / T / state_row(S, prm.lay.Q);
      const long long t = state_paired(prm.lay.Q) ? (off % (2 * T)) / 2 : off % T;
      H[u] += prm.perturb * prm.geo[(row * kGeoStride + 9) * T + t];
    }
#pragma unroll
    for (int d1 = 0; d1 < 3; ++d1) sT[qpt * 27 + (c * 3 + d1) * 3 + d2] = H[c * 3 + d1];
  }
  __syncthreads();
  for (int r = threadIdx.x; r < 3 * N3; r += blockDim.x) {
    int a = r / 3, c = r % 3;
    double sum = 0.0;
    for (int qpt = 0; qpt < Q3; ++qpt) {
      double ga[3];
      tab_grad<N, Q>(sI, sDv, a, qpt, ga);
      const double* d = sT + qpt * 27 + c * 9;
#pragma unroll
      for (int d1 = 0; d1 < 3; ++d1)
#pragma unroll
        for (int d2 = 0; d2 < 3; ++d2) sum += ga[d1] * d[d1 * 3 + d2] * ga[d2];
    }
    prm.out[(e * 3 + c) * N3 + a] = sum;
  }
}

// Element matrix entries (a, ca, b, cb) in the reference COO order
// (coo_numeric, assembly.hpp:202-224).  One CTA per element; shared holds
// the full 81-entry tensor per point.
template <int P, int Q>
__global__ void assemble_element_kernel(DiagParams prm) {
  constexpr int N = P + 1, N3 = N * N * N, Q3 = Q * Q * Q, M = 3 * N3;
  extern __shared__ double smem[];
  double* sI = smem;
  double* sDv = smem + Q * N;
  double* sT = smem + 2 * Q * N;  // Q3 * 81
  long long e = blockIdx.x;
  for (int r = threadIdx.x; r < Q * N; r += blockDim.x) {
    sI[r] = prm.interp[r];
    sDv[r] = prm.deriv[r];
  }
  for (int qpt = threadIdx.x; qpt < Q3; qpt += blockDim.x) point_tensor(prm, e, qpt, sT + qpt * 81);
  __syncthreads();
  for (int r = threadIdx.x; r < M * M; r += blockDim.x) {
    int row = r / M, col = r % M;
    int a = row / 3, ca = row % 3, b = col / 3, cb = col % 3;
    double sum = 0.0;
    for (int qpt = 0; qpt < Q3; ++qpt) {
      double ga[3], gb[3];
      tab_grad<N, Q>(sI, sDv, a, qpt, ga);
      tab_grad<N, Q>(sI, sDv, b, qpt, gb);
      const double* drow = sT + qpt * 81 + (ca * 3) * 9 + cb * 3;
      sum += ga[0] * (drow[0] * gb[0] + drow[1] * gb[1] + drow[2] * gb[2]);
      sum += ga[1] * (drow[9] * gb[0] + drow[10] * gb[1] + drow[11] * gb[2]);
      sum += ga[2] * (drow[18] * gb[0] + drow[19] * gb[1] + drow[20] * gb[2]);
    }
    prm.out[e * (long long)(M * M) + r] = sum;
  }
}

// p = 1 element matrices (the coarse level's, coo_numeric assembly.hpp:
// 188-230): K[(a,ca),(b,cb)] = sum_q sum_i g_a,i(q) sum_j D_q[(ca,i),(cb,j)]
// g_b,j(q).  Per chunk of points, D_q by one q-function probe per thread
// (point, column) and the node gradients into shared memory; then thread
// (point group, column (ca, b, cb)) forms t_i = sum_j D_q[(ca,i),(cb,j)] g_b,j
// and accumulates all 8 rows a (the g_a,i are warp-uniform broadcasts); the
// 4 point groups are reduced in fixed order.  ~40 k flops per element and no
// materialised intermediate (shared-memory traffic was the limiter).
constexpr int kQ1AsmThreads = 288;
constexpr int kQ1AsmChunk = 27;
template <int Q, int ST>
__global__ void __launch_bounds__(kQ1AsmThreads, 2) assemble_element_q1_kernel(DiagParams prm) {
  constexpr int N = 2, N3 = 8, Q3 = Q * Q * Q, M = 3 * N3, QC = kQ1AsmChunk;
  extern __shared__ double smem[];
  double* sD = smem;              // QC x 81; reused for the group reduction
  double* sG = sD + QC * 81;      // QC x 8 x 3
  const long long e = blockIdx.x;
  const int tid = threadIdx.x;
  constexpr int S = device_state_stride(ST);
  const int combo = tid % 72, grp = tid / 72;  // 72 columns (ca, b, cb) x 4 point groups
  const int ca = combo / 24, bc = combo - 24 * ca, b = bc / 3, cb = bc - 3 * b;
  double acc[N3] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int q0 = 0; q0 < Q3; q0 += QC) {
    const int qn = Q3 - q0 < QC ? Q3 - q0 : QC;
    for (int w = tid; w < qn * 9; w += kQ1AsmThreads) {  // D_q column u of point ql
      const int ql = w / 9, u = w - 9 * ql, qpt = q0 + ql;
      const long long off = state_offset(prm.lay, e, qpt, S);
      double st[S];
#pragma unroll
      for (int s = 0; s < S; ++s) st[s] = prm.state[off + state_pair_off(s, prm.lay.T, prm.lay.Q)];
      double G[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, H[9];
      G[u] = 1.0;
      if constexpr (ST == kStorageCurrent)
        jacobian_qf(prm.mu, prm.lambda, G, st, H);
      else
        jacobian_qf_initial<ST>(prm.mu, prm.lambda, G, st, H);
      if (prm.perturb != 0.0) {  // + eps w detJ G (as point_tensor)
        const long long T = prm.lay.T, row = off / T / state_row(S, prm.lay.Q);
        const long long t = state_paired(prm.lay.Q) ? (off % (2 * T)) / 2 : off % T;
        H[u] += prm.perturb * prm.geo[(row * kGeoStride + 9) * T + t];
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) sD[ql * 81 + k * 9 + u] = H[k];
    }
    // node gradients at the chunk's points (dense tabulation, basis.hpp:439-447)
    for (int w = tid; w < qn * N3; w += kQ1AsmThreads) {
      const int ql = w / N3, a = w - N3 * ql, qpt = q0 + ql;
      const int i = a & 1, j = (a >> 1) & 1, k = a >> 2;
      const int qa = qpt % Q, qb = (qpt / Q) % Q, qc = qpt / (Q * Q);
      const double bi = prm.interp[qa * N + i], bj = prm.interp[qb * N + j], bk = prm.interp[qc * N + k];
      const double di = prm.deriv[qa * N + i], dj = prm.deriv[qb * N + j], dk = prm.deriv[qc * N + k];
      sG[(ql * N3 + a) * 3 + 0] = di * bj * bk;
      sG[(ql * N3 + a) * 3 + 1] = bi * dj * bk;
      sG[(ql * N3 + a) * 3 + 2] = bi * bj * dk;
    }
    __syncthreads();
    for (int ql = grp; ql < qn; ql += 4) {
      const double* d = sD + ql * 81 + (ca * 3) * 9 + cb * 3;
      const double* gb = sG + (ql * N3 + b) * 3;
      const double g0 = gb[0], g1 = gb[1], g2 = gb[2];
      const double t0 = d[0] * g0 + d[1] * g1 + d[2] * g2;
      const double t1 = d[9] * g0 + d[10] * g1 + d[11] * g2;
      const double t2 = d[18] * g0 + d[19] * g1 + d[20] * g2;
      const double* g = sG + ql * N3 * 3;
#pragma unroll
      for (int a = 0; a < N3; ++a) acc[a] += g[a * 3 + 0] * t0 + g[a * 3 + 1] * t1 + g[a * 3 + 2] * t2;
    }
    __syncthreads();
  }
  // reduce the 4 point groups in fixed order ([grp][combo][a] over the D + G buffers)
  double* red = sD;
#pragma unroll
  for (int a = 0; a < N3; ++a) red[(grp * 72 + combo) * N3 + a] = acc[a];
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int idx = tid + h * kQ1AsmThreads;  // (a ca) * 24 + (b cb)
    const int rowi = idx / M, col = idx - rowi * M, a = rowi / 3, car = rowi - 3 * a;
    const int cmb = car * 24 + col;
    double v = 0.0;
#pragma unroll
    for (int g = 0; g < 4; ++g) v += red[(g * 72 + cmb) * N3 + a];
    prm.out[e * (long long)(M * M) + idx] = v;
  }
}

}  // namespace hxg
