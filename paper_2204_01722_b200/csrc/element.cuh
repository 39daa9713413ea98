// Sum-factorised tensor-product basis on one element, one thread per
// quadrature column (qx, qy) holding all qz in registers
// (grad_slab / grad_transpose_slab, basis.hpp:319-355).
//
// Contractions along z stay in registers; x and y go through two per-element
// shared-memory slabs S1, S2 of Q^3 doubles.  Every thread of the CTA must
// call these (they contain __syncthreads()).
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"

namespace hxg {

template <int P, int Q>
struct Dims {
  static constexpr int N = P + 1;
  static constexpr int N3 = N * N * N;
  static constexpr int Q2 = Q * Q;
  static constexpr int Q3 = Q * Q * Q;
  static constexpr int BX = brick_x(Q), BY = brick_y(Q), BZ = brick_z(Q);
  static constexpr int NE = BX * BY * BZ;  // elements per brick
  static constexpr int T = NE * Q2;        // threads per CTA
  // Per-element shared scratch: U (3 N^3 nodal values) + S1 + S2.
  static constexpr int ELEM_SMEM = 3 * N3 + 2 * Q3;
  // Basis tables in shared memory: B (Q x N), Dc (Q x Q).
  static constexpr int TAB = Q * N + Q * Q;
};

// Forward: nodal U (N^3, x-fastest) of one component -> reference gradient
// g[d][qz] at this thread's column.  interp (x, y, z), then the collocated
// derivative per direction (basis.hpp:319-335).
// U(k, j, i) = U[k * KS + j * JS + i * IS]: compact per-element storage
// (KS, JS, IS) = (N^2, N, 1) or a view into a brick node block.
template <int P, int Q, int KS = (P + 1) * (P + 1), int JS = P + 1, int IS = 1>
__device__ __forceinline__ void grad_column(const double* __restrict__ sB,
                                            const double* __restrict__ sD,
                                            const double* U, double* S1, double* S2, int qx,
                                            int qy, double g[3][Q]) {
  constexpr int N = P + 1;
  // x: S1[k][j][a] = sum_i B[a][i] U[k][j][i]
  if (qy < N) {
    double b[N];
#pragma unroll
    for (int i = 0; i < N; ++i) b[i] = sB[qx * N + i];
    const double* Uj = U + qy * JS;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) s += b[i] * Uj[k * KS + i * IS];
      S1[(k * N + qy) * Q + qx] = s;
    }
  }
  __syncthreads();
  // y then z in registers.
  double t2[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) s += sB[qy * N + j] * S1[(k * N + j) * Q + qx];
    t2[k] = s;
  }
  double v[Q];
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < N; ++k) s += sB[c * N + k] * t2[k];
    v[c] = s;
    S2[(c * Q + qy) * Q + qx] = s;
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      sx += sD[qx * Q + r] * S2[(c * Q + qy) * Q + r];
      sy += sD[qy * Q + r] * S2[(c * Q + r) * Q + qx];
      sz += sD[c * Q + r] * v[r];
    }
    g[0][c] = sx;
    g[1][c] = sy;
    g[2][c] = sz;
  }
}

// Backward: h[d][qz] at this thread's column -> nodal output of one
// component, written by threads (i = qx < N, j = qy < N) through
// out(k, j, i, value).  Exact adjoint of grad_column (basis.hpp:339-355).
template <int P, int Q, class Out>
__device__ __forceinline__ void grad_transpose_column(const double* __restrict__ sB,
                                                      const double* __restrict__ sD, double* S1,
                                                      double* S2, int qx, int qy,
                                                      const double h[3][Q], Out&& out) {
  constexpr int N = P + 1;
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    S1[(c * Q + qy) * Q + qx] = h[0][c];
    S2[(c * Q + qy) * Q + qx] = h[1][c];
  }
  __syncthreads();
  double acc[Q];
#pragma unroll
  for (int c = 0; c < Q; ++c) {
    double sx = 0.0, sy = 0.0, sz = 0.0;
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      sx += sD[r * Q + qx] * S1[(c * Q + qy) * Q + r];
      sy += sD[r * Q + qy] * S2[(c * Q + r) * Q + qx];
      sz += sD[r * Q + c] * h[2][r];
    }
    acc[c] = (sx + sy) + sz;
  }
  double w[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < Q; ++c) s += sB[c * N + k] * acc[c];
    w[k] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < N; ++k) S1[(k * Q + qy) * Q + qx] = w[k];
  __syncthreads();
  if (qy < N) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < Q; ++b) s += sB[b * N + qy] * S1[(k * Q + b) * Q + qx];
      S2[(k * N + qy) * Q + qx] = s;
    }
  }
  __syncthreads();
  if (qx < N && qy < N) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < Q; ++a) s += sB[a * N + qx] * S2[(k * N + qy) * Q + a];
      out(k, qy, qx, s);
    }
  }
  __syncthreads();
}

}  // namespace hxg
