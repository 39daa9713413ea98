// Shared definitions for the B200 FP64 matrix-free p-multigrid library.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "hexmg_b200.h"

namespace hxg {

// Error carried across the C-ABI (hxg_last_error); the C++ drop-in layer
// rethrows the reference's exception types from it (errors.hpp:9-104).
struct Error : std::runtime_error {
  int code;
  int element = -1, point = -1;
  double jacobian = 0.0;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(HXG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define HXG_CUDA(x) ::hxg::cuda_check((x), #x)

// Supported (P, Q) pairs: fine levels (p, p+1) and the coarse levels the
// p-halving schedule builds on the fine rule (multigrid.hpp:15-19, :244).
constexpr int kMaxP = 4;
constexpr int kMaxQ = 5;

// Per-qpt scalars of the reference's Current storage (material.hpp:70-78,
// :145-148): [w detJ, dxi/dx (9, row-major), tau (00,11,22,01,02,12),
// lambda log J] -- the byte model and hxg_op_export_state use this layout.
constexpr int kRefStateScalars = 17;
// Stored on the device: the same data in 16 scalars,
// [sqrt(w detJ) dxi/dx (9), tau (6), mu - lambda log J]: w detJ folds into
// the two dxi/dx products of the Jacobian q-function (sqrt(w) on each side),
// one scalar less to stream and ~20 fewer flops per point.  w detJ itself is
// the geometry's (undeformed) weight, kept in the geometric factors.
constexpr int kStateStride = 16;
// JacobianStorage (material.hpp:66-78) and its per-point scalars: the
// reference's strides; on the device Current uses kStateStride, the initial
// variants their reference layout.
constexpr int kStorageCurrent = 0, kStorageInitialNative = 1, kStorageInitialTuned = 2,
              kStorageInitialAD = 3;
__host__ __device__ constexpr int ref_state_stride(int storage) {
  return storage == kStorageInitialNative ? 19
         : storage == kStorageInitialTuned ? 26
         : storage == kStorageInitialAD    ? 25
                                           : kRefStateScalars;
}
__host__ __device__ constexpr int device_state_stride(int storage) {
  return storage == kStorageCurrent ? kStateStride : ref_state_stride(storage);
}
constexpr int kMaxStateStride = 26;
// In HBM the scalars of a point are paired (q <= 4): row r = brick Q + qz
// holds ceil(S/2) pair-planes of T points x 2 doubles, so scalar s of point
// t sits at r SP T + (s/2) 2T + 2t + s%2 (SP = S rounded up to even) and a
// thread streams its point's state with 16-byte loads (Q2 apply 332.7 ->
// 318.0 us).  q = 5 (the Q4 hierarchy) keeps one plane per scalar,
// r S T + s T + t (paired it measured 3.5 % slower there).
__host__ __device__ constexpr bool state_paired(int q) { return q != 5; }
__host__ __device__ constexpr int state_pad(int S) { return (S + 1) & ~1; }
__host__ __device__ constexpr int state_row(int S, int q) {
  return state_paired(q) ? state_pad(S) : S;
}
template <class I>
__host__ __device__ constexpr I state_lane(I t, int q) {
  return state_paired(q) ? 2 * t : t;
}
__host__ __device__ inline long long state_pair_off(int s, int T, int q) {
  return state_paired(q) ? (long long)(s >> 1) * 2 * T + (s & 1) : (long long)s * T;
}
// Geometry per qpt: dxi/dX (9, row-major) then w * detJ (mesh.hpp:169-189).
constexpr int kGeoStride = 10;

// Brick of elements processed by one CTA; depends only on Q so every level
// of a hierarchy (which shares the fine quadrature, multigrid.hpp:229-249)
// shares one quadrature-data layout.
__host__ __device__ constexpr int brick_x(int q) { return q == 2 ? 4 : q == 3 ? 4 : 2; }
__host__ __device__ constexpr int brick_y(int q) { return q == 2 ? 4 : q == 3 ? 4 : 2; }
#ifndef HXG_BRICK_Z3
#define HXG_BRICK_Z3 2
#endif
__host__ __device__ constexpr int brick_z(int q) {
  return q == 2 ? 4 : q == 3 ? HXG_BRICK_Z3 : q == 4 ? 2 : 1;
}

// Quadrature-data layout in HBM: brick-blocked structure-of-arrays so that
// the thread owning column (element, qx, qy) reads one coalesced double per
// (brick, qz, scalar) row:
//   offset(brick, qz, s, t) = ((brick * Q + qz) * S + s) * T + t,
//   t = (qy * Q + qx) * NE + local_element,  NE = BX*BY*BZ,  T = NE*Q^2.
// Elements are the fastest index so a warp holds one column position of
// many elements: per-element shared slabs are then hit with a constant odd
// stride (bank-conflict free) while the state loads stay coalesced.
struct QLayout {
  int cells[3] = {1, 1, 1};
  int Q = 2;
  int B[3] = {1, 1, 1};
  int nb[3] = {1, 1, 1};
  int T = 0;

  __host__ __device__ long long num_bricks() const { return (long long)nb[0] * nb[1] * nb[2]; }
  // Doubles per scalar-stride unit of one brick (Q * T).
  __host__ __device__ long long brick_points() const { return (long long)Q * T; }
  __host__ __device__ long long total_points() const { return num_bricks() * brick_points(); }

  static QLayout make(const int cells_[3], int q) {
    QLayout l;
    l.Q = q;
    l.B[0] = brick_x(q);
    l.B[1] = brick_y(q);
    l.B[2] = brick_z(q);
    for (int d = 0; d < 3; ++d) {
      l.cells[d] = cells_[d];
      l.nb[d] = (cells_[d] + l.B[d] - 1) / l.B[d];
    }
    l.T = l.B[0] * l.B[1] * l.B[2] * q * q;
    return l;
  }

  // Element (reference order e = ex + cx (ey + cy ez)) and point q (x-fastest)
  // -> (brick, qz, t) coordinates for host-side permutations.
  void locate(long long e, int qpt, long long& brick, int& qz, int& t) const {
    long long ex = e % cells[0], ey = (e / cells[0]) % cells[1], ez = e / ((long long)cells[0] * cells[1]);
    long long bx = ex / B[0], by = ey / B[1], bz = ez / B[2];
    int lx = (int)(ex - bx * B[0]), ly = (int)(ey - by * B[1]), lz = (int)(ez - bz * B[2]);
    brick = bx + nb[0] * (by + (long long)nb[1] * bz);
    int le = lx + B[0] * (ly + B[1] * lz);
    int qx = qpt % Q, qy = (qpt / Q) % Q;
    qz = qpt / (Q * Q);
    t = (qy * Q + qx) * (B[0] * B[1] * B[2]) + le;
  }
};

// Box-mesh description on device: element counts, order, nodes per dim
// (BoxMesh, mesh.hpp:19-33); restriction indices are analytic
// (build_restriction, mesh.hpp:119-138).
struct BoxDev {
  int cells[3];
  int p;
  int npd[3];
  __host__ __device__ long long num_nodes() const { return (long long)npd[0] * npd[1] * npd[2]; }
  __host__ __device__ long long num_elements() const {
    return (long long)cells[0] * cells[1] * cells[2];
  }
};

inline BoxDev make_box(const int cells[3], int p) {
  BoxDev b;
  b.p = p;
  for (int d = 0; d < 3; ++d) {
    b.cells[d] = cells[d];
    b.npd[d] = p * cells[d] + 1;
  }
  return b;
}

}  // namespace hxg
