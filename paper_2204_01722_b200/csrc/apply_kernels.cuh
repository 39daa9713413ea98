// Element-level kernels of the composed operator y = E^T B^T D B E x
// (operator.hpp:146-215): one CTA per brick of elements, one thread per
// quadrature column.  Shared by the two-pass path and the fused brick path.
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"
#include "element.cuh"
#include "qfunction.cuh"
#include "qfunction_initial.cuh"

namespace hxg {

enum ApplyMode { kJacobian = 0, kResidual = 1, kEnergy = 2, kResidualBox = 3 };

struct ElemParams {
  BoxDev box;
  QLayout lay;
  const double* x;         // input L-vector
  const uint8_t* mask;     // constraint mask (jacobian input masking), may be null
  double* evec;            // E-vector output (e, c, a) for the two-pass path
  const double* tab;       // B (Q x N) then Dc (Q x Q)
  const double* state;     // shared quadrature state (blocked)
  double* state_out;       // residual: written state
  const double* geo;       // residual/energy: geometry (blocked, 10 per qpt)
  double mu, lambda, perturb;
  int storage;               // JacobianStorage (the kernel's ST template argument)
  unsigned long long* fail;  // residual: min over e*Q^3+q of inverted points
  double* energy_part;       // energy: per-element partial sums
};

// Brick coordinates of this CTA's thread: element e (or -1 when padding).
template <int Q>
struct ThreadPos {
  int le, qx, qy;
  long long e;
  long long brick;
};

template <int P, int Q>
__device__ __forceinline__ ThreadPos<Q> thread_pos(const QLayout& lay, long long brick) {
  using D = Dims<P, Q>;
  ThreadPos<Q> tp;
  // Thread t = (qy Q + qx) NE + le: elements fastest (QLayout).
  int t = threadIdx.x;
  tp.le = t % D::NE;
  tp.qx = (t / D::NE) % Q;
  tp.qy = t / (D::NE * Q);
  tp.brick = brick;
  long long bx = brick % lay.nb[0], by = (brick / lay.nb[0]) % lay.nb[1],
            bz = brick / ((long long)lay.nb[0] * lay.nb[1]);
  int lx = tp.le % D::BX, ly = (tp.le / D::BX) % D::BY, lz = tp.le / (D::BX * D::BY);
  long long ex = bx * D::BX + lx, ey = by * D::BY + ly, ez = bz * D::BZ + lz;
  if (ex < lay.cells[0] && ey < lay.cells[1] && ez < lay.cells[2])
    tp.e = ex + lay.cells[0] * (ey + (long long)lay.cells[1] * ez);
  else
    tp.e = -1;
  return tp;
}

// Gathers the element's 3 N^3 nodal values into U[c][a] (mesh.hpp:88-101),
// zeroing constrained entries (operator.hpp:189-193) when mask != null.
template <int P, int Q>
__device__ __forceinline__ void gather_element(const BoxDev& box, long long e, const double* x,
                                               const uint8_t* mask, double* U, int lane,
                                               int nlanes) {
  constexpr int N = P + 1, N3 = N * N * N;
  if (e < 0) {
    for (int r = lane; r < 3 * N3; r += nlanes) U[r] = 0.0;
    return;
  }
  long long ex = e % box.cells[0], ey = (e / box.cells[0]) % box.cells[1],
            ez = e / ((long long)box.cells[0] * box.cells[1]);
  for (int r = lane; r < 3 * N3; r += nlanes) {
    int a = r / 3, c = r % 3;
    int i = a % N, j = (a / N) % N, k = a / (N * N);
    long long node = (P * ex + i) + box.npd[0] * ((P * ey + j) + (long long)box.npd[1] * (P * ez + k));
    long long dof = 3 * node + c;
    double v = x[dof];
    if (mask && mask[dof]) v = 0.0;
    U[c * N3 + a] = v;
  }
}

template <int P, int Q>
__device__ __forceinline__ void load_tables(const double* tab, double* sTab) {
  using D = Dims<P, Q>;
  for (int r = threadIdx.x; r < D::TAB; r += blockDim.x) sTab[r] = tab[r];
}

// Two-pass element kernel: gather -> grad -> q-function -> grad^T -> E-vector.
// ST = JacobianStorage: the state stride and the q-function pair.
template <int P, int Q, int MODE, int ST = kStorageCurrent>
__global__ void __launch_bounds__(Dims<P, Q>::T) element_apply_kernel(ElemParams prm) {
  constexpr int S = device_state_stride(ST), SP = state_row(S, Q);
  using D = Dims<P, Q>;
  constexpr int N = D::N, N3 = D::N3;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sD = smem + Q * N;
  ThreadPos<Q> tp = thread_pos<P, Q>(prm.lay, blockIdx.x);
  double* U = smem + D::TAB + tp.le * D::ELEM_SMEM;
  double* S1 = U + 3 * N3;
  double* S2 = S1 + D::Q3;
  load_tables<P, Q>(prm.tab, smem);
  gather_element<P, Q>(prm.box, tp.e, prm.x, MODE == kJacobian ? prm.mask : nullptr, U,
                       tp.qy * Q + tp.qx, D::Q2);
  __syncthreads();

  double g[3][3][Q];  // [component][direction][qz]
#pragma unroll
  for (int c = 0; c < 3; ++c) grad_column<P, Q>(sB, sD, U + c * N3, S1, S2, tp.qx, tp.qy, g[c]);
  // S1/S2 are rewritten by the first transpose before every thread has
  // finished reading the last forward slab.
  __syncthreads();

  const long long T = prm.lay.T;
  const long long base = prm.lay.brick_points() * tp.brick;
  if (MODE == kJacobian) {
#pragma unroll
    for (int qz = 0; qz < Q; ++qz) {
      double st[S];
      const double* sp = prm.state + (base + (long long)qz * T) * SP + state_lane(threadIdx.x, Q);
#pragma unroll
      for (int s = 0; s < S; ++s) st[s] = __ldg(sp + state_pair_off(s, (int)T, Q));
      double G[9], H[9];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) G[3 * c + d] = g[c][d][qz];
      if constexpr (ST == kStorageCurrent)
        jacobian_qf(prm.mu, prm.lambda, G, st, H);
      else
        jacobian_qf_initial<ST>(prm.mu, prm.lambda, G, st, H);
      if (prm.perturb != 0.0) {  // fault-injection hook: + eps w detJ G
        const double wdet = prm.geo[(base + (long long)qz * T) * kGeoStride + 9 * T + threadIdx.x];
#pragma unroll
        for (int k = 0; k < 9; ++k) H[k] += prm.perturb * wdet * G[k];
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) g[c][d][qz] = H[3 * c + d];
    }
  } else if (MODE == kResidual) {
#pragma unroll
    for (int qz = 0; qz < Q; ++qz) {
      double geo[kGeoStride];
      const double* gp = prm.geo + (base + (long long)qz * T) * kGeoStride + threadIdx.x;
#pragma unroll
      for (int s = 0; s < kGeoStride; ++s) geo[s] = __ldg(gp + s * T);
      double G[9], H[9], st[ref_state_stride(ST)];
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) G[3 * c + d] = g[c][d][qz];
      double J;
      if constexpr (ST == kStorageCurrent)
        J = residual_qf(prm.mu, prm.lambda, G, geo, geo[9], H, st);
      else
        J = residual_qf_initial<ST>(prm.mu, prm.lambda, G, geo, geo[9], H, st);
      double* so = prm.state_out + (base + (long long)qz * T) * SP + state_lane(threadIdx.x, Q);
      if (!(J > 0.0)) {
        if (tp.e >= 0) {
          unsigned long long idx =
              (unsigned long long)tp.e * D::Q3 + (unsigned long long)(tp.qx + Q * (tp.qy + Q * qz));
          atomicMin(prm.fail, idx);
          so[0] = J;  // read back by the host for the error report
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) H[k] = 0.0;
      } else if (tp.e >= 0) {
        if constexpr (ST == kStorageCurrent) {
          double sp[kStateStride];
          pack_state(prm.mu, st, sp);
#pragma unroll
          for (int s = 0; s < kStateStride; ++s) so[state_pair_off(s, (int)T, Q)] = sp[s];
        } else {
#pragma unroll
          for (int s = 0; s < S; ++s) so[state_pair_off(s, (int)T, Q)] = st[s];
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) g[c][d][qz] = H[3 * c + d];
    }
  }

  double* ev = prm.evec;
  const long long e = tp.e;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    grad_transpose_column<P, Q>(sB, sD, S1, S2, tp.qx, tp.qy, g[c],
                                [&](int k, int j, int i, double v) {
                                  if (e >= 0) ev[(e * 3 + c) * N3 + (k * N + j) * N + i] = v;
                                });
  }
}

// Total strain energy partials (operator.hpp:287-315): per-element sums over
// q of w * psi(grad_u), grad_u = G dxi/dX; inverted points recorded in fail.
template <int P, int Q>
__global__ void __launch_bounds__(Dims<P, Q>::T) element_energy_kernel(ElemParams prm) {
  using D = Dims<P, Q>;
  constexpr int N3 = D::N3;
  extern __shared__ double smem[];
  double* sB = smem;
  double* sD = smem + Q * D::N;
  ThreadPos<Q> tp = thread_pos<P, Q>(prm.lay, blockIdx.x);
  double* U = smem + D::TAB + tp.le * D::ELEM_SMEM;
  double* S1 = U + 3 * N3;
  double* S2 = S1 + D::Q3;
  double* red = smem + D::TAB + D::NE * D::ELEM_SMEM;  // T doubles
  load_tables<P, Q>(prm.tab, smem);
  gather_element<P, Q>(prm.box, tp.e, prm.x, nullptr, U, tp.qy * Q + tp.qx, D::Q2);
  __syncthreads();
  double g[3][3][Q];
#pragma unroll
  for (int c = 0; c < 3; ++c) grad_column<P, Q>(sB, sD, U + c * N3, S1, S2, tp.qx, tp.qy, g[c]);
  const long long T = prm.lay.T;
  const long long base = prm.lay.brick_points() * tp.brick;
  double psum[Q];
#pragma unroll
  for (int qz = 0; qz < Q; ++qz) {
    const double* gp = prm.geo + (base + (long long)qz * T) * kGeoStride + threadIdx.x;
    double xi[9];
#pragma unroll
    for (int s = 0; s < 9; ++s) xi[s] = __ldg(gp + s * T);
    double w = __ldg(gp + 9 * T);
    double gu[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        double s = g[i][0][qz] * xi[0 + j];
        s = s + g[i][1][qz] * xi[3 + j];
        s = s + g[i][2][qz] * xi[6 + j];
        gu[3 * i + j] = s;
      }
    double J;
    double psi = energy_density(prm.mu, prm.lambda, gu, &J);
    if (!(J > 0.0) && tp.e >= 0) {
      unsigned long long idx =
          (unsigned long long)tp.e * D::Q3 + (unsigned long long)(tp.qx + Q * (tp.qy + Q * qz));
      atomicMin(prm.fail, idx);
    }
    psum[qz] = w * psi;
  }
  // Per-element sum in reference point order q = qx + Q (qy + Q qz).
  for (int qz = 0; qz < Q; ++qz) {
    red[threadIdx.x] = psum[qz];
    __syncthreads();
    if (tp.qx == 0 && tp.qy == 0 && tp.e >= 0) {
      double s = qz == 0 ? 0.0 : prm.energy_part[tp.e];
      for (int r = 0; r < D::Q2; ++r) s += red[tp.le + r * D::NE];  // column r = qy Q + qx
      prm.energy_part[tp.e] = s;
    }
    __syncthreads();
  }
}

}  // namespace hxg
