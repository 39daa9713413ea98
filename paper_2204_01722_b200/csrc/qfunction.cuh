// Neo-Hookean pointwise q-functions, Current storage (material.hpp:126-194),
// as straight-line FP64 device code on 3x3 row-major registers.
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"

namespace hxg {

// Jacobian action (material.hpp:179-194) on the stored state
// st = [A = sqrt(w detJ) dxi/dx (9), tau (00,11,22,01,02,12), h = mu - lambda log J]:
//   grad_du = G dxi/dx, deps = sym(grad_du),
//   k = grad_du tau + lambda tr(deps) I + 2 (mu - lambda log J) deps,
//   H = w detJ * k dxi/dx^T
// computed as gd = G A (= sqrt(w) grad_du), k~ from gd (linear: = sqrt(w) k),
// H = k~ A^T.
__device__ __forceinline__ void jacobian_qf(double /*mu*/, double lambda, const double G[9],
                                            const double st[kStateStride], double H[9]) {
  const double* xi = st;
  double gd[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = G[3 * i + 0] * xi[0 + j];
      s = s + G[3 * i + 1] * xi[3 + j];
      s = s + G[3 * i + 2] * xi[6 + j];
      gd[3 * i + j] = s;
    }
  const double tau[9] = {st[9], st[12], st[13], st[12], st[10], st[14], st[13], st[14], st[11]};
  double k[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = gd[3 * i + 0] * tau[0 + j];
      s = s + gd[3 * i + 1] * tau[3 + j];
      s = s + gd[3 * i + 2] * tau[6 + j];
      k[3 * i + j] = s;
    }
  // + lambda tr(deps) I + 2 h sym(gd): the symmetric part once per pair
  const double tr = lambda * (gd[0] + gd[4] + gd[8]);
  const double h = st[15], h2 = h + h;
  k[0] += fma(h2, gd[0], tr);
  k[4] += fma(h2, gd[4], tr);
  k[8] += fma(h2, gd[8], tr);
  const double s01 = h * (gd[1] + gd[3]), s02 = h * (gd[2] + gd[6]), s12 = h * (gd[5] + gd[7]);
  k[1] += s01;
  k[3] += s01;
  k[2] += s02;
  k[6] += s02;
  k[5] += s12;
  k[7] += s12;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = k[3 * i + 0] * xi[3 * j + 0];
      s = s + k[3 * i + 1] * xi[3 * j + 1];
      s = s + k[3 * i + 2] * xi[3 * j + 2];
      H[3 * i + j] = s;
    }
}

// Reference-layout state (residual_qf's output) -> stored state.
__device__ __forceinline__ void pack_state(double mu, const double r[kRefStateScalars],
                                           double st[kStateStride]) {
  const double sw = sqrt(r[0]);
#pragma unroll
  for (int k = 0; k < 9; ++k) st[k] = sw * r[1 + k];
#pragma unroll
  for (int k = 0; k < 6; ++k) st[9 + k] = r[10 + k];
  st[15] = mu - r[16];
}

__device__ __forceinline__ double det3(const double m[9]) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}

// Residual q-function (material.hpp:126-150).  Returns J; when J <= 0 the
// outputs are unspecified and the caller records the inverted point.
// DIAG: dxi/dX is diagonal (box meshes); only its diagonal is read and the
// products with its zero entries are skipped (the same values: those terms
// add exact zeros).
template <bool DIAG = false>
__device__ __forceinline__ double residual_qf(double mu, double lambda, const double G[9],
                                              const double dxidX[9], double wdet, double H[9],
                                              double st[kRefStateScalars]) {
  double F[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s;
      if constexpr (DIAG) {
        s = G[3 * i + j] * dxidX[4 * j];
      } else {
        s = G[3 * i + 0] * dxidX[0 + j];
        s = s + G[3 * i + 1] * dxidX[3 + j];
        s = s + G[3 * i + 2] * dxidX[6 + j];
      }
      F[3 * i + j] = s + (i == j ? 1.0 : 0.0);
    }
  const double J = det3(F);
  if (!(J > 0.0)) return J;
  const double logJ = log(J);
  // inv3 via adjugate (tensor3.hpp:94-110).
  double r[9] = {F[4] * F[8] - F[5] * F[7], F[2] * F[7] - F[1] * F[8], F[1] * F[5] - F[2] * F[4],
                 F[5] * F[6] - F[3] * F[8], F[0] * F[8] - F[2] * F[6], F[2] * F[3] - F[0] * F[5],
                 F[3] * F[7] - F[4] * F[6], F[1] * F[6] - F[0] * F[7], F[0] * F[4] - F[1] * F[3]};
  const double inv_det = 1.0 / J;
#pragma unroll
  for (int k = 0; k < 9; ++k) r[k] *= inv_det;
  double xi[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if constexpr (DIAG) {
        xi[3 * i + j] = dxidX[4 * i] * r[3 * i + j];
      } else {
        double s = dxidX[3 * i + 0] * r[0 + j];
        s = s + dxidX[3 * i + 1] * r[3 + j];
        s = s + dxidX[3 * i + 2] * r[6 + j];
        xi[3 * i + j] = s;
      }
    }
  double tau[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = F[3 * i + 0] * F[3 * j + 0];
      s = s + F[3 * i + 1] * F[3 * j + 1];
      s = s + F[3 * i + 2] * F[3 * j + 2];
      tau[3 * i + j] = mu * (s - (i == j ? 1.0 : 0.0));
    }
  const double d = lambda * logJ;
  tau[0] += d;
  tau[4] += d;
  tau[8] += d;
  st[0] = wdet;
#pragma unroll
  for (int k = 0; k < 9; ++k) st[1 + k] = xi[k];
  st[10] = tau[0];
  st[11] = tau[4];
  st[12] = tau[8];
  st[13] = tau[1];
  st[14] = tau[2];
  st[15] = tau[5];
  st[16] = d;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double s = tau[3 * i + 0] * xi[3 * j + 0];
      s = s + tau[3 * i + 1] * xi[3 * j + 1];
      s = s + tau[3 * i + 2] * xi[3 * j + 2];
      H[3 * i + j] = wdet * s;
    }
  return J;
}

// Strain energy density (material.hpp:38-48); returns J via *jout.
__device__ __forceinline__ double energy_density(double mu, double lambda, const double grad_u[9],
                                                 double* jout) {
  double F[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) F[k] = grad_u[k] + ((k % 4) == 0 ? 1.0 : 0.0);
  const double J = det3(F);
  *jout = J;
  if (!(J > 0.0)) return 0.0;
  const double lj = log(J);
  double tb = 0.0;
#pragma unroll
  for (int k = 0; k < 9; ++k) tb += F[k] * F[k];
  const double te = 0.5 * (tb - 3.0);
  return 0.5 * lambda * lj * lj - mu * lj + mu * te;
}

}  // namespace hxg
