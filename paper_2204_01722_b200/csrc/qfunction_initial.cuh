// Neo-Hookean q-functions of the "initial configuration" Jacobian storage
// variants (material.hpp:66-78, :152-175, :196-239): the state holds the
// undeformed mapping and grad_X u, and the Jacobian action re-derives the
// second Piola-Kirchhoff stress (and its directional derivative) per point.
//   InitialNative (19): [w detJ, dxi/dX (9), grad_X u (9)]
//   InitialTuned  (26): native + C^-1 (sym 6) + lambda log J
//   InitialAD     (25): native + S (sym 6); dS by forward-mode dual numbers
// The state is kept in the reference's per-point layout (these variants are
// the paper's Table III comparison, not the production path; Current uses
// the fused kernel).
#pragma once

#include <cuda_runtime.h>

#include "common.hpp"

namespace hxg {

// Forward-mode dual number (dual.hpp:9-40): value + directional derivative.
struct Dual {
  double v, d;
  __device__ Dual() : v(0.0), d(0.0) {}
  __device__ Dual(double x) : v(x), d(0.0) {}  // constants lift with zero derivative
  __device__ Dual(double x, double dx) : v(x), d(dx) {}
};
__device__ __forceinline__ Dual operator+(Dual a, Dual b) { return {a.v + b.v, a.d + b.d}; }
__device__ __forceinline__ Dual operator-(Dual a, Dual b) { return {a.v - b.v, a.d - b.d}; }
__device__ __forceinline__ Dual operator*(Dual a, Dual b) { return {a.v * b.v, a.v * b.d + a.d * b.v}; }
__device__ __forceinline__ Dual operator/(Dual a, Dual b) {
  const double inv = 1.0 / b.v;
  return {a.v * inv, (a.d - a.v * b.d * inv) * inv};
}
__device__ __forceinline__ Dual lg(Dual a) { return {::log(a.v), a.d / a.v}; }
__device__ __forceinline__ double lg(double a) { return ::log(a); }

namespace qi {

// 3x3 row-major helpers, generic over double / Dual.
template <class T>
__device__ __forceinline__ T det3(const T m[9]) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}
// inv3 via adjugate / det (tensor3.hpp:94-110).
template <class T>
__device__ __forceinline__ void inv3(const T m[9], T r[9]) {
  r[0] = m[4] * m[8] - m[5] * m[7];
  r[1] = m[2] * m[7] - m[1] * m[8];
  r[2] = m[1] * m[5] - m[2] * m[4];
  r[3] = m[5] * m[6] - m[3] * m[8];
  r[4] = m[0] * m[8] - m[2] * m[6];
  r[5] = m[2] * m[3] - m[0] * m[5];
  r[6] = m[3] * m[7] - m[4] * m[6];
  r[7] = m[1] * m[6] - m[0] * m[7];
  r[8] = m[0] * m[4] - m[1] * m[3];
  const T inv_det = T(1.0) / det3(m);
#pragma unroll
  for (int k = 0; k < 9; ++k) r[k] = r[k] * inv_det;
}
// c = a b, c = a^T b, c = a b^T
template <class T>
__device__ __forceinline__ void mul(const T a[9], const T b[9], T c[9]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[3 * i + j] = a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
}
template <class T>
__device__ __forceinline__ void mul_tn(const T a[9], const T b[9], T c[9]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[3 * i + j] = a[i] * b[j] + a[3 + i] * b[3 + j] + a[6 + i] * b[6 + j];
}
template <class T>
__device__ __forceinline__ void mul_nt(const T a[9], const T b[9], T c[9]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      c[3 * i + j] = a[3 * i] * b[3 * j] + a[3 * i + 1] * b[3 * j + 1] + a[3 * i + 2] * b[3 * j + 2];
}
__device__ __forceinline__ void unpack_sym(const double* s, double m[9]) {  // (00,11,22,01,02,12)
  m[0] = s[0]; m[4] = s[1]; m[8] = s[2];
  m[1] = m[3] = s[3];
  m[2] = m[6] = s[4];
  m[5] = m[7] = s[5];
}
__device__ __forceinline__ void pack_sym(const double m[9], double* s) {
  s[0] = m[0]; s[1] = m[4]; s[2] = m[8]; s[3] = m[1]; s[4] = m[2]; s[5] = m[5];
}

// S(E) = mu I + (lambda log J - mu) C^-1, C = I + 2E (material.hpp:110-121).
template <class T>
__device__ __forceinline__ void second_piola(double mu, double lambda, const T e[9], T s[9]) {
  T c[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) c[k] = T((k % 4) == 0 ? 1.0 : 0.0) + T(2.0) * e[k];
  const T log_j = T(0.5) * lg(det3(c));
  T ci[9];
  inv3(c, ci);
  const T coeff = T(lambda) * log_j - T(mu);
#pragma unroll
  for (int k = 0; k < 9; ++k) s[k] = T(mu) * T((k % 4) == 0 ? 1.0 : 0.0) + coeff * ci[k];
}

}  // namespace qi

// Residual q-function of the initial variants (material.hpp:152-175):
// writes the variant's reference-layout state, returns J (<= 0: inverted,
// outputs unspecified).
template <int ST>
__device__ __forceinline__ double residual_qf_initial(double mu, double lambda, const double G[9],
                                                      const double dxidX[9], double wdet,
                                                      double H[9], double* st) {
  double gu[9], f[9];
  qi::mul(G, dxidX, gu);
#pragma unroll
  for (int k = 0; k < 9; ++k) f[k] = gu[k] + ((k % 4) == 0 ? 1.0 : 0.0);
  const double j = qi::det3(f);
  if (!(j > 0.0)) return j;
  const double log_j = ::log(j);
  double c[9], ci[9], s[9];
  qi::mul_tn(f, f, c);
  qi::inv3(c, ci);
  const double coeff = lambda * log_j - mu;
#pragma unroll
  for (int k = 0; k < 9; ++k) s[k] = mu * ((k % 4) == 0 ? 1.0 : 0.0) + coeff * ci[k];
  st[0] = wdet;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    st[1 + k] = dxidX[k];
    st[10 + k] = gu[k];
  }
  if (ST == kStorageInitialTuned) {
    qi::pack_sym(ci, st + 19);
    st[25] = lambda * log_j;
  } else if (ST == kStorageInitialAD) {
    qi::pack_sym(s, st + 19);
  }
  double fs[9], h[9];
  qi::mul(f, s, fs);
  qi::mul_nt(fs, dxidX, h);
#pragma unroll
  for (int k = 0; k < 9; ++k) H[k] = wdet * h[k];
  return j;
}

// Jacobian q-function of the initial variants (material.hpp:196-239).
template <int ST>
__device__ __forceinline__ void jacobian_qf_initial(double mu, double lambda, const double G[9],
                                                    const double* st, double H[9]) {
  const double wdet = st[0];
  const double* dxidX = st + 1;
  const double* gu = st + 10;
  double f[9], df[9], ftdf[9], de[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) f[k] = gu[k] + ((k % 4) == 0 ? 1.0 : 0.0);
  qi::mul(G, dxidX, df);
  qi::mul_tn(f, df, ftdf);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) de[3 * i + jj] = 0.5 * (ftdf[3 * i + jj] + ftdf[3 * jj + i]);
  double s[9], ds[9];
  if (ST == kStorageInitialAD) {
    qi::unpack_sym(st + 19, s);
    // E = sym(grad_u) + grad_u^T grad_u / 2, seeded with direction dE.
    double gtg[9];
    qi::mul_tn(gu, gu, gtg);
    Dual e[9], sd[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int jj = 0; jj < 3; ++jj) {
        const int k = 3 * i + jj;
        e[k] = Dual(0.5 * (gu[k] + gu[3 * jj + i]) + 0.5 * gtg[k], de[k]);
      }
    qi::second_piola<Dual>(mu, lambda, e, sd);
#pragma unroll
    for (int k = 0; k < 9; ++k) ds[k] = sd[k].d;
  } else {
    double ci[9], lambda_log_j;
    if (ST == kStorageInitialTuned) {
      qi::unpack_sym(st + 19, ci);
      lambda_log_j = st[25];
    } else {
      double c[9];
      qi::mul_tn(f, f, c);
      qi::inv3(c, ci);
      lambda_log_j = 0.5 * lambda * ::log(qi::det3(c));
    }
    const double coeff = lambda_log_j - mu;
#pragma unroll
    for (int k = 0; k < 9; ++k) s[k] = mu * ((k % 4) == 0 ? 1.0 : 0.0) + coeff * ci[k];
    // dS = lambda (C^-1 : dE) C^-1 - 2 (lambda log J - mu) C^-1 dE C^-1
    double cde = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) cde += ci[k] * de[k];
    double t1[9], t2[9];
    qi::mul(ci, de, t1);
    qi::mul(t1, ci, t2);
#pragma unroll
    for (int k = 0; k < 9; ++k) ds[k] = (lambda * cde) * ci[k] - (2.0 * coeff) * t2[k];
  }
  double a[9], b[9], h[9];
  qi::mul(df, s, a);
  qi::mul(f, ds, b);
#pragma unroll
  for (int k = 0; k < 9; ++k) a[k] += b[k];
  qi::mul_nt(a, dxidX, h);
#pragma unroll
  for (int k = 0; k < 9; ++k) H[k] = wdet * h[k];
}

}  // namespace hxg
