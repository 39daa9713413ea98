// Host-side problem setup: quadrature, 1D Lagrange basis, box-mesh geometry,
// Dirichlet masks and traction loads.  These restate the reference's setup
// (quadrature.hpp, basis.hpp:134-175, mesh.hpp:35-232, operator.hpp:36-55,
// :381-443); they run once per problem and feed device tabulations.
#include "setup.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <stdexcept>

#include "common.hpp"

namespace hxg {

namespace {

// P_n and P_n' by the three-term recurrence.
void legendre(int n, double x, double& p, double& dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  dp = n * (x * p1 - p0) / (x * x - 1.0);
}

}  // namespace

Rule gauss_legendre(int q) {
  if (q < 1) throw Error(HXG_ERR_INVALID_ARGUMENT, "quadrature size must be >= 1");
  Rule r;
  r.points.assign(q, 0.0);
  r.weights.assign(q, 0.0);
  for (int i = 0; i < (q + 1) / 2; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (q + 0.5));
    double p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre(q, x, p, dp);
      double dx = p / dp;
      x -= dx;
      if (std::abs(dx) < 1e-16) break;
    }
    legendre(q, x, p, dp);
    double w = 2.0 / ((1.0 - x * x) * dp * dp);
    r.points[q - 1 - i] = x;
    r.points[i] = -x;
    r.weights[i] = r.weights[q - 1 - i] = w;
  }
  if (q % 2 == 1) r.points[q / 2] = 0.0;
  return r;
}

std::vector<double> gauss_lobatto(int p) {
  if (p < 1) throw Error(HXG_ERR_INVALID_ARGUMENT, "basis order must be >= 1");
  int n = p + 1;
  std::vector<double> x(n, 0.0);
  x[0] = -1.0;
  x[n - 1] = 1.0;
  for (int i = 1; i <= (n - 1) / 2; ++i) {
    double y = std::cos(M_PI * i / p);
    for (int it = 0; it < 100; ++it) {
      double pp, dp;
      legendre(p, y, pp, dp);
      double d2p = (2.0 * y * dp - p * (p + 1.0) * pp) / (1.0 - y * y);
      double dy = dp / d2p;
      y -= dy;
      if (std::abs(dy) < 1e-16) break;
    }
    x[n - 1 - i] = std::abs(y);
    x[i] = -std::abs(y);
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
  return x;
}

// Lagrange cardinal values (and derivatives) on `nodes` at `points`, the
// barycentric form with the collocated special case.
void lagrange_tabulate(const std::vector<double>& nodes, const std::vector<double>& points,
                       std::vector<double>* vals, std::vector<double>* ders) {
  int n = (int)nodes.size();
  std::vector<double> bary(n, 1.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (j != i) bary[i] /= nodes[i] - nodes[j];
  if (vals) vals->assign(points.size() * n, 0.0);
  if (ders) ders->assign(points.size() * n, 0.0);
  for (size_t r = 0; r < points.size(); ++r) {
    double y = points[r];
    int hit = -1;
    for (int i = 0; i < n; ++i)
      if (std::abs(y - nodes[i]) < 1e-13) hit = i;
    if (hit >= 0) {
      if (vals) (*vals)[r * n + hit] = 1.0;
      if (ders) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) {
          if (i == hit) continue;
          double d = (bary[i] / bary[hit]) / (nodes[hit] - nodes[i]);
          (*ders)[r * n + i] = d;
          s += d;
        }
        (*ders)[r * n + hit] = -s;
      }
      continue;
    }
    double l = 1.0, s = 0.0;
    for (int j = 0; j < n; ++j) {
      l *= y - nodes[j];
      s += 1.0 / (y - nodes[j]);
    }
    for (int i = 0; i < n; ++i) {
      double v = bary[i] * l / (y - nodes[i]);
      if (vals) (*vals)[r * n + i] = v;
      if (ders) (*ders)[r * n + i] = v * (s - 1.0 / (y - nodes[i]));
    }
  }
}

Basis build_basis(int p, const Rule& rule) {
  if (p < 1) throw Error(HXG_ERR_INVALID_ARGUMENT, "basis order must be >= 1");
  int q = (int)rule.points.size();
  if (q < p + 1)
    throw Error(HXG_ERR_INVALID_ARGUMENT,
                "need at least p + 1 quadrature points for full column rank");
  Basis b;
  b.p = p;
  b.q = q;
  b.nodes = gauss_lobatto(p);
  b.rule = rule;
  lagrange_tabulate(b.nodes, rule.points, &b.interp, &b.deriv);
  int n = p + 1;
  // pinv = (B^T B)^-1 B^T by Gaussian elimination with partial pivoting.
  std::vector<double> a(n * n, 0.0), rhs(n * q, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int r = 0; r < q; ++r) s += b.interp[r * n + i] * b.interp[r * n + j];
      a[i * n + j] = s;
    }
  for (int i = 0; i < n; ++i)
    for (int r = 0; r < q; ++r) rhs[i * q + r] = b.interp[r * n + i];
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a[i * n + k]) > std::abs(a[piv * n + k])) piv = i;
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(a[k * n + j], a[piv * n + j]);
      for (int j = 0; j < q; ++j) std::swap(rhs[k * q + j], rhs[piv * q + j]);
    }
    for (int i = k + 1; i < n; ++i) {
      double f = a[i * n + k] / a[k * n + k];
      for (int j = k; j < n; ++j) a[i * n + j] -= f * a[k * n + j];
      for (int j = 0; j < q; ++j) rhs[i * q + j] -= f * rhs[k * q + j];
    }
  }
  for (int k = n - 1; k >= 0; --k)
    for (int j = 0; j < q; ++j) {
      double s = rhs[k * q + j];
      for (int i = k + 1; i < n; ++i) s -= a[k * n + i] * rhs[i * q + j];
      rhs[k * q + j] = s / a[k * n + k];
    }
  b.pinv = rhs;
  b.colloc.assign(q * q, 0.0);
  for (int r = 0; r < q; ++r)
    for (int c = 0; c < q; ++c) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += b.deriv[r * n + i] * b.pinv[i * q + c];
      b.colloc[r * q + c] = s;
    }
  return b;
}

Basis build_basis(int p, int q) { return build_basis(p, gauss_legendre(q)); }

std::array<std::vector<double>, 3> box_axes(const double extents[3], const int cells[3], int p) {
  auto lob = gauss_lobatto(p);
  std::array<std::vector<double>, 3> axis;
  for (int d = 0; d < 3; ++d) {
    if (!(extents[d] > 0.0)) throw Error(HXG_ERR_INVALID_ARGUMENT, "box extents must be positive");
    if (cells[d] < 1) throw Error(HXG_ERR_INVALID_ARGUMENT, "element counts must be >= 1");
    int m = p * cells[d] + 1;
    axis[d].assign(m, 0.0);
    double h = extents[d] / cells[d];
    for (int e = 0; e < cells[d]; ++e)
      for (int i = 0; i <= p; ++i) axis[d][e * p + i] = (e + 0.5 * (lob[i] + 1.0)) * h;
    axis[d].back() = extents[d];
  }
  return axis;
}

// Geometric factors by pushing element node coordinates through the
// six-contraction gradient, as compute_geometric_factors (mesh.hpp:193-232).
void geometry(const double extents[3], const int cells[3], int p, const Basis& b,
              std::vector<double>& dxidX, std::vector<double>& weight) {
  if (b.p != p) throw Error(HXG_ERR_INVALID_ARGUMENT, "geometry basis order must match mesh order");
  auto axis = box_axes(extents, cells, p);
  int n = p + 1, q = b.q, nq = q * q * q;
  long long E = (long long)cells[0] * cells[1] * cells[2];
  dxidX.assign((size_t)E * nq * 9, 0.0);
  weight.assign((size_t)E * nq, 0.0);
  std::vector<double> in(n * n * n), t1(q * n * n), t2(q * q * n), v(nq), g(nq);
  auto contract = [&](const double* M, int rows, int cols, int dim, const double* src,
                      std::array<int, 3> shape, double* dst) {
    int n0 = shape[0], n1 = shape[1], n2 = shape[2];
    if (dim == 0) {
      for (int k = 0; k < n2; ++k)
        for (int j = 0; j < n1; ++j)
          for (int a = 0; a < rows; ++a) {
            double s = 0.0;
            for (int i = 0; i < n0; ++i) s += M[a * cols + i] * src[i + n0 * (j + n1 * k)];
            dst[a + rows * (j + n1 * k)] = s;
          }
    } else if (dim == 1) {
      for (int k = 0; k < n2; ++k)
        for (int bb = 0; bb < rows; ++bb)
          for (int i = 0; i < n0; ++i) {
            double s = 0.0;
            for (int j = 0; j < n1; ++j) s += M[bb * cols + j] * src[i + n0 * (j + n1 * k)];
            dst[i + n0 * (bb + rows * k)] = s;
          }
    } else {
      for (int c = 0; c < rows; ++c)
        for (int j = 0; j < n1; ++j)
          for (int i = 0; i < n0; ++i) {
            double s = 0.0;
            for (int k = 0; k < n2; ++k) s += M[c * cols + k] * src[i + n0 * (j + n1 * k)];
            dst[i + n0 * (j + n1 * c)] = s;
          }
    }
  };
  const double* w = b.rule.weights.data();
  std::vector<double> A(nq * 9);
  for (long long e = 0; e < E; ++e) {
    long long ex = e % cells[0], ey = (e / cells[0]) % cells[1], ez = e / ((long long)cells[0] * cells[1]);
    for (int c = 0; c < 3; ++c) {
      for (int k = 0; k <= p; ++k)
        for (int j = 0; j <= p; ++j)
          for (int i = 0; i <= p; ++i) {
            long long gi[3] = {p * ex + i, p * ey + j, p * ez + k};
            in[i + n * (j + n * k)] = axis[c][gi[c]];
          }
      contract(b.interp.data(), q, n, 0, in.data(), {n, n, n}, t1.data());
      contract(b.interp.data(), q, n, 1, t1.data(), {q, n, n}, t2.data());
      contract(b.interp.data(), q, n, 2, t2.data(), {q, q, n}, v.data());
      for (int d = 0; d < 3; ++d) {
        contract(b.colloc.data(), q, q, d, v.data(), {q, q, q}, g.data());
        for (int pt = 0; pt < nq; ++pt) A[pt * 9 + c * 3 + d] = g[pt];
      }
    }
    for (int pt = 0; pt < nq; ++pt) {
      const double* m = &A[pt * 9];
      double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                   m[2] * (m[3] * m[7] - m[4] * m[6]);
      if (!(det > 0.0))
        throw Error(HXG_ERR_INVALID_ARGUMENT, "degenerate element " + std::to_string(e));
      double r[9] = {m[4] * m[8] - m[5] * m[7], m[2] * m[7] - m[1] * m[8], m[1] * m[5] - m[2] * m[4],
                     m[5] * m[6] - m[3] * m[8], m[0] * m[8] - m[2] * m[6], m[2] * m[3] - m[0] * m[5],
                     m[3] * m[7] - m[4] * m[6], m[1] * m[6] - m[0] * m[7], m[0] * m[4] - m[1] * m[3]};
      double inv_det = 1.0 / det;
      double* dst = &dxidX[((size_t)e * nq + pt) * 9];
      for (int k = 0; k < 9; ++k) dst[k] = r[k] * inv_det;
      int qa = pt % q, qb = (pt / q) % q, qc = pt / (q * q);
      weight[(size_t)e * nq + pt] = w[qa] * w[qb] * w[qc] * det;
    }
  }
}

// Dirichlet mask from fixed faces, all components (build_constraints,
// operator.hpp:36-55 with select_boundary_nodes, mesh.hpp:151-164).
void face_mask(const int cells[3], int p, int fixed_face_mask, std::vector<uint8_t>& mask) {
  int npd[3] = {p * cells[0] + 1, p * cells[1] + 1, p * cells[2] + 1};
  long long nn = (long long)npd[0] * npd[1] * npd[2];
  mask.assign((size_t)nn * 3, 0);
  for (long long node = 0; node < nn; ++node) {
    int g[3] = {(int)(node % npd[0]), (int)((node / npd[0]) % npd[1]),
                (int)(node / ((long long)npd[0] * npd[1]))};
    bool fixed = false;
    for (int f = 0; f < 6; ++f) {
      if (!(fixed_face_mask & (1 << f))) continue;
      int axis = f / 2;
      int at = (f % 2) ? npd[axis] - 1 : 0;
      if (g[axis] == at) fixed = true;
    }
    if (fixed)
      for (int c = 0; c < 3; ++c) mask[(size_t)node * 3 + c] = 1;
  }
}

// Consistent traction load on one face (assemble_traction_load,
// operator.hpp:381-443) with geometry order = solution order.
void traction_load(const double extents[3], const int cells[3], int p, const Basis& b, int face,
                   const double traction[3], std::vector<double>& load) {
  auto axis_c = box_axes(extents, cells, p);
  int npd[3] = {p * cells[0] + 1, p * cells[1] + 1, p * cells[2] + 1};
  long long nn = (long long)npd[0] * npd[1] * npd[2];
  load.assign((size_t)nn * 3, 0.0);
  if (face < 0) return;
  int axis = face / 2, t1 = (axis + 1) % 3, t2 = (axis + 2) % 3;
  bool at_max = face % 2 == 1;
  int elem_a = at_max ? cells[axis] - 1 : 0;
  int fixed = at_max ? p : 0;
  int q = b.q, n = p + 1;
  auto coord = [&](const int gi[3], int c) { return axis_c[c][gi[c]]; };
  for (int e2 = 0; e2 < cells[t2]; ++e2)
    for (int e1 = 0; e1 < cells[t1]; ++e1)
      for (int q2 = 0; q2 < q; ++q2)
        for (int qa = 0; qa < q; ++qa) {
          double tan1[3] = {0, 0, 0}, tan2[3] = {0, 0, 0};
          for (int j = 0; j <= p; ++j)
            for (int i = 0; i <= p; ++i) {
              int gi[3];
              gi[axis] = p * elem_a + fixed;
              gi[t1] = p * e1 + i;
              gi[t2] = p * e2 + j;
              double di = b.deriv[qa * n + i] * b.interp[q2 * n + j];
              double dj = b.interp[qa * n + i] * b.deriv[q2 * n + j];
              for (int c = 0; c < 3; ++c) {
                tan1[c] += di * coord(gi, c);
                tan2[c] += dj * coord(gi, c);
              }
            }
          double cr[3] = {tan1[1] * tan2[2] - tan1[2] * tan2[1], tan1[2] * tan2[0] - tan1[0] * tan2[2],
                          tan1[0] * tan2[1] - tan1[1] * tan2[0]};
          double area = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
          double ds = b.rule.weights[qa] * b.rule.weights[q2] * area;
          for (int j = 0; j <= p; ++j)
            for (int i = 0; i <= p; ++i) {
              int gi[3];
              gi[axis] = p * elem_a + fixed;
              gi[t1] = p * e1 + i;
              gi[t2] = p * e2 + j;
              long long node = gi[0] + (long long)npd[0] * (gi[1] + (long long)npd[1] * gi[2]);
              double phi = b.interp[qa * n + i] * b.interp[q2 * n + j];
              for (int c = 0; c < 3; ++c) load[(size_t)node * 3 + c] += phi * traction[c] * ds;
            }
        }
}

}  // namespace hxg
