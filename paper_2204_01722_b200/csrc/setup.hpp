// Host-side setup (quadrature, basis, geometry, constraints, loads).
#pragma once

#include <array>
#include <cstdint>
#include <vector>

namespace hxg {

struct Rule {
  std::vector<double> points, weights;
};

// Basis1D (basis.hpp:117-130): tabulations are row-major (points x nodes).
struct Basis {
  int p = 0, q = 0;
  std::vector<double> nodes;
  Rule rule;
  std::vector<double> interp, deriv, pinv, colloc;
};

Rule gauss_legendre(int q);
std::vector<double> gauss_lobatto(int p);
void lagrange_tabulate(const std::vector<double>& nodes, const std::vector<double>& points,
                       std::vector<double>* vals, std::vector<double>* ders);
Basis build_basis(int p, const Rule& rule);
Basis build_basis(int p, int q);
std::array<std::vector<double>, 3> box_axes(const double extents[3], const int cells[3], int p);
void geometry(const double extents[3], const int cells[3], int p, const Basis& b,
              std::vector<double>& dxidX, std::vector<double>& weight);
void face_mask(const int cells[3], int p, int fixed_face_mask, std::vector<uint8_t>& mask);
void traction_load(const double extents[3], const int cells[3], int p, const Basis& b, int face,
                   const double traction[3], std::vector<double>& load);

}  // namespace hxg
