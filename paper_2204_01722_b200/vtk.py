"""Legacy ASCII VTK writer (vtk.hpp:15-66): lattice points of the box mesh
(build_box_mesh node coordinates, mesh.hpp:35-60), each element split into
p^3 tri-linear sub-cells (type 12), the displacement as point vectors.
Same bytes as the reference for the same field (12 significant digits)."""
from __future__ import annotations

import numpy as np


def box_coords(extents, cells, order, lobatto):
    """Node coordinates (node-major xyz) of build_box_mesh (mesh.hpp:35-60)."""
    axes = []
    for d in range(3):
        h = extents[d] / cells[d]
        a = np.empty(order * cells[d] + 1)
        for e in range(cells[d]):
            for i in range(order + 1):
                a[e * order + i] = (e + 0.5 * (lobatto[i] + 1.0)) * h
        a[-1] = extents[d]  # no roundoff drift at the far boundary
        axes.append(a)
    z, y, x = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], 1)


def _g(v):
    return "%.12g" % v


def write_vtk(stream, extents, cells, order, u):
    """write_vtk (vtk.hpp:15-55)."""
    from .hexmg import build_lagrange_basis
    u = np.asarray(u.detach().cpu() if hasattr(u, "detach") else u, np.float64).ravel()
    npd = [order * c + 1 for c in cells]
    nn = npd[0] * npd[1] * npd[2]
    if u.size != 3 * nn:
        raise ValueError("displacement field size mismatch")
    X = box_coords(extents, cells, order, build_lagrange_basis(order).nodes)
    p = order
    ncell = cells[0] * cells[1] * cells[2] * p ** 3
    w = stream.write
    w("# vtk DataFile Version 3.0\nhexmg displacement field\nASCII\nDATASET UNSTRUCTURED_GRID\n")
    w(f"POINTS {nn} double\n")
    w("".join(f"{_g(a)} {_g(b)} {_g(c)}\n" for a, b, c in X))
    w(f"CELLS {ncell} {ncell * 9}\n")

    def idx(gx, gy, gz):
        return gx + npd[0] * (gy + npd[1] * gz)

    lines = []
    for ez in range(cells[2]):
        for ey in range(cells[1]):
            for ex in range(cells[0]):
                for k in range(p):
                    for j in range(p):
                        for i in range(p):
                            x0, y0, z0 = p * ex + i, p * ey + j, p * ez + k
                            lines.append(
                                f"8 {idx(x0, y0, z0)} {idx(x0 + 1, y0, z0)} {idx(x0 + 1, y0 + 1, z0)} "
                                f"{idx(x0, y0 + 1, z0)} {idx(x0, y0, z0 + 1)} {idx(x0 + 1, y0, z0 + 1)} "
                                f"{idx(x0 + 1, y0 + 1, z0 + 1)} {idx(x0, y0 + 1, z0 + 1)}\n")
    w("".join(lines))
    w(f"CELL_TYPES {ncell}\n" + "12\n" * ncell)
    w(f"POINT_DATA {nn}\nVECTORS displacement double\n")
    U = u.reshape(-1, 3)
    w("".join(f"{_g(a)} {_g(b)} {_g(c)}\n" for a, b, c in U))


def write_vtk_file(path, extents, cells, order, u):
    """write_vtk_file (vtk.hpp:57-64)."""
    try:
        with open(path, "w") as f:
            write_vtk(f, extents, cells, order, u)
    except OSError:
        raise OSError(f"cannot open '{path}' for writing") from None
