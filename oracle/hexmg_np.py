"""ORACLE / TEST INFRASTRUCTURE ONLY — numpy restatement of the reference hot path.

This module restates, in vectorised numpy, the algorithm of the reference
header library ``hexmg`` (/root/reference/proj/include/hexmg) for the FP64
matrix-free p-multigrid path.  It is a *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg may import
it.  The product (``paper_2204_01722_b200``) never does and fails loudly when
its CUDA library is missing.

Parity pinning: every function here is checked in ``tests/test_oracle.py``
against the reference itself, compiled unmodified into
``oracle/_ref/libhexmg_ref.so`` (see ``oracle/Makefile``), and against the
golden fixtures in ``tests/golden/`` generated from that library by
``tests/golden/gen_golden.py``.

Layouts follow the reference exactly:
  L-vector   interleaved ``3*node + c``                 (mesh.hpp:24, :98)
  E-vector   (e, c, a) with x-fastest a                 (basis.hpp:177-197)
  Q-grads    (e, c, d, q)                               (basis.hpp:221-244)
  state      (e, q, 17) = [w detJ, dxi/dx(9), tau(6), lambda log J]
                                                        (material.hpp:136-150)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# Quadrature (quadrature.hpp:20-86)
# --------------------------------------------------------------------------


def _legendre_with_deriv(n: int, x: float):
    """P_n(x), P_n'(x) by the three-term recurrence (quadrature.hpp:20-31)."""
    if n == 0:
        return 1.0, 0.0
    p0, p1 = 1.0, x
    for k in range(2, n + 1):
        p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k
        p0, p1 = p1, p2
    dp = n * (x * p1 - p0) / (x * x - 1.0)
    return p1, dp


def gauss_legendre(q: int):
    """q-point Gauss-Legendre rule, symmetrised (quadrature.hpp:37-60)."""
    if q < 1:
        raise ValueError("quadrature size must be >= 1")
    pts = [0.0] * q
    wts = [0.0] * q
    for i in range((q + 1) // 2):
        x = math.cos(math.pi * (i + 0.75) / (q + 0.5))
        for _ in range(100):
            p, dp = _legendre_with_deriv(q, x)
            dx = p / dp
            x -= dx
            if abs(dx) < 1e-16:
                break
        _, dp = _legendre_with_deriv(q, x)
        w = 2.0 / ((1.0 - x * x) * dp * dp)
        pts[q - 1 - i] = x
        pts[i] = -x
        wts[i] = wts[q - 1 - i] = w
    if q % 2 == 1:
        pts[q // 2] = 0.0
    return np.array(pts), np.array(wts)


def gauss_lobatto_nodes(p: int):
    """p+1 GLL nodes (quadrature.hpp:64-86)."""
    if p < 1:
        raise ValueError("basis order must be >= 1")
    n = p + 1
    x = [0.0] * n
    x[0], x[n - 1] = -1.0, 1.0
    for i in range(1, (n - 1) // 2 + 1):
        y = math.cos(math.pi * i / p)
        for _ in range(100):
            pp, dp = _legendre_with_deriv(p, y)
            d2p = (2.0 * y * dp - p * (p + 1.0) * pp) / (1.0 - y * y)
            dy = dp / d2p
            y -= dy
            if abs(dy) < 1e-16:
                break
        x[n - 1 - i] = abs(y)
        x[i] = -abs(y)
    if n % 2 == 1:
        x[n // 2] = 0.0
    return np.array(x)


# --------------------------------------------------------------------------
# Basis (basis.hpp:13-175)
# --------------------------------------------------------------------------


def _lagrange_tab(nodes, points, derivs: bool):
    """Barycentric Lagrange values / derivatives (basis.hpp:16-59)."""
    n = len(nodes)
    bary = np.ones(n)
    for i in range(n):
        for j in range(n):
            if j != i:
                bary[i] /= nodes[i] - nodes[j]
    vals = np.zeros((len(points), n))
    ders = np.zeros((len(points), n))
    for r, y in enumerate(points):
        hit = -1
        for i in range(n):
            if abs(y - nodes[i]) < 1e-13:
                hit = i
        if hit >= 0:
            vals[r, hit] = 1.0
            s = 0.0
            for i in range(n):
                if i == hit:
                    continue
                ders[r, i] = (bary[i] / bary[hit]) / (nodes[hit] - nodes[i])
                s += ders[r, i]
            ders[r, hit] = -s
            continue
        l, s = 1.0, 0.0
        for j in range(n):
            l *= y - nodes[j]
            s += 1.0 / (y - nodes[j])
        for i in range(n):
            vals[r, i] = bary[i] * l / (y - nodes[i])
            ders[r, i] = vals[r, i] * (s - 1.0 / (y - nodes[i]))
    return ders if derivs else vals


def lagrange_values(nodes, points):
    return _lagrange_tab(nodes, points, False)


@dataclass
class Basis1D:
    """basis.hpp:117-130."""

    order: int
    nodes: np.ndarray
    points: np.ndarray
    weights: np.ndarray
    interp: np.ndarray  # q x n
    deriv: np.ndarray  # q x n
    pinv: np.ndarray  # n x q
    colloc: np.ndarray  # q x q

    @property
    def n(self):
        return self.order + 1

    @property
    def q(self):
        return len(self.points)


def build_lagrange_basis(p: int, q: int | None = None, rule=None) -> Basis1D:
    """basis.hpp:134-175 (pinv by normal equations, colloc = deriv * pinv)."""
    if p < 1:
        raise ValueError("basis order must be >= 1")
    if rule is None:
        rule = gauss_legendre(p + 1 if q is None else q)
    pts, wts = rule
    if len(pts) < p + 1:
        raise ValueError("need at least p + 1 quadrature points for full column rank")
    nodes = gauss_lobatto_nodes(p)
    interp = lagrange_values(nodes, pts)
    deriv = _lagrange_tab(nodes, pts, True)
    pinv = np.linalg.solve(interp.T @ interp, interp.T)
    colloc = deriv @ pinv
    return Basis1D(p, nodes, pts, wts, interp, deriv, pinv, colloc)


def _contract(M, x, axis_from_fast: int, transpose: bool):
    """detail::contract (basis.hpp:250-285) on batched (..., n2, n1, n0) arrays.

    axis_from_fast = 0 contracts the x-fastest axis (last numpy axis)."""
    A = M.T if transpose else M
    ax = x.ndim - 1 - axis_from_fast
    y = np.tensordot(x, A, axes=([ax], [1]))  # contracted axis moved to end
    return np.moveaxis(y, -1, ax)


def grad_ref(b: Basis1D, ev):
    """Six-contraction gradient (basis.hpp:319-335).

    ev: (E, 3, n, n, n) [z, y, x] -> (E, 3, 3, q, q, q)."""
    v = _contract(b.interp, ev, 0, False)
    v = _contract(b.interp, v, 1, False)
    v = _contract(b.interp, v, 2, False)
    return np.stack([_contract(b.colloc, v, d, False) for d in range(3)], axis=2)


def grad_transpose_ref(b: Basis1D, qg):
    """Exact adjoint (basis.hpp:339-355). qg: (E, 3, 3, q,q,q) -> (E,3,n,n,n)."""
    acc = _contract(b.colloc, qg[:, :, 0], 0, True)
    acc = acc + _contract(b.colloc, qg[:, :, 1], 1, True)
    acc = acc + _contract(b.colloc, qg[:, :, 2], 2, True)
    t = _contract(b.interp, acc, 2, True)
    t = _contract(b.interp, t, 1, True)
    return _contract(b.interp, t, 0, True)


def dense_tabulation(b: Basis1D):
    """basis.hpp:424-451: grad[d] is (q^3, n^3) with x-fastest rows/cols."""
    B, D = b.interp, b.deriv
    # rows (qc, qb, qa) -> qa fastest; cols (k, j, i) -> i fastest.
    q, n = b.q, b.n
    t_interp = np.einsum("ck,bj,ai->cbakji", B, B, B).reshape(q**3, n**3)
    t0 = np.einsum("ck,bj,ai->cbakji", B, B, D).reshape(q**3, n**3)
    t1 = np.einsum("ck,bj,ai->cbakji", B, D, B).reshape(q**3, n**3)
    t2 = np.einsum("ck,bj,ai->cbakji", D, B, B).reshape(q**3, n**3)
    return t_interp, [t0, t1, t2]


# --------------------------------------------------------------------------
# Mesh, restriction, geometry (mesh.hpp:19-232)
# --------------------------------------------------------------------------


@dataclass
class BoxMesh:
    extents: tuple
    counts: tuple
    order: int
    npd: tuple  # nodes per dim
    coords: np.ndarray  # (num_nodes, 3)

    @property
    def num_nodes(self):
        return self.npd[0] * self.npd[1] * self.npd[2]

    @property
    def num_elements(self):
        return self.counts[0] * self.counts[1] * self.counts[2]


def build_box_mesh(extents, counts, order) -> BoxMesh:
    """mesh.hpp:35-71."""
    lob = gauss_lobatto_nodes(order)
    axes = []
    npd = []
    for d in range(3):
        m = order * counts[d] + 1
        npd.append(m)
        h = extents[d] / counts[d]
        a = np.zeros(m)
        for e in range(counts[d]):
            for i in range(order + 1):
                a[e * order + i] = (e + 0.5 * (lob[i] + 1.0)) * h
        a[-1] = extents[d]
        axes.append(a)
    Z, Y, X = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
    coords = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    return BoxMesh(tuple(extents), tuple(counts), order, tuple(npd), coords)


def build_restriction(mesh: BoxMesh):
    """mesh.hpp:119-138: (E, n^3) int32 node indices + multiplicity."""
    p = mesh.order
    cx, cy, cz = mesh.counts
    nx, ny, _ = mesh.npd
    ez, ey, ex = np.meshgrid(np.arange(cz), np.arange(cy), np.arange(cx), indexing="ij")
    k, j, i = np.meshgrid(np.arange(p + 1), np.arange(p + 1), np.arange(p + 1), indexing="ij")
    gx = p * ex.reshape(-1, 1) + i.reshape(1, -1)
    gy = p * ey.reshape(-1, 1) + j.reshape(1, -1)
    gz = p * ez.reshape(-1, 1) + k.reshape(1, -1)
    idx = (gx + nx * (gy + ny * gz)).astype(np.int32)
    mult = np.bincount(idx.ravel(), minlength=mesh.num_nodes).astype(np.int32)
    return idx, mult


def gather(idx, u, n):
    """ElementRestriction::gather (mesh.hpp:88-101) -> (E, 3, n, n, n)."""
    U = u.reshape(-1, 3)
    ev = U[idx]  # (E, n^3, 3)
    return np.ascontiguousarray(ev.transpose(0, 2, 1)).reshape(idx.shape[0], 3, n, n, n)


def scatter_add(idx, ev, num_nodes):
    """ElementRestriction::scatter_add (mesh.hpp:105-116), element order."""
    E = idx.shape[0]
    vals = ev.reshape(E, 3, -1).transpose(0, 2, 1).reshape(-1, 3)
    out = np.zeros((num_nodes, 3))
    flat = idx.ravel()
    for c in range(3):
        out[:, c] = np.bincount(flat, weights=vals[:, c], minlength=num_nodes)
    return out.ravel()


def select_boundary_nodes(mesh: BoxMesh, face: int):
    """mesh.hpp:151-164; face in (-x,+x,-y,+y,-z,+z) order."""
    axis = face // 2
    fixed = mesh.npd[axis] - 1 if face % 2 == 1 else 0
    gz, gy, gx = np.meshgrid(
        np.arange(mesh.npd[2]), np.arange(mesh.npd[1]), np.arange(mesh.npd[0]), indexing="ij"
    )
    g = [gx.ravel(), gy.ravel(), gz.ravel()]
    return np.nonzero(g[axis] == fixed)[0]


def build_constraints(mesh: BoxMesh, fixed_faces):
    """operator.hpp:36-55 (all components fixed, zero values)."""
    mask = np.zeros(3 * mesh.num_nodes, dtype=np.uint8)
    for f in fixed_faces:
        nodes = select_boundary_nodes(mesh, f)
        for c in range(3):
            mask[3 * nodes + c] = 1
    return mask


def compute_geometric_factors(mesh: BoxMesh, basis: Basis1D):
    """mesh.hpp:193-232: dxidX (E, nq, 3, 3) and weight (E, nq)."""
    idx, _ = build_restriction(mesh)
    n, q = basis.n, basis.q
    ev = gather(idx, mesh.coords.ravel(), n)
    g = grad_ref(basis, ev)  # (E, 3c, 3d, q, q, q)
    E = idx.shape[0]
    A = g.reshape(E, 3, 3, q**3).transpose(0, 3, 1, 2)  # (E, nq, c, d) = dX_c/dxi_d
    det = np.linalg.det(A)
    if not np.all(det > 0):
        raise ValueError("degenerate element")
    Ainv = _inv3(A)
    w = basis.weights
    W = np.einsum("c,b,a->cba", w, w, w).ravel()
    return Ainv, W[None, :] * det


# --------------------------------------------------------------------------
# 3x3 helpers (tensor3.hpp) vectorised over leading axes
# --------------------------------------------------------------------------


def _det3(m):
    return (
        m[..., 0, 0] * (m[..., 1, 1] * m[..., 2, 2] - m[..., 1, 2] * m[..., 2, 1])
        - m[..., 0, 1] * (m[..., 1, 0] * m[..., 2, 2] - m[..., 1, 2] * m[..., 2, 0])
        + m[..., 0, 2] * (m[..., 1, 0] * m[..., 2, 1] - m[..., 1, 1] * m[..., 2, 0])
    )


def _inv3(m):
    """Adjugate inverse (tensor3.hpp:94-110)."""
    r = np.empty_like(m)
    r[..., 0, 0] = m[..., 1, 1] * m[..., 2, 2] - m[..., 1, 2] * m[..., 2, 1]
    r[..., 0, 1] = m[..., 0, 2] * m[..., 2, 1] - m[..., 0, 1] * m[..., 2, 2]
    r[..., 0, 2] = m[..., 0, 1] * m[..., 1, 2] - m[..., 0, 2] * m[..., 1, 1]
    r[..., 1, 0] = m[..., 1, 2] * m[..., 2, 0] - m[..., 1, 0] * m[..., 2, 2]
    r[..., 1, 1] = m[..., 0, 0] * m[..., 2, 2] - m[..., 0, 2] * m[..., 2, 0]
    r[..., 1, 2] = m[..., 0, 2] * m[..., 1, 0] - m[..., 0, 0] * m[..., 1, 2]
    r[..., 2, 0] = m[..., 1, 0] * m[..., 2, 1] - m[..., 1, 1] * m[..., 2, 0]
    r[..., 2, 1] = m[..., 0, 1] * m[..., 2, 0] - m[..., 0, 0] * m[..., 2, 1]
    r[..., 2, 2] = m[..., 0, 0] * m[..., 1, 1] - m[..., 0, 1] * m[..., 1, 0]
    return r * (1.0 / _det3(m))[..., None, None]


SYM_IDX = [(0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2)]  # material.hpp:82


def lame_from_young_poisson(E, nu):
    """material.hpp:27-36."""
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    return mu, lam


class InvertedElementError(RuntimeError):
    def __init__(self, j, element=-1, point=-1):
        super().__init__(f"non-positive deformation jacobian {j} in element {element} at point {point}")
        self.jacobian, self.element, self.point = j, element, point


def residual_qfunction(mu, lam, G, dxidX, wdet):
    """residual_qpoint, Current storage (material.hpp:126-150).

    G: (..., 3c, 3d) reference gradient; returns (H, state(...,17))."""
    grad_u = G @ dxidX
    F = np.eye(3) + grad_u
    J = _det3(F)
    bad = ~(J > 0)
    if np.any(bad):
        first = np.flatnonzero(bad.ravel())[0]
        raise InvertedElementError(J.ravel()[first], *np.unravel_index(first, J.shape))
    logJ = np.log(J)
    dxidx = dxidX @ _inv3(F)
    b = F @ np.swapaxes(F, -1, -2)
    tau = mu * (b - np.eye(3))
    d = lam * logJ
    for i in range(3):
        tau[..., i, i] += d
    state = np.empty(G.shape[:-2] + (17,))
    state[..., 0] = wdet
    state[..., 1:10] = dxidx.reshape(dxidx.shape[:-2] + (9,))
    for k, (i, j) in enumerate(SYM_IDX):
        state[..., 10 + k] = tau[..., i, j]
    state[..., 16] = d
    H = wdet[..., None, None] * (tau @ np.swapaxes(dxidx, -1, -2))
    return H, state


def jacobian_qfunction(mu, lam, G, state):
    """jacobian_qpoint, Current storage (material.hpp:179-194)."""
    wdet = state[..., 0]
    dxidx = state[..., 1:10].reshape(state.shape[:-1] + (3, 3))
    tau = np.empty(state.shape[:-1] + (3, 3))
    for k, (i, j) in enumerate(SYM_IDX):
        tau[..., i, j] = state[..., 10 + k]
        tau[..., j, i] = state[..., 10 + k]
    llj = state[..., 16]
    grad_du = G @ dxidx
    deps = 0.5 * (grad_du + np.swapaxes(grad_du, -1, -2))
    k = grad_du @ tau
    tr = lam * np.trace(deps, axis1=-2, axis2=-1)
    c = 2.0 * (mu - llj)
    k = k + c[..., None, None] * deps
    for i in range(3):
        k[..., i, i] += tr
    return wdet[..., None, None] * (k @ np.swapaxes(dxidx, -1, -2))


# --------------------------------------------------------------------------
# Initial-configuration JacobianStorage variants (material.hpp:66-78,
# :152-175, :196-239): state [w, dxi/dX (9), grad_X u (9), +C^-1 sym + lambda
# log J (Tuned) | +S sym (AD)].  Strides 19 / 26 / 25.
# --------------------------------------------------------------------------
STATE_SCALARS = {0: 17, 1: 19, 2: 26, 3: 25}


class _Dual:
    """Forward-mode dual arrays (dual.hpp:9-40): value + directional derivative."""

    def __init__(self, v, d):
        self.v, self.d = v, d

    def __getitem__(self, k):
        return _Dual(self.v[k], self.d[k])

    def __add__(self, o):
        o = _lift(o)
        return _Dual(self.v + o.v, self.d + o.d)

    __radd__ = __add__

    def __sub__(self, o):
        o = _lift(o)
        return _Dual(self.v - o.v, self.d - o.d)

    def __rsub__(self, o):
        return _lift(o) - self

    def __mul__(self, o):
        o = _lift(o)
        return _Dual(self.v * o.v, self.v * o.d + self.d * o.v)

    __rmul__ = __mul__

    def __truediv__(self, o):
        o = _lift(o)
        inv = 1.0 / o.v
        return _Dual(self.v * inv, (self.d - self.v * o.d * inv) * inv)

    def __rtruediv__(self, o):
        return _lift(o) / self


def _lift(o):
    return o if isinstance(o, _Dual) else _Dual(o, np.zeros_like(o) if np.ndim(o) else 0.0)


def _dual_inv3(m):
    """Adjugate inverse (tensor3.hpp:94-110) of a dual (..., 3, 3)."""
    adj = [[m[..., 1, 1] * m[..., 2, 2] - m[..., 1, 2] * m[..., 2, 1],
            m[..., 0, 2] * m[..., 2, 1] - m[..., 0, 1] * m[..., 2, 2],
            m[..., 0, 1] * m[..., 1, 2] - m[..., 0, 2] * m[..., 1, 1]],
           [m[..., 1, 2] * m[..., 2, 0] - m[..., 1, 0] * m[..., 2, 2],
            m[..., 0, 0] * m[..., 2, 2] - m[..., 0, 2] * m[..., 2, 0],
            m[..., 0, 2] * m[..., 1, 0] - m[..., 0, 0] * m[..., 1, 2]],
           [m[..., 1, 0] * m[..., 2, 1] - m[..., 1, 1] * m[..., 2, 0],
            m[..., 0, 1] * m[..., 2, 0] - m[..., 0, 0] * m[..., 2, 1],
            m[..., 0, 0] * m[..., 1, 1] - m[..., 0, 1] * m[..., 1, 0]]]
    inv_det = 1.0 / _det3(m)
    ent = [[a * inv_det for a in row] for row in adj]
    v = np.stack([np.stack([a.v for a in row], -1) for row in ent], -2)
    d = np.stack([np.stack([a.d for a in row], -1) for row in ent], -2)
    return _Dual(v, d)


def _dual_second_piola(mu, lam, e):
    """S(E) = mu I + (lambda log J - mu) C^-1, C = I + 2E (material.hpp:110-121), dual E."""
    c = _Dual(np.eye(3) + 2.0 * e.v, 2.0 * e.d)
    dj = _det3(c)
    log_j = 0.5 * _Dual(np.log(dj.v), dj.d / dj.v)
    ci = _dual_inv3(c)
    coeff = lam * log_j - mu
    return _Dual(mu * np.eye(3) + coeff.v[..., None, None] * ci.v,
                 coeff.v[..., None, None] * ci.d + coeff.d[..., None, None] * ci.v)


def _sym(m):
    return 0.5 * (m + np.swapaxes(m, -1, -2))


def _unpack_sym(v):
    m = np.empty(v.shape[:-1] + (3, 3))
    for k, (i, j) in enumerate(SYM_IDX):
        m[..., i, j] = v[..., k]
        m[..., j, i] = v[..., k]
    return m


def residual_qfunction_initial(storage, mu, lam, G, dxidX, wdet):
    """residual_qpoint, initial-configuration storages (material.hpp:152-175)."""
    grad_u = G @ dxidX
    F = np.eye(3) + grad_u
    J = _det3(F)
    bad = ~(J > 0)
    if np.any(bad):
        first = np.flatnonzero(bad.ravel())[0]
        raise InvertedElementError(J.ravel()[first], *np.unravel_index(first, J.shape))
    log_j = np.log(J)
    C = np.swapaxes(F, -1, -2) @ F
    Ci = _inv3(C)
    coeff = lam * log_j - mu
    S = mu * np.eye(3) + coeff[..., None, None] * Ci
    st = np.zeros(G.shape[:-2] + (STATE_SCALARS[storage],))
    st[..., 0] = wdet
    st[..., 1:10] = np.broadcast_to(dxidX, G.shape).reshape(G.shape[:-2] + (9,))
    st[..., 10:19] = grad_u.reshape(G.shape[:-2] + (9,))
    for k, (i, j) in enumerate(SYM_IDX):
        if storage == 2:
            st[..., 19 + k] = Ci[..., i, j]
        elif storage == 3:
            st[..., 19 + k] = S[..., i, j]
    if storage == 2:
        st[..., 25] = lam * log_j
    H = wdet[..., None, None] * ((F @ S) @ np.swapaxes(dxidX, -1, -2))
    return H, st


def jacobian_qfunction_initial(storage, mu, lam, G, st):
    """jacobian_qpoint, initial-configuration storages (material.hpp:196-239)."""
    wdet = st[..., 0]
    dxidX = st[..., 1:10].reshape(st.shape[:-1] + (3, 3))
    grad_u = st[..., 10:19].reshape(st.shape[:-1] + (3, 3))
    F = np.eye(3) + grad_u
    dF = G @ dxidX
    dE = _sym(np.swapaxes(F, -1, -2) @ dF)
    if storage == 3:
        S = _unpack_sym(st[..., 19:25])
        E = _sym(grad_u) + 0.5 * (np.swapaxes(grad_u, -1, -2) @ grad_u)
        dS = _dual_second_piola(mu, lam, _Dual(E, dE)).d
    else:
        if storage == 2:
            Ci, llj = _unpack_sym(st[..., 19:25]), st[..., 25]
        else:
            C = np.swapaxes(F, -1, -2) @ F
            Ci, llj = _inv3(C), 0.5 * lam * np.log(_det3(C))
        coeff = llj - mu
        S = mu * np.eye(3) + coeff[..., None, None] * Ci
        cde = np.einsum("...ij,...ij->...", Ci, dE)
        dS = (lam * cde)[..., None, None] * Ci - (2.0 * coeff)[..., None, None] * ((Ci @ dE) @ Ci)
    return wdet[..., None, None] * ((dF @ S + F @ dS) @ np.swapaxes(dxidX, -1, -2))


# --------------------------------------------------------------------------
# Composed operator (operator.hpp:70-354)
# --------------------------------------------------------------------------


def _qgrad_to_pts(qg):
    """(E, 3c, 3d, q,q,q) -> (E, nq, 3c, 3d)."""
    E = qg.shape[0]
    return qg.reshape(E, 3, 3, -1).transpose(0, 3, 1, 2)


def _pts_to_qgrad(H, q):
    E = H.shape[0]
    return np.ascontiguousarray(H.transpose(0, 2, 3, 1)).reshape(E, 3, 3, q, q, q)


class Operator:
    """MatrixFreeOperator (operator.hpp:70-373); storage = JacobianStorage id."""

    def __init__(self, mesh: BoxMesh, basis: Basis1D, dxidX, weight, mu, lam, mask, state_ref=None,
                 storage=0):
        self.storage = storage
        self.mesh, self.basis = mesh, basis
        self.idx, self.mult = build_restriction(mesh)
        self.dxidX, self.weight = dxidX, weight
        self.mu, self.lam = mu, lam
        self.mask = mask
        self.state_ref = state_ref if state_ref is not None else {"state": None}
        self.external_load = None
        self.load_scale = 1.0

    @property
    def size(self):
        return 3 * self.mesh.num_nodes

    @property
    def state(self):
        return self.state_ref["state"]

    def apply_residual(self, u):
        b = self.basis
        ev = gather(self.idx, u, b.n)
        G = _qgrad_to_pts(grad_ref(b, ev))
        try:
            if self.storage:
                H, st = residual_qfunction_initial(self.storage, self.mu, self.lam, G, self.dxidX,
                                                   self.weight)
            else:
                H, st = residual_qfunction(self.mu, self.lam, G, self.dxidX, self.weight)
        except InvertedElementError as err:
            raise InvertedElementError(err.jacobian, err.element, err.point) from None
        self.state_ref["state"] = st
        out = scatter_add(self.idx, grad_transpose_ref(b, _pts_to_qgrad(H, b.q)), self.mesh.num_nodes)
        if self.external_load is not None:
            out = out - self.load_scale * self.external_load
        if self.mask is not None:
            out[self.mask != 0] = 0.0
        return out

    def apply_jacobian(self, du):
        if self.state is None:
            raise RuntimeError("quadrature state not initialized")
        b = self.basis
        x = du.copy()
        if self.mask is not None:
            x[self.mask != 0] = 0.0
        ev = gather(self.idx, x, b.n)
        G = _qgrad_to_pts(grad_ref(b, ev))
        H = self._jacobian_qf(G, self.state)
        out = scatter_add(self.idx, grad_transpose_ref(b, _pts_to_qgrad(H, b.q)), self.mesh.num_nodes)
        if self.mask is not None:
            out[self.mask != 0] = du[self.mask != 0]
        return out

    def _jacobian_qf(self, G, st):
        if self.storage:
            return jacobian_qfunction_initial(self.storage, self.mu, self.lam, G, st)
        return jacobian_qfunction(self.mu, self.lam, G, st)

    def pointwise_tensor(self):
        """D[e,q,(c1,d1),(c2,d2)] by probing (operator.hpp:233-243)."""
        st = self.state
        E, nq = st.shape[:2]
        D = np.zeros((E, nq, 9, 9))
        for c2 in range(3):
            for d2 in range(3):
                unit = np.zeros((E, nq, 3, 3))
                unit[..., c2, d2] = 1.0
                h = self._jacobian_qf(unit, st)
                D[..., :, c2 * 3 + d2] = h.reshape(E, nq, 9)
        return D

    def extract_diagonal(self):
        """operator.hpp:247-283."""
        _, grads = dense_tabulation(self.basis)
        g = np.stack(grads, axis=-1)  # (nq, npe, 3d)
        D = self.pointwise_tensor().reshape(self.state.shape[0], -1, 3, 3, 3, 3)
        Dcc = np.einsum("eqcacb->eqcab", D)  # D[(c,d1),(c,d2)]
        contrib = np.einsum("qad,eqcdf,qaf->eac", g, Dcc, g)  # (E, npe, 3)
        out = np.zeros((self.mesh.num_nodes, 3))
        flat = self.idx.ravel()
        for c in range(3):
            out[:, c] = np.bincount(flat, weights=contrib[:, :, c].ravel(), minlength=self.mesh.num_nodes)
        out = out.ravel()
        if self.mask is not None:
            out[self.mask != 0] = 1.0
        return out

    def assemble_dense(self):
        """Assembled Jacobian as the reference's coo_symbolic/coo_numeric
        (assembly.hpp:142-230) would produce, returned dense (small sizes)."""
        _, grads = dense_tabulation(self.basis)
        g = np.stack(grads, axis=-1)  # (nq, npe, 3)
        E = self.state.shape[0]
        D = self.pointwise_tensor().reshape(E, -1, 3, 3, 3, 3)  # e q ca d1 cb d2
        Ke = np.einsum("qad,eqcdfg,qbg->eacbf", g, D, g)  # (E, a, ca, b, cb)
        npe = g.shape[1]
        Ke = Ke.reshape(E, 3 * npe, 3 * npe)
        dofs = (3 * self.idx[:, :, None] + np.arange(3)[None, None, :]).reshape(E, -1)
        n = self.size
        A = np.zeros((n, n))
        fixed = self.mask != 0 if self.mask is not None else np.zeros(n, bool)
        for e in range(E):
            d = dofs[e]
            keep = ~fixed[d]
            dk = d[keep]
            A[np.ix_(dk, dk)] += Ke[e][np.ix_(keep, keep)]
        A[fixed, fixed] = 1.0
        return A


def traction_load(mesh: BoxMesh, basis: Basis1D, face: int, traction):
    """assemble_traction_load (operator.hpp:381-443), geometry order == order."""
    p = mesh.order
    axis = face // 2
    t1, t2 = (axis + 1) % 3, (axis + 2) % 3
    at_max = face % 2 == 1
    elem_a = mesh.counts[axis] - 1 if at_max else 0
    fixed = p if at_max else 0
    q = basis.q
    B, Dv, w = basis.interp, basis.deriv, basis.weights
    load = np.zeros(3 * mesh.num_nodes)
    coords = mesh.coords
    nx, ny, _ = mesh.npd

    def node(gi):
        return gi[0] + nx * (gi[1] + ny * gi[2])

    for e2 in range(mesh.counts[t2]):
        for e1 in range(mesh.counts[t1]):
            for q2 in range(q):
                for qa in range(q):
                    tan1 = np.zeros(3)
                    tan2 = np.zeros(3)
                    for j in range(p + 1):
                        for i in range(p + 1):
                            gi = [0, 0, 0]
                            gi[axis] = p * elem_a + fixed
                            gi[t1] = p * e1 + i
                            gi[t2] = p * e2 + j
                            nd = node(gi)
                            di = Dv[qa, i] * B[q2, j]
                            dj = B[qa, i] * Dv[q2, j]
                            tan1 += di * coords[nd]
                            tan2 += dj * coords[nd]
                    area = np.linalg.norm(np.cross(tan1, tan2))
                    ds = w[qa] * w[q2] * area
                    for j in range(p + 1):
                        for i in range(p + 1):
                            gi = [0, 0, 0]
                            gi[axis] = p * elem_a + fixed
                            gi[t1] = p * e1 + i
                            gi[t2] = p * e2 + j
                            nd = node(gi)
                            phi = B[qa, i] * B[q2, j]
                            load[3 * nd : 3 * nd + 3] += phi * np.asarray(traction) * ds
    return load


# --------------------------------------------------------------------------
# Transfers, smoother, CG, Lanczos, V-cycle (multigrid.hpp, smoother.hpp, cg.hpp)
# --------------------------------------------------------------------------


def default_schedule(p):
    """multigrid.hpp:15-19."""
    out = [p]
    while out[-1] > 1:
        out.append((out[-1] + 1) // 2)
    return out


class Prolongation:
    """multigrid.hpp:25-74 (and ctof / 1/m from build_hierarchy :254-266)."""

    def __init__(self, fine_order, coarse_order, idx_f, idx_c, mult_f, nn_f, nn_c):
        self.ctof = lagrange_values(gauss_lobatto_nodes(coarse_order), gauss_lobatto_nodes(fine_order))
        self.nf, self.nc = fine_order + 1, coarse_order + 1
        self.idx_f, self.idx_c = idx_f, idx_c
        self.inv_m = 1.0 / mult_f
        self.nn_f, self.nn_c = nn_f, nn_c

    def apply(self, xc):
        ev = gather(self.idx_c, xc, self.nc)
        for ax in range(3):
            ev = _contract(self.ctof, ev, ax, False)
        xf = scatter_add(self.idx_f, ev, self.nn_f).reshape(-1, 3)
        return (xf * self.inv_m[:, None]).ravel()

    def apply_transpose(self, xf):
        s = (xf.reshape(-1, 3) * self.inv_m[:, None]).ravel()
        ev = gather(self.idx_f, s, self.nf)
        for ax in (2, 1, 0):
            ev = _contract(self.ctof, ev, ax, True)
        return scatter_add(self.idx_c, ev, self.nn_c)


def rough_seed(n, mask=None):
    """cg.hpp:138-147: mt19937(0x9e3779b9) stream."""
    rng = np.random.RandomState(0x9E3779B9)
    raw = rng.randint(0, 2**32, size=n, dtype=np.uint64).astype(np.float64)
    v = 2.0 * (raw * (1.0 / 4294967296.0)) - 1.0
    if mask is not None:
        v[mask != 0] = 0.0
    return v


def lanczos_eigs(alphas, betas):
    """cg.hpp:56-73 (eigenvalues of the CG/Lanczos tridiagonal)."""
    k = len(alphas)
    if k == 0:
        return 0.0, 0.0
    T = np.zeros((k, k))
    T[0, 0] = 1.0 / alphas[0]
    for i in range(1, k):
        T[i, i] = 1.0 / alphas[i] + betas[i - 1] / alphas[i - 1]
        off = math.sqrt(betas[i - 1]) / alphas[i - 1]
        T[i, i - 1] = T[i - 1, i] = off
    ev = np.linalg.eigvalsh(T)
    return float(ev.min()), float(ev.max())


@dataclass
class CgReport:
    iterations: int = 0
    converged: bool = False
    history: list = field(default_factory=list)
    eig_min: float = 0.0
    eig_max: float = 0.0


def cg_solve(A, M, b, x, rtol, max_iterations):
    """cg.hpp:81-134 (natural-norm PCG)."""
    r = b - A(x)
    z = M(r)
    rz = float(r @ z)
    rep = CgReport()
    nat0 = math.sqrt(rz)
    if nat0 == 0.0:
        rep.converged = True
        return rep
    rep.history.append(nat0)
    p = z.copy()
    alphas, betas = [], []
    for _ in range(max_iterations):
        ap = A(p)
        pap = float(p @ ap)
        if pap <= 0:
            raise RuntimeError("indefinite")
        alpha = rz / pap
        alphas.append(alpha)
        x += alpha * p
        r -= alpha * ap
        z = M(r)
        rz_new = float(r @ z)
        rep.iterations += 1
        nat = math.sqrt(max(rz_new, 0.0))
        if nat > 0:
            rep.history.append(nat)
        if nat <= rtol * nat0:
            rep.converged = True
            break
        if rz_new <= 0:
            rep.converged = rz_new == 0
            break
        beta = rz_new / rz
        betas.append(beta)
        p = z + beta * p
        rz = rz_new
    betas = betas[: max(len(alphas) - 1, 0)]
    rep.eig_min, rep.eig_max = lanczos_eigs(alphas, betas)
    return rep


def estimate_lambda_max(A, M, seed, iterations=10):
    """cg.hpp:152-184."""
    r = seed.copy()
    z = M(r)
    rz = float(r @ z)
    alphas, betas = [], []
    if rz <= 0:
        return 1.0
    p = z.copy()
    for it in range(iterations):
        ap = A(p)
        pap = float(p @ ap)
        if pap <= 0:
            break
        alpha = rz / pap
        alphas.append(alpha)
        r -= alpha * ap
        z = M(r)
        rz_new = float(r @ z)
        if rz_new <= 0:
            break
        if it + 1 < iterations:
            betas.append(rz_new / rz)
        p = z + (rz_new / rz) * p
        rz = rz_new
    if not alphas:
        return 1.0
    return lanczos_eigs(alphas, betas[: len(alphas) - 1])[1]


class Chebyshev:
    """smoother.hpp:15-63 (degree 2 on [0.1, 1.1] lambda_max)."""

    def __init__(self, A, diag, mask, degree=2):
        self.inv_diag = 1.0 / diag
        self.degree = degree
        seed = rough_seed(len(diag), mask)
        self.lambda_max = estimate_lambda_max(A, lambda r: self.inv_diag * r, seed, 10)
        self.lo, self.hi = 0.1 * self.lambda_max, 1.1 * self.lambda_max

    def apply(self, A, b, x):
        theta = 0.5 * (self.hi + self.lo)
        delta = 0.5 * (self.hi - self.lo)
        sigma = theta / delta
        rho = 1.0 / sigma
        r = b - A(x)
        d = self.inv_diag * r / theta
        for k in range(1, self.degree + 1):
            x += d
            if k == self.degree:
                break
            r = b - A(x)
            rho_new = 1.0 / (2.0 * sigma - rho)
            d = rho_new * rho * d + (2.0 * rho_new / delta) * self.inv_diag * r
            rho = rho_new
        return x


class Hierarchy:
    """MultigridHierarchy + build_hierarchy (multigrid.hpp:88-268) with a
    dense Cholesky coarse solve (the reference uses sparse SimplicialLLT; both
    are exact)."""

    def __init__(self, extents, counts, order, q, fixed_faces, mu, lam, fine_op: Operator):
        self.levels = []
        sched = default_schedule(order)
        state_ref = fine_op.state_ref
        for s, p in enumerate(sched):
            if s == 0:
                op = fine_op
            else:
                mesh = build_box_mesh(extents, counts, p)
                basis = build_lagrange_basis(p, rule=(fine_op.basis.points, fine_op.basis.weights))
                op = Operator(mesh, basis, fine_op.dxidX, fine_op.weight, mu, lam,
                              build_constraints(mesh, fixed_faces), state_ref)
            self.levels.insert(0, op)
        self.transfers = [None]
        for k in range(1, len(self.levels)):
            f, c = self.levels[k], self.levels[k - 1]
            self.transfers.append(Prolongation(f.mesh.order, c.mesh.order, f.idx, c.idx, f.mult,
                                               f.mesh.num_nodes, c.mesh.num_nodes))

    def setup_numeric(self):
        import scipy.linalg as sla

        self.smoothers = [None]
        for k in range(1, len(self.levels)):
            op = self.levels[k]
            self.smoothers.append(Chebyshev(op.apply_jacobian, op.extract_diagonal(), op.mask))
        self.coarse_matrix = self.levels[0].assemble_dense()
        self.chol = sla.cho_factor(self.coarse_matrix, lower=True)

    def cycle(self, k, b, x):
        import scipy.linalg as sla

        if k == 0:
            x[:] = sla.cho_solve(self.chol, b)
            return x
        op = self.levels[k]
        A = op.apply_jacobian
        x = self.smoothers[k].apply(A, b, x)
        r = b - A(x)
        rc = self.transfers[k].apply_transpose(r)
        cm = self.levels[k - 1].mask
        rc[cm != 0] = 0.0
        ec = self.cycle(k - 1, rc, np.zeros_like(rc))
        corr = self.transfers[k].apply(ec)
        corr[op.mask != 0] = 0.0
        x += corr
        return self.smoothers[k].apply(A, b, x)

    def v_cycle(self, b, x):
        x = self.cycle(len(self.levels) - 1, b, x)
        m = self.levels[-1].mask
        x[m != 0] = b[m != 0]
        return x

    def precondition(self, r):
        return self.v_cycle(r, np.zeros_like(r))


@dataclass
class Problem:
    """The configured pieces FemProblem (problem.hpp:19-58) builds, restated."""

    mesh: BoxMesh
    basis: Basis1D
    op: Operator
    load: np.ndarray
    fixed_faces: tuple
    mu: float
    lam: float
    extents: tuple
    counts: tuple


def make_problem(extents, counts, order, q=0, fixed_faces=(0,), traction_face=-1,
                 traction=(0.0, 0.0, 0.0), young=1.0, poisson=0.3, storage=0) -> Problem:
    q = q or order + 1
    mesh = build_box_mesh(extents, counts, order)
    basis = build_lagrange_basis(order, q)
    dxidX, weight = compute_geometric_factors(mesh, basis)
    mu, lam = lame_from_young_poisson(young, poisson)
    mask = build_constraints(mesh, fixed_faces)
    op = Operator(mesh, basis, dxidX, weight, mu, lam, mask, storage=storage)
    load = np.zeros(op.size)
    if traction_face >= 0:
        load = traction_load(mesh, basis, traction_face, traction)
    op.external_load = load
    return Problem(mesh, basis, op, load, tuple(fixed_faces), mu, lam, tuple(extents), tuple(counts))
