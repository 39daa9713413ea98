"""Slab-partitioned p-multigrid PCG across ranks.

The reference is single-process; the paper runs the same
algorithm distributed, with PETSc star-forest sums of the shared nodes after
every operator application.  Here each rank owns a
contiguous slab of elements along x (``partition.slab_partition``) and holds
the hexmg objects of its slab on its GPU; this module composes the reference
algorithm from them:

* operator apply (operator.hpp:184-215): local apply, then the interface
  planes of the neighbouring slabs are summed (``partition.exchange_faces``:
  one grouped send/recv per face over NCCL);
* Jacobi diagonal (operator.hpp:247-283): local diagonal + the same exchange;
* p-transfer (multigrid.hpp:25-74): the local transfers use the local
  multiplicities, which on an interface plane are half the global ones, so
  prolongation = local prolong, exchange, x 1/2 on the planes; restriction =
  x 1/2 on the planes, local restrict, exchange (both exact scalings);
* Chebyshev smoothing (smoother.hpp:41-62) and lambda_max from 10
  CG-Lanczos steps (cg.hpp:152-184) on the distributed operator, started from
  the GLOBAL rough_seed stream sliced to the slab (cg.hpp:138-147), so
  lambda_max does not depend on the partition;
* coarse solve (coarse_solver.hpp:16-47): the slab coarse matrices are
  summed into the global p = 1 matrix (one all-reduce of its values at each
  numeric setup), every rank factorises it (replicated, the fallback of
  SURVEY.md §8(e)) and each V-cycle all-reduces the coarse right-hand side;
* PCG (cg.hpp:81-134): dots over owned entries (a shared plane belongs to the
  lower rank), one all-reduce per dot, two per iteration.

The level operations come from a *backend* (duck-typed):
``levels`` (orders, coarse first), ``size(k)``, ``npd(k)``, ``mask(k)``,
``apply(k, x)``, ``diagonal(k)``, ``prolong(kc, xc)``, ``restrict(kc, xf)``,
``coarse_csr()``, ``coarse_solver(row_ptr, cols, npd)``, ``device`` and, for
the Newton driver, ``residual(u)`` and ``set_time(t)``.
``SlabBackend`` is the GPU one (libhexmg_b200 through the C-ABI); the CPU
tests plug the numpy oracle in the same place.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from dist_partition_model import Block, exchange_block, exchange_faces


# --------------------------------------------------------------------------
# communication helpers
# --------------------------------------------------------------------------
class SlabComm:
    """Rank / world / process group plus the slab-interface primitives."""

    def __init__(self, rank=0, world=1, dist=None):
        self.rank, self.world, self.dist = rank, world, dist if world > 1 else None
        self._owned = {}

    def exchange(self, y, npd):
        if self.dist is not None:
            exchange_faces(y, npd, self.rank, self.world, self.dist)
        return y

    def scale_interfaces(self, y, npd, factor):
        """y *= factor on the node planes shared with a neighbouring slab."""
        if self.world == 1:
            return y
        nx, ny, nz = npd
        v = y.view(nz, ny, nx, 3)
        if self.rank > 0:
            v[:, :, 0, :] *= factor
        if self.rank + 1 < self.world:
            v[:, :, nx - 1, :] *= factor
        return y

    def owned(self, npd, device):
        key = (tuple(npd), str(device))
        if key not in self._owned:
            nx, ny, nz = npd
            m = torch.ones(nz, ny, nx, 3, dtype=torch.bool, device=device)
            if self.rank > 0:
                m[:, :, 0, :] = False
            self._owned[key] = m.reshape(-1)
        return self._owned[key]

    def dot(self, x, y, npd):
        """x . y over owned entries, summed over ranks (one f64 all-reduce)."""
        m = self.owned(npd, x.device)
        local = torch.dot(x[m], y[m]).reshape(1)
        if self.dist is not None:
            self.dist.all_reduce(local)
        return float(local.item())

    def all_reduce_(self, t):
        if self.dist is not None:
            self.dist.all_reduce(t)
        return t


class BlockComm(SlabComm):
    """The same primitives for a px x py x pz block partition
    (``partition.block_partition``): interface sums one direction after the
    other, interface scaling per shared direction (a node on k partition
    planes has 2^k times the local multiplicity), ownership by the lower
    block in every direction."""

    def __init__(self, block: Block, dist=None):
        super().__init__(block.rank, block.world, dist)
        self.block = block

    def _planes(self, v, d, npd):
        n = npd[d]
        out = []
        if self.block.neighbour(d, -1) is not None:
            out.append(0)
        if self.block.neighbour(d, +1) is not None:
            out.append(n - 1)
        sl = [(lambda i: v[:, :, i, :]), (lambda i: v[:, i, :, :]), (lambda i: v[i, :, :, :])][d]
        return [sl(i) for i in out]

    def exchange(self, y, npd):
        if self.dist is not None:
            exchange_block(y, npd, self.block, self.dist)
        return y

    def scale_interfaces(self, y, npd, factor):
        if self.world == 1:
            return y
        v = y.view(npd[2], npd[1], npd[0], 3)
        for d in range(3):
            for pl in self._planes(v, d, npd):
                pl *= factor
        return y

    def owned(self, npd, device):
        key = (tuple(npd), str(device))
        if key not in self._owned:
            m = torch.ones(npd[2], npd[1], npd[0], 3, dtype=torch.bool, device=device)
            if self.block.neighbour(0, -1) is not None:
                m[:, :, 0, :] = False
            if self.block.neighbour(1, -1) is not None:
                m[:, 0, :, :] = False
            if self.block.neighbour(2, -1) is not None:
                m[0, :, :, :] = False
            self._owned[key] = m.reshape(-1)
        return self._owned[key]


def global_rough_seed_slice(global_npd, node0, local_npd, mask=None):
    """rough_seed (cg.hpp:138-147, mt19937(0x9e3779b9)) of the GLOBAL vector,
    restricted to this block's nodes (node0: first global node per direction,
    or the x offset alone for a slab); constrained entries zeroed."""
    n = 3 * global_npd[0] * global_npd[1] * global_npd[2]
    raw = np.random.RandomState(0x9E3779B9).randint(0, 2**32, size=n, dtype=np.uint64)
    v = 2.0 * (raw.astype(np.float64) * (1.0 / 4294967296.0)) - 1.0
    v = v.reshape(global_npd[2], global_npd[1], global_npd[0], 3)
    x0, y0, z0 = (node0, 0, 0) if np.isscalar(node0) else node0
    v = np.ascontiguousarray(v[z0:z0 + local_npd[2], y0:y0 + local_npd[1],
                               x0:x0 + local_npd[0], :]).ravel()
    if mask is not None:
        v[np.asarray(mask, bool)] = 0.0
    return v


def lanczos_eigs(alphas, betas):
    """Eigenvalues of the CG/Lanczos tridiagonal (cg.hpp:56-73)."""
    k = len(alphas)
    if k == 0:
        return 0.0, 0.0
    T = np.zeros((k, k))
    T[0, 0] = 1.0 / alphas[0]
    for i in range(1, k):
        T[i, i] = 1.0 / alphas[i] + betas[i - 1] / alphas[i - 1]
        T[i, i - 1] = T[i - 1, i] = math.sqrt(betas[i - 1]) / alphas[i - 1]
    ev = np.linalg.eigvalsh(T)
    return float(ev.min()), float(ev.max())


def q1_lattice_pattern(npd, mask):
    """coo_symbolic (assembly.hpp:142-176) of the global p = 1 operator: the
    27-point node stencil x 3 components, sorted columns; constrained rows
    keep only their diagonal and constrained columns are dropped."""
    nx, ny, nz = npd
    n = 3 * nx * ny * nz
    mask = np.asarray(mask, bool)
    node = np.arange(nx * ny * nz)
    gx, gy, gz = node % nx, (node // nx) % ny, node // (nx * ny)
    cols = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((gx + dx >= 0) & (gx + dx < nx) & (gy + dy >= 0) & (gy + dy < ny) &
                      (gz + dz >= 0) & (gz + dz < nz))
                nb = np.where(ok, node + dx + nx * (dy + ny * dz), -1)
                for c in range(3):
                    cols.append(np.where(ok, 3 * nb + c, -1))
    C = np.stack(cols, 1)                         # (nodes, 81) sorted (node-major, c fastest)
    C = np.repeat(C, 3, axis=0)                   # rows 3 node + c
    rows = np.arange(n)
    keep = C >= 0
    keep &= ~mask[np.where(C >= 0, C, 0)]         # drop constrained columns
    keep[mask] = False
    keep[mask, :] = False
    diag = np.zeros_like(keep)
    # constrained rows: the diagonal alone (its column is itself constrained)
    rc = np.nonzero(mask)[0]
    C[rc, 0] = rc
    diag[rc, 0] = True
    keep |= diag
    counts = keep.sum(1)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    colidx = C[keep]
    return row_ptr, colidx.astype(np.int64)


# --------------------------------------------------------------------------
# the distributed hierarchy
# --------------------------------------------------------------------------
class DistributedHierarchy:
    """MultigridHierarchy (multigrid.hpp:88-194) over slab-partitioned
    levels; ``global_cells`` is the whole box, ``x0`` this slab's first
    element along x (or a block's first element per direction, a 3-tuple),
    ``global_mask_fn(order)`` the global constraint mask of a level (for the
    coarse pattern)."""

    def __init__(self, backend, comm: SlabComm, global_cells, x0, global_mask_fn, degree=2,
                 pre_smooth=1, post_smooth=1):
        self.b, self.comm = backend, comm
        self.global_cells, self.x0 = tuple(global_cells), x0
        self.e0 = (x0, 0, 0) if np.isscalar(x0) else tuple(x0)
        self.global_mask_fn = global_mask_fn
        self.degree, self.pre, self.post = degree, pre_smooth, post_smooth
        self.L = len(backend.levels)
        self.inv_diag = [None] * self.L
        self.lambda_max = [0.0] * self.L
        self._coarse = None

    # -- distributed primitives --------------------------------------------
    def npd(self, k):
        return self.b.npd(k)

    def global_npd(self, k):
        p = self.b.levels[k]
        c = self.global_cells
        return (p * c[0] + 1, p * c[1] + 1, p * c[2] + 1)

    def apply(self, k, x):
        return self.comm.exchange(self.b.apply(k, x), self.npd(k))

    def dot(self, k, x, y):
        return self.comm.dot(x, y, self.npd(k))

    def prolong(self, kc, xc):
        xf = self.comm.exchange(self.b.prolong(kc, xc), self.npd(kc + 1))
        return self.comm.scale_interfaces(xf, self.npd(kc + 1), 0.5)

    def restrict_to(self, kc, xf):
        t = self.comm.scale_interfaces(xf.clone(), self.npd(kc + 1), 0.5)
        return self.comm.exchange(self.b.restrict(kc, t), self.npd(kc))

    # -- setup ----------------------------------------------------------------
    def _estimate_lambda_max(self, k, iterations=10):
        """estimate_lambda_max (cg.hpp:152-184) on the distributed D^-1 A."""
        p = self.b.levels[k]
        seed = global_rough_seed_slice(self.global_npd(k), tuple(p * e for e in self.e0), self.npd(k),
                                       self.b.mask(k).cpu().numpy())
        r = torch.as_tensor(seed, dtype=torch.float64, device=self.b.device)
        inv = self.inv_diag[k]
        z = inv * r
        rz = self.dot(k, r, z)
        if rz <= 0.0:
            return 1.0
        pv = z.clone()
        alphas, betas = [], []
        for it in range(iterations):
            ap = self.apply(k, pv)
            pap = self.dot(k, pv, ap)
            if pap <= 0.0:
                break
            alpha = rz / pap
            alphas.append(alpha)
            r -= alpha * ap
            z = inv * r
            rz_new = self.dot(k, r, z)
            if rz_new <= 0.0:
                break
            if it + 1 < iterations:
                betas.append(rz_new / rz)
            pv = z + (rz_new / rz) * pv
            rz = rz_new
        if not alphas:
            return 1.0
        return lanczos_eigs(alphas, betas[: len(alphas) - 1])[1]

    def _coarse_symbolic(self):
        gnpd = self.global_npd(0)
        gmask = np.asarray(self.global_mask_fn(1), bool)
        self._gmask0 = gmask
        row_ptr, cols = q1_lattice_pattern(gnpd, gmask)
        n = len(row_ptr) - 1
        keys_g = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr)) * n + cols
        lrp, lcols, _ = self.b.coarse_csr()
        lnpd = self.npd(0)
        lrows = np.repeat(np.arange(len(lrp) - 1, dtype=np.int64), np.diff(lrp))

        def to_global(d):
            node, c = d // 3, d % 3
            ix, iy, iz = node % lnpd[0], (node // lnpd[0]) % lnpd[1], node // (lnpd[0] * lnpd[1])
            ex, ey, ez = self.e0  # p = 1: node offset = element offset
            return 3 * ((ix + ex) + gnpd[0] * ((iy + ey) + gnpd[1] * (iz + ez))) + c

        rg, cg = to_global(lrows), to_global(np.asarray(lcols, np.int64))
        lkeys = rg * n + cg
        slots = np.searchsorted(keys_g, lkeys)
        # local constrained identity rows are re-imposed globally after the sum
        ok = (slots < len(keys_g)) & (keys_g[np.minimum(slots, len(keys_g) - 1)] == lkeys)
        ok &= ~gmask[rg] & ~gmask[cg]
        self._slots = slots[ok]
        self._lsel = np.nonzero(ok)[0]
        self._nnz = len(keys_g)
        self._diag_slots = row_ptr[:-1][gmask]  # constrained rows hold only their diagonal
        self._coarse = self.b.coarse_solver(row_ptr, cols, gnpd)
        self._gn = n
        # this slab's coarse entries inside the global vector, owned first
        idx = to_global(np.arange(self.b.size(0), dtype=np.int64))
        self._coarse_idx = torch.as_tensor(idx, device=self.b.device)
        self._coarse_owned = self.comm.owned(lnpd, self.b.device)

    def setup_numeric(self):
        """setup_numeric (multigrid.hpp:100-113), distributed."""
        for k in range(1, self.L):
            d = self.comm.exchange(self.b.diagonal(k), self.npd(k))
            if bool((d == 0).any()):
                raise RuntimeError("invalid smoother: zero diagonal entry")
            self.inv_diag[k] = 1.0 / d
            self.lambda_max[k] = self._estimate_lambda_max(k)
        if self._coarse is None:
            self._coarse_symbolic()
        if hasattr(self.b, "coarse_vals"):  # device-resident values (GPU backend)
            lvals = self.b.coarse_vals()
        else:
            lvals = torch.as_tensor(np.asarray(self.b.coarse_csr()[2]), dtype=torch.float64,
                                    device=self.b.device)
        if not hasattr(self, "_slots_t"):
            dev = self.b.device
            self._slots_t = torch.as_tensor(self._slots, device=dev)
            self._lsel_t = torch.as_tensor(self._lsel, device=dev)
            self._diag_t = torch.as_tensor(self._diag_slots, device=dev)
        gv = torch.zeros(self._nnz, dtype=torch.float64, device=self.b.device)
        gv[self._slots_t] = lvals[self._lsel_t]
        self.comm.all_reduce_(gv)
        gv[self._diag_t] = 1.0
        self._coarse.factorize(gv if gv.is_cuda else gv.numpy())

    # -- cycle ------------------------------------------------------------------
    def coarse_solve(self, b):
        g = torch.zeros(self._gn, dtype=torch.float64, device=b.device)
        m = self._coarse_owned
        g[self._coarse_idx[m]] = b[m]
        self.comm.all_reduce_(g)
        x = self._coarse.solve(g)
        return x[self._coarse_idx].clone()

    def smooth(self, k, b, x, x_zero):
        """ChebyshevSmoother::apply (smoother.hpp:41-62), degree 2 on
        [0.1, 1.1] lambda_max."""
        lo, hi = 0.1 * self.lambda_max[k], 1.1 * self.lambda_max[k]
        theta, delta = 0.5 * (hi + lo), 0.5 * (hi - lo)
        sigma = theta / delta
        rho = 1.0 / sigma
        inv = self.inv_diag[k]
        if x_zero:  # A 0 = 0 (bitwise)
            d = inv * b / theta
            x.copy_(d)
        else:
            r = b - self.apply(k, x)
            d = inv * r / theta
            x += d
        for _ in range(2, self.degree + 1):
            r = b - self.apply(k, x)
            rho_new = 1.0 / (2.0 * sigma - rho)
            d = (rho_new * rho) * d + (2.0 * rho_new / delta) * (inv * r)
            x += d
            rho = rho_new
        return x

    def cycle(self, k, b, x, x_zero=True):
        if k == 0:
            x.copy_(self.coarse_solve(b))
            return x
        for i in range(self.pre):
            self.smooth(k, b, x, x_zero and i == 0)
        r = b - self.apply(k, x) if not (x_zero and self.pre == 0) else b.clone()
        rc = self.restrict_to(k - 1, r)
        rc[self.b.mask(k - 1)] = 0.0
        ec = torch.zeros_like(rc)
        self.cycle(k - 1, rc, ec, True)
        corr = self.prolong(k - 1, ec)
        corr[self.b.mask(k)] = 0.0
        x += corr
        for _ in range(self.post):
            self.smooth(k, b, x, False)
        return x

    def v_cycle(self, b):
        """v_cycle / preconditioner (multigrid.hpp:137-152)."""
        k = self.L - 1
        x = torch.zeros_like(b)
        self.cycle(k, b, x, True)
        m = self.b.mask(k)
        x[m] = b[m]
        return x


def distributed_pcg(h: DistributedHierarchy, b, rtol=1e-8, max_iterations=500, precond="mg"):
    """cg_solve (cg.hpp:81-134) on the fine level of ``h``: natural-norm
    stopping sqrt(r.z) <= rtol sqrt(r0.z0); two all-reduces per iteration."""
    k = h.L - 1
    A = lambda v: h.apply(k, v)  # noqa: E731
    M = h.v_cycle if precond == "mg" else (lambda v: v.clone())
    x = torch.zeros_like(b)
    r = b.clone()
    z = M(r)
    rz = h.dot(k, r, z)
    if rz < 0.0:
        raise RuntimeError(f"operator is not positive definite (p^T A p = {rz})")
    hist = [math.sqrt(max(rz, 0.0))]
    rep = dict(iterations=0, converged=False)
    if hist[0] == 0.0:
        rep.update(converged=True, x=x, history=hist, eig_min=0.0, eig_max=0.0)
        return rep
    p = z.clone()
    alphas, betas = [], []
    for _ in range(max_iterations):
        ap = A(p)
        pap = h.dot(k, p, ap)
        if pap <= 0.0:
            raise RuntimeError(f"operator is not positive definite (p^T A p = {pap})")
        alpha = rz / pap
        alphas.append(alpha)
        x += alpha * p
        r -= alpha * ap
        z = M(r)
        rz_new = h.dot(k, r, z)
        rep["iterations"] += 1
        nat = math.sqrt(max(rz_new, 0.0))
        if nat > 0.0:
            hist.append(nat)
        if nat <= rtol * hist[0]:
            rep["converged"] = True
            break
        if rz_new <= 0.0:
            rep["converged"] = rz_new == 0.0
            break
        beta = rz_new / rz
        betas.append(beta)
        p = z + beta * p
        rz = rz_new
    rep["eig_min"], rep["eig_max"] = lanczos_eigs(alphas, betas[: max(len(alphas) - 1, 0)])
    rep.update(x=x, history=hist)
    return rep


class StepRejected(RuntimeError):
    """StepRejectedError (errors.hpp) of the distributed driver."""


def _critical_point_line_search(g_eval, g0):
    """critical_point_line_search (nonlinear.hpp:77-129)."""
    trial, halvings = 1.0, 0
    g1 = g_eval(trial)
    while not math.isfinite(g1) and halvings < 5:
        trial *= 0.5
        g1 = g_eval(trial)
        halvings += 1
    if not math.isfinite(g1):
        raise StepRejected("residual not evaluable along the search direction")
    if g0 >= 0.0 or g1 == g0:
        alpha = trial
    else:
        alpha = min(max(trial * g0 / (g0 - g1), 0.1), 2.0)
        if halvings > 0:
            alpha = min(alpha, trial)
    if alpha == trial:
        return alpha
    ga = g_eval(alpha)
    while not math.isfinite(ga) and halvings < 5:
        alpha *= 0.5
        ga = g_eval(alpha)
        halvings += 1
    if not math.isfinite(ga):
        raise StepRejected("residual not evaluable at the line search result")
    return alpha


def distributed_newton(h: DistributedHierarchy, u, max_iterations=50, rtol=1e-8, atol=1e-10,
                       linear_rtol=1e-3, linear_max_iterations=500, use_line_search=True,
                       load_step=0, time=1.0):
    """newton_solve (nonlinear.hpp:162-216) on the slab-partitioned system:
    the residual is the backend's local residual + interface exchange (and
    leaves the shared quadrature state at the evaluated iterate), norms and
    line-search slopes are owned-entry dots, the p-MG is rebuilt at every
    linearisation point.  An inverted element on any rank reads as NaN on
    every rank (max all-reduce of the failure flag)."""
    k = h.L - 1
    npd = h.npd(k)

    def residual(v):
        bad = torch.zeros(1, dtype=torch.float64, device=v.device)
        f = None
        try:
            f = h.b.residual(v)
        except Exception as exc:  # noqa: BLE001  (InvertedElementError of either backend)
            if "nvert" not in type(exc).__name__:
                raise
            bad += 1.0
        if h.comm.dist is not None:
            h.comm.dist.all_reduce(bad, op=h.comm.dist.ReduceOp.MAX)
        if bad.item() > 0:
            return None
        return h.comm.exchange(f, npd)

    def norm(v):
        return math.sqrt(max(h.dot(k, v, v), 0.0))

    f = residual(u)
    if f is None:
        raise StepRejected("inverted element at the initial iterate")
    fnorm0 = norm(f)
    rep = dict(converged=False, iterations=0, total_cg_iterations=0, records=[])
    if fnorm0 <= atol:
        rep.update(converged=True, final_fnorm=fnorm0)
        return rep
    for it in range(1, max_iterations + 1):
        h.setup_numeric()
        cg = distributed_pcg(h, -f, rtol=linear_rtol, max_iterations=linear_max_iterations)
        du = cg["x"]
        rep["total_cg_iterations"] += cg["iterations"]
        last = {}

        def g_eval(a):
            ft = residual(u + a * du)
            if ft is None:
                return float("nan")
            last["f"] = ft
            g = h.dot(k, ft, du)
            return g if math.isfinite(g) else float("nan")

        if use_line_search:
            alpha = _critical_point_line_search(g_eval, h.dot(k, f, du))
        else:
            if not math.isfinite(g_eval(1.0)):
                raise StepRejected("residual not evaluable at the full Newton step")
            alpha = 1.0
        u += alpha * du
        f = last["f"]  # the search's last evaluation was at the accepted point
        fnorm = norm(f)
        rep["records"].append(dict(load_step=load_step, time=time, iteration=it, fnorm=fnorm,
                                   fnorm_rel=fnorm / fnorm0, cg_iterations=cg["iterations"],
                                   alpha=alpha))
        rep["iterations"] = it
        if fnorm <= max(rtol * fnorm0, atol):
            rep["converged"] = True
            break
    f = residual(u)
    rep["final_fnorm"] = norm(f)
    return rep


def distributed_solve(h: DistributedHierarchy, load_steps=1, max_bisections=3, **newton):
    """FemProblem::solve (problem.hpp:118-127): load_continuation
    (nonlinear.hpp:325-366) from u = 0 with whole-face zero Dirichlet values;
    the backend scales the external load (set_time)."""
    k = h.L - 1
    u = torch.zeros(h.b.size(k), dtype=torch.float64, device=h.b.device)
    saved = u.clone()
    steps, t_done = [], 0.0
    for step in range(1, load_steps + 1):
        target, bisections, t_try = step / load_steps, 0, step / load_steps
        while True:
            h.b.set_time(t_try)
            u.copy_(saved)
            u[h.b.mask(k)] = 0.0
            ok = False
            try:
                r = distributed_newton(h, u, load_step=step, time=t_try, **newton)
                ok = r["converged"]
                if ok:
                    steps.append(r)
            except StepRejected:
                ok = False
            if ok:
                t_done = t_try
                saved.copy_(u)
                if t_try == target:
                    break
                t_try = target
            else:
                bisections += 1
                if bisections > max_bisections:
                    raise StepRejected(f"load step failed after {max_bisections} bisections")
                t_try = 0.5 * (t_done + t_try)
    return dict(u=u, steps=steps, newton_iterations=sum(r["iterations"] for r in steps),
                cg_iterations=sum(r["total_cg_iterations"] for r in steps),
                final_fnorm=steps[-1]["final_fnorm"] if steps else 0.0)


# --------------------------------------------------------------------------
# GPU backend: the slab's hexmg objects through the C-ABI
# --------------------------------------------------------------------------
class SlabBackend:
    """Level operations of one slab on this rank's GPU (libhexmg_b200)."""

    def __init__(self, prob, fixed_faces):
        from .hexmg import constraint_mask

        self.prob = prob
        self.mg = prob.hierarchy
        self.device = torch.device("cuda", torch.cuda.current_device())
        L = self.mg.num_levels()
        sched = [prob.order]
        while sched[-1] > 1:
            sched.append((sched[-1] + 1) // 2)
        self.levels = sched[::-1]
        self._ops = [self.mg.level_operator(k) for k in range(L)]
        self._masks = [torch.as_tensor(constraint_mask(prob.cells, p, fixed_faces)[0] != 0,
                                       device=self.device) for p in self.levels]

    def size(self, k):
        return self.mg.level_size(k)

    def npd(self, k):
        p, c = self.levels[k], self.prob.cells
        return (p * c[0] + 1, p * c[1] + 1, p * c[2] + 1)

    def mask(self, k):
        return self._masks[k]

    def apply(self, k, x):
        return self._ops[k].apply_jacobian(x)

    def diagonal(self, k):
        return self._ops[k].extract_diagonal()

    def prolong(self, kc, xc):
        return self.mg.prolong(kc, xc)

    def restrict(self, kc, xf):
        return self.mg.restrict_to(kc, xf)

    def coarse_csr(self):
        self.mg.assemble_coarse()
        return self.mg.coarse_csr()

    def coarse_vals(self):
        """Re-assembled coarse values, left on the device."""
        self.mg.assemble_coarse()
        return self.mg.coarse_vals_device()

    def coarse_solver(self, row_ptr, cols, npd):
        from .hexmg import CoarseCholesky

        return CoarseCholesky(row_ptr, cols, npd)

    def residual(self, u):
        """apply_residual (operator.hpp:146-180): local residual; writes the
        quadrature state every level shares."""
        return self.prob.op.apply_residual(u)

    def set_time(self, t):
        self.prob.op.set_load_scale(t)
