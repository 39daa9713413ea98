"""Slab partition of the box across ranks and the interface-plane exchange
(SURVEY.md §8(e)).

The reference is single-process; the paper's distributed version
sums interface-node contributions with a PETSc star forest after every
operator apply.  Here the box of ``cells_x`` elements
is cut into contiguous slabs along x, one per rank; each rank owns the
elements of its slab and holds every lattice node of the slab, so the only
shared entries are the node planes between neighbouring slabs.  After a local
apply, neighbours swap their partial sums on the shared plane and both add
(lower-rank partial + upper-rank partial): the shared entries end up bitwise
identical on both ranks.  Dot products count each shared node once (owned by
the lower rank) and are summed with one all-reduce.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    cells: tuple  # local element counts (cx, cy, cz)
    x0: int       # first global element index along x
    order: int

    @property
    def npd(self):
        p = self.order
        return (p * self.cells[0] + 1, p * self.cells[1] + 1, p * self.cells[2] + 1)

    @property
    def node_x0(self):
        """Global lattice x-index of this slab's first node plane."""
        return self.order * self.x0


def slab_partition(global_cells, world, rank, order):
    """Split ``global_cells[0]`` elements along x as evenly as possible."""
    cx = global_cells[0]
    base, extra = divmod(cx, world)
    sizes = [base + (1 if r < extra else 0) for r in range(world)]
    if min(sizes) < 1:
        raise ValueError("more ranks than element layers along x")
    x0 = sum(sizes[:rank])
    return Slab(rank, world, (sizes[rank], global_cells[1], global_cells[2]), x0, order)


def exchange_faces(y, npd, rank, world, dist):
    """Sum the shared x-interface planes of the L-vector ``y`` (torch tensor,
    interleaved 3 per node, x fastest) with the neighbouring slabs."""
    import torch

    nx, ny, nz = npd
    v = y.view(nz, ny, nx, 3)
    # gloo moves host buffers only (the single-GPU multi-rank test mode)
    host = y.is_cuda and dist.get_backend() == "gloo"
    stage = (lambda t: t.cpu()) if host else (lambda t: t)
    ops, bufs = [], {}
    if rank + 1 < world:
        send_hi = stage(v[:, :, nx - 1, :].contiguous())
        recv_hi = torch.empty_like(send_hi)
        ops += [dist.P2POp(dist.isend, send_hi, rank + 1), dist.P2POp(dist.irecv, recv_hi, rank + 1)]
        bufs["hi"] = (send_hi, recv_hi)
    if rank > 0:
        send_lo = stage(v[:, :, 0, :].contiguous())
        recv_lo = torch.empty_like(send_lo)
        ops += [dist.P2POp(dist.isend, send_lo, rank - 1), dist.P2POp(dist.irecv, recv_lo, rank - 1)]
        bufs["lo"] = (send_lo, recv_lo)
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    if "hi" in bufs:
        s, r = bufs["hi"]
        v[:, :, nx - 1, :] = (s + r).to(y.device)  # this rank is the lower one
    if "lo" in bufs:
        s, r = bufs["lo"]
        v[:, :, 0, :] = (r + s).to(y.device)  # the neighbour is the lower one
    return y


@dataclass(frozen=True)
class Block:
    """One rank's block of a px x py x pz element partition of the box
    (2 x 2 x 2 for the cfg5 cube).  Ranks are numbered x
    fastest; ``e0`` is the block's first global element per direction."""
    rank: int
    dims: tuple    # (px, py, pz)
    coords: tuple  # (cx, cy, cz)
    cells: tuple   # local element counts
    e0: tuple      # first global element index per direction
    order: int

    @property
    def world(self):
        return self.dims[0] * self.dims[1] * self.dims[2]

    @property
    def npd(self):
        p = self.order
        return tuple(p * c + 1 for c in self.cells)

    @property
    def node0(self):
        """Global lattice index of this block's first node per direction."""
        return tuple(self.order * e for e in self.e0)

    def neighbour(self, d, step):
        """Rank of the neighbouring block along direction d (step -1 / +1),
        or None at the box boundary."""
        c = list(self.coords)
        c[d] += step
        if not 0 <= c[d] < self.dims[d]:
            return None
        return c[0] + self.dims[0] * (c[1] + self.dims[1] * c[2])


def _split(n, parts, i):
    base, extra = divmod(n, parts)
    sizes = [base + (1 if r < extra else 0) for r in range(parts)]
    if min(sizes) < 1:
        raise ValueError("more blocks than element layers")
    return sizes[i], sum(sizes[:i])


def block_partition(global_cells, dims, rank, order):
    """Split the box into dims[0] x dims[1] x dims[2] contiguous element
    blocks, each direction as evenly as possible; rank -> block, x fastest."""
    px, py, pz = dims
    if not 0 <= rank < px * py * pz:
        raise ValueError("rank outside the partition")
    coords = (rank % px, (rank // px) % py, rank // (px * py))
    cells, e0 = [], []
    for d in range(3):
        n, o = _split(global_cells[d], dims[d], coords[d])
        cells.append(n)
        e0.append(o)
    return Block(rank, tuple(dims), coords, tuple(cells), tuple(e0), order)


def exchange_block(y, npd, block: Block, dist):
    """Sum the interface node planes of a block-partitioned L-vector with
    the face neighbours, one direction after the other (x, then y, then z):
    after the x pass the x-shared nodes hold their pairwise sums on both
    sides, the y pass then sums those, and so on, so nodes on partition
    edges and corners collect all (up to 8) contributions -- the same value,
    bitwise, on every rank that holds them."""
    import torch

    nx, ny, nz = npd
    v = y.view(nz, ny, nx, 3)
    host = y.is_cuda and dist.get_backend() == "gloo"
    stage = (lambda t: t.cpu()) if host else (lambda t: t)
    n = (nx, ny, nz)
    for d in range(3):
        def plane(i, d=d):
            return (v[:, :, i, :] if d == 0 else v[:, i, :, :] if d == 1 else v[i, :, :, :])
        ops, bufs = [], {}
        hi, lo = block.neighbour(d, +1), block.neighbour(d, -1)
        if hi is not None:
            s = stage(plane(n[d] - 1).contiguous())
            r = torch.empty_like(s)
            ops += [dist.P2POp(dist.isend, s, hi), dist.P2POp(dist.irecv, r, hi)]
            bufs["hi"] = (s, r)
        if lo is not None:
            s = stage(plane(0).contiguous())
            r = torch.empty_like(s)
            ops += [dist.P2POp(dist.isend, s, lo), dist.P2POp(dist.irecv, r, lo)]
            bufs["lo"] = (s, r)
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if "hi" in bufs:
            s, r = bufs["hi"]
            plane(n[d] - 1).copy_((s + r).to(y.device))  # this block is the lower one
        if "lo" in bufs:
            s, r = bufs["lo"]
            plane(0).copy_((r + s).to(y.device))
    return y


def owned_mask(npd, rank, world):
    """Boolean mask over the local L-vector of the entries this rank owns
    (shared planes belong to the lower rank)."""
    import torch

    nx, ny, nz = npd
    m = torch.ones(nz, ny, nx, 3, dtype=torch.bool)
    if rank > 0:
        m[:, :, 0, :] = False
    return m.reshape(-1)


def global_dot(x, y, owned, dist):
    """x . y over owned entries, all-reduced (one f64): the CG/Lanczos dots
    of SURVEY.md §8(e)."""
    import torch

    local = torch.sum(x[owned] * y[owned]).reshape(1).to(torch.float64)
    if dist is not None:
        dist.all_reduce(local)
    return float(local.item())
