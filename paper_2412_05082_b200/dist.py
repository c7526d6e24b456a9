"""Slab domain decomposition across GPUs: one process per GPU, torch.distributed
(NCCL on GPUs, gloo on CPU) for the ghost-row exchange, the C-ABI library for every computation.

The mesh is cut along the slowest axis (y in 2D, z in 3D) at cell boundaries: rank r owns the node
rows [c_r k, c_{r+1} k) clipped to the interior [1, kN-1], with c_r = round(r N / R).  Each rank stores
a window of rows (owned rows plus `ghost` rows on each side, clipped at the domain boundary) in one
contiguous array; a "row" is n^(d-1) values.  Before a smoothing step each rank sends its first /
last `ghost` owned rows to its lower / upper neighbour (contiguous slices: no pack kernels).
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Slab:
    rank: int
    nranks: int
    k: int
    N: int
    ghost: int
    own_lo: int      # node rows owned: [own_lo, own_hi)
    own_hi: int
    win_lo: int      # node rows held in the window: [win_lo, win_hi)
    win_hi: int

    @property
    def n(self):
        return self.k * self.N - 1

    @property
    def row0(self):
        """global interior row index of local row 0"""
        return self.win_lo - 1

    @property
    def lrows(self):
        return self.win_hi - self.win_lo

    @property
    def own_local(self):
        """local row slice of the owned rows"""
        return slice(self.own_lo - self.win_lo, self.own_hi - self.win_lo)


def partition(N, k, nranks, ghost):
    """Slabs of every rank; requires every slab to own at least `ghost` rows (single-hop halos)."""
    KN = k * N
    cuts = [round(r * N / nranks) for r in range(nranks + 1)]
    slabs = []
    for r in range(nranks):
        lo = max(1, cuts[r] * k)
        hi = min(KN, cuts[r + 1] * k)
        if hi - lo < ghost and nranks > 1:
            raise ValueError(f"slab {r} owns {hi - lo} rows < ghost width {ghost}; use fewer ranks")
        slabs.append(Slab(r, nranks, k, N, ghost, lo, hi, max(1, lo - ghost), min(KN, hi + ghost)))
    return slabs


def exchange_ghosts(x_ext, slab, row_len, group=None):
    """Fill the ghost rows of x_ext (1D tensor, window layout) from the neighbours' owned rows.

    Uses torch.distributed point-to-point (isend/irecv) on contiguous row slices; works with NCCL
    (GPU tensors) and gloo (CPU tensors).  Returns the number of bytes received.
    """
    import torch.distributed as dist
    g = slab.ghost
    ops = []
    recv_bytes = 0
    rows = x_ext.view(-1, row_len)
    lo_ghost = slab.own_lo - slab.win_lo           # ghost rows below the owned range
    hi_ghost = slab.win_hi - slab.own_hi
    if slab.rank > 0 and lo_ghost > 0:
        ops.append(dist.P2POp(dist.isend, rows[lo_ghost:lo_ghost + g], slab.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, rows[0:lo_ghost], slab.rank - 1, group))
        recv_bytes += rows[0:lo_ghost].numel() * rows.element_size()
    if slab.rank < slab.nranks - 1 and hi_ghost > 0:
        top = slab.own_hi - slab.win_lo
        ops.append(dist.P2POp(dist.isend, rows[top - g:top], slab.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, rows[top:top + hi_ghost], slab.rank + 1, group))
        recv_bytes += rows[top:top + hi_ghost].numel() * rows.element_size()
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return recv_bytes
