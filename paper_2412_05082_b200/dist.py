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


# ----------------------------------------------------------------------------------------------------------
# Distributed multigrid and Krylov drivers.  Every computation is a C-ABI call on the rank's
# window (c0ip_slab_* for the distributed levels, c0ip_vcycle_level for the replicated coarse part,
# c0ip_vec_axpby / c0ip_vec_dots for the Krylov vectors); torch.distributed carries the ghost-row exchanges
# (one per smoothing step / MVS colour / residual / transfer), the coarse-level all-gather (agglomeration) and
# the all-reduced dot products.  On one GPU per rank the group is NCCL; the 2-rank tests run both ranks on one
# GPU with gloo, staging the exchanged rows through host memory.

def _host_staged(t):
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend() == "gloo"


def exchange(x_ext, slab, row_len, group=None):
    """exchange_ghosts, with gloo + CUDA tensors staged through host memory (both ranks on one GPU)."""
    if slab.nranks == 1:
        return 0
    if not _host_staged(x_ext):
        return exchange_ghosts(x_ext, slab, row_len, group)
    h = x_ext.cpu()
    nbytes = exchange_ghosts(h, slab, row_len, group)
    rows, hrows = x_ext.view(-1, row_len), h.view(-1, row_len)
    lo, hi = slab.own_lo - slab.win_lo, slab.own_hi - slab.win_lo
    if lo > 0:
        rows[:lo].copy_(hrows[:lo])
    if hi < rows.shape[0]:
        rows[hi:].copy_(hrows[hi:])
    return nbytes


def start_exchange(x_ext, slab, row_len, group=None):
    """Post the ghost-row exchange without waiting (NCCL: the receive completes on NCCL's stream); returns a
    finisher that makes the current stream wait for it.  gloo with CUDA tensors (one-GPU tests) is host-staged
    and completes here."""
    import torch.distributed as dist
    if slab.nranks == 1:
        return lambda: None
    if _host_staged(x_ext) or dist.get_backend() == "gloo":
        exchange(x_ext, slab, row_len, group)
        return lambda: None
    g = slab.ghost
    rows = x_ext.view(-1, row_len)
    lo_ghost, hi_ghost = slab.own_lo - slab.win_lo, slab.win_hi - slab.own_hi
    ops = []
    if slab.rank > 0 and lo_ghost > 0:
        ops.append(dist.P2POp(dist.isend, rows[lo_ghost:lo_ghost + g], slab.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, rows[0:lo_ghost], slab.rank - 1, group))
    if slab.rank < slab.nranks - 1 and hi_ghost > 0:
        top = slab.own_hi - slab.win_lo
        ops.append(dist.P2POp(dist.isend, rows[top - g:top], slab.rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, rows[top:top + hi_ghost], slab.rank + 1, group))
    works = dist.batch_isend_irecv(ops) if ops else []

    def finish():
        for w in works:
            w.wait()
    return finish


def avs_step_overlapped(ctx, level, omega, slab, row_len, b_ext, x_ext, r_ext, group=None):
    """One additive smoothing step on a slab with the halo exchange overlapped (SURVEY.md §8e "Overlap"): the
    residual of the interior owned rows (whose stencil needs no ghost row) runs while the ghost rows travel;
    then the residual of the two boundary strips and the FDM update (c0ip_slab_fdm).  Same result as
    c0ip_slab_avs_step, bitwise."""
    k = ctx.degree
    s = slab
    KN = k * s.N
    finish = start_exchange(x_ext, s, row_len, group)
    in_lo, in_hi = s.own_lo + 2 * k, s.own_hi - 2 * k
    r_lo, r_hi = max(1, s.own_lo - (2 * k - 2)), min(KN, s.own_hi + 2 * k - 2)
    if in_hi > in_lo:
        ctx.slab_apply(level, s.row0, s.lrows, in_lo, in_hi, x_ext, r_ext, b_ext=b_ext)
    finish()
    if in_hi > in_lo:
        ctx.slab_apply(level, s.row0, s.lrows, r_lo, in_lo, x_ext, r_ext, b_ext=b_ext)
        ctx.slab_apply(level, s.row0, s.lrows, in_hi, r_hi, x_ext, r_ext, b_ext=b_ext)
    else:
        ctx.slab_apply(level, s.row0, s.lrows, r_lo, r_hi, x_ext, r_ext, b_ext=b_ext)
    ctx.slab_fdm(level, omega, s.row0, s.lrows, s.own_lo, s.own_hi, r_ext, x_ext)
    return x_ext


def allreduce_sum(vals, device, group=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(vals), dtype=torch.float64)
    if dist.get_backend() != "gloo":
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [float(v) for v in t.cpu()]


class DistLevel:
    def __init__(self, ctx, level, nranks, rank, ghost, dtype, device):
        import torch
        info = ctx.level_info(level)
        self.level, self.N, self.n = level, info["cells"], info["n_1d"]
        self.k, self.d = ctx.degree, ctx.dim
        self.row = self.n ** (self.d - 1)
        self.slab = partition(self.N, self.k, nranks, ghost)[rank]
        self.slabs = partition(self.N, self.k, nranks, ghost)
        size = self.slab.lrows * self.row
        self.x, self.b, self.r = (torch.zeros(size, dtype=dtype, device=device) for _ in range(3))

    def owned(self, v):
        return v.view(-1, self.row)[self.slab.own_local].reshape(-1)


class DistMG:
    """The V-cycle of Algorithm 1 on slabs: levels L, L-1, ... stay distributed while every
    rank owns at least `min_cells` cells of the level (single-hop halos) and the level has the fused slab
    kernels (N >= 8); below, the restricted residual is all-gathered (agglomeration) and every rank runs the
    remaining coarse cycle redundantly (c0ip_vcycle_level, deterministic), then prolongates onto its own rows.
    FP64 cycle (the FP32 cycle's data conversion happens inside the replicated part only)."""

    def __init__(self, ctx, mg_kind="avs", steps=2, omega=0.25, symmetric=True, group=None, min_cells=4):
        import torch
        import torch.distributed as dist
        from . import api
        self.ctx, self.group = ctx, group
        self.rank, self.nranks = dist.get_rank(group), dist.get_world_size(group)
        self.kind, self.steps, self.omega, self.symmetric = mg_kind, steps, omega, symmetric
        self.device = ctx.device
        k, d = ctx.degree, ctx.dim
        self.ghost = 4 * k - 2
        self.levels = {}
        lvl = ctx.finest_level
        while lvl > 1:
            N = ctx.level_info(lvl)["cells"]
            if N < 8 or N // self.nranks < max(min_cells, 1) or N % self.nranks:
                break
            self.levels[lvl] = DistLevel(ctx, lvl, self.nranks, self.rank, self.ghost, torch.float64, self.device)
            lvl -= 1
        if not self.levels:
            raise ValueError("the finest level is too small to distribute over this many ranks")
        self.lowest = min(self.levels)
        self.coarse_mg = api.MG(mg_kind, steps, omega, symmetric=symmetric)
        self.ncolors = 2 ** (d + 1)
        nc = ctx.level_info(self.lowest - 1)["n_dofs"]
        self.c_full = torch.zeros(nc, dtype=torch.float64, device=self.device)
        self.e_full = torch.zeros(nc, dtype=torch.float64, device=self.device)
        self.exchanges = 0

    def _xchg(self, lev, v):
        self.exchanges += 1
        exchange(v, lev.slab, lev.row, self.group)

    def smooth(self, lev, x, b, reverse=False):
        s = lev.slab
        for _ in range(self.steps):
            if self.kind == "mvs":
                order = range(self.ncolors - 1, -1, -1) if reverse else range(self.ncolors)
                for c in order:
                    self._xchg(lev, x)
                    self.ctx.slab_mvs_color(lev.level, self.omega, c, s.row0, s.lrows, s.own_lo, s.own_hi, b, x, lev.r)
            else:
                self.exchanges += 1
                avs_step_overlapped(self.ctx, lev.level, self.omega, s, lev.row, b, x, lev.r, self.group)

    def residual(self, lev, x, b, r):
        """owned rows of r = b - A x (ghosts of x exchanged first)"""
        s = lev.slab
        self._xchg(lev, x)
        self.ctx.slab_apply(lev.level, s.row0, s.lrows, s.own_lo, s.own_hi, x, r, b_ext=b)

    def apply(self, lev, x, y):
        s = lev.slab
        self._xchg(lev, x)
        self.ctx.slab_apply(lev.level, s.row0, s.lrows, s.own_lo, s.own_hi, x, y)

    def _gather_coarse(self, lev_c_level, part_rows, src):
        """all-gather the owned coarse node rows [lo, hi) of every rank into self.c_full"""
        import torch
        import torch.distributed as dist
        info = self.ctx.level_info(lev_c_level)
        n, row = info["n_1d"], info["n_1d"] ** (self.ctx.dim - 1)
        cells = info["cells"]
        parts = partition(cells, self.ctx.degree, self.nranks, 0)
        mx = max(p.own_hi - p.own_lo for p in parts) * row
        mine = parts[self.rank]
        buf = torch.zeros(mx, dtype=torch.float64, device=self.device)
        buf[: (mine.own_hi - mine.own_lo) * row] = src.view(-1, row)[mine.own_lo - 1: mine.own_hi - 1].reshape(-1)
        staged = _host_staged(buf)
        sendb = buf.cpu() if staged else buf
        outs = [torch.zeros_like(sendb) for _ in range(self.nranks)]
        dist.all_gather(outs, sendb, group=self.group)
        full = self.c_full.view(-1, row)
        for p, o in zip(parts, outs):
            full[p.own_lo - 1: p.own_hi - 1] = o[: (p.own_hi - p.own_lo) * row].view(-1, row).to(self.device)
        return parts

    def cycle(self, level, x, b):
        """x = MG_level(0, b) on the rank's window of a distributed level (owned rows valid on return)."""
        lev = self.levels[level]
        s = lev.slab
        x.zero_()
        self._xchg(lev, b)                               # the smoothers read b on the patch rows beyond the owned ones
        self.smooth(lev, x, b)
        self.residual(lev, x, b, lev.r)
        self._xchg(lev, lev.r)                           # the restriction reads fine rows below the owned ones
        if level - 1 in self.levels:
            cl = self.levels[level - 1]
            cs = cl.slab
            self.ctx.slab_restrict(level, s.row0, s.lrows, lev.r, cs.row0, cs.lrows, cs.own_lo, cs.own_hi, cl.b)
            self.cycle(level - 1, cl.x, cl.b)
            self._xchg(cl, cl.x)                         # the prolongation reads coarse rows around the owned ones
            self.ctx.slab_prolongate_add(level, cs.row0, cs.lrows, cl.x, s.row0, s.lrows, s.own_lo, s.own_hi, x)
        else:
            info = self.ctx.level_info(level - 1)
            nc = info["n_1d"]
            parts = partition(info["cells"], self.ctx.degree, self.nranks, 0)
            mine = parts[self.rank]
            self.c_full.zero_()
            self.ctx.slab_restrict(level, s.row0, s.lrows, lev.r, 0, nc, mine.own_lo, mine.own_hi, self.c_full)
            self._gather_coarse(level - 1, None, self.c_full)
            self.ctx.vcycle_level(self.coarse_mg, level - 1, self.c_full, self.e_full)
            self.ctx.slab_prolongate_add(level, 0, nc, self.e_full, s.row0, s.lrows, s.own_lo, s.own_hi, x)
        self.smooth(lev, x, b, reverse=self.symmetric and self.kind == "mvs")
        return x


class DistPCG:
    """MG-preconditioned CG in FP64 on slabs (Saad Alg. 9.1 as c0ip_pcg): vectors are windows of
    the finest level, the update arithmetic runs in the library (c0ip_vec_axpby / c0ip_vec_dots on the owned rows),
    dot products are all-reduced, the preconditioner is DistMG.cycle."""

    def __init__(self, mgd):
        self.m = mgd
        self.lev = mgd.levels[mgd.ctx.finest_level]

    def dot2(self, a, b, c=None, d=None):
        o = self.lev.owned
        v = self.m.ctx.dots(o(a), o(b)) if c is None else self.m.ctx.dots(o(a), o(b), o(c), o(d))
        return allreduce_sum(v, self.m.device, self.m.group)

    def solve(self, b_ext, rtol=1e-8, max_iter=200):
        import torch
        ctx, lev, o = self.m.ctx, self.lev, self.lev.owned
        x = torch.zeros_like(b_ext)
        r, z, p, Ap = (torch.zeros_like(b_ext) for _ in range(4))
        self.m.residual(lev, x, b_ext, r)
        self.m.cycle(lev.level, z, r)
        ctx.axpby(1.0, o(z), 0.0, o(p))
        rz, rr = self.dot2(r, z, r, r)
        hist = [rr ** 0.5]
        n = 0
        while n < max_iter and hist[-1] > rtol * hist[0]:
            self.m.apply(lev, p, Ap)
            alpha = rz / self.dot2(p, Ap)[0]
            ctx.axpby(alpha, o(p), 1.0, o(x))
            ctx.axpby(-alpha, o(Ap), 1.0, o(r))
            n += 1
            hist.append(self.dot2(r, r)[0] ** 0.5)
            if hist[-1] <= rtol * hist[0]:
                break
            self.m.cycle(lev.level, z, r)
            rz_new = self.dot2(r, z)[0]
            ctx.axpby(1.0, o(z), rz_new / rz, o(p))
            rz = rz_new
        return x, n, hist


class DistGMRES:
    """Flexible right-preconditioned GMRES(m) in FP64 on slabs (the paper's outer solver for the
    multiplicative smoother; c0ip_gmres on one GPU): Arnoldi with classical Gram-Schmidt and one
    re-orthogonalisation (CGS2: the j+1 projections of a step are one all-reduce), Givens rotations on the host,
    the preconditioner is DistMG.cycle (same-order MVS cycle when symmetric=False).  Vectors are windows of the
    finest level; every vector update runs in the library (c0ip_vec_axpby / c0ip_vec_dots on the owned rows)."""

    def __init__(self, mgd, restart=30):
        self.m = mgd
        self.lev = mgd.levels[mgd.ctx.finest_level]
        self.restart = restart

    def _dots(self, pairs):
        o = self.lev.owned
        vals = []
        for i in range(0, len(pairs), 2):
            chunk = pairs[i:i + 2]
            if len(chunk) == 2:
                vals += list(self.m.ctx.dots(o(chunk[0][0]), o(chunk[0][1]), o(chunk[1][0]), o(chunk[1][1])))
            else:
                vals += list(self.m.ctx.dots(o(chunk[0][0]), o(chunk[0][1])))
        return allreduce_sum(vals, self.m.device, self.m.group)

    def solve(self, b_ext, rtol=1e-8, max_iter=200):
        import math
        import torch
        ctx, lev, o = self.m.ctx, self.lev, self.lev.owned
        x = torch.zeros_like(b_ext)
        w = torch.zeros_like(b_ext)
        V = [torch.zeros_like(b_ext) for _ in range(self.restart + 1)]
        Z = [torch.zeros_like(b_ext) for _ in range(self.restart)]
        self.m.residual(lev, x, b_ext, V[0])
        beta = math.sqrt(self._dots([(V[0], V[0])])[0])
        r0, rn, hist, it = beta, beta, [beta], 0
        while it < max_iter and rn > rtol * r0 and beta > 0:
            mm = min(self.restart, max_iter - it)
            ctx.axpby(0.0, o(V[0]), 1.0 / beta, o(V[0]))
            H = [[0.0] * mm for _ in range(mm + 1)]
            cs, sn, g = [0.0] * mm, [0.0] * mm, [0.0] * (mm + 1)
            g[0] = beta
            jd = 0
            for j in range(mm):
                self.m.cycle(lev.level, Z[j], V[j])
                self.m.apply(lev, Z[j], w)
                for _ in range(2):                                   # CGS2
                    hs = self._dots([(w, V[i]) for i in range(j + 1)])
                    for i in range(j + 1):
                        H[i][j] += hs[i]
                        ctx.axpby(-hs[i], o(V[i]), 1.0, o(w))
                H[j + 1][j] = math.sqrt(self._dots([(w, w)])[0])
                ctx.axpby(1.0 / H[j + 1][j] if H[j + 1][j] > 0 else 0.0, o(w), 0.0, o(V[j + 1]))
                for i in range(j):
                    t = cs[i] * H[i][j] + sn[i] * H[i + 1][j]
                    H[i + 1][j] = -sn[i] * H[i][j] + cs[i] * H[i + 1][j]
                    H[i][j] = t
                den = math.hypot(H[j][j], H[j + 1][j])
                cs[j], sn[j] = H[j][j] / den, H[j + 1][j] / den
                H[j][j], H[j + 1][j] = den, 0.0
                g[j + 1] = -sn[j] * g[j]
                g[j] = cs[j] * g[j]
                it += 1
                jd = j + 1
                rn = abs(g[j + 1])
                hist.append(rn)
                if rn <= rtol * r0:
                    break
            y = [0.0] * jd
            for i in range(jd - 1, -1, -1):
                y[i] = (g[i] - sum(H[i][l] * y[l] for l in range(i + 1, jd))) / H[i][i]
            for i in range(jd):
                ctx.axpby(y[i], o(Z[i]), 1.0, o(x))
            self.m.residual(lev, x, b_ext, V[0])
            beta = math.sqrt(self._dots([(V[0], V[0])])[0])
        return x, it, hist
