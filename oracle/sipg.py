"""Poisson with the symmetric interior penalty DG method (SIPG) -- the comparison workload of PAPER.md:752-816
(Fig. 5): -Delta u = f, u = 0 on the boundary (weakly, Nitsche), discontinuous Q_k.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:813 names the method ("discretized using the symmetric interior penalty method") but not its
parameters; reading Q30: the standard SIPG form
    a(u, v) = sum_K int_K grad u . grad v + sum_e int_e (sigma_P / h_e) [u][v] - {d_n u}[v] - [u]{d_n v}
with [u] = u^- n^- + u^+ n^+ (normal component), {d_n u} the mean normal derivative, one-sided on boundary
facets, sigma_P = k(k+1) on interior and 2 k(k+1) on boundary facets (the boundary convention of reading Q27),
h_e = h.  DoFs: per cell the (k+1)^d Gauss-Lobatto nodes (discontinuous), numbering x fastest with the 1D
index c (k+1) + m.  A vertex patch holds all (2k+2)^d DoFs of its 2^d cells; the operator
restricted to a patch is exactly L_v (x) M_v + M_v (x) L_v (rank 2), so fast diagonalisation is exact
(PAPER.md:351-365).  This module assembles by d-dimensional quadrature (never the Kronecker form) and solves
the patches with dense Cholesky (never FDM).
"""
import itertools

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .basis import Basis1D, gauss_legendre, gauss_lobatto_points
from .mesh import patch_vertices, color_patches
from .operator import _tensor


def sipg_sigma(k):
    """Reading Q30: sigma_P = k (k+1) (interior facets; twice that on boundary facets)."""
    return float(k * (k + 1))


def _cell_ids(k, d, N, cells):
    """[ncells, (k+1)^d] DG DoF ids of the cells (x fastest, 1D index c (k+1) + m)."""
    n1 = N * (k + 1)
    offs = np.array(list(itertools.product(range(k + 1), repeat=d)))[:, ::-1]
    j = cells[:, None, :] * (k + 1) + offs[None, :, :]
    return (j * (n1 ** np.arange(d))).sum(-1)


def assemble_sipg(k, d, N, sigma=None, bfac=2.0):
    """Global SIPG matrix (CSR, size (N(k+1))^d) by d-dimensional cell and facet quadrature."""
    sigma = sipg_sigma(k) if sigma is None else sigma
    h = 1.0 / N
    bas = Basis1D(k)
    nq = k + 2
    t, w = gauss_legendre(nq)
    V, D1 = bas.eval(t, 0), bas.eval(t, 1) / h
    W = _tensor([w[None, :]] * d).ravel() * h ** d
    K = 0.0
    for a in range(d):
        G = _tensor([D1 if ax == a else V for ax in range(d)])
        K = K + (G * W) @ G.T
    Wf = _tensor([w[None, :]] * (d - 1)).ravel() * h ** (d - 1) if d > 1 else np.ones(1)

    def trace(axis, tn, der):
        tabs = [V] * d
        tabs = list(tabs)
        tabs[axis] = bas.eval(tn, der) / h ** der
        return _tensor(tabs)

    def face(axis, kind):
        if kind == "interior":
            J = np.vstack([trace(axis, 1.0, 0), -trace(axis, 0.0, 0)])         # [u] (normal of K^-: +e)
            Dn = np.vstack([0.5 * trace(axis, 1.0, 1), 0.5 * trace(axis, 0.0, 1)])  # {d_n u} along +e
            s = sigma
        elif kind == "lower":
            J, Dn, s = trace(axis, 0.0, 0), -trace(axis, 0.0, 1), bfac * sigma       # n = -e
        else:
            J, Dn, s = trace(axis, 1.0, 0), trace(axis, 1.0, 1), bfac * sigma         # n = +e
        JW, DW = J * Wf, Dn * Wf
        return (s / h) * (JW @ J.T) - JW @ Dn.T - DW @ J.T

    cells = np.array(list(itertools.product(range(N), repeat=d)))[:, ::-1]
    rows, cols, vals = [], [], []

    def add(ids, Mat):
        rows.append(np.repeat(ids, Mat.shape[1], axis=1).ravel())
        cols.append(np.tile(ids, (1, Mat.shape[0])).ravel())
        vals.append(np.broadcast_to(Mat.ravel(), (ids.shape[0], Mat.size)).ravel())

    add(_cell_ids(k, d, N, cells), K)
    for a in range(d):
        lo, up = cells[cells[:, a] == 0], cells[cells[:, a] == N - 1]
        add(_cell_ids(k, d, N, lo), face(a, "lower"))
        add(_cell_ids(k, d, N, up), face(a, "upper"))
        cm = cells[cells[:, a] < N - 1]
        cp = cm.copy(); cp[:, a] += 1
        add(np.hstack([_cell_ids(k, d, N, cm), _cell_ids(k, d, N, cp)]), face(a, "interior"))
    n = (N * (k + 1)) ** d
    rows = np.concatenate(rows); cols = np.concatenate(cols); vals = np.concatenate(vals)
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def sipg_matrices_1d(k, N, sigma=None, bfac=2.0):
    """1D DG mass M and SIPG stiffness L (dense, N(k+1) square) by 1D quadrature (PAPER.md:323-332 analogue)."""
    A = assemble_sipg(k, 1, N, sigma, bfac).toarray()
    h = 1.0 / N
    bas = Basis1D(k)
    t, w = gauss_legendre(k + 2)
    V = bas.eval(t, 0)
    Mc = (V * w) @ V.T * h
    M = np.kron(np.eye(N), Mc)
    return M, A


def sipg_load(k, d, N, f):
    """b_i = int f phi_i over the DG cells (Gauss k+3 points per cell and axis)."""
    h = 1.0 / N
    nq = k + 3
    bas = Basis1D(k)
    t, w = gauss_legendre(nq)
    Phi = _tensor([bas.eval(t, 0)] * d)
    W = _tensor([w[None, :]] * d).ravel() * h ** d
    cells = np.array(list(itertools.product(range(N), repeat=d)))[:, ::-1]
    tq = np.array(list(itertools.product(range(nq), repeat=d)))[:, ::-1]
    coords = [(cells[:, a][:, None] + t[tq[:, a]][None, :]) * h for a in range(d)]
    contrib = (f(*coords) * W) @ Phi.T
    b = np.zeros((N * (k + 1)) ** d)
    np.add.at(b, _cell_ids(k, d, N, cells).ravel(), contrib.ravel())
    return b


def sipg_paper_load(d):
    """-Delta prod sin(pi x_a) = d pi^2 prod sin(pi x_a) (u* vanishes on the boundary)."""
    def f(*xs):
        out = d * np.pi ** 2
        for x in xs:
            out = out * np.sin(np.pi * x)
        return out
    return f


def sipg_dof_coords(k, N):
    t = gauss_lobatto_points(k)
    return np.array([(c + t[m]) / N for c in range(N) for m in range(k + 1)])


def sipg_patch_dofs(k, d, N, v):
    n1 = N * (k + 1)
    ranges = [np.arange((va - 1) * (k + 1), (va + 1) * (k + 1)) for va in v]
    idx = np.zeros([2 * k + 2] * d, dtype=np.int64)
    for a in range(d):
        shape = [1] * d; shape[d - 1 - a] = 2 * k + 2
        idx = idx + (ranges[a] * n1 ** a).reshape(shape)
    return idx.ravel()


class SipgPatchSolvers:
    """Dense Cholesky inverses of the exact patch matrices A_v = R_v A R_v^T, grouped by the
    axis-variant tuple; same interface as smoothers.PatchSolvers (dofs, solve, d, N) so that smoothers.avs_step /
    mvs_step apply the vertex-patch smoothers of PAPER.md:206-239 to the SIPG operator."""

    def __init__(self, k, d, N, A):
        from .discretization import patch_variant
        self.k, self.d, self.N = k, d, N
        self.verts = patch_vertices(d, N)
        self.dofs = np.array([sipg_patch_dofs(k, d, N, v) for v in self.verts], dtype=np.int64)
        keys = [tuple(patch_variant(va, N) for va in v) for v in self.verts]
        self.groups = {}
        A = A.tocsr()
        for key in sorted(set(keys)):
            ids = np.array([i for i, kk in enumerate(keys) if kk == key])
            g = self.dofs[ids[0]]
            Av = A[g][:, g].toarray()
            fac = sla.cho_factor(Av)
            Ainv = sla.cho_solve(fac, np.eye(len(g)))
            self.groups[key] = (ids, 0.5 * (Ainv + Ainv.T), Av)

    def solve(self, ids, R):
        out = np.empty_like(R)
        for key, (gids, Ainv, Av) in self.groups.items():
            mask = np.isin(ids, gids)
            if mask.any():
                Rg = R[mask]
                U = Rg @ Ainv
                out[mask] = U + (Rg - U @ Av) @ Ainv
        return out


def sipg_embedding_1d(k, Nc):
    """DG embedding (PAPER.md:177 analogue): coarse cell polynomials evaluated at the nodes of its 2 fine cells."""
    t = gauss_lobatto_points(k)
    bas = Basis1D(k)
    Nf = 2 * Nc
    E = np.zeros((Nf * (k + 1), Nc * (k + 1)))
    for cf in range(Nf):
        cc = cf // 2
        for m in range(k + 1):
            tl = ((cf % 2) + t[m]) * 0.5
            E[cf * (k + 1) + m, cc * (k + 1): (cc + 1) * (k + 1)] = bas.eval(tl, 0)[:, 0]
    return E


class SipgHierarchy:
    """Levels 1..L of the SIPG workload (N = 2^l cells per axis) with the attributes multigrid.vcycle /
    precondition use (Ac, ps, Pc, L, dtype): rediscretised A_l, exact patch solvers, DG embeddings P_l."""

    def __init__(self, k, d, L):
        from .mesh import level_cells
        self.k, self.d, self.L, self.dtype = k, d, L, np.float64
        self.Ac, self.ps, self.Pc = {}, {}, {}
        for l in range(1, L + 1):
            N = level_cells(l)
            self.Ac[l] = assemble_sipg(k, d, N)
            self.ps[l] = SipgPatchSolvers(k, d, N, self.Ac[l])
            if l > 1:
                E = sp.csr_matrix(sipg_embedding_1d(k, N // 2))
                P = E
                for _ in range(d - 1):
                    P = sp.kron(E, P)
                self.Pc[l] = P.tocsr()
        self.A = self.Ac
