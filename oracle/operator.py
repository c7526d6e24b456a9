"""Assembled C0IP operator by d-dimensional quadrature (Eq. bfc0ip).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

This is the *definition* of A_ell written out: cell integrals of the full Hessian
contraction  int_K grad^2 u : grad^2 v  (including the mixed 2 d_xy u d_xy v terms,
PAPER.md:53, 119) plus, on every facet, the penalty, consistency and adjoint
consistency terms  (sigma/h_e)[d_n u][d_n v] - {d_n^2 u}[d_n v] - [d_n u]{d_n^2 v}
 with the jump/mean of PAPER.md:87-106 (one-sided on boundary
facets, reading Q26) and h_e = h on interior, h/2 on boundary facets (reading Q27).  It does
NOT use the Kronecker form of PAPER.md:314-342; the Kronecker identity is a
test that compares the two.

Numbering: full nodes j_a = 0..kN per axis, interior index
i_a = j_a - 1, global id sum_a i_a n^a with n = kN-1 (x fastest).
"""
import itertools
import numpy as np
import scipy.sparse as sp

from .basis import Basis1D, gauss_legendre
from .discretization import BOUNDARY_PENALTY


def _tensor(tables):
    """kron(T_{d-1}, ..., T_0): row = local dof (x fastest), col = point (x fastest)."""
    out = np.ones((1, 1))
    for T in tables[::-1]:
        out = np.kron(out, T)
    return out


def reference_cell_matrix(k, d, h, nq=None):
    """(k+1)^d square matrix of sum_{a,b} int_K d_ab u d_ab v on a box cell of widths h (scalar: a cube;
    sequence: per-axis widths of a graded / anisotropic cell)."""
    hs = np.broadcast_to(np.asarray(h, dtype=np.float64), (d,))
    bas = Basis1D(k)
    nq = nq or (k + 2)
    t, w = gauss_legendre(nq)
    V, D1r, D2r = bas.eval(t, 0), bas.eval(t, 1), bas.eval(t, 2)
    W = _tensor([w[None, :]] * d).ravel() * np.prod(hs)
    K = 0.0
    for a in range(d):
        for b in range(d):
            tabs = []
            for ax in range(d):
                if a == b:
                    tabs.append(D2r / hs[ax] ** 2 if ax == a else V)
                else:
                    tabs.append(D1r / hs[ax] if ax in (a, b) else V)
            H = _tensor(tabs)                      # [nl, Q]: d_ab phi_m at points
            K = K + (H * W) @ H.T
    return K


def graded_face_matrix(k, d, axis, kind, sigma, ht, hm, hp=None, nq=None, bfac=BOUNDARY_PENALTY):
    """Face matrix of a facet perpendicular to `axis` on a graded Cartesian mesh: ht = the d
    widths of the facet's cells (only the tangential ones are used), hm / hp = the normal widths of the lower /
    upper cell; h_e = harmonic mean 2 hm hp / (hm + hp) on an interior facet, h / bfac on a
    boundary facet (reading Q27).  kind as in reference_face_matrix."""
    bas = Basis1D(k)
    nq = nq or (k + 2)
    t, w = gauss_legendre(nq)
    V = bas.eval(t, 0)
    ht = np.asarray(ht, dtype=np.float64)
    tang = [ax for ax in range(d) if ax != axis]
    Wf = _tensor([w[None, :]] * (d - 1)).ravel() * np.prod(ht[tang]) if d > 1 else np.ones(1)

    def trace(tn, der, hn):
        tabs = [V] * d
        tabs = list(tabs)
        tabs[axis] = bas.eval(tn, der) / hn ** der
        return _tensor(tabs)

    if kind == "interior":
        J = np.vstack([trace(1.0, 1, hm), -trace(0.0, 1, hp)])
        Mn = np.vstack([0.5 * trace(1.0, 2, hm), 0.5 * trace(0.0, 2, hp)])
        he = 2.0 * hm * hp / (hm + hp)
    elif kind == "lower":
        J, Mn, he = -trace(0.0, 1, hm), trace(0.0, 2, hm), hm / bfac
    elif kind == "upper":
        J, Mn, he = trace(1.0, 1, hm), trace(1.0, 2, hm), hm / bfac
    else:
        raise ValueError(kind)
    JW, MW = J * Wf, Mn * Wf
    return (sigma / he) * (JW @ J.T) - JW @ Mn.T - MW @ J.T


def reference_face_matrix(k, d, h, axis, kind, sigma, nq=None, bfac=BOUNDARY_PENALTY):
    """Face matrix for a facet perpendicular to `axis`.

    kind='interior': (2 nl)^2 on [dofs of lower cell K^- | dofs of upper cell K^+].
    kind='lower'/'upper': nl^2 on the one cell touching the boundary facet x_axis=0 / =1;
    penalty sigma/h_e with h_e = h/bfac there (reading Q27).
    """
    bas = Basis1D(k)
    nq = nq or (k + 2)
    t, w = gauss_legendre(nq)
    V = bas.eval(t, 0)
    Wf = _tensor([w[None, :]] * (d - 1)).ravel() * h ** (d - 1) if d > 1 else np.ones(1)

    def trace(tn, der):
        """[nl, Qf]: d^der/dx_axis^der phi_m at face points (normal coordinate tn)."""
        col = bas.eval(tn, der) / h ** der           # [k+1, 1]
        tabs = [V] * d
        tabs = list(tabs)
        tabs[axis] = col
        return _tensor(tabs)

    if kind == "interior":
        Jm, Jp = trace(1.0, 1), -trace(0.0, 1)          # outward normals +e (K^-), -e (K^+)
        Mm, Mp = 0.5 * trace(1.0, 2), 0.5 * trace(0.0, 2)
        J = np.vstack([Jm, Jp]); Mn = np.vstack([Mm, Mp])
    elif kind == "lower":
        J, Mn = -trace(0.0, 1), trace(0.0, 2)
        sigma = bfac * sigma
    elif kind == "upper":
        J, Mn = trace(1.0, 1), trace(1.0, 2)
        sigma = bfac * sigma
    else:
        raise ValueError(kind)
    JW, MW = J * Wf, Mn * Wf
    return (sigma / h) * (JW @ J.T) - JW @ Mn.T - MW @ J.T


def _local_full_ids(k, d, N, cells):
    """[ncells, nl] full-node ids (j-numbering, nn=kN+1 per axis) of the cells' local dofs."""
    nn = k * N + 1
    offs = np.array(list(itertools.product(range(k + 1), repeat=d)))[:, ::-1]   # x fastest
    j = cells[:, None, :] * k + offs[None, :, :]                                   # [nc, nl, d]
    strides = nn ** np.arange(d)
    return (j * strides).sum(-1)


def assemble_full(k, d, N, sigma, cells=None, bfac=BOUNDARY_PENALTY, nodes=None):
    """COO->CSR of the C0IP form over full nodes (boundary nodes included).

    cells: optional [m, d] int array of included cells (a window); all faces whose adjacent
    cells are all included are added.  Default: every cell (the global matrix).
    nodes: optional list of d arrays of cell boundaries (graded / anisotropic Cartesian mesh):
    every cell and facet matrix is then integrated with its own widths (graded_face_matrix).
    """
    if nodes is not None:
        return _assemble_full_graded(k, d, N, sigma, bfac, [np.asarray(x, dtype=np.float64) for x in nodes])
    h = 1.0 / N
    nn = k * N + 1
    if cells is None:
        cells = np.array(list(itertools.product(range(N), repeat=d)))[:, ::-1]
    cells = np.asarray(cells, dtype=np.int64)
    inset = np.zeros((N,) * d, dtype=bool)
    inset[tuple(cells[:, ::-1].T)] = True                # indexed [c_{d-1},...,c_0]
    rows, cols, vals = [], [], []

    def add(ids, Mat):
        rows.append(np.repeat(ids, Mat.shape[1], axis=1).ravel())
        cols.append(np.tile(ids, (1, Mat.shape[0])).ravel())
        vals.append(np.broadcast_to(Mat.ravel(), (ids.shape[0], Mat.size)).ravel())

    Kc = reference_cell_matrix(k, d, h)
    ids = _local_full_ids(k, d, N, cells)
    add(ids, Kc)
    for a in range(d):
        Fi = reference_face_matrix(k, d, h, a, "interior", sigma)
        Fl = reference_face_matrix(k, d, h, a, "lower", sigma, bfac=bfac)
        Fu = reference_face_matrix(k, d, h, a, "upper", sigma, bfac=bfac)
        lo = cells[cells[:, a] == 0]
        if len(lo):
            add(_local_full_ids(k, d, N, lo), Fl)
        up = cells[cells[:, a] == N - 1]
        if len(up):
            add(_local_full_ids(k, d, N, up), Fu)
        cand = cells[cells[:, a] < N - 1]
        nb = cand.copy(); nb[:, a] += 1
        ok = inset[tuple(nb[:, ::-1].T)]
        if ok.any():
            idm = _local_full_ids(k, d, N, cand[ok]); idp = _local_full_ids(k, d, N, nb[ok])
            add(np.hstack([idm, idp]), Fi)
    rows = np.concatenate(rows); cols = np.concatenate(cols); vals = np.concatenate(vals)
    return sp.csr_matrix((vals, (rows, cols)), shape=(nn ** d, nn ** d))


def _assemble_full_graded(k, d, N, sigma, bfac, nodes):
    nn = k * N + 1
    hs = [np.diff(x) for x in nodes]
    cells = np.array(list(itertools.product(range(N), repeat=d)))[:, ::-1]
    rows, cols, vals = [], [], []
    cache = {}

    def add(ids, Mat):
        rows.append(np.repeat(ids, Mat.shape[1], axis=1).ravel())
        cols.append(np.tile(ids, (1, Mat.shape[0])).ravel())
        vals.append(np.broadcast_to(Mat.ravel(), (ids.shape[0], Mat.size)).ravel())

    for c in cells:
        hc = tuple(hs[a][c[a]] for a in range(d))
        key = ("cell", hc)
        if key not in cache:
            cache[key] = reference_cell_matrix(k, d, hc)
        add(_local_full_ids(k, d, N, c[None, :]), cache[key])
        for a in range(d):
            if c[a] == 0:
                add(_local_full_ids(k, d, N, c[None, :]),
                    graded_face_matrix(k, d, a, "lower", sigma, hc, hc[a], bfac=bfac))
            if c[a] == N - 1:
                add(_local_full_ids(k, d, N, c[None, :]),
                    graded_face_matrix(k, d, a, "upper", sigma, hc, hc[a], bfac=bfac))
            else:
                nb = c.copy(); nb[a] += 1
                Fi = graded_face_matrix(k, d, a, "interior", sigma, hc, hc[a], hs[a][c[a] + 1], bfac=bfac)
                add(np.hstack([_local_full_ids(k, d, N, c[None, :]), _local_full_ids(k, d, N, nb[None, :])]), Fi)
    rows = np.concatenate(rows); cols = np.concatenate(cols); vals = np.concatenate(vals)
    return sp.csr_matrix((vals, (rows, cols)), shape=(nn ** d, nn ** d))


def interior_full_ids(k, d, N):
    """Full-node ids of the interior nodes, in interior (i) order, x fastest."""
    nn = k * N + 1
    n = k * N - 1
    idx = np.zeros((n,) * d, dtype=np.int64)
    strides = nn ** np.arange(d)
    # idx[i_{d-1}, ..., i_0] = sum_a (i_a + 1) nn^a
    for a in range(d):
        shape = [1] * d; shape[d - 1 - a] = n
        idx = idx + ((np.arange(n) + 1) * strides[a]).reshape(shape)
    return idx.ravel()


def assemble(k, d, N, sigma, bfac=BOUNDARY_PENALTY, nodes=None):
    """A_ell over interior DoFs (CSR), boundary rows/cols eliminated (reading Q26); nodes: graded mesh."""
    Af = assemble_full(k, d, N, sigma, bfac=bfac, nodes=nodes)
    keep = interior_full_ids(k, d, N)
    return Af[keep][:, keep].tocsr()


def rhs_load(k, d, N, f, nq=None, nodes=None):
    """b_i = int f phi_i (Eq. bfandrhs) by tensor Gauss quadrature per cell.

    f(*coords) takes d arrays of physical coordinates.  nq defaults to k+3.
    nodes: optional per-axis cell boundaries (graded mesh).
    """
    nodes = [np.arange(N + 1) / N] * d if nodes is None else [np.asarray(x, dtype=np.float64) for x in nodes]
    hs = [np.diff(x) for x in nodes]
    nq = nq or (k + 3)
    bas = Basis1D(k)
    t, w = gauss_legendre(nq)
    Phi = _tensor([bas.eval(t, 0)] * d)                      # [nl, Q]
    W0 = _tensor([w[None, :]] * d).ravel()
    cells = np.array(list(itertools.product(range(N), repeat=d)))[:, ::-1]
    tq = np.array(list(itertools.product(range(nq), repeat=d)))[:, ::-1]   # x fastest points
    coords = [nodes[a][cells[:, a]][:, None] + t[tq[:, a]][None, :] * hs[a][cells[:, a]][:, None] for a in range(d)]
    vol = np.prod([hs[a][cells[:, a]] for a in range(d)], axis=0)            # [ncells]
    fv = f(*coords)                                          # [ncells, Q]
    contrib = (fv * W0[None, :] * vol[:, None]) @ Phi.T      # [ncells, nl]
    nn = k * N + 1
    bf = np.zeros(nn ** d)
    np.add.at(bf, _local_full_ids(k, d, N, cells).ravel(), contrib.ravel())
    return bf[interior_full_ids(k, d, N)]


def paper_load(d):
    """f = Delta^2 prod sin(pi x_a) = d^2 pi^4 prod sin(pi x_a) (readings Q1, Q8)."""
    def f(*xs):
        out = (d * d) * np.pi ** 4
        for x in xs:
            out = out * np.sin(np.pi * x)
        return out
    return f


def paper_solution(d):
    """u*(x) = prod_a sin(pi x_a), the analytical solution of the experiments."""
    def u(*xs):
        out = 1.0
        for x in xs:
            out = out * np.sin(np.pi * x)
        return out
    return u


def boundary_data_load(k, d, N, sigma, nq=None, bfac=BOUNDARY_PENALTY, nodes=None):
    """Nitsche boundary-data part of F for d_n u = g on the boundary (reading Q8b).

    PAPER.md:488 fixes u* = prod sin(pi x_a) as the solution; u* = 0 on the boundary but its
    normal derivative g = d_n u* is not zero, so the clamped condition d_n u = g is imposed weakly
    by the terms that the boundary facets of Eq. bfc0ip (one-sided jump/mean
    PAPER.md:100-106) generate with [d_n u] -> d_n u - g:
        F_bd(v) = sum_{e in F^bd} int_e g ( (sigma/h_e) d_n v - d_n^2 v ) ds,
    with h_e = h/bfac (reading Q27).  On the facet x_a = 0 (outward normal -e_a) and x_a = 1
    (normal +e_a): g = d_n u* = -pi prod_{b != a} sin(pi x_b).  Facet quadrature: k+3 Gauss points
    per cell and tangential axis.
    """
    nodes = [np.arange(N + 1) / N] * d if nodes is None else [np.asarray(x, dtype=np.float64) for x in nodes]
    hs = [np.diff(x) for x in nodes]
    nq = nq or (k + 3)
    bas = Basis1D(k)
    t, w = gauss_legendre(nq)
    V = bas.eval(t, 0)
    Wf0 = _tensor([w[None, :]] * (d - 1)).ravel() if d > 1 else np.ones(1)
    tq = np.array(list(itertools.product(range(nq), repeat=d - 1)))[:, ::-1] if d > 1 else np.zeros((1, 0), int)
    nn = k * N + 1
    bf = np.zeros(nn ** d)
    for a in range(d):
        for side in (0, 1):
            tn = float(side)
            sgn = 1.0 if side == 1 else -1.0
            hn = hs[a][0 if side == 0 else N - 1]                  # normal width of the boundary cells
            # traces on the facet: [nl, Qf] for d_n phi and d_n^2 phi (x fastest over the cell's dofs)
            tabs1 = [V] * d; tabs1[a] = sgn * bas.eval(tn, 1) / hn
            tabs2 = [V] * d; tabs2[a] = bas.eval(tn, 2) / hn ** 2
            Dn1, Dn2 = _tensor(tabs1), _tensor(tabs2)
            cells = np.array(list(itertools.product(range(N), repeat=d)))[:, ::-1]
            cells = cells[cells[:, a] == (0 if side == 0 else N - 1)]
            others = [b for b in range(d) if b != a]
            g = -np.pi * np.ones((len(cells), len(Wf0)))
            area = np.ones(len(cells))
            for j, b in enumerate(others):
                hb = hs[b][cells[:, b]]
                g = g * np.sin(np.pi * (nodes[b][cells[:, b]][:, None] + t[tq[:, j]][None, :] * hb[:, None]))
                area = area * hb
            contrib = (g * Wf0[None, :] * area[:, None]) @ ((bfac * sigma / hn) * Dn1 - Dn2).T   # [ncells, nl]
            np.add.at(bf, _local_full_ids(k, d, N, cells).ravel(), contrib.ravel())
    return bf[interior_full_ids(k, d, N)]


def paper_rhs(k, d, N, sigma, bfac=BOUNDARY_PENALTY, nodes=None):
    """F of the solve experiments: int f v with f = Delta^2 u* plus the
    boundary-data terms of boundary_data_load, so that u_h -> u* = prod sin(pi x_a)."""
    return (rhs_load(k, d, N, paper_load(d), nodes=nodes) +
            boundary_data_load(k, d, N, sigma, bfac=bfac, nodes=nodes))


def dof_coords_graded(k, X):
    """Physical coordinates of the interior 1D DoFs of the graded mesh with cell boundaries X."""
    from .basis import gauss_lobatto_points
    X = np.asarray(X, dtype=np.float64)
    t = gauss_lobatto_points(k)
    N = len(X) - 1
    return np.array([X[c] + t[m] * (X[c + 1] - X[c]) for c in range(N) for m in range(k)][1:])


def dof_coords(k, N, i):
    """Physical coordinate of interior 1D DoF index i (node j = i+1), SURVEY.md C1."""
    from .basis import gauss_lobatto_points
    t = gauss_lobatto_points(k)
    j = np.asarray(i) + 1
    return (j // k + t[j % k]) / N


def residual_on_box(k, d, N, sigma, x, b, box_lo, box_hi):
    """r = b - A x on the interior-DoF box [box_lo, box_hi) (per axis, interior indices).

    Assembles the form only on a window of cells around the box (every cell and facet
    that touches a box node's basis function), so it is exact at any N.  Used for
    sampled parity at sizes where the global CSR does not fit.
    """
    n = k * N - 1
    nn = k * N + 1
    box_lo = np.asarray(box_lo); box_hi = np.asarray(box_hi)
    j_lo, j_hi = box_lo + 1, box_hi                          # full-node range [j_lo, j_hi]
    c_lo = np.maximum((j_lo - 1) // k - 1, 0)                # cells touching the box nodes ...
    c_hi = np.minimum(j_hi // k + 1, N - 1)                  # ... and their facet neighbours
    rng = [np.arange(c_lo[a], c_hi[a] + 1) for a in range(d)]
    cells = np.array(list(itertools.product(*rng[::-1])))[:, ::-1]
    Af = assemble_full(k, d, N, sigma, cells)
    # rows: box nodes (full ids); columns: every node in the window cells
    box_axes = [np.arange(box_lo[a], box_hi[a]) for a in range(d)]
    bi = np.array(list(itertools.product(*box_axes[::-1])))[:, ::-1]          # interior idx
    rows_full = ((bi + 1) * nn ** np.arange(d)).sum(-1)
    rows_int = (bi * n ** np.arange(d)).sum(-1)
    sub = Af[rows_full].tocoo()
    jc = np.stack([(sub.col // nn ** a) % nn for a in range(d)], -1)
    interior = np.all((jc >= 1) & (jc <= nn - 2), axis=1)
    ic = ((jc - 1) * n ** np.arange(d)).sum(-1)
    Ax = np.zeros(len(rows_full))
    np.add.at(Ax, sub.row[interior], sub.data[interior] * x[ic[interior]])
    return (b[rows_int] - Ax), rows_int


def energy_error(k, d, N, sigma, uh, hess_u, nq=None):
    """Mesh-dependent energy error |u - u_h|_h of Eq. hnorm:

    sum_K |u - u_h|^2_{H^2(K)} + sum_e (sigma/h_e) ||[d_n (u - u_h)]||^2_{L^2(e)}.
    u must be in H^2_0 and smooth (no jumps, d_n u = 0 on the boundary), so the facet part
    reduces to the jumps of u_h.  hess_u(*coords) -> array [..., d, d].
    """
    h = 1.0 / N
    nq = nq or (k + 3)
    bas = Basis1D(k)
    t, w = gauss_legendre(nq)
    V, D1, D2 = bas.eval(t, 0), bas.eval(t, 1) / h, bas.eval(t, 2) / h ** 2
    W = _tensor([w[None, :]] * d).ravel() * h ** d
    cells = np.array(list(itertools.product(range(N), repeat=d)))[:, ::-1]
    nn = k * N + 1
    uf = np.zeros(nn ** d)
    uf[interior_full_ids(k, d, N)] = uh
    U = uf[_local_full_ids(k, d, N, cells)]                         # [ncells, nl]
    tq = np.array(list(itertools.product(range(nq), repeat=d)))[:, ::-1]
    coords = [(cells[:, a][:, None] + t[tq[:, a]][None, :]) * h for a in range(d)]
    Hu = hess_u(*coords)                                            # [ncells, Q, d, d]
    bulk = 0.0
    for a in range(d):
        for b in range(d):
            tabs = []
            for ax in range(d):
                if a == b:
                    tabs.append(D2 if ax == a else V)
                else:
                    tabs.append(D1 if ax in (a, b) else V)
            Hh = U @ _tensor(tabs)                                  # [ncells, Q]
            bulk += (((Hu[..., a, b] - Hh) ** 2) * W).sum()
    face = 0.0
    for a in range(d):
        for kind in ("interior", "lower", "upper"):
            # penalty-only face matrix: (sigma/h) J J^T  ==  face matrix with b-terms removed
            Fs = reference_face_matrix(k, d, h, a, kind, sigma) - reference_face_matrix(k, d, h, a, kind, 0.0)
            if kind == "interior":
                cm = cells[cells[:, a] < N - 1]; cp = cm.copy(); cp[:, a] += 1
                Uf = np.hstack([uf[_local_full_ids(k, d, N, cm)], uf[_local_full_ids(k, d, N, cp)]])
            else:
                sel = cells[cells[:, a] == (0 if kind == "lower" else N - 1)]
                Uf = uf[_local_full_ids(k, d, N, sel)]
            face += np.einsum("ci,ij,cj->", Uf, Fs, Uf)
    return np.sqrt(bulk + face)
