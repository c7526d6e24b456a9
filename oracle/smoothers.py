"""Vertex-patch Schwarz smoothers with the separable surrogate local solver.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

AVS:      x <- x + omega sum_v R_v^T A~_v^{-1} R_v (b - A x)
coloured MVS: for each colour c in order,
                              x <- x + omega sum_{v in c} R_v^T A~_v^{-1} R_v (b - A x)
(sign "+" per reading Q2).  A~_v is the separable surrogate of Eq. localsolverbila
(PAPER.md:369-384): A~_v = sum_a B_{v,a} (x) (x)_{b!=a} M_{v,b}, built from principal
submatrices of the 1D matrices in numpy.kron order (z,y,x; x fastest,
reading Q17).  The oracle inverts A~_v densely (Cholesky solve against the identity, refined once)
-- never by fast diagonalisation -- and applies the explicit inverse to all patches of a variant
tuple as one matrix product followed by one step of iterative refinement.  The exact local solver
A_v = R_v A R_v^T (Table 1) is available for tests.
"""
import numpy as np
import scipy.linalg as sla

from .discretization import global_matrices_1d, patch_range_1d, patch_variant
from .mesh import patch_vertices, all_patch_dofs, color_patches, patch_dofs, n_dofs_1d


def _kron_all(mats):
    """kron(m_{d-1}, ..., m_0) for mats = [m_0 (x), m_1 (y), ...]."""
    out = np.ones((1, 1))
    for m in mats[::-1]:
        out = np.kron(out, m)
    return out


class PatchSolvers:
    """Dense Cholesky factors of A~_v per variant tuple, plus the patch DoF maps."""

    def __init__(self, k, d, N, sigma, exact_A=None, nodes=None):
        """nodes: optional per-axis cell boundaries (graded mesh): the 1D matrices are per axis and
        every patch has its own blocks (group key = vertex tuple instead of the axis-variant tuple)."""
        self.k, self.d, self.N = k, d, N
        mats = [[X.toarray() for X in global_matrices_1d(k, N, sigma, nodes=None if nodes is None else nodes[a])]
                for a in range(d)]
        self.verts = patch_vertices(d, N)
        self.dofs = all_patch_dofs(k, d, N)
        self.groups = {}          # variant tuple -> (patch ids, factor, dense matrix)
        if nodes is None:
            keys = [tuple(patch_variant(va, N) for va in v) for v in self.verts]
        else:
            keys = [tuple(int(va) for va in v) for v in self.verts]
        for key in sorted(set(keys)):
            ids = np.array([i for i, kk in enumerate(keys) if kk == key])
            v0 = self.verts[ids[0]]
            if exact_A is None:
                Ms = [mats[a][0][np.ix_(patch_range_1d(k, va), patch_range_1d(k, va))] for a, va in enumerate(v0)]
                Bs = [mats[a][2][np.ix_(patch_range_1d(k, va), patch_range_1d(k, va))] for a, va in enumerate(v0)]
                At = 0.0
                for a in range(d):
                    At = At + _kron_all([Bs[b] if b == a else Ms[b] for b in range(d)])
            else:
                g = self.dofs[ids[0]]
                At = exact_A[np.ix_(g, g)].toarray() if hasattr(exact_A, "toarray") else exact_A[np.ix_(g, g)]
            fac = sla.cho_factor(At)
            eye = np.eye(At.shape[0])
            Ainv = sla.cho_solve(fac, eye)
            Ainv = Ainv + sla.cho_solve(fac, eye - At @ Ainv)      # one refinement step
            self.groups[key] = (ids, 0.5 * (Ainv + Ainv.T), At)
        self.exact = exact_A is not None

    def solve(self, ids, R):
        """U[i] = A~_{v_i}^{-1} R[i] for patches ids (rows of R): U = R A~^{-1} (A~ symmetric), then one
        step of iterative refinement U += (R - U A~) A~^{-1}."""
        out = np.empty_like(R)
        for key, (gids, Ainv, At) in self.groups.items():
            mask = np.isin(ids, gids)
            if not mask.any():
                continue
            Rg = R[mask]
            U = Rg @ Ainv
            out[mask] = U + (Rg - U @ At) @ Ainv
        return out


def avs_step(A, ps, x, b, omega):
    """One additive vertex-patch smoothing step (reading Q2)."""
    r = b - A @ x
    ids = np.arange(len(ps.dofs))
    U = ps.solve(ids, r[ps.dofs])
    xn = x.copy()
    np.add.at(xn, ps.dofs.ravel(), omega * U.ravel())
    return xn


def mvs_step(A, ps, x, b, omega, reverse=False):
    """One coloured multiplicative step: residual recomputed per colour."""
    x = x.copy()
    cols = color_patches(ps.d, ps.N)
    order = range(len(cols) - 1, -1, -1) if reverse else range(len(cols))
    for c in order:
        ids = cols[c]
        if len(ids) == 0:
            continue
        r = b - A @ x
        U = ps.solve(ids, r[ps.dofs[ids]])
        np.add.at(x, ps.dofs[ids].ravel(), omega * U.ravel())
    return x


def smooth(A, ps, x, b, kind, steps, omega, reverse=False):
    for _ in range(steps):
        x = avs_step(A, ps, x, b, omega) if kind == "avs" else mvs_step(A, ps, x, b, omega, reverse)
    return x


def avs_delta_sample(k, d, N, sigma, x, b, omega, sample):
    """delta = x' - x of one AVS step at the interior DoF ids `sample`, without a global matrix.

    For every sampled DoF: its <= 2^d patches, the residual on those patches' DoFs from a
    local window assembly (operator.residual_on_box), dense surrogate solves, and the sum
    (PAPER.md:206-213).  Exact at any N.
    """
    from .operator import residual_on_box
    import itertools
    M, L, B = (X.tocsr() for X in global_matrices_1d(k, N, sigma))
    n = n_dofs_1d(k, N)

    def block(X, va):
        rr = patch_range_1d(k, va)
        return X[rr][:, rr].toarray()
    out = np.zeros(len(sample))
    for s, g in enumerate(sample):
        i = [(g // n ** a) % n for a in range(d)]
        j = [ia + 1 for ia in i]
        # vertices whose patch contains node j along each axis
        vs_axes = []
        for ja in j:
            if ja % k == 0:
                vs_axes.append([ja // k])
            else:
                vs_axes.append([ja // k, ja // k + 1])
        vs_axes = [[v for v in va if 1 <= v <= N - 1] for va in vs_axes]
        lo = [min(vv) for vv in vs_axes]; hi = [max(vv) for vv in vs_axes]
        box_lo = np.array([(lo[a] - 1) * k for a in range(d)])
        box_hi = np.array([(hi[a] + 1) * k - 1 for a in range(d)])
        r_box, ids_box = residual_on_box(k, d, N, sigma, x, b, box_lo, box_hi)
        pos = {gid: p for p, gid in enumerate(ids_box)}
        for v in itertools.product(*vs_axes):
            pd = patch_dofs(k, d, N, v)
            rv = r_box[[pos[q] for q in pd]]
            At = 0.0
            for a in range(d):
                At = At + _kron_all([block(B, v[bb]) if bb == a else block(M, v[bb])
                                     for bb in range(d)])
            fac = sla.cho_factor(At)
            u = sla.cho_solve(fac, rv)
            u = u + sla.cho_solve(fac, rv - At @ u)      # one refinement step
            loc = int(np.nonzero(pd == g)[0][0])
            out[s] += omega * u[loc]
    return out
