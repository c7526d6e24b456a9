"""Transfers, V-cycle (Alg. 1) and MG-preconditioned CG.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Transfers: prolongation = matrix of the natural embedding V_{l-1} -> V_l,
E_ij = phi^coarse_j(x^fine_i) over interior nodes, P = kron(E,..,E) (x fastest); the
restriction is P^T.  A_l is rediscretised on every level.

V-cycle (PAPER.md:158-176 with readings Q12, Q13): at the coarsest level (N=2, one
patch) a single smoothing step from zero; else pre-smooth, restrict the residual,
recurse with zero guess, prolongate-add, post-smooth (reversed colour order for MVS when
`symmetric`, reading Q11).  The FP32 cycle is the same code on float32 copies of every
array (reading Q21): the residual is converted at entry, the correction at exit
(PAPER.md:749).

PCG: textbook preconditioned CG (Saad Alg. 9.1) in FP64, x0 = 0 (reading Q19), stop at
||r_n|| <= rtol ||r_0|| on the recursively updated residual;
nu = -8 / log10((||r_n||/||r_0||)^(1/n)) (reading Q7).
"""
import numpy as np
import scipy.sparse as sp

from .basis import Basis1D, gauss_lobatto_points
from .operator import assemble
from .smoothers import PatchSolvers, smooth
from .mesh import level_cells


def default_omega(d, kind, exact=False):
    """Damping of the experiments: AVS 1/4 in 2D, 0.1 in 3D;
    MVS 1 with exact local solvers, 0.7 in 3D and, where the paper
    gives no value (2D, inexact local solvers), 0.8 (reading Q28)."""
    if kind == "avs":
        return 0.25 if d == 2 else 0.1
    if exact:
        return 1.0
    return 0.8 if d == 2 else 0.7


def embedding_1d(k, Nc, nodes_f=None):
    """E (n_f x n_c): coarse global basis (Nc cells) evaluated at the fine (2Nc) interior nodes.
    nodes_f: optional cell boundaries of the fine graded mesh (2Nc + 1 values); the coarse mesh is every second
    boundary (nested refinement)."""
    Nf = 2 * Nc
    t = gauss_lobatto_points(k)
    bas = Basis1D(k)
    nf, nc = k * Nf - 1, k * Nc - 1
    Xf = np.arange(Nf + 1) / Nf if nodes_f is None else np.asarray(nodes_f, dtype=np.float64)
    Xc = Xf[::2]
    E = np.zeros((nf, nc))
    for i in range(nf):
        j = i + 1
        cf = min(j // k, Nf - 1)
        x = Xf[cf] + t[j - cf * k] * (Xf[cf + 1] - Xf[cf])
        c = cf // 2
        tl = (x - Xc[c]) / (Xc[c + 1] - Xc[c])
        vals = bas.eval(tl, 0)[:, 0]
        for m in range(k + 1):
            jc = c * k + m
            if 1 <= jc <= k * Nc - 1:
                E[i, jc - 1] += vals[m]
    E[np.abs(E) < 1e-15] = 0.0
    return E


def prolongation(k, d, Nc, nodes_f=None):
    """P = kron(E_{d-1}, ..., E_0) (x fastest); nodes_f: per-axis fine cell boundaries of a graded mesh."""
    Es = [sp.csr_matrix(embedding_1d(k, Nc, None if nodes_f is None else nodes_f[a])) for a in range(d)]
    P = Es[0]
    for a in range(1, d):
        P = sp.kron(Es[a], P)      # kron(E_y, E_x) etc.: x fastest
    return P.tocsr()


class Hierarchy:
    """Levels 1..L (N = 2^l, reading Q9) with A_l, patch solvers and P_l (coarse l-1 -> l)."""

    def __init__(self, k, d, L, sigma, dtype=np.float64, nodes=None):
        """nodes: optional per-axis cell boundaries of the finest level (graded mesh); level l uses
        every 2^(L-l)-th boundary."""
        self.k, self.d, self.L, self.sigma = k, d, L, sigma
        self.A, self.ps, self.P = {}, {}, {}
        for l in range(1, L + 1):
            N = level_cells(l)
            nl = None if nodes is None else [np.asarray(x)[:: 2 ** (L - l)] for x in nodes]
            self.A[l] = assemble(k, d, N, sigma, nodes=nl)
            self.ps[l] = PatchSolvers(k, d, N, sigma, nodes=nl)
            if l > 1:
                self.P[l] = prolongation(k, d, level_cells(l - 1), nodes_f=nl)
        self.set_dtype(dtype)

    def set_dtype(self, dtype):
        """FP32 cycle: every array rounded from the FP64 values (reading Q21)."""
        self.dtype = dtype
        self.Ac = {l: A.astype(dtype) for l, A in self.A.items()}
        self.Pc = {l: P.astype(dtype) for l, P in self.P.items()}
        for ps in self.ps.values():
            if not hasattr(ps, "groups64"):
                ps.groups64 = ps.groups
            ps.groups = {key: (ids, Ainv.astype(dtype), At.astype(dtype))
                         for key, (ids, Ainv, At) in ps.groups64.items()}


def vcycle(h, l, x, b, kind, steps, omega, symmetric=True):
    """MG_l(x, b) of Algorithm 1 with readings Q12/Q13/Q11."""
    A, ps = h.Ac[l], h.ps[l]
    if l == 1:
        return smooth(A, ps, np.zeros_like(b), b, kind, 1, omega)
    x = smooth(A, ps, x, b, kind, steps, omega)
    bc = h.Pc[l].T @ (b - A @ x)
    e = vcycle(h, l - 1, np.zeros_like(bc), bc, kind, steps, omega, symmetric)
    x = x + h.Pc[l] @ e
    return smooth(A, ps, x, b, kind, steps, omega, reverse=(symmetric and kind == "mvs"))


def precondition(h, r64, kind, steps, omega, symmetric=True):
    """z = MG_L(0, r): convert r to the cycle dtype at entry, z to FP64 at exit."""
    rc = r64.astype(h.dtype)
    z = vcycle(h, h.L, np.zeros_like(rc), rc, kind, steps, omega, symmetric)
    return z.astype(np.float64)


def pcg(A, b, prec, rtol=1e-8, max_iter=200, x0=None):
    """Preconditioned CG (Saad Alg. 9.1).  Returns x, iterations n, residual-norm history."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - A @ x
    z = prec(r)
    p = z.copy()
    rz = r @ z
    hist = [np.linalg.norm(r)]
    n = 0
    while n < max_iter and hist[-1] > rtol * hist[0]:
        Ap = A @ p
        alpha = rz / (p @ Ap)
        x = x + alpha * p
        r = r - alpha * Ap
        n += 1
        hist.append(np.linalg.norm(r))
        if hist[-1] <= rtol * hist[0]:
            break
        z = prec(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, n, np.array(hist)


def gmres(A, b, prec, rtol=1e-8, max_iter=200, restart=50, x0=None):
    """Flexible right-preconditioned restarted GMRES, FGMRES(m) (Saad, Iterative Methods for Sparse
    Linear Systems, Alg. 9.6; with a fixed preconditioner it is right-preconditioned GMRES, Alg. 9.5):
    modified Gram-Schmidt Arnoldi on A M^{-1}, Givens rotations for the least-squares problem, x
    updated from the stored preconditioned vectors Z at the end of every cycle.  PAPER.md:487 (GMRES
    outer solver for the multiplicative smoother, rtol 1e-8 relative to ||r_0||).  Returns x,
    iterations n (Arnoldi steps), history of the least-squares residual norms |g_{j+1}| (the true
    residual norm in exact arithmetic)."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - A @ x
    beta = np.linalg.norm(r)
    hist = [beta]
    r0 = beta
    n = 0
    # stopping test on the least-squares residual |g_{j+1}| (the recursively updated residual, as in
    # PCG): the true residual of a smooth solution is only known to ~eps || |A| |x| ||
    while n < max_iter and hist[-1] > rtol * r0:
        m = min(restart, max_iter - n)
        V = [r / beta]
        Z = []
        H = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        j_done = 0
        for j in range(m):
            z = prec(V[j])
            Z.append(z)
            w = A @ z
            for i in range(j + 1):                     # modified Gram-Schmidt
                H[i, j] = w @ V[i]
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            V.append(w / H[j + 1, j] if H[j + 1, j] > 0 else w)
            for i in range(j):                         # apply the previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            n += 1
            j_done = j + 1
            hist.append(abs(g[j + 1]))
            if hist[-1] <= rtol * r0:
                break
        y = np.linalg.solve(np.triu(H[:j_done, :j_done]), g[:j_done])
        for i in range(j_done):
            x = x + y[i] * Z[i]
        r = b - A @ x
        beta = np.linalg.norm(r)
    return x, n, np.array(hist)


def fractional_iterations(hist):
    """nu = -8 / log10(rbar), rbar = (||r_n||/||r_0||)^(1/n) (reading Q7)."""
    n = len(hist) - 1
    if n == 0:
        return 0.0
    ratio = hist[-1] / hist[0]
    if ratio == 0.0:
        return 0.0
    return -8.0 / np.log10(ratio ** (1.0 / n))


def solve_paper(d, k, L, kind, steps, exact=False, omega=None, cycle_dtype=np.float64, rtol=1e-8):
    """One solve of the paper's experiment protocol: x0 = 0, F =
    operator.paper_rhs (reading Q8b), boundary penalty per reading Q27.  AVS: CG with the symmetric
    cycle; MVS: GMRES (FGMRES(50)) with the same-order cycle (reading Q11).  `steps` pre- and
    post-smoothing steps, omega = default_omega unless given; exact=True uses A_v = R_v A R_v^T
    (Table 1).  Returns (iterations, nu, Hierarchy)."""
    from .operator import paper_rhs
    from .smoothers import PatchSolvers
    from .discretization import default_sigma
    s = default_sigma(k)
    h = Hierarchy(k, d, L, s)
    if exact:
        for l in h.A:
            h.ps[l] = PatchSolvers(k, d, level_cells(l), s, exact_A=h.A[l])
    h.set_dtype(cycle_dtype)
    om = default_omega(d, kind, exact) if omega is None else omega
    b = paper_rhs(k, d, level_cells(L), s)
    if kind == "avs":
        _, n, hist = pcg(h.A[L], b, lambda r: precondition(h, r, kind, steps, om), rtol=rtol)
    else:
        _, n, hist = gmres(h.A[L], b, lambda r: precondition(h, r, kind, steps, om, symmetric=False),
                           rtol=rtol, restart=50)
    return n, fractional_iterations(hist), h
