"""Pins for the graded / anisotropic Cartesian meshes of the oracle ("the
discretization only requires shape regular, locally uniform cells", PAPER.md:131 harmonic-mean h_e)."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle.discretization import global_matrices_1d, graded_nodes, default_sigma
from oracle.operator import assemble, paper_rhs, paper_solution, dof_coords_graded
from oracle.multigrid import embedding_1d, Hierarchy, pcg, precondition, fractional_iterations

NODES = {2: [graded_nodes(4, 0.5), graded_nodes(4, -0.4)],
         3: [graded_nodes(3, 0.5), graded_nodes(3, -0.4), graded_nodes(3, 0.2)]}


def _kron_form(mats):
    d = len(mats)
    if d == 2:
        (Mx, Lx, Bx), (My, Ly, By) = mats
        return np.kron(My, Bx) + 2 * np.kron(Ly, Lx) + np.kron(By, Mx)
    (Mx, Lx, Bx), (My, Ly, By), (Mz, Lz, Bz) = mats
    kr = lambda a, b, c: np.kron(np.kron(a, b), c)
    return (kr(Mz, My, Bx) + kr(Mz, By, Mx) + kr(Bz, My, Mx) +
            2 * (kr(Mz, Ly, Lx) + kr(Lz, Ly, Mx) + kr(Lz, My, Lx)))


@pytest.mark.parametrize("d,k", [(2, 2), (2, 3), (2, 4), (3, 2)])
def test_graded_kronecker_identity_spd(d, k):
    """The d-dimensional cell/facet quadrature on graded cells (per-axis widths, harmonic-mean h_e) equals the
    Kronecker form of PAPER.md:314-342 built from the graded 1D matrices; the matrix is symmetric positive
    definite."""
    nodes = NODES[d]
    N = len(nodes[0]) - 1
    s = default_sigma(k)
    A = assemble(k, d, N, s, nodes=nodes).toarray()
    mats = [[X.toarray() for X in global_matrices_1d(k, N, s, nodes=nodes[a])] for a in range(d)]
    K = _kron_form(mats)
    assert np.abs(A - K).max() <= 1e-12 * np.abs(A).max()
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0


def test_uniform_nodes_reduce_to_uniform():
    k, N, s = 3, 5, default_sigma(3)
    X = np.linspace(0, 1, N + 1)
    for a, b in zip(global_matrices_1d(k, N, s), global_matrices_1d(k, N, s, nodes=X)):
        assert np.abs((a - b).toarray()).max() <= 1e-13 * np.abs(a.toarray()).max()
    A, G = assemble(k, 2, N, s), assemble(k, 2, N, s, nodes=[X, X])
    assert np.abs((A - G).toarray()).max() <= 1e-12 * np.abs(A.toarray()).max()


@pytest.mark.parametrize("k", [3, 4])
def test_graded_manufactured_solution(k):
    """PAPER.md:488 on an anisotropically graded mesh: u_h -> u* = prod sin(pi x_a) at nodal rate >= k."""
    errs = []
    for N in (4, 8, 16):
        nodes = [graded_nodes(N, 0.5), graded_nodes(N, -0.4)]
        s = default_sigma(k)
        u = spla.spsolve(assemble(k, 2, N, s, nodes=nodes).tocsc(), paper_rhs(k, 2, N, s, nodes=nodes))
        xs = [dof_coords_graded(k, X) for X in nodes]
        XX, YY = np.meshgrid(xs[0], xs[1])
        errs.append(np.abs(u - paper_solution(2)(XX.ravel(), YY.ravel())).max())
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates >= k - 0.3), rates


@pytest.mark.parametrize("k", [2, 3, 5])
def test_graded_embedding_reproduces_polynomials(k):
    """The natural embedding on nested graded meshes: the coarse interpolant of p in Q_k with
    p(0) = p(1) = 0 evaluated at the fine DoFs is the fine interpolant."""
    Xf = graded_nodes(6, 0.6)
    E = embedding_1d(k, 3, nodes_f=Xf)
    xc, xf = dof_coords_graded(k, Xf[::2]), dof_coords_graded(k, Xf)
    for deg in range(2, k + 1):
        p = lambda x: x * (1 - x) * (x + 0.3) ** (deg - 2)
        assert np.abs(E @ p(xc) - p(xf)).max() < 1e-12


def test_graded_mg_pcg_converges():
    """MG-PCG with the AVS cycle on a graded hierarchy reaches 1e-8 and stays within 1.5x the uniform count."""
    k, L, s = 3, 5, default_sigma(3)
    nodes = [graded_nodes(2 ** L, 0.5), graded_nodes(2 ** L, -0.4)]
    hg = Hierarchy(k, 2, L, s, nodes=nodes)
    b = paper_rhs(k, 2, 2 ** L, s, nodes=nodes)
    x, n, hist = pcg(hg.A[L], b, lambda r: precondition(hg, r, "avs", 2, 0.25))
    hu = Hierarchy(k, 2, L, s)
    _, nu, _ = pcg(hu.A[L], paper_rhs(k, 2, 2 ** L, s), lambda r: precondition(hu, r, "avs", 2, 0.25))
    assert hist[-1] <= 1e-8 * hist[0] and n <= 1.5 * nu + 1, (n, nu)
    xd = spla.spsolve(hg.A[L].tocsc(), b)
    assert np.linalg.norm(x - xd) <= 1e-6 * np.linalg.norm(xd)
