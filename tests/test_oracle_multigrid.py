"""Pins for transfers, V-cycle and PCG of the oracle."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle.multigrid import (embedding_1d, prolongation, Hierarchy, vcycle, precondition, pcg,
                              fractional_iterations)
from oracle.operator import dof_coords, rhs_load, paper_load, paper_rhs
from oracle.mesh import level_cells
from oracle.discretization import default_sigma
from c0ip_inputs import uniform
from golden_io import read_matrices


def test_embedding_golden_appendix_A():
    g = read_matrices("k2_N2_sigma6_1d.txt")
    assert np.allclose(embedding_1d(2, 2), g["E"], atol=1e-15)


@pytest.mark.parametrize("k", range(2, 8))
def test_embedding_reproduces_polynomials(k):
    """E maps the coarse interpolant of p in Q_k (p(0)=p(1)=0) to the fine one."""
    Nc = 3
    E = embedding_1d(k, Nc)
    xc = dof_coords(k, Nc, np.arange(k * Nc - 1)); xf = dof_coords(k, 2 * Nc, np.arange(2 * k * Nc - 1))
    for deg in range(2, k + 1):
        p = lambda x: x * (1 - x) * (x + 0.3) ** (deg - 2)
        assert np.abs(E @ p(xc) - p(xf)).max() < 1e-12


def test_prolongation_restriction_adjoint():
    """<P c, f> = <c, P^T f> and the kron order is x fastest."""
    k, Nc = 3, 3
    P = prolongation(k, 2, Nc)
    c = uniform(P.shape[1], 1); f = uniform(P.shape[0], 2)
    assert abs((P @ c) @ f - c @ (P.T @ f)) < 1e-13 * np.abs(f).sum()
    xc = dof_coords(k, Nc, np.arange(k * Nc - 1)); xf = dof_coords(k, 2 * Nc, np.arange(2 * k * Nc - 1))
    u = lambda x, y: x * (1 - x) * y * y * (1 - y)
    cc = u(xc[None, :], xc[:, None]).ravel(); ff = u(xf[None, :], xf[:, None]).ravel()
    assert np.abs(P @ cc - ff).max() < 1e-13


@pytest.fixture(scope="module")
def h2():
    return Hierarchy(2, 2, 3, default_sigma(2))


def test_vcycle_fixed_point(h2):
    """b = A x*, x = x* -> x*."""
    L = 3
    xs = uniform(h2.A[L].shape[0], 5)
    out = vcycle(h2, L, xs.copy(), h2.A[L] @ xs, "avs", 2, 0.25)
    assert np.abs(out - xs).max() <= 1e-12 * np.abs(xs).max()


@pytest.mark.parametrize("kind,steps,omega", [("avs", 2, 0.25), ("mvs", 1, 1.0)])
def test_preconditioner_symmetric(h2, kind, steps, omega):
    """Reading Q11: AVS cycle and the reversed-post-order MVS cycle are symmetric (CG-valid)."""
    n = h2.A[3].shape[0]
    r1, r2 = uniform(n, 11), uniform(n, 12)
    lhs = precondition(h2, r1, kind, steps, omega) @ r2
    rhs = r1 @ precondition(h2, r2, kind, steps, omega)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    assert precondition(h2, r1, kind, steps, omega) @ r1 > 0


@pytest.mark.parametrize("nratio,n,nu", [(1e-8, 10, 10.0), (1e-4, 2, 4.0), (1e-16, 8, 4.0)])
def test_fractional_iterations_arithmetic(nratio, n, nu):
    """SPEC.md:480-482 (reading Q7)."""
    hist = np.r_[1.0, np.ones(n - 1), nratio]
    assert abs(fractional_iterations(hist) - nu) < 1e-12


def test_cfg1_pcg_matches_direct(h2):
    """cfg1 (2D, Q2, 8x8): MG-PCG to 1e-8 equals the dense direct solve."""
    L = 3
    A = h2.A[L]
    b = paper_rhs(2, 2, level_cells(L), default_sigma(2))
    x, n, hist = pcg(A, b, lambda r: precondition(h2, r, "avs", 2, 0.25))
    xd = spla.spsolve(A.tocsc(), b)
    assert hist[-1] <= 1e-8 * hist[0]
    assert np.linalg.norm(x - xd) <= 1e-6 * np.linalg.norm(xd)
    assert np.linalg.norm(b - A @ x) <= 1.0001e-8 * np.linalg.norm(b)


@pytest.mark.parametrize("k", [2, 3, 4])
def test_mixed_precision_iterations(k):
    """PAPER.md:747 (goddeke2007: FP32 V-cycle inside FP64 CG reaches the FP64 accuracy with the same
    iteration count): the oracle's FP32 cycle (every table rounded, reading Q21) within 1 iteration."""
    L = 5
    h = Hierarchy(k, 2, L, default_sigma(k))
    b = paper_rhs(k, 2, level_cells(L), default_sigma(k))
    _, n64, _ = pcg(h.A[L], b, lambda r: precondition(h, r, "avs", 2, 0.25))
    h.set_dtype(np.float32)
    x32, n32, hist = pcg(h.A[L], b, lambda r: precondition(h, r, "avs", 2, 0.25))
    assert abs(n32 - n64) <= 1, (n32, n64)
    assert np.linalg.norm(b - h.A[L] @ x32) <= 1.01e-8 * np.linalg.norm(b)


def test_two_grid_h_independent():
    """Two-grid (exact coarse solve) iteration counts settle as h -> 0 (MG approximation +
    smoothing property); the full V-cycle ν is recorded in DESIGN.md against Tables 2-3."""
    from oracle.smoothers import smooth
    k = 2
    nus = []
    for L in (5, 6):
        h = Hierarchy(k, 2, L, default_sigma(k))
        A, P = h.A[L], h.P[L]
        lu = spla.splu(h.A[L - 1].tocsc())

        def tg(r):
            x = smooth(A, h.ps[L], np.zeros_like(r), r, "avs", 2, 0.25)
            x = x + P @ lu.solve(P.T @ (r - A @ x))
            return smooth(A, h.ps[L], x, r, "avs", 2, 0.25)
        b = paper_rhs(k, 2, level_cells(L), default_sigma(k))
        nus.append(fractional_iterations(pcg(A, b, tg)[2]))
    assert abs(nus[1] - nus[0]) < 1.5 and nus[1] < 20


# ------------------------------------------------------------------------------ GMRES
def test_gmres_matches_direct_solve_and_is_monotone():
    """Textbook properties: the solution of a small nonsymmetric system (np.linalg.solve), and the
    minimal-residual property -- the residual history never increases within a cycle."""
    from oracle.multigrid import gmres
    rng = np.random.default_rng(3)
    n = 40
    A = np.eye(n) * 4 + rng.standard_normal((n, n)) * 0.3
    b = rng.standard_normal(n)
    x, it, hist = gmres(A, b, lambda v: v, rtol=1e-12, max_iter=200, restart=60)
    assert np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-10 * np.linalg.norm(np.linalg.solve(A, b))
    assert np.all(np.diff(hist[:it + 1]) <= 1e-12 * hist[0])
    assert np.linalg.norm(b - A @ x) <= 1e-11 * np.linalg.norm(b)


def test_gmres_terminates_in_number_of_distinct_eigenvalues():
    """Krylov theory: for a diagonalisable A with m distinct eigenvalues GMRES (no restart) reaches
    the exact solution in at most m steps."""
    from oracle.multigrid import gmres
    rng = np.random.default_rng(4)
    Q, _ = np.linalg.qr(rng.standard_normal((30, 30)))
    lam = np.repeat([1.0, 2.5, 7.0, 11.0], [10, 8, 7, 5])
    A = Q @ np.diag(lam) @ Q.T
    b = rng.standard_normal(30)
    x, it, hist = gmres(A, b, lambda v: v, rtol=1e-13, max_iter=30, restart=30)
    assert it <= 4
    assert np.linalg.norm(b - A @ x) <= 1e-11 * np.linalg.norm(b)


def test_gmres_right_preconditioning_exact_inverse():
    """With M^{-1} = A^{-1} right-preconditioned GMRES converges in one step."""
    from oracle.multigrid import gmres
    rng = np.random.default_rng(5)
    A = np.eye(20) * 3 + rng.standard_normal((20, 20)) * 0.5
    Ai = np.linalg.inv(A)
    b = rng.standard_normal(20)
    x, it, hist = gmres(A, b, lambda v: Ai @ v, rtol=1e-12)
    assert it == 1
    assert np.allclose(x, np.linalg.solve(A, b), rtol=1e-10, atol=1e-12)


def test_gmres_with_nonsymmetric_mvs_cycle_solves_cfg1():
    """The paper's MVS protocol: GMRES around the same-order (nonsymmetric) MVS V-cycle
    on cfg1 reaches the direct solution; its iteration count is level-independent-ish and small."""
    from oracle.multigrid import gmres, Hierarchy, precondition
    h = Hierarchy(2, 2, 3, default_sigma(2))
    A = h.A[3]
    rng = np.random.default_rng(6)
    b = rng.standard_normal(A.shape[0])
    prec = lambda r: precondition(h, r, "mvs", 1, 1.0, symmetric=False)
    x, it, hist = gmres(A, b, prec, rtol=1e-10)
    xd = np.linalg.solve(A.toarray(), b)
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)
    assert it <= 15


# ------------------------------------------------------------------------------ the paper's iteration counts
# (d, k, L, smoother, steps, exact) -> (paper nu, allowed deviation).  PAPER.md Table 1 (exact local
# solvers) and Table 2 (FDM surrogate); the protocol and the
# readings (Q8b boundary data, Q27 boundary penalty, Q28 MVS damping) are DESIGN.md §2 / §2b.
PAPER_GATES = {
    "table2_avs2_k2_L7": ((2, 2, 7, "avs", 2, False), 19.2, 2.0),
    "table2_avs2_k4_L6": ((2, 4, 6, "avs", 2, False), 9.2, 1.0),
    "table2_mvs1_k4_L6": ((2, 4, 6, "mvs", 1, False), 4.2, 1.0),
    "table1_avs2_k4_L6": ((2, 4, 6, "avs", 2, True), 10.3, 1.0),
    "table1_mvs1_k4_L6": ((2, 4, 6, "mvs", 1, True), 2.9, 1.0),
    "table2_avs2_k4_L5": ((2, 4, 5, "avs", 2, False), None, None),   # level-uniformity partner
    # Table 3 (3D): the paper's 3D level L has 2^(L-1) cells per axis (reading Q9b),
    # i.e. the oracle's level L-1; omega 0.1 (AVS) / 0.7 (MVS)
    "table3_avs1_k2_L5": ((3, 2, 4, "avs", 1, False), 29.8, 2.0),
    "table3_mvs1_k2_L5": ((3, 2, 4, "mvs", 1, False), 9.1, 1.0),
}


def _gate_job(args):
    from oracle.multigrid import solve_paper
    n, nu, _ = solve_paper(*args)
    return nu


@pytest.fixture(scope="module")
def paper_nu():
    from concurrent.futures import ProcessPoolExecutor
    keys = list(PAPER_GATES)
    with ProcessPoolExecutor(min(8, len(keys))) as ex:
        vals = list(ex.map(_gate_job, [PAPER_GATES[k][0] for k in keys]))
    return dict(zip(keys, vals))


@pytest.mark.parametrize("name", [k for k, v in PAPER_GATES.items() if v[1] is not None])
def test_paper_iteration_counts(paper_nu, name):
    """The oracle's multigrid reproduces the paper's fractional iteration counts nu."""
    _, ref, tol = PAPER_GATES[name]
    assert abs(paper_nu[name] - ref) <= tol, (name, paper_nu[name], ref)


def test_paper_level_uniformity(paper_nu):
    """convergence uniform in the mesh level -- nu(L+1) - nu(L) <= 1 (k=4, L=5 -> 6)."""
    assert paper_nu["table2_avs2_k4_L6"] - paper_nu["table2_avs2_k4_L5"] <= 1.0
