"""Pins for the Poisson SIPG comparison workload of the oracle (Fig. 5)."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse.linalg as spla

from oracle.sipg import (assemble_sipg, sipg_matrices_1d, sipg_load, sipg_paper_load, sipg_dof_coords,
                         SipgPatchSolvers, sipg_embedding_1d, sipg_sigma)
from oracle.smoothers import avs_step
from c0ip_inputs import uniform


@pytest.mark.parametrize("d,k,N", [(2, 2, 3), (2, 3, 4), (2, 5, 2), (3, 2, 2), (3, 3, 2)])
def test_sipg_kronecker_rank2_spd(d, k, N):
    """The d-dimensional SIPG quadrature equals the rank-2 (rank-d) Kronecker sum of the 1D matrices
    (Eq. laplacianfdm: A = A_1 (x) M_2 + M_1 (x) A_2); symmetric positive definite."""
    A = assemble_sipg(k, d, N).toarray()
    M, L = sipg_matrices_1d(k, N)
    if d == 2:
        K = np.kron(M, L) + np.kron(L, M)
    else:
        K = np.kron(np.kron(M, M), L) + np.kron(np.kron(M, L), M) + np.kron(np.kron(L, M), M)
    assert np.abs(A - K).max() <= 1e-12 * np.abs(A).max()
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0


def test_sipg_small_penalty_not_coercive():
    """SIPG needs sigma large enough: 1% of the reading-Q30 penalty gives an indefinite matrix."""
    k, N = 3, 4
    M, L = sipg_matrices_1d(k, N, sigma=0.01 * sipg_sigma(k))
    assert np.linalg.eigvalsh(L).min() < 0


@pytest.mark.parametrize("k", [2, 3])
def test_sipg_manufactured_solution(k):
    """-Delta u = d pi^2 prod sin: the DG solution converges to prod sin(pi x_a) at nodal rate >= k + 1."""
    errs = []
    for N in (4, 8, 16):
        u = spla.spsolve(assemble_sipg(k, 2, N).tocsc(), sipg_load(k, 2, N, sipg_paper_load(2)))
        x = sipg_dof_coords(k, N)
        X, Y = np.meshgrid(x, x)
        errs.append(np.abs(u - (np.sin(np.pi * X) * np.sin(np.pi * Y)).ravel()).max())
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates >= k + 1 - 0.3), rates


def test_sipg_patch_solve_is_fdm_exact():
    """the SIPG patch matrix is exactly L_v (x) M_v + M_v (x) L_v, so the fast diagonalisation
    (LAPACK generalized eigenvectors) reproduces the dense patch inverse -- the FDM of f3 is exact."""
    k, N = 3, 5
    A = assemble_sipg(k, 2, N)
    ps = SipgPatchSolvers(k, 2, N, A)
    M, L = sipg_matrices_1d(k, N)
    v = (2, 3)
    pid = (v[1] - 1) * (N - 1) + (v[0] - 1)
    rr = [np.arange((va - 1) * (k + 1), (va + 1) * (k + 1)) for va in v]
    Sx = [sla.eigh(L[np.ix_(r, r)], M[np.ix_(r, r)]) for r in rr]
    r = uniform((2 * k + 2) ** 2, 3)
    T = r.reshape(2 * k + 2, 2 * k + 2)                     # [y][x]
    T = Sx[1][1].T @ T @ Sx[0][1]
    T = T / (Sx[1][0][:, None] + Sx[0][0][None, :])
    T = Sx[1][1] @ T @ Sx[0][1].T
    u = ps.solve(np.array([pid]), r[None, :])[0]
    assert np.linalg.norm(u - T.ravel()) <= 1e-10 * np.linalg.norm(u)


def test_sipg_embedding_reproduces_cellwise_polynomials():
    """DG embedding: a piecewise polynomial of degree k on the coarse cells is reproduced on the fine cells."""
    k, Nc = 3, 3
    E = sipg_embedding_1d(k, Nc)
    xc, xf = sipg_dof_coords(k, Nc), sipg_dof_coords(k, 2 * Nc)
    cc = np.repeat(np.arange(Nc), k + 1)
    cf = np.repeat(np.arange(2 * Nc), k + 1) // 2
    p = lambda x, c: (x + 0.2 * c) ** k - c
    assert np.abs(E @ p(xc, cc) - p(xf, cf)).max() < 1e-12


def test_sipg_avs_one_patch_is_exact_solve():
    """N = 2 (one patch holding every DoF): one AVS step with omega = 1 from x is the direct solve."""
    k = 2
    A = assemble_sipg(k, 2, 2)
    ps = SipgPatchSolvers(k, 2, 2, A)
    b = uniform(A.shape[0], 4)
    x = uniform(A.shape[0], 5)
    assert np.linalg.norm(avs_step(A, ps, x, b, 1.0) - spla.spsolve(A.tocsc(), b)) <= 1e-10 * np.linalg.norm(b)
