"""Pins for the oracle's assembled C0IP operator."""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse.linalg as spla
from numpy.polynomial import Polynomial as Pn

from oracle.operator import (assemble, rhs_load, residual_on_box, dof_coords, energy_error,
                             paper_load)
from oracle.discretization import global_matrices_1d, default_sigma
from c0ip_inputs import random_xb


def _kron_sum(k, d, N, s):
    M, L, B = (X.toarray() for X in global_matrices_1d(k, N, s))
    K = np.kron
    if d == 2:
        return K(M, B) + 2 * K(L, L) + K(B, M)
    return (K(K(M, M), B) + K(K(M, B), M) + K(K(B, M), M)
            + 2 * (K(K(M, L), L) + K(K(L, L), M) + K(K(L, M), L)))


@pytest.mark.parametrize("d,k,N", [(2, k, N) for k in (2, 3, 4, 5) for N in (2, 3, 4, 8) if (k * N) <= 24]
                         + [(3, k, N) for k in (2, 3) for N in (2, 3, 4) if k * N <= 9])
def test_kronecker_identity(d, k, N):
    """Independent d-dim quadrature == Kronecker sum of Eq. c0iptensorvp(3D)."""
    s = default_sigma(k)
    A = assemble(k, d, N, s).toarray()
    K = _kron_sum(k, d, N, s)
    assert np.abs(A - K).max() <= 1e-12 * np.abs(K).max()


@pytest.mark.parametrize("d,k,N", [(2, 2, 4), (2, 5, 4), (3, 2, 3), (3, 3, 2)])
def test_symmetric_positive_definite(d, k, N):
    """Coercivity: A symmetric, Cholesky succeeds, no null vector."""
    A = assemble(k, d, N, default_sigma(k)).toarray()
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    sla.cholesky(A)
    x = np.zeros(A.shape[0])
    assert np.all(A @ x == 0)


_p = Pn([0, 0, 1]) * Pn([1, -1]) ** 2          # x^2 (1-x)^2  in H^2_0(0,1)


@pytest.mark.parametrize("k,N", [(4, 4), (4, 8), (5, 4), (6, 2)])
def test_polynomial_exactness(k, N):
    """Consistency: u = p(x)p(y) in Q_4 cap H^2_0 is reproduced exactly for k>=4.

    A wrong sign or a dropped consistency / adjoint-consistency / boundary term breaks this.
    """
    A = assemble(k, 2, N, default_sigma(k))
    p2, p4 = _p.deriv(2), _p.deriv(4)
    f = lambda x, y: p4(x) * _p(y) + 2 * p2(x) * p2(y) + _p(x) * p4(y)       # Delta^2 u
    u = spla.spsolve(A.tocsc(), rhs_load(k, 2, N, f))
    xs = dof_coords(k, N, np.arange(k * N - 1))
    ui = np.outer(_p(xs), _p(xs)).ravel()
    assert np.abs(u - ui).max() <= 1e-9 * np.abs(ui).max()


def test_polynomial_exactness_3d():
    k, N = 4, 2
    A = assemble(k, 3, N, default_sigma(k))
    p2, p4 = _p.deriv(2), _p.deriv(4)
    f = lambda x, y, z: (p4(x) * _p(y) * _p(z) + _p(x) * p4(y) * _p(z) + _p(x) * _p(y) * p4(z)
                         + 2 * (p2(x) * p2(y) * _p(z) + _p(x) * p2(y) * p2(z) + p2(x) * _p(y) * p2(z)))
    u = spla.spsolve(A.tocsc(), rhs_load(k, 3, N, f))
    xs = dof_coords(k, N, np.arange(k * N - 1))
    ui = np.einsum("i,j,k->ijk", _p(xs), _p(xs), _p(xs)).ravel()
    assert np.abs(u - ui).max() <= 1e-9 * np.abs(ui).max()


@pytest.mark.parametrize("k", [2, 3])
def test_energy_error_rate(k):
    """Eq. energyerror: |u-u_h|_h = O(h^{k-1}); u = sin^2(pi x) sin^2(pi y)."""
    pi = np.pi
    s2 = lambda x: np.sin(pi * x) ** 2
    ds2 = lambda x: pi * np.sin(2 * pi * x)
    dds2 = lambda x: 2 * pi ** 2 * np.cos(2 * pi * x)
    d4s2 = lambda x: -8 * pi ** 4 * np.cos(2 * pi * x)
    f = lambda x, y: d4s2(x) * s2(y) + 2 * dds2(x) * dds2(y) + s2(x) * d4s2(y)

    def hess(x, y):
        H = np.empty(x.shape + (2, 2))
        H[..., 0, 0] = dds2(x) * s2(y); H[..., 1, 1] = s2(x) * dds2(y)
        H[..., 0, 1] = H[..., 1, 0] = ds2(x) * ds2(y)
        return H
    errs = []
    for N in (8, 16, 32):
        s = default_sigma(k)
        u = spla.spsolve(assemble(k, 2, N, s).tocsc(), rhs_load(k, 2, N, f))
        errs.append(energy_error(k, 2, N, s, u, hess))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(rates >= k - 1 - 0.15)


@pytest.mark.parametrize("d,k,Ns", [(2, 3, (4, 8, 16)), (2, 4, (4, 8, 16)), (3, 2, (2, 4, 8))])
def test_paper_rhs_solution_is_prod_sin(d, k, Ns):
    """the experiments' F yields the analytical solution u* = prod sin(pi x_a).  u* is not
    clamped (d_n u* != 0), so F carries the Nitsche boundary data (reading Q8b); with it the discrete
    solution converges to u* (nodal max error at rate >= k, one order above the energy rate k-1 of
    Eq. energyerror) -- a sign or factor error in the boundary data stops it."""
    from oracle.operator import paper_rhs, paper_solution
    nod = []
    for N in Ns:
        s = default_sigma(k)
        u = spla.spsolve(assemble(k, d, N, s).tocsc(), paper_rhs(k, d, N, s))
        from oracle.operator import dof_coords
        xs = np.meshgrid(*[dof_coords(k, N, np.arange(k * N - 1))] * d, indexing="ij")[::-1]
        nod.append(np.abs(u - paper_solution(d)(*[x.ravel() for x in xs])).max())
    rates = np.log2(np.array(nod[:-1]) / np.array(nod[1:]))
    assert np.all(rates >= k - 0.3), rates          # nodal error: at least the energy rate + 1


def test_rhs_partition_of_unity():
    k, N = 3, 4
    b = rhs_load(k, 2, N, lambda x, y: 0 * x + 2.5)
    # sum over interior basis functions misses the boundary nodes; add them back via full sum
    # check instead: f = const times bubble-free interior => sum b <= 2.5 and b symmetric
    assert b.sum() < 2.5 and np.allclose(b.reshape(11, 11), b.reshape(11, 11).T)
    assert np.all(rhs_load(k, 2, N, lambda x, y: 0 * x) == 0)


def test_paper_load_quadrature_converged():
    """doubling the order changes b by < 1e-10 relative (k+3 points default)."""
    k, N = 3, 8
    b1 = rhs_load(k, 2, N, paper_load(2))
    b2 = rhs_load(k, 2, N, paper_load(2), nq=2 * (k + 3))
    assert np.abs(b1 - b2).max() <= 1e-10 * np.abs(b2).max()


@pytest.mark.parametrize("d,k,N", [(2, 3, 6), (3, 2, 4)])
def test_window_rows_equal_global(d, k, N):
    """Window assembly (used for sampled parity at full size) == global CSR rows."""
    s = default_sigma(k)
    A = assemble(k, d, N, s)
    x, b = random_xb(k, d, N)
    r = b - A @ x
    n = k * N - 1
    for lo, hi in [((0,) * d, (k + 1,) * d), ((k - 1,) * d, (3 * k,) * d), ((n - 2 * k,) * d, (n,) * d)]:
        rb, ids = residual_on_box(k, d, N, s, x, b, np.array(lo), np.array(hi))
        assert np.abs(rb - r[ids]).max() <= 1e-12 * np.abs(r).max()
