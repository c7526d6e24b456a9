"""Pins for the oracle's basis and 1D matrices."""
import numpy as np
import pytest
import sympy as sy

from oracle.basis import gauss_lobatto_points, Basis1D, gauss_legendre
from oracle.discretization import (global_matrices_1d, element_matrices_1d, default_sigma,
                                   patch_range_1d)
from golden_io import read_matrices


def test_gauss_lobatto_k2_k3():
    # k=2: {0, 1/2, 1}; k=3: 0, (1 -+ 1/sqrt5)/2, 1 (roots of P_3')
    assert np.allclose(gauss_lobatto_points(2), [0, 0.5, 1], atol=1e-15)
    s = 1 / np.sqrt(5)
    assert np.allclose(gauss_lobatto_points(3), [0, (1 - s) / 2, (1 + s) / 2, 1], atol=1e-15)


@pytest.mark.parametrize("k", range(2, 8))
def test_lagrange_partition_of_unity_and_kronecker(k):
    b = Basis1D(k)
    assert np.allclose(b.eval(b.points), np.eye(k + 1), atol=1e-12)
    t = np.linspace(0, 1, 17)
    assert np.allclose(b.eval(t).sum(0), 1.0, atol=1e-13)
    assert np.allclose(b.eval(t, 1).sum(0), 0.0, atol=1e-10)


@pytest.mark.parametrize("nq", range(1, 9))
def test_gauss_rule_exactness(nq):
    t, w = gauss_legendre(nq)
    for p in range(2 * nq):
        assert abs((w * t ** p).sum() - 1.0 / (p + 1)) < 1e-14


def _exact_1d(k, N, sigma, bfac=2):
    """Independent exact construction with sympy (symbolic integration, GL nodes in radicals).
    bfac: boundary-facet penalty factor (reading Q27: 2; 1)."""
    t = sy.symbols("t")
    nodes = [sy.Integer(0)] + sorted(sy.solve(sy.diff(sy.legendre(k, 2 * t - 1), t), t),
                                     key=lambda e: float(e)) + [sy.Integer(1)]
    ell = []
    for i, ti in enumerate(nodes):
        p = sy.Integer(1)
        for j, tj in enumerate(nodes):
            if j != i:
                p = p * (t - tj) / (ti - tj)
        ell.append(sy.expand(p))
    h = sy.Rational(1, N)
    nn = k * N + 1
    Mf = sy.zeros(nn, nn); Lf = sy.zeros(nn, nn); Bf = sy.zeros(nn, nn)
    for c in range(N):
        for m in range(k + 1):
            for q in range(k + 1):
                gm, gq = c * k + m, c * k + q
                Mf[gm, gq] += h * sy.integrate(ell[m] * ell[q], (t, 0, 1))
                Lf[gm, gq] += sy.integrate(sy.diff(ell[m], t) * sy.diff(ell[q], t), (t, 0, 1)) / h
                Bf[gm, gq] += sy.integrate(sy.diff(ell[m], t, 2) * sy.diff(ell[q], t, 2), (t, 0, 1)) / h ** 3
    d1 = lambda m, x: sy.diff(ell[m], t).subs(t, x) / h
    d2 = lambda m, x: sy.diff(ell[m], t, 2).subs(t, x) / h ** 2
    for f in range(N + 1):
        a = {}; b = {}
        if f > 0:   # left cell, t=1, outward +e
            for m in range(k + 1):
                g = (f - 1) * k + m
                a[g] = a.get(g, 0) + d1(m, 1)
                b[g] = b.get(g, 0) + (d2(m, 1) if f == N else d2(m, 1) / 2)
        if f < N:   # right cell, t=0, outward -e
            for m in range(k + 1):
                g = f * k + m
                a[g] = a.get(g, 0) - d1(m, 0)
                b[g] = b.get(g, 0) + (d2(m, 0) if f == 0 else d2(m, 0) / 2)
        sf = sigma * (bfac if f in (0, N) else 1)
        for i in a:
            for j in a:
                Bf[i, j] += sf / h * a[i] * a[j] - a[i] * b[j] - b[i] * a[j]
    sl = slice(1, nn - 1)
    return [np.array(X[sl, sl].evalf(30).tolist(), dtype=float) for X in (Mf, Lf, Bf)]


def test_golden_k2_N2_appendix_A():
    """SURVEY.md Appendix A (boundary penalty = interior penalty, bfac=1)."""
    g = read_matrices("k2_N2_sigma6_1d.txt")
    M, L, B = (X.toarray() for X in global_matrices_1d(2, 2, 6.0, bfac=1.0))
    assert np.allclose(M, g["M"], rtol=0, atol=1e-13)
    assert np.allclose(L, g["L"], rtol=0, atol=1e-12)
    assert np.allclose(B, g["B"], rtol=1e-14, atol=1e-10)
    assert np.allclose(np.linalg.eigvalsh(B), [137.2648, 768.0, 3222.7352], atol=1e-4)


def test_golden_k2_N2_boundary_penalty_2():
    """tests/golden/k2_N2_sigma6_bfac2_1d.txt (exact rationals by tests/golden/make_bfac2.py, sympy
    only): reading Q27 adds (sigma/h) a a^T once more on each boundary facet."""
    g = read_matrices("k2_N2_sigma6_bfac2_1d.txt")
    M, L, B = (X.toarray() for X in global_matrices_1d(2, 2, 6.0))
    assert np.allclose(M, g["M"], rtol=0, atol=1e-13)
    assert np.allclose(B, g["B"], rtol=1e-14, atol=1e-10)


def test_cell_mass_spec_example():
    # Q2 cell mass (h/30)[[4,2,-1],[2,16,2],[-1,2,4]]
    h = 0.37
    Mc, _, _ = element_matrices_1d(2, h)
    assert np.allclose(Mc, h / 30 * np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]), atol=1e-15)


@pytest.mark.parametrize("k,N", [(2, 2), (2, 3), (3, 2), (3, 4)])
def test_sympy_exact_matrices(k, N):
    sigma = default_sigma(k)
    Me, Le, Be = _exact_1d(k, N, sigma)
    M, L, B = (X.toarray() for X in global_matrices_1d(k, N, sigma))
    assert np.allclose(M, Me, rtol=0, atol=1e-14 * np.abs(Me).max())
    assert np.allclose(L, Le, rtol=0, atol=1e-13 * np.abs(Le).max())
    assert np.allclose(B, Be, rtol=0, atol=1e-12 * np.abs(Be).max())


@pytest.mark.parametrize("k", range(2, 8))
def test_invariants(k):
    N = 5
    s = default_sigma(k)
    Mf, Lf, Bf = (X.toarray() for X in global_matrices_1d(k, N, s, eliminate=False))
    assert np.abs(Lf.sum(1)).max() < 1e-9 * np.abs(Lf).max()
    for X in (Mf, Lf, Bf):
        assert np.abs(X - X.T).max() <= 1e-13 * np.abs(X).max()
    # quadrature-order invariance
    M2, L2, B2 = (X.toarray() for X in global_matrices_1d(k, N, s, nq=k + 5))
    M1, L1, B1 = (X.toarray() for X in global_matrices_1d(k, N, s))
    assert np.abs(B2 - B1).max() <= 1e-12 * np.abs(B1).max()
    assert np.abs(M2 - M1).max() <= 1e-12 * np.abs(M1).max()


@pytest.mark.parametrize("k", range(2, 8))
def test_coercivity_default_sigma(k):
    """Coercivity (reading Q4): B SPD for sigma=k(k+1), N=2..16; fails for 0.01x."""
    for N in (2, 3, 4, 8, 16):
        B = global_matrices_1d(k, N, default_sigma(k))[2].toarray()
        assert np.linalg.eigvalsh(B).min() > 0
    B = global_matrices_1d(k, 8, 0.01 * default_sigma(k))[2].toarray()
    assert np.linalg.eigvalsh(B).min() < 0


@pytest.mark.parametrize("k", [2, 4, 7])
def test_translation_invariance_patch_blocks(k):
    """three distinct (M,L,B) patch blocks per level: left, interior, right."""
    N = 8
    mats = global_matrices_1d(k, N, default_sigma(k))
    blocks = [[X[np.ix_(patch_range_1d(k, v), patch_range_1d(k, v))].toarray() for X in mats]
              for v in range(1, N)]
    for v in range(2, N - 2):
        for a, b in zip(blocks[1], blocks[v - 1]):
            assert np.array_equal(a, b) or np.abs(a - b).max() < 1e-12 * np.abs(a).max()
    assert np.abs(blocks[0][2] - blocks[1][2]).max() > 1e-3 * np.abs(blocks[1][2]).max()
    # left/right mirror symmetry
    J = np.eye(2 * k - 1)[::-1]
    assert np.abs(J @ blocks[0][2] @ J - blocks[-1][2]).max() < 1e-12 * np.abs(blocks[-1][2]).max()
