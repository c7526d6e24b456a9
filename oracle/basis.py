"""Q_k Lagrange basis on the reference interval [0,1] and Gauss quadrature.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:66 (Sec. 2, Eq. fespace) fixes tensor-product Lagrange elements of degree k
but not their support points; reading Q18 takes Gauss-Lobatto points,
the deal.II FE_Q default.  Quadrature is Gauss-Legendre.
"""
import numpy as np
from numpy.polynomial import Polynomial, Legendre
from numpy.polynomial import legendre as npleg


def gauss_lobatto_points(k):
    """k+1 Gauss-Lobatto points on [0,1]: 0, 1 and the roots of P_k'(2t-1)."""
    if k < 1:
        raise ValueError("degree must be >= 1")
    inner = Legendre.basis(k).deriv().roots() if k >= 2 else np.array([])
    pts = np.concatenate(([-1.0], np.sort(np.real(inner)), [1.0]))
    return 0.5 * (pts + 1.0)


def lagrange_polynomials(points):
    """Lagrange polynomials l_i(t) = prod_{j!=i} (t - t_j)/(t_i - t_j) as numpy Polynomials."""
    polys = []
    for i, ti in enumerate(points):
        p = Polynomial([1.0])
        for j, tj in enumerate(points):
            if j != i:
                p = p * Polynomial([-tj, 1.0]) / (ti - tj)
        polys.append(p)
    return polys


def gauss_legendre(nq):
    """nq-point Gauss-Legendre rule on [0,1] (exact for degree 2*nq-1)."""
    x, w = npleg.leggauss(nq)
    return 0.5 * (x + 1.0), 0.5 * w


class Basis1D:
    """Reference basis: values and first/second derivatives of l_0..l_k (w.r.t. t in [0,1])."""

    def __init__(self, k):
        self.k = k
        self.points = gauss_lobatto_points(k)
        self.polys = lagrange_polynomials(self.points)
        self.d1 = [p.deriv(1) for p in self.polys]
        self.d2 = [p.deriv(2) for p in self.polys]

    def eval(self, t, der=0):
        """Array [k+1, len(t)] of l_m^{(der)}(t)."""
        t = np.atleast_1d(np.asarray(t, dtype=np.float64))
        src = (self.polys, self.d1, self.d2)[der] if der <= 2 else [p.deriv(der) for p in self.polys]
        return np.array([p(t) for p in src])
