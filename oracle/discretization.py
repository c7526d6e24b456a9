"""1D matrices M, L, B of the C0IP discretisation (Eq. matrix1d).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

On N uniform cells of [0,1] (h = 1/N) with the Q_k Lagrange basis (support points per
reading Q18), global nodes j = 0..kN.  Following PAPER.md:323-332 and Eqs. bulk1/bulk3,
ev, eh:

  M_ij = int phi_j phi_i,   L_ij = int phi_j' phi_i',
  B_ij = sum_cells int phi_j'' phi_i''
       + sum_faces [ (sigma/h_f) a_i a_j - b_j a_i - a_j b_i ]

with a = [phi'] the jump of the derivative (sum of outward normal derivatives,
PAPER.md:87-97) and b = {phi''} the mean of the second derivative; on the two boundary
facets the one-sided definitions of PAPER.md:100-106 (reading Q26): a = d_n phi,
b = d_n^2 phi.  h_f = harmonic mean of the adjacent cell widths, i.e. h on an
interior facet.  On a boundary facet the harmonic-mean rule names a single cell; reading Q27
 takes h_f = h/2 there, i.e. the boundary (Nitsche) penalty is BOUNDARY_PENALTY x
the interior one (the variant that reproduces PAPER.md Tables 1-2).
sigma is an input (reading Q4: default k(k+1)).  Rows/columns of nodes 0 and kN are
eliminated (u = 0 strongly, reading Q26).
"""
import numpy as np
import scipy.sparse as sp

from .basis import Basis1D, gauss_legendre


BOUNDARY_PENALTY = 2.0   # reading Q27: sigma/h_f on boundary facets with h_f = h/2


def default_sigma(k, penalty_scale=1.0):
    """Reading Q4: sigma = penalty_scale * k (k+1)."""
    return penalty_scale * k * (k + 1)


def element_matrices_1d(k, h, nq=None):
    """Cell matrices (k+1)x(k+1) on a cell of width h by Gauss quadrature (nq >= k+1 exact)."""
    bas = Basis1D(k)
    nq = nq or (k + 2)
    t, w = gauss_legendre(nq)
    v, d1, d2 = bas.eval(t, 0), bas.eval(t, 1) / h, bas.eval(t, 2) / h ** 2
    Mc = (v * w) @ v.T * h
    Lc = (d1 * w) @ d1.T * h
    Bc = (d2 * w) @ d2.T * h
    return Mc, Lc, Bc


def face_vectors_1d(k, h):
    """Jump/mean vectors of the reference basis at a face.

    Returns dict with
      'interior': (a, b) of length 2k+1 on nodes of [left cell | right cell] (shared vertex once)
      'lower'   : (a, b) of length k+1 on the nodes of the first cell (face at x=0, n = -e)
      'upper'   : (a, b) of length k+1 on the nodes of the last cell  (face at x=1, n = +e)
    """
    bas = Basis1D(k)
    d1_0, d1_1 = bas.eval(0.0, 1)[:, 0] / h, bas.eval(1.0, 1)[:, 0] / h
    d2_0, d2_1 = bas.eval(0.0, 2)[:, 0] / h ** 2, bas.eval(1.0, 2)[:, 0] / h ** 2
    a = np.zeros(2 * k + 1)
    b = np.zeros(2 * k + 1)
    # left cell K^- (outward normal +e): its local node m sits at global offset m
    a[: k + 1] += d1_1
    b[: k + 1] += 0.5 * d2_1
    # right cell K^+ (outward normal -e): d_{n+} v = -v'(x_f^+), d^2_{n+} v = v''
    a[k:] += -d1_0
    b[k:] += 0.5 * d2_0
    return {
        "interior": (a, b),
        "lower": (-d1_0, d2_0.copy()),
        "upper": (d1_1.copy(), d2_1.copy()),
    }


def global_matrices_1d(k, N, sigma, eliminate=True, nq=None, bfac=BOUNDARY_PENALTY, nodes=None):
    """Global 1D M, L, B (scipy CSR).  Size (kN+1)^2, or (kN-1)^2 after elimination.

    bfac: boundary-facet penalty factor (reading Q27; bfac=1 is SURVEY.md Appendix A).
    nodes: optional cell boundaries x_0 = 0 < x_1 < ... < x_N = 1 of a graded mesh (PAPER.md:73,
    131): cell c has width h_c = x_{c+1} - x_c, the interior facet between cells c-1 and c uses the harmonic mean
    h_f = 2 h_{c-1} h_c / (h_{c-1} + h_c) of the adjacent widths, a boundary facet h_f = h_c / bfac
    (reading Q27).  Default: uniform, h = 1/N."""
    hs = np.full(N, 1.0 / N) if nodes is None else np.diff(np.asarray(nodes, dtype=np.float64))
    assert len(hs) == N and np.all(hs > 0)
    nn = k * N + 1
    rows, cols, vm, vl, vb = [], [], [], [], []
    loc = np.arange(k + 1)
    for c in range(N):
        Mc, Lc, Bc = element_matrices_1d(k, hs[c], nq)
        g = c * k + loc
        rr, cc = np.meshgrid(g, g, indexing="ij")
        rows.append(rr.ravel()); cols.append(cc.ravel())
        vm.append(Mc.ravel()); vl.append(Lc.ravel()); vb.append(Bc.ravel())
    zeros = lambda n: np.zeros(n)
    for f in range(N + 1):
        if f == 0:
            a, b = face_vectors_1d(k, hs[0])["lower"]; g = loc; h_f = hs[0] / bfac
        elif f == N:
            a, b = face_vectors_1d(k, hs[N - 1])["upper"]; g = (N - 1) * k + loc; h_f = hs[N - 1] / bfac
        else:
            fl, fr = face_vectors_1d(k, hs[f - 1]), face_vectors_1d(k, hs[f])
            # jump / mean across the facet with the two cells' own scalings
            a = np.zeros(2 * k + 1); b = np.zeros(2 * k + 1)
            a[: k + 1] += fl["upper"][0]; b[: k + 1] += 0.5 * fl["upper"][1]
            a[k:] += fr["lower"][0]; b[k:] += 0.5 * fr["lower"][1]
            g = (f - 1) * k + np.arange(2 * k + 1)
            h_f = 2.0 * hs[f - 1] * hs[f] / (hs[f - 1] + hs[f])
        F = (sigma / h_f) * np.outer(a, a) - np.outer(a, b) - np.outer(b, a)
        rr, cc = np.meshgrid(g, g, indexing="ij")
        rows.append(rr.ravel()); cols.append(cc.ravel())
        vm.append(zeros(F.size)); vl.append(zeros(F.size)); vb.append(F.ravel())
    rows = np.concatenate(rows); cols = np.concatenate(cols)
    mk = lambda v: sp.csr_matrix((np.concatenate(v), (rows, cols)), shape=(nn, nn))
    M, L, B = mk(vm), mk(vl), mk(vb)
    if eliminate:
        keep = np.arange(1, nn - 1)
        M, L, B = (X[keep][:, keep].tocsr() for X in (M, L, B))
    return M, L, B


def graded_nodes(N, beta=0.0):
    """Cell boundaries of a graded 1D mesh on [0,1]: x_c = phi(c/N), phi(t) = t + beta t (1 - t) (|beta| < 1,
    monotone); nested: the boundaries of the N/2-cell mesh are every second one."""
    t = np.arange(N + 1) / N
    return t + beta * t * (1.0 - t)


def patch_range_1d(k, v):
    """0-based interior indices of the 1D patch of vertex v (1..N-1): [(v-1)k, (v+1)k-2]."""
    return np.arange((v - 1) * k, (v + 1) * k - 1)


def patch_variant(v, N):
    """Axis variant: 'both' if N==2, 'left' v=1, 'right' v=N-1, else 'interior'."""
    if N == 2:
        return "both"
    if v == 1:
        return "left"
    if v == N - 1:
        return "right"
    return "interior"
