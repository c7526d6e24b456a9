"""Pins for maps, colours, surrogate solves and smoothers."""
import itertools

import numpy as np
import pytest
import scipy.linalg as sla

from oracle.mesh import (patch_vertices, patch_dofs, all_patch_dofs, color_patches, color_of,
                         n_colors)
from oracle.operator import assemble
from oracle.discretization import global_matrices_1d, default_sigma, patch_range_1d
from oracle.smoothers import PatchSolvers, avs_step, mvs_step, avs_delta_sample
from c0ip_inputs import random_xb


# ---------------------------------------------------------------- maps
def test_counts_spec_examples():
    assert (2 * 4 - 1) ** 2 == 49
    assert len(patch_vertices(2, 2)) == 1
    assert len(patch_vertices(3, 4)) == 27
    assert len(patch_vertices(3, 8)) == 343
    assert [tuple(v) for v in patch_vertices(2, 4)] == [(x, y) for y in (1, 2, 3) for x in (1, 2, 3)]
    assert np.array_equal(patch_dofs(2, 2, 2, (1, 1)), np.arange(9))
    assert len(patch_dofs(3, 2, 8, (2, 3))) == 25 and len(patch_dofs(2, 3, 4, (1, 2, 3))) == 27


def test_colour_split_spec_example():
    """class (1,1) on the 3x3 vertex grid splits {(1,1),(3,3)} | {(1,3),(3,1)}."""
    verts = patch_vertices(2, 4)
    cls = color_patches(2, 4)
    sets = [set(tuple(verts[i]) for i in c) for c in cls]
    assert {(1, 1), (3, 3)} in sets and {(1, 3), (3, 1)} in sets


def test_cfg1_colour_sizes():
    """2D N=8 colour sizes [5,4,6,6,6,6,8,8]; N=2: only colour 6 (2D) / 14 (3D)."""
    assert [len(c) for c in color_patches(2, 8)] == [5, 4, 6, 6, 6, 6, 8, 8]
    assert [len(c) for c in color_patches(2, 2)] == [0] * 6 + [1, 0]
    assert [len(c) for c in color_patches(3, 2)] == [0] * 14 + [1, 0]
    assert n_colors(2) == 8 and n_colors(3) == 16


@pytest.mark.parametrize("d,k,N", [(2, 2, 9), (2, 3, 6), (3, 2, 6)])
def test_colour_partition_and_independence(d, k, N):
    """Partition + A-orthogonality of same-colour patches (brute force on the assembled A):
    patches of one colour share no DoF and A couples none of their DoFs."""
    cols = color_patches(d, N)
    allp = np.sort(np.concatenate(cols))
    assert np.array_equal(allp, np.arange((N - 1) ** d))
    A = assemble(k, d, N, default_sigma(k)).tocsr()
    dofs = all_patch_dofs(k, d, N)
    for c in cols:
        for p, q in itertools.combinations(c, 2):
            assert not set(dofs[p]) & set(dofs[q])
            assert abs(A[dofs[p]][:, dofs[q]]).max() == 0.0


def test_patch_map_is_tensor_of_1d_ranges():
    k, N = 3, 5
    n = k * N - 1
    for v in patch_vertices(2, N):
        g = patch_dofs(k, 2, N, v)
        rx, ry = patch_range_1d(k, v[0]), patch_range_1d(k, v[1])
        assert np.array_equal(g, (ry[:, None] * n + rx[None, :]).ravel())


# ---------------------------------------------------------------- surrogate (F4, F5)
@pytest.mark.parametrize("d,k", [(2, 2), (2, 4), (2, 7), (3, 2), (3, 4)])
def test_surrogate_equals_fdm(d, k):
    """Dense Cholesky surrogate solve == FDM (Eq. inverse) via LAPACK dsygv."""
    N = 6
    s = default_sigma(k)
    ps = PatchSolvers(k, d, N, s)
    M, L, B = (X.toarray() for X in global_matrices_1d(k, N, s))
    rng = np.random.default_rng(3)
    for key, (ids, fac, At) in ps.groups.items():
        v = ps.verts[ids[0]]
        S, lam = [], []
        for a in range(d):
            rr = patch_range_1d(k, v[a])
            w, Q = sla.eigh(B[np.ix_(rr, rr)], M[np.ix_(rr, rr)])
            S.append(Q); lam.append(w)
        r = rng.standard_normal((2 * k - 1) ** d)
        # FDM: (S_z x S_y x S_x) diag(1/sum lam) (..)^T r  (x fastest)
        T = r.reshape([2 * k - 1] * d)
        for a in range(d):
            T = np.moveaxis(np.tensordot(S[a].T, np.moveaxis(T, d - 1 - a, 0), 1), 0, d - 1 - a)
        D = sum(np.meshgrid(*[lam[a] for a in range(d)][::-1], indexing="ij"))
        T = T / D
        for a in range(d):
            T = np.moveaxis(np.tensordot(S[a], np.moveaxis(T, d - 1 - a, 0), 1), 0, d - 1 - a)
        u = ps.solve(np.array([ids[0]]), r[None, :])[0]
        assert np.linalg.norm(u - T.ravel()) <= 1e-11 * np.linalg.norm(u)


@pytest.mark.parametrize("d,k", [(2, 2), (2, 5), (3, 3)])
def test_surrogate_spectral_bounds(d, k):
    """spec(A~_v^{-1} A_v) in [1, d] (dropping the PSD 2L(x)L terms)."""
    N = 6
    s = default_sigma(k)
    A = assemble(k, d, N, s)
    ps = PatchSolvers(k, d, N, s)
    for key, (ids, fac, At) in ps.groups.items():
        g = ps.dofs[ids[0]]
        Av = A[g][:, g].toarray()
        w = sla.eigh(Av, At, eigvals_only=True)
        assert w.min() >= 1 - 1e-9 and w.max() <= d + 1e-9


# ---------------------------------------------------------------- smoothers (C7)
def _setup(d, k, N):
    s = default_sigma(k)
    A = assemble(k, d, N, s)
    ps = PatchSolvers(k, d, N, s)
    x, b = random_xb(k, d, N)
    return A, ps, x, b, s


@pytest.mark.parametrize("kind", ["avs", "mvs"])
def test_fixed_point(kind):
    A, ps, x, b, s = _setup(2, 3, 6)
    b = A @ x
    xn = avs_step(A, ps, x, b, 0.25) if kind == "avs" else mvs_step(A, ps, x, b, 1.0)
    assert np.abs(xn - x).max() <= 1e-12 * np.abs(x).max()


@pytest.mark.parametrize("d,k", [(2, 2), (2, 5), (3, 2)])
def test_one_patch_brute_force(d, k):
    """N=2 (one patch, R_v = I): AVS = x + w A~^{-1}(b - Ax); exact local solver, w=1 -> A^{-1} b."""
    N = 2
    A, ps, x, b, s = _setup(d, k, N)
    M, L, B = (X.toarray() for X in global_matrices_1d(k, N, s))
    K = np.kron
    At = K(M, B) + K(B, M) if d == 2 else K(K(M, M), B) + K(K(M, B), M) + K(K(B, M), M)
    xn = avs_step(A, ps, x, b, 0.3)
    ref = x + 0.3 * np.linalg.solve(At, b - A @ x)
    assert np.linalg.norm(xn - ref) <= 1e-11 * np.linalg.norm(ref)
    assert np.linalg.norm(mvs_step(A, ps, x, b, 0.3) - ref) <= 1e-11 * np.linalg.norm(ref)
    pse = PatchSolvers(k, d, N, s, exact_A=A)
    xe = avs_step(A, pse, x, b, 1.0)
    xs = np.linalg.solve(A.toarray(), b)
    assert np.linalg.norm(xe - xs) <= 1e-10 * np.linalg.norm(xs)


def test_avs_error_propagation_A_symmetric():
    """<S e1, e2>_A = <e1, S e2>_A for AVS (makes CG valid)."""
    A, ps, x, b, s = _setup(2, 2, 6)
    rng = np.random.default_rng(0)
    e1, e2 = rng.standard_normal((2, A.shape[0]))
    z = np.zeros(A.shape[0])
    S = lambda e: avs_step(A, ps, e, z, 0.25)
    lhs = S(e1) @ (A @ e2); rhs = e1 @ (A @ S(e2))
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def test_mvs_intra_colour_permutation():
    """permuting patches inside a colour changes x' only by rounding."""
    A, ps, x, b, s = _setup(2, 3, 8)
    ref = mvs_step(A, ps, x, b, 1.0)
    import oracle.smoothers as sm
    orig = sm.color_patches
    sm.color_patches = lambda d, N: [c[::-1] for c in orig(d, N)]
    try:
        perm = mvs_step(A, ps, x, b, 1.0)
    finally:
        sm.color_patches = orig
    assert np.abs(perm - ref).max() <= 1e-13 * np.abs(ref).max()


def test_mvs_reverse_differs_and_colour_order_matters():
    """Reading Q25: colour order defines a different (valid) smoother."""
    A, ps, x, b, s = _setup(2, 2, 8)
    assert np.abs(mvs_step(A, ps, x, b, 1.0) - mvs_step(A, ps, x, b, 1.0, reverse=True)).max() > 1e-6


@pytest.mark.parametrize("d,k,N", [(2, 3, 7), (3, 2, 5)])
def test_sampled_delta_matches_full_step(d, k, N):
    A, ps, x, b, s = _setup(d, k, N)
    delta = avs_step(A, ps, x, b, 0.25) - x
    sample = np.array([0, 5, len(x) // 2, len(x) - 1])
    ds = avs_delta_sample(k, d, N, s, x, b, 0.25, sample)
    assert np.abs(ds - delta[sample]).max() <= 1e-11 * np.abs(delta).max()


def test_avs_smoother_contracts_energy():
    """||x'-x*||_A < ||x-x*||_A (2D, k=2, N=8)."""
    A, ps, x, b, s = _setup(2, 2, 8)
    xs = np.linalg.solve(A.toarray(), b)
    e0, e1 = x - xs, avs_step(A, ps, x, b, 0.25) - xs
    assert e1 @ (A @ e1) < e0 @ (A @ e0)
