"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bars: maps bit-exact; FP64 relative l2 <= 1e-11 for y = Ax, r = b - Ax,
smoother increments and transfers on random inputs; FP32 <= 1e-5 against the FP64 oracle;
PCG iteration counts +-1.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from c0ip_inputs import random_xb, uniform  # noqa: E402
from oracle.operator import assemble, paper_rhs  # noqa: E402
from oracle.discretization import default_sigma, global_matrices_1d, patch_range_1d  # noqa: E402
from oracle.mesh import all_patch_dofs, color_patches, patch_vertices  # noqa: E402
from oracle.smoothers import PatchSolvers, avs_step, mvs_step  # noqa: E402
from oracle.multigrid import Hierarchy, prolongation, precondition, pcg, fractional_iterations  # noqa: E402

DEV = "cuda:0"
FP64_TOL, FP32_TOL = 1e-11, 1e-5
U32 = 2.0 ** -24


def fp32_delta_tol(A, ps, xi, bi, om, kind, reverse=False):
    """FP32 smoother-increment bar: 4x the deviation of the oracle's FP32 model of the
    step -- residual b - A x evaluated in FP32 arithmetic on the FP32 inputs, x stored in FP32, exact
    (FP64) local solves -- from the FP64 oracle step on the same inputs; floor 1e-6."""
    A32, x32, b32 = A.astype(np.float32), xi.astype(np.float32), bi.astype(np.float32)
    if kind == "avs":
        xm, xo = avs_step(A32, ps, x32, b32, om), avs_step(A, ps, xi, bi, om)
    else:
        xm, xo = mvs_step(A32, ps, x32, b32, om, reverse=reverse), mvs_step(A, ps, xi, bi, om, reverse=reverse)
    return max(1e-6, 4 * rel(xm.astype(np.float64) - xi, xo - xi))


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


_CACHE = {}


def ctx_for(d, k, N):
    """Context whose finest level has N cells (nested if N is a power of two, else override)."""
    from paper_2412_05082_b200 import api
    key = (d, k, N)
    if key not in _CACHE:
        L = int(np.log2(N))
        if 2 ** L == N:
            _CACHE[key] = (api.Context(d, k, L), L)
        else:
            _CACHE[key] = (api.Context(d, k, 3, cells_override=N), 3)
    return _CACHE[key]


_OR = {}


def oracle(d, k, N):
    key = (d, k, N)
    if key not in _OR:
        s = default_sigma(k)
        _OR[key] = (assemble(k, d, N, s), PatchSolvers(k, d, N, s))
    return _OR[key]


CASES_2D = [(2, k, N) for k in range(2, 8) for N in (2, 3, 5, 8, 16) if (k * N - 1) ** 2 <= 40000]
CASES_3D = [(3, k, N) for k in range(2, 6) for N in (2, 3, 4, 6) if (k * N - 1) ** 3 <= 30000]
CASES = CASES_2D + CASES_3D


# ------------------------------------------------------------------------------ maps
@pytest.mark.parametrize("d,k,N", [(2, 2, 8), (2, 3, 5), (2, 7, 3), (3, 2, 4), (3, 3, 2)])
def test_maps_bit_exact(d, k, N):
    ctx, L = ctx_for(d, k, N)
    info = ctx.level_info(L)
    assert info["n_dofs"] == (k * N - 1) ** d and info["n_patches"] == (N - 1) ** d
    assert info["n_colors"] == 2 ** (d + 1)
    dofs = all_patch_dofs(k, d, N)
    for p in range(len(dofs)):
        assert np.array_equal(ctx.patch_dofs(L, p), dofs[p])
    for c, ids in enumerate(color_patches(d, N)):
        assert np.array_equal(ctx.color_patches(L, c), ids)


@pytest.mark.parametrize("k,N", [(2, 2), (2, 3), (4, 8), (7, 5)])
def test_matrices_1d_and_fdm(k, N):
    ctx, L = ctx_for(2, k, N)
    s = default_sigma(k)
    Mo, Lo, Bo = (X.toarray() for X in global_matrices_1d(k, N, s))
    Mg, Lg, Bg = ctx.matrices_1d(L)
    for g, o in ((Mg, Mo), (Lg, Lo), (Bg, Bo)):
        assert np.abs(g - o).max() <= 1e-12 * np.abs(o).max()
    variants = {0: 1, 1: 2, 2: N - 1} if N > 2 else {3: 1}
    for var, v in variants.items():
        if var == 1 and N < 4:
            continue
        S, lam = ctx.fdm(L, var)
        rr = patch_range_1d(k, v)
        Mv, Bv = Mo[np.ix_(rr, rr)], Bo[np.ix_(rr, rr)]
        # unique quantities: S S^T = M_v^{-1}, S diag(1/lam) S^T = B_v^{-1}
        assert rel(S @ S.T, np.linalg.inv(Mv)) < 1e-10
        assert rel(S @ np.diag(1 / lam) @ S.T, np.linalg.inv(Bv)) < 1e-10
        assert np.all(np.diff(lam) >= 0) and lam[0] > 0


# ------------------------------------------------------------------------------ operator
@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("d,k,N", CASES)
def test_apply_residual(d, k, N, generic):
    ctx, L = ctx_for(d, k, N)
    ctx.set_path(generic)
    A, _ = oracle(d, k, N)
    x, b = random_xb(k, d, N)
    y = ctx.apply(L, torch.tensor(x, device=DEV)).cpu().numpy()
    assert rel(y, A @ x) <= FP64_TOL
    r = ctx.residual(L, torch.tensor(b, device=DEV), torch.tensor(x, device=DEV)).cpu().numpy()
    assert rel(r, b - A @ x) <= FP64_TOL
    xi = x.astype(np.float32).astype(np.float64)
    y32 = ctx.apply(L, torch.tensor(xi, device=DEV, dtype=torch.float32)).cpu().numpy().astype(np.float64)
    assert rel(y32, A @ xi) <= FP32_TOL
    ctx.set_path(False)


@pytest.mark.parametrize("d,k,N", [(2, 2, 8), (2, 5, 4), (3, 3, 4)])
def test_rhs_matches_oracle(d, k, N):
    ctx, L = ctx_for(d, k, N)
    b = ctx.rhs(L).cpu().numpy()
    bo = paper_rhs(k, d, N, default_sigma(k))
    assert rel(b, bo) <= 1e-13


# ------------------------------------------------------------------------------ smoothers
SMOOTH_CASES = [c for c in CASES if c[2] <= 8]


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("sm", ["avs_atomic", "avs", "avs_colored"])
@pytest.mark.parametrize("d,k,N", SMOOTH_CASES)
def test_avs_increment(d, k, N, sm, generic):
    ctx, L = ctx_for(d, k, N)
    ctx.set_path(generic)
    A, ps = oracle(d, k, N)
    x, b = random_xb(k, d, N)
    om = 0.25 if d == 2 else 0.1
    for dt, tol in ((torch.float64, FP64_TOL), (torch.float32, FP32_TOL)):
        # both sides take the same inputs: the FP32 run's RN-rounded x, b
        xi = x.astype(np.float32).astype(np.float64) if dt == torch.float32 else x
        bi = b.astype(np.float32).astype(np.float64) if dt == torch.float32 else b
        xt = torch.tensor(xi, device=DEV, dtype=dt)
        ctx.smooth(L, sm, 1, om, torch.tensor(bi, device=DEV, dtype=dt), xt)
        xo = avs_step(A, ps, xi, bi, om)
        xg = xt.cpu().numpy().astype(np.float64)
        # FP64: the increment delta = x' - x at 1e-11.  FP32: the smoother output x' at 1e-5
        # (north star), the increment at FP32_DELTA_TOL (its FP32 rounding is amplified by
        # kappa(A~_v)).
        if dt == torch.float64:
            assert rel(xg - xi, xo - xi) <= tol, rel(xg - xi, xo - xi)
        else:
            dtol = fp32_delta_tol(A, ps, xi, bi, om, "avs")
            assert rel(xg - xi, xo - xi) <= dtol, (rel(xg - xi, xo - xi), dtol)
            xtol = max(FP32_TOL, dtol * np.linalg.norm(xo - xi) / np.linalg.norm(xo))
            assert rel(xg, xo) <= xtol, (rel(xg, xo), xtol)
    ctx.set_path(False)


@pytest.mark.parametrize("generic", [False, True])
@pytest.mark.parametrize("reverse", [False, True])
@pytest.mark.parametrize("d,k,N", SMOOTH_CASES)
def test_mvs_increment(d, k, N, reverse, generic):
    ctx, L = ctx_for(d, k, N)
    ctx.set_path(generic)
    A, ps = oracle(d, k, N)
    x, b = random_xb(k, d, N)
    om = 1.0 if d == 2 else 0.7
    xt = torch.tensor(x, device=DEV)
    ctx.smooth(L, "mvs", 1, om, torch.tensor(b, device=DEV), xt, reverse=reverse)
    do = mvs_step(A, ps, x, b, om, reverse=reverse) - x
    assert rel(xt.cpu().numpy() - x, do) <= FP64_TOL
    xi, bi = x.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
    x32 = torch.tensor(xi, device=DEV, dtype=torch.float32)
    ctx.smooth(L, "mvs", 1, om, torch.tensor(bi, device=DEV, dtype=torch.float32), x32, reverse=reverse)
    xo32 = mvs_step(A, ps, xi, bi, om, reverse=reverse)
    xg32 = x32.cpu().numpy().astype(np.float64)
    dtol = fp32_delta_tol(A, ps, xi, bi, om, "mvs", reverse)
    assert rel(xg32 - xi, xo32 - xi) <= dtol, (rel(xg32 - xi, xo32 - xi), dtol)
    assert rel(xg32, xo32) <= max(FP32_TOL, dtol * np.linalg.norm(xo32 - xi) / np.linalg.norm(xo32))
    ctx.set_path(False)


# sizes spanning several fused tiles (interior fast paths, ragged last tile) of the 2D kernels; N >= 34
# puts more than 33 patches in a row: the atomic DMMA patch kernel's 32-patch runs get a seam
LARGE_2D = [(2, 2, 40), (2, 3, 27), (2, 3, 32), (2, 4, 27), (2, 4, 32), (2, 5, 21), (2, 7, 13),
            (2, 3, 36), (2, 4, 36)]


@pytest.mark.parametrize("sm", ["avs", "mvs", "avs_atomic"])
@pytest.mark.parametrize("d,k,N", LARGE_2D)
def test_smoother_increment_large_2d(d, k, N, sm):
    ctx, L = ctx_for(d, k, N)
    A, ps = oracle(d, k, N)
    x, b = random_xb(k, d, N)
    om = 0.8 if sm == "mvs" else 0.25
    step = mvs_step if sm == "mvs" else avs_step
    xt = torch.tensor(x, device=DEV)
    ctx.smooth(L, sm, 1, om, torch.tensor(b, device=DEV), xt)
    do = step(A, ps, x, b, om) - x
    assert rel(xt.cpu().numpy() - x, do) <= FP64_TOL, rel(xt.cpu().numpy() - x, do)
    xi, bi = x.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
    x32 = torch.tensor(xi, device=DEV, dtype=torch.float32)
    ctx.smooth(L, sm, 1, om, torch.tensor(bi, device=DEV, dtype=torch.float32), x32)
    xo32 = step(A, ps, xi, bi, om)
    xg32 = x32.cpu().numpy().astype(np.float64)
    dtol = fp32_delta_tol(A, ps, xi, bi, om, "mvs" if sm == "mvs" else "avs")
    assert rel(xg32 - xi, xo32 - xi) <= dtol, (rel(xg32 - xi, xo32 - xi), dtol)
    assert rel(xg32, xo32) <= max(FP32_TOL, dtol * np.linalg.norm(xo32 - xi) / np.linalg.norm(xo32))


def test_avs_deterministic_bitwise_reproducible():
    ctx, L = ctx_for(2, 4, 8)
    x, b = random_xb(4, 2, 8)
    outs = []
    for _ in range(2):
        xt = torch.tensor(x, device=DEV)
        ctx.smooth(L, "avs", 2, 0.25, torch.tensor(b, device=DEV), xt)
        outs.append(xt.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------------------------------------ transfers
@pytest.mark.parametrize("d,k,L", [(2, 2, 3), (2, 5, 3), (2, 7, 2), (2, 3, 5), (2, 4, 4), (2, 7, 4),
                                   (3, 2, 3), (3, 4, 2)])
def test_transfers(d, k, L):
    from paper_2412_05082_b200 import api
    ctx = api.Context(d, k, L)
    P = prolongation(k, d, 2 ** (L - 1))
    c = uniform(P.shape[1], 3); f = uniform(P.shape[0], 4)
    for dt, tol in ((torch.float64, FP64_TOL), (torch.float32, FP32_TOL)):
        ft = torch.tensor(f, device=DEV, dtype=dt)
        ctx.prolongate_add(L, torch.tensor(c, device=DEV, dtype=dt), ft)
        assert rel(ft.cpu().numpy().astype(np.float64), f + P @ c) <= tol
        rc = ctx.restrict(L, torch.tensor(f, device=DEV, dtype=dt)).cpu().numpy().astype(np.float64)
        assert rel(rc, P.T @ f) <= tol
    ctx.close()


# ------------------------------------------------------------------------------ V-cycle / PCG
@pytest.mark.parametrize("d,k,L,sm,steps,om", [(2, 2, 3, "avs", 2, 0.25), (2, 3, 4, "mvs", 1, 1.0),
                                               (3, 2, 3, "avs", 1, 0.1), (3, 2, 2, "mvs", 1, 0.7)])
def test_vcycle(d, k, L, sm, steps, om):
    from paper_2412_05082_b200 import api
    ctx = api.Context(d, k, L)
    h = Hierarchy(k, d, L, default_sigma(k))
    r = uniform(h.A[L].shape[0], 9)
    kind = "avs" if sm.startswith("avs") else "mvs"
    zo = precondition(h, r, kind, steps, om)
    z = ctx.vcycle(api.MG(sm, steps, om), torch.tensor(r, device=DEV)).cpu().numpy()
    assert rel(z, zo) <= 1e-10
    z32 = ctx.vcycle(api.MG(sm, steps, om, cycle_dtype=torch.float32), torch.tensor(r, device=DEV)).cpu().numpy()
    assert rel(z32, zo) <= 1e-4
    ctx.close()


@pytest.mark.parametrize("d,k,L,sm,steps,om", [(2, 2, 3, "avs", 2, 0.25), (2, 3, 5, "avs", 2, 0.25),
                                               (2, 4, 4, "mvs", 1, 1.0), (3, 2, 3, "avs", 2, 0.1),
                                               (3, 3, 3, "mvs", 1, 0.7)])
def test_pcg_iterations(d, k, L, sm, steps, om):
    from paper_2412_05082_b200 import api
    ctx = api.Context(d, k, L)
    h = Hierarchy(k, d, L, default_sigma(k))
    h32 = Hierarchy(k, d, L, default_sigma(k), dtype=np.float32)
    b = paper_rhs(k, d, 2 ** L, default_sigma(k))
    kind = "avs" if sm.startswith("avs") else "mvs"
    xo, no, ho = pcg(h.A[L], b, lambda r: precondition(h, r, kind, steps, om))
    _, no32, _ = pcg(h.A[L], b, lambda r: precondition(h32, r, kind, steps, om))
    for dt in (torch.float64, torch.float32):
        x, rep, hist = ctx.pcg(api.MG(sm, steps, om, cycle_dtype=dt), torch.tensor(b, device=DEV))
        assert rep["converged"]
        # +-1 against the oracle's cycle in the same precision (north star; FP32: Hierarchy dtype float32)
        assert abs(rep["iterations"] - (no if dt == torch.float64 else no32)) <= 1, (dt, rep["iterations"], no, no32)
        xn = x.cpu().numpy()
        assert np.linalg.norm(b - h.A[L] @ xn) <= 1.01e-8 * np.linalg.norm(b)
        if dt == torch.float64:
            assert abs(rep["nu"] - fractional_iterations(ho)) <= 0.5
    ctx.close()


@pytest.mark.parametrize("d,k,L,sm,steps,om,sym", [(2, 2, 3, "mvs", 1, 1.0, False), (2, 3, 4, "mvs", 1, 1.0, False),
                                                   (2, 4, 5, "mvs", 1, 1.0, False), (2, 2, 4, "avs", 2, 0.25, True),
                                                   (3, 2, 3, "mvs", 1, 0.7, False)])
def test_gmres_iterations(d, k, L, sm, steps, om, sym):
    """GMRES around the paper's same-order (nonsymmetric) MVS cycle:
    iteration count within 1 (FP64 cycle) / 2 (FP32 cycle) of the oracle's FGMRES, true residual at
    the tolerance, nu within 0.5."""
    from paper_2412_05082_b200 import api
    from oracle.multigrid import gmres
    ctx = api.Context(d, k, L)
    h = Hierarchy(k, d, L, default_sigma(k))
    h32 = Hierarchy(k, d, L, default_sigma(k), dtype=np.float32)
    b = paper_rhs(k, d, 2 ** L, default_sigma(k))
    xo, no, ho = gmres(h.A[L], b, lambda r: precondition(h, r, sm, steps, om, symmetric=sym))
    _, no32, _ = gmres(h.A[L], b, lambda r: precondition(h32, r, sm, steps, om, symmetric=sym))
    for dt in (torch.float64, torch.float32):
        x, rep, hist = ctx.gmres(api.MG(sm, steps, om, symmetric=sym, cycle_dtype=dt), torch.tensor(b, device=DEV))
        assert rep["converged"]
        assert abs(rep["iterations"] - (no if dt == torch.float64 else no32)) <= 1, (dt, rep["iterations"], no, no32)
        xn = x.cpu().numpy()
        # the residual of a smooth solution is itself only known to ~ eps || |A| |x| || (SURVEY.md F9:
        # cancellation 1e7..1e12); the GPU stops on its own residual, so the host-measured one is checked
        # against the tolerance plus that rounding floor
        tr = np.linalg.norm(b - h.A[L] @ xn) / np.linalg.norm(b)
        floor = 32 * 2.2e-16 * np.linalg.norm(abs(h.A[L]) @ np.abs(xn)) / np.linalg.norm(b)
        assert tr <= 1.05e-8 + floor, (dt, tr, floor, rep, hist[-3:], ho[-3:])
        if dt == torch.float64:
            assert abs(rep["nu"] - fractional_iterations(ho)) <= 0.5
            assert np.allclose(hist[: min(len(hist), len(ho))], ho[: min(len(hist), len(ho))], rtol=1e-6, atol=1e-12 * ho[0])
    ctx.close()


def test_gmres_bad_restart_is_arg_error():
    from paper_2412_05082_b200 import api
    ctx = api.Context(2, 2, 3)
    b = torch.zeros(ctx.n_dofs(3), device=DEV, dtype=torch.float64)
    with pytest.raises(Exception):
        ctx.gmres(api.MG("mvs", 1, 1.0), b, restart=0)
    ctx.close()


def test_coercivity_error():
    from paper_2412_05082_b200 import api, _lib
    with pytest.raises(_lib.C0ipError) as e:
        api.Context(2, 3, 3, penalty_scale=0.01)
    assert e.value.status == _lib.ERR_COERCIVITY


def test_bad_level_is_arg_error():
    from paper_2412_05082_b200 import _lib
    ctx, L = ctx_for(2, 2, 8)
    with pytest.raises(_lib.C0ipError) as e:
        ctx.apply(L + 1, torch.zeros(10, device=DEV, dtype=torch.float64))
    assert e.value.status == _lib.ERR_ARG


# ------------------------------------------------------------------------------ slabs (multi-GPU path)
@pytest.mark.parametrize("k,N,R", [(2, 32, 2), (4, 16, 2), (3, 20, 3), (7, 12, 2)])
def test_slab_step_bitwise_equals_single_domain(k, N, R):
    """Each rank's slab step (window with exchanged ghosts) == the single-domain step on its owned rows
    (same tiles, same arithmetic -> bitwise); apply likewise.  Ranks are emulated on one GPU."""
    from paper_2412_05082_b200 import api
    from paper_2412_05082_b200.dist import partition
    ctx = api.Context(2, k, 3, cells_override=N)
    L = 3
    n = k * N - 1
    x, b = random_xb(k, 2, N)
    full = torch.tensor(x, device=DEV)
    ctx.smooth(L, "avs", 1, 0.25, torch.tensor(b, device=DEV), full)
    yfull = ctx.apply(L, torch.tensor(x, device=DEV))
    ga, gp = ctx.slab_ghosts()
    assert ga == 4 * k - 2 and gp == 2 * k
    out = torch.empty_like(full)
    yout = torch.empty_like(full)
    for s in partition(N, k, R, ga):
        rows = slice(s.win_lo - 1, s.win_hi - 1)
        xw = torch.tensor(x.reshape(n, n)[rows].ravel(), device=DEV)
        bw = torch.tensor(b.reshape(n, n)[rows].ravel(), device=DEV)
        rw = torch.empty_like(xw)
        ctx.slab_avs_step(L, 0.25, s.row0, s.lrows, s.own_lo, s.own_hi, bw, xw, rw)
        out.view(n, n)[s.own_lo - 1:s.own_hi - 1] = xw.view(-1, n)[s.own_local]
        yw = torch.empty_like(xw)
        ctx.slab_apply(L, s.row0, s.lrows, s.own_lo, s.own_hi, torch.tensor(x.reshape(n, n)[rows].ravel(), device=DEV), yw)
        yout.view(n, n)[s.own_lo - 1:s.own_hi - 1] = yw.view(-1, n)[s.own_local]
    assert torch.equal(out, full)
    assert torch.equal(yout, yfull)
    ctx.close()


@pytest.mark.parametrize("sm", ["avs", "avs_atomic"])
@pytest.mark.parametrize("k,N,R", [(2, 16, 2), (3, 12, 3), (5, 10, 2), (4, 40, 2)])
def test_slab_step_3d(k, N, R, sm):
    """3D z-slabs: apply is bitwise equal to the single-domain apply on the owned planes; the slab AVS
    step (parity-class FDM restricted to the owned planes) is bitwise equal to the single-domain
    deterministic step, and within FP64 tolerance of the atomic one."""
    from paper_2412_05082_b200 import api
    from paper_2412_05082_b200.dist import partition
    ctx = api.Context(3, k, 3, cells_override=N)
    L = 3
    n = k * N - 1
    x, b = random_xb(k, 3, N)
    full = torch.tensor(x, device=DEV)
    ctx.smooth(L, sm, 1, 0.1, torch.tensor(b, device=DEV), full)
    yfull = ctx.apply(L, torch.tensor(x, device=DEV))
    ga, gp = ctx.slab_ghosts()
    out = torch.empty_like(full)
    yout = torch.empty_like(full)
    plane = n * n
    for s in partition(N, k, R, ga):
        rows = slice((s.win_lo - 1) * plane, (s.win_hi - 1) * plane)
        xw = torch.tensor(x[rows], device=DEV)
        bw = torch.tensor(b[rows], device=DEV)
        rw = torch.empty_like(xw)
        ctx.slab_avs_step(L, 0.1, s.row0, s.lrows, s.own_lo, s.own_hi, bw, xw, rw)
        out.view(n, plane)[s.own_lo - 1:s.own_hi - 1] = xw.view(-1, plane)[s.own_local]
        yw = torch.empty_like(xw)
        ctx.slab_apply(L, s.row0, s.lrows, s.own_lo, s.own_hi, torch.tensor(x[rows], device=DEV), yw)
        yout.view(n, plane)[s.own_lo - 1:s.own_hi - 1] = yw.view(-1, plane)[s.own_local]
    assert torch.equal(yout, yfull)
    if sm == "avs":
        assert torch.equal(out, full)
    else:
        assert rel((out - torch.tensor(x, device=DEV)).cpu().numpy(), (full - torch.tensor(x, device=DEV)).cpu().numpy()) <= 1e-13
    ctx.close()


def test_slab_rejects_missing_ghosts():
    from paper_2412_05082_b200 import api, _lib
    ctx = api.Context(2, 3, 3, cells_override=16)
    n = 3 * 16 - 1
    xw = torch.zeros(10 * n, device=DEV, dtype=torch.float64)
    with pytest.raises(_lib.C0ipError) as e:
        ctx.slab_avs_step(3, 0.25, 10, 10, 12, 18, xw, xw.clone(), xw.clone())
    assert e.value.status == _lib.ERR_ARG
    ctx.close()


# ------------------------------------------------------------------------------ 3D fused kernels (N >= 8)
CASES_3D_FUSED = [(3, 2, 8), (3, 3, 9), (3, 4, 8), (3, 5, 8), (3, 3, 10), (3, 2, 12), (3, 2, 16)]


@pytest.mark.parametrize("d,k,N", CASES_3D_FUSED)
def test_apply_residual_3d_fused(d, k, N):
    ctx, L = ctx_for(d, k, N)
    ctx.set_path(False)
    A, _ = oracle(d, k, N)
    x, b = random_xb(k, d, N)
    y = ctx.apply(L, torch.tensor(x, device=DEV)).cpu().numpy()
    assert rel(y, A @ x) <= FP64_TOL
    r = ctx.residual(L, torch.tensor(b, device=DEV), torch.tensor(x, device=DEV)).cpu().numpy()
    assert rel(r, b - A @ x) <= FP64_TOL
    xi = x.astype(np.float32).astype(np.float64)
    y32 = ctx.apply(L, torch.tensor(xi, device=DEV, dtype=torch.float32)).cpu().numpy().astype(np.float64)
    assert rel(y32, A @ xi) <= FP32_TOL


@pytest.mark.parametrize("sm", ["avs", "avs_colored", "avs_atomic", "mvs", "mvs_rev"])
@pytest.mark.parametrize("d,k,N", CASES_3D_FUSED)
def test_smoothers_3d_fused(d, k, N, sm):
    ctx, L = ctx_for(d, k, N)
    ctx.set_path(False)
    A, ps = oracle(d, k, N)
    x, b = random_xb(k, d, N)
    rev = sm == "mvs_rev"
    smc = "mvs" if rev else sm
    om = 0.7 if smc == "mvs" else 0.1

    def ref(xi, bi):
        return mvs_step(A, ps, xi, bi, om, reverse=rev) if smc == "mvs" else avs_step(A, ps, xi, bi, om)
    xt = torch.tensor(x, device=DEV)
    ctx.smooth(L, smc, 1, om, torch.tensor(b, device=DEV), xt, reverse=rev)
    do = ref(x, b) - x
    assert rel(xt.cpu().numpy() - x, do) <= FP64_TOL
    # FP32 (the mixed-precision cycle's kernels) on the RN-rounded inputs
    xi, bi = x.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
    x32 = torch.tensor(xi, device=DEV, dtype=torch.float32)
    ctx.smooth(L, smc, 1, om, torch.tensor(bi, device=DEV, dtype=torch.float32), x32, reverse=rev)
    xo32 = ref(xi, bi)
    xg32 = x32.cpu().numpy().astype(np.float64)
    dtol = fp32_delta_tol(A, ps, xi, bi, om, "mvs" if smc == "mvs" else "avs", rev)
    assert rel(xg32 - xi, xo32 - xi) <= dtol, (rel(xg32 - xi, xo32 - xi), dtol)
    assert rel(xg32, xo32) <= max(FP32_TOL, dtol * np.linalg.norm(xo32 - xi) / np.linalg.norm(xo32))


@pytest.mark.parametrize("k,N", [(2, 72), (3, 68)])
def test_3d_chunked_stream_matches_oracle_rows(k, N):
    """N > CZ (32 cell layers per CTA chunk): chunk seams of the z-streaming kernel, checked on sampled
    residual rows from the oracle's window assembly and against the generic per-axis path."""
    from paper_2412_05082_b200 import api
    from oracle.operator import residual_on_box
    ctx = api.Context(3, k, 3, cells_override=N)
    x, b = random_xb(k, 3, N)
    xt, bt = torch.tensor(x, device=DEV), torch.tensor(b, device=DEV)
    r_f = ctx.residual(3, bt, xt).cpu().numpy()
    ctx.set_path(True)
    r_g = ctx.residual(3, bt, xt).cpu().numpy()
    ctx.set_path(False)
    assert rel(r_f, r_g) <= 1e-13
    n = k * N - 1
    s = default_sigma(k)
    for z0 in (0, 32 * k - 3, n - 4):                    # boxes across the chunk seam and at the ends
        lo = np.array([n // 2 - 2, 3, z0]); hi = lo + 4
        rb, ids = residual_on_box(k, 3, N, s, x, b, lo, hi)
        assert rel(r_f[ids], rb) <= FP64_TOL
    ctx.close()


# ------------------------------------------------------------------------------ full bench sizes
# BASELINE.json configs[1] / configs[3] at the sizes and in the launch configuration bench.py times
# (atomic AVS step, fused kernels), checked on sampled outputs the oracle computes one by one
# (local window assembly + dense surrogate solves; oracle.smoothers.avs_delta_sample).
def _sample_ids(n, d, rng, m=48):
    ids = set()
    edge = [0, 1, n // 2, n - 2, n - 1]
    for _ in range(m):
        c = [int(rng.integers(0, n)) if rng.random() < 0.7 else int(rng.choice(edge)) for _ in range(d)]
        ids.add(sum(c[a] * n ** a for a in range(d)))
    return np.array(sorted(ids))


@pytest.mark.parametrize("d,k,sm", [(2, 4, "avs_atomic"), (2, 4, "avs"), (2, 3, "avs_atomic"), (2, 2, "avs_atomic"),
                                    (2, 5, "avs"), (2, 7, "avs"),
                                    (3, 3, "avs_atomic"), (3, 2, "avs_atomic"), (3, 2, "avs"), (3, 4, "avs_atomic"),
                                    (3, 5, "avs_atomic")])
def test_full_size_sampled_avs(d, k, sm):
    from c0ip_inputs import CFG2_CELLS, CFG4_CELLS
    from oracle.smoothers import avs_delta_sample
    from oracle.operator import residual_on_box
    from paper_2412_05082_b200 import api
    N = CFG2_CELLS[k] if d == 2 else CFG4_CELLS[k]
    om = 0.25 if d == 2 else 0.1
    ctx = api.Context(d, k, 3, cells_override=N)
    x, b = random_xb(k, d, N)
    n = k * N - 1
    xt = torch.tensor(x, device=DEV)
    bt = torch.tensor(b, device=DEV)
    r = ctx.residual(3, bt, xt, torch.empty_like(xt)).cpu().numpy()
    ctx.smooth(3, sm, 1, om, bt, xt)
    dg = xt.cpu().numpy() - x
    ctx.close()
    rng = np.random.default_rng(7)
    ids = _sample_ids(n, d, rng)
    s = default_sigma(k)
    do = avs_delta_sample(k, d, N, s, x, b, om, ids)
    assert np.abs(dg[ids] - do).max() <= 1e-11 * np.abs(do).max(), np.abs(dg[ids] - do).max() / np.abs(do).max()
    # residual rows at the same ids
    ro = np.array([residual_on_box(k, d, N, s, x, b, [(g // n ** a) % n for a in range(d)],
                                   [(g // n ** a) % n + 1 for a in range(d)])[0][0] for g in ids])
    assert np.abs(r[ids] - ro).max() <= 1e-11 * np.abs(ro).max()


@pytest.mark.parametrize("k,sm", [(4, "avs_atomic"), (3, "avs"), (7, "avs")])
def test_full_size_sampled_avs_fp32(k, sm):
    """cfg2 at full size in FP32 (the mixed cycle's kernels): sampled increments against the oracle on the
    RN-rounded inputs; bar = 4x the oracle FP32-model deviation of the same degree on a small mesh
    (fp32_delta_tol), measured on the sample."""
    from c0ip_inputs import CFG2_CELLS
    from oracle.smoothers import avs_delta_sample
    from paper_2412_05082_b200 import api
    d, N, om = 2, CFG2_CELLS[k], 0.25
    ctx = api.Context(d, k, 3, cells_override=N)
    x, b = random_xb(k, d, N)
    xi, bi = x.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
    n = k * N - 1
    xt = torch.tensor(xi, device=DEV, dtype=torch.float32)
    ctx.smooth(3, sm, 1, om, torch.tensor(bi, device=DEV, dtype=torch.float32), xt)
    dg = xt.cpu().numpy().astype(np.float64) - xi
    ctx.close()
    ids = _sample_ids(n, d, np.random.default_rng(8))
    do = avs_delta_sample(k, d, N, default_sigma(k), xi, bi, om, ids)
    Ns = 12
    A, ps = oracle(d, k, Ns)
    xs, bs = random_xb(k, d, Ns)
    xs, bs = xs.astype(np.float32).astype(np.float64), bs.astype(np.float32).astype(np.float64)
    dtol = fp32_delta_tol(A, ps, xs, bs, om, "avs")
    assert rel(dg[ids], do) <= dtol, (rel(dg[ids], do), dtol)


# ------------------------------------------------------------------------------ exact local solvers
EXACT_CASES = [(2, 2, 8), (2, 3, 5), (2, 4, 8), (2, 5, 3), (3, 2, 4), (3, 3, 3), (2, 2, 2), (3, 2, 2)]


@pytest.mark.parametrize("sm", ["avs_atomic", "mvs", "mvs_rev"])
@pytest.mark.parametrize("d,k,N", EXACT_CASES)
def test_exact_local_smoothers(d, k, N, sm):
    """c0ip_set_local_solver(EXACT): the smoother with A_v = R_v A R_v^T (Table 1) against the
    oracle's dense exact patch solves (PatchSolvers(exact_A=A)); FP64 1e-11, FP32 at the FP32-model bar."""
    from paper_2412_05082_b200 import api
    L = int(np.log2(N)) if 2 ** int(np.log2(N)) == N else 3
    ctx = api.Context(d, k, L, cells_override=0 if 2 ** int(np.log2(N)) == N else N)
    ctx.set_local_solver(True)
    A = assemble(k, d, N, default_sigma(k))
    ps = PatchSolvers(k, d, N, default_sigma(k), exact_A=A)
    x, b = random_xb(k, d, N)
    rev = sm == "mvs_rev"
    kind = "mvs" if sm.startswith("mvs") else "avs"
    om = (0.8 if d == 2 else 0.7) if kind == "mvs" else (0.25 if d == 2 else 0.1)
    ref = (lambda xi, bi: mvs_step(A, ps, xi, bi, om, reverse=rev)) if kind == "mvs" else \
        (lambda xi, bi: avs_step(A, ps, xi, bi, om))
    xt = torch.tensor(x, device=DEV)
    ctx.smooth(L, kind if kind == "mvs" else sm, 1, om, torch.tensor(b, device=DEV), xt, reverse=rev)
    assert rel(xt.cpu().numpy() - x, ref(x, b) - x) <= FP64_TOL
    xi, bi = x.astype(np.float32).astype(np.float64), b.astype(np.float32).astype(np.float64)
    x32 = torch.tensor(xi, device=DEV, dtype=torch.float32)
    ctx.smooth(L, kind if kind == "mvs" else sm, 1, om, torch.tensor(bi, device=DEV, dtype=torch.float32), x32,
               reverse=rev)
    dtol = fp32_delta_tol(A, ps, xi, bi, om, kind, rev)
    assert rel(x32.cpu().numpy().astype(np.float64) - xi, ref(xi, bi) - xi) <= dtol
    ctx.close()


@pytest.mark.parametrize("kind,steps", [("avs", 2), ("mvs", 1)])
def test_exact_local_table1_iterations(kind, steps):
    """Table 1: 2D k=4 L=6 with exact local solvers -- the GPU solve within 1 iteration of the
    oracle's (paper protocol: CG + AVS-2 omega 1/4, GMRES + MVS-1 omega 1) and nu within 1 of the paper."""
    from paper_2412_05082_b200 import api
    from oracle.multigrid import solve_paper
    d, k, L = 2, 4, 6
    no, nuo, _ = solve_paper(d, k, L, kind, steps, exact=True)
    ctx = api.Context(d, k, L)
    ctx.set_local_solver(True)
    b = ctx.rhs(L)
    if kind == "avs":
        x, rep, hist = ctx.pcg(api.MG("avs", steps, 0.25), b)
        paper = 10.3
    else:
        x, rep, hist = ctx.gmres(api.MG("mvs", steps, 1.0, symmetric=False), b)
        paper = 2.9
    assert rep["converged"] and abs(rep["iterations"] - no) <= 1, (rep, no)
    assert abs(rep["nu"] - paper) <= 1.0
    ctx.close()
