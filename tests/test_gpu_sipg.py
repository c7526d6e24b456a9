"""GPU parity for the Poisson SIPG comparison workload: c0ip_create_sipg
against oracle/sipg.py on the same seeded inputs."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.sipg import (assemble_sipg, SipgPatchSolvers, sipg_embedding_1d, sipg_load, sipg_paper_load,  # noqa: E402
                         SipgHierarchy)
from oracle.smoothers import avs_step, mvs_step  # noqa: E402
from oracle.multigrid import pcg, precondition  # noqa: E402

DEV = "cuda:0"


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def inputs(n, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    return g.uniform(-1, 1, n)


@pytest.mark.parametrize("d,k,N", [(2, 2, 8), (2, 3, 4), (2, 5, 4), (3, 2, 4), (3, 3, 2)])
def test_sipg_operator_and_smoothers(d, k, N):
    from paper_2412_05082_b200 import api
    L = int(np.log2(N))
    ctx = api.Context(d, k, L, sipg=True)
    A = assemble_sipg(k, d, N)
    n = A.shape[0]
    assert ctx.n_dofs(L) == n
    x, b = inputs(n, 20241205), inputs(n, 20241206)
    xt, bt = torch.tensor(x, device=DEV), torch.tensor(b, device=DEV)
    assert rel(ctx.apply(L, xt).cpu().numpy(), A @ x) <= 1e-11
    assert rel(ctx.residual(L, bt, xt).cpu().numpy(), b - A @ x) <= 1e-11
    assert rel(ctx.rhs(L).cpu().numpy(), sipg_load(k, d, N, sipg_paper_load(d))) <= 1e-13
    ps = SipgPatchSolvers(k, d, N, A)
    for p in (0, len(ps.dofs) - 1):
        assert np.array_equal(ctx.patch_dofs(L, p), ps.dofs[p])
    om = 0.25 if d == 2 else 0.125
    for sm in ("avs_atomic", "avs", "avs_colored", "mvs"):
        xg = torch.tensor(x, device=DEV)
        ctx.smooth(L, sm, 1, 1.0 if sm == "mvs" else om, bt, xg)
        ref = mvs_step(A, ps, x, b, 1.0) if sm == "mvs" else avs_step(A, ps, x, b, om)
        assert rel(xg.cpu().numpy() - x, ref - x) <= 1e-11, sm
    ctx.close()


@pytest.mark.parametrize("d,k,L", [(2, 3, 3), (3, 2, 2)])
def test_sipg_transfers(d, k, L):
    from paper_2412_05082_b200 import api
    ctx = api.Context(d, k, L, sipg=True)
    import scipy.sparse as sp
    E = sp.csr_matrix(sipg_embedding_1d(k, 2 ** (L - 1)))
    P = E
    for _ in range(d - 1):
        P = sp.kron(E, P)
    c, f = inputs(P.shape[1], 1), inputs(P.shape[0], 2)
    ft = torch.tensor(f, device=DEV)
    ctx.prolongate_add(L, torch.tensor(c, device=DEV), ft)
    assert rel(ft.cpu().numpy(), f + P @ c) <= 1e-12
    assert rel(ctx.restrict(L, torch.tensor(f, device=DEV)).cpu().numpy(), P.T @ f) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("d,k,L,kind,steps,om", [(2, 3, 4, "avs", 2, 0.25), (2, 2, 4, "mvs", 1, 1.0),
                                                 (3, 2, 3, "avs", 1, 0.125)])
def test_sipg_pcg_iterations(d, k, L, kind, steps, om):
    """MG-PCG for the SIPG Poisson problem: iteration count within 1 of the oracle's V-cycle + CG."""
    from paper_2412_05082_b200 import api
    h = SipgHierarchy(k, d, L)
    b = sipg_load(k, d, 2 ** L, sipg_paper_load(d))
    _, no, _ = pcg(h.A[L], b, lambda r: precondition(h, r, kind, steps, om))
    ctx = api.Context(d, k, L, sipg=True)
    x, rep, hist = ctx.pcg(api.MG(kind, steps, om), torch.tensor(b, device=DEV))
    assert rep["converged"] and abs(rep["iterations"] - no) <= 1, (rep, no)
    assert np.linalg.norm(b - h.A[L] @ x.cpu().numpy()) <= 1.01e-8 * np.linalg.norm(b)
    ctx.close()
