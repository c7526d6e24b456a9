"""GPU parity on graded / anisotropic Cartesian meshes: the C-ABI path
(c0ip_create_graded, generic per-axis kernels, per-vertex FDM factors) against the oracle on the same meshes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from c0ip_inputs import random_xb  # noqa: E402
from oracle.discretization import default_sigma, graded_nodes  # noqa: E402
from oracle.operator import assemble, paper_rhs  # noqa: E402
from oracle.smoothers import PatchSolvers, avs_step, mvs_step  # noqa: E402
from oracle.multigrid import Hierarchy, prolongation, pcg, precondition  # noqa: E402

DEV = "cuda:0"
BETAS = (0.5, -0.4, 0.3)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def nodes_for(d, N):
    return [graded_nodes(N, BETAS[a]) for a in range(d)]


CASES = [(2, 2, 8), (2, 3, 8), (2, 4, 4), (2, 5, 4), (3, 2, 4), (3, 3, 2)]


@pytest.mark.parametrize("d,k,N", CASES)
def test_graded_operator_rhs_smoothers(d, k, N):
    from paper_2412_05082_b200 import api
    L = int(np.log2(N))
    nodes = nodes_for(d, N)
    ctx = api.Context(d, k, L, nodes=nodes)
    s = default_sigma(k)
    A = assemble(k, d, N, s, nodes=nodes)
    x, b = random_xb(k, d, N)
    xt, bt = torch.tensor(x, device=DEV), torch.tensor(b, device=DEV)
    assert rel(ctx.apply(L, xt).cpu().numpy(), A @ x) <= 1e-11
    assert rel(ctx.residual(L, bt, xt).cpu().numpy(), b - A @ x) <= 1e-11
    assert rel(ctx.rhs(L).cpu().numpy(), paper_rhs(k, d, N, s, nodes=nodes)) <= 1e-13
    ps = PatchSolvers(k, d, N, s, nodes=nodes)
    om_a, om_m = (0.25, 0.8) if d == 2 else (0.1, 0.7)
    for sm, ref in (("avs_atomic", lambda: avs_step(A, ps, x, b, om_a)), ("avs", lambda: avs_step(A, ps, x, b, om_a)),
                    ("mvs", lambda: mvs_step(A, ps, x, b, om_m))):
        xg = torch.tensor(x, device=DEV)
        ctx.smooth(L, sm, 1, om_m if sm == "mvs" else om_a, bt, xg)
        assert rel(xg.cpu().numpy() - x, ref() - x) <= 1e-11, sm
    xi = x.astype(np.float32).astype(np.float64)
    y32 = ctx.apply(L, torch.tensor(xi, device=DEV, dtype=torch.float32)).cpu().numpy().astype(np.float64)
    assert rel(y32, A @ xi) <= 1e-5
    ctx.close()


@pytest.mark.parametrize("d,k,L", [(2, 3, 4), (3, 2, 3)])
def test_graded_transfers(d, k, L):
    from paper_2412_05082_b200 import api
    N = 2 ** L
    nodes = nodes_for(d, N)
    ctx = api.Context(d, k, L, nodes=nodes)
    P = prolongation(k, d, N // 2, nodes_f=nodes)
    c = np.random.default_rng(1).standard_normal(P.shape[1])
    f = np.random.default_rng(2).standard_normal(P.shape[0])
    ft = torch.tensor(f, device=DEV)
    ctx.prolongate_add(L, torch.tensor(c, device=DEV), ft)
    assert rel(ft.cpu().numpy(), f + P @ c) <= 1e-12
    assert rel(ctx.restrict(L, torch.tensor(f, device=DEV)).cpu().numpy(), P.T @ f) <= 1e-12
    ctx.close()


@pytest.mark.parametrize("d,k,L,kind,steps,om", [(2, 3, 5, "avs", 2, 0.25), (2, 4, 4, "mvs", 1, 0.8),
                                                 (3, 2, 3, "avs", 2, 0.1)])
def test_graded_pcg_iterations(d, k, L, kind, steps, om):
    """MG-PCG on the graded hierarchy: iteration count within 1 of the oracle's, FP64 cycle."""
    from paper_2412_05082_b200 import api
    N = 2 ** L
    nodes = nodes_for(d, N)
    s = default_sigma(k)
    h = Hierarchy(k, d, L, s, nodes=nodes)
    b = paper_rhs(k, d, N, s, nodes=nodes)
    xo, no, ho = pcg(h.A[L], b, lambda r: precondition(h, r, kind, steps, om))
    ctx = api.Context(d, k, L, nodes=nodes)
    x, rep, hist = ctx.pcg(api.MG(kind, steps, om), torch.tensor(b, device=DEV))
    assert rep["converged"] and abs(rep["iterations"] - no) <= 1, (rep, no)
    assert np.linalg.norm(b - h.A[L] @ x.cpu().numpy()) <= 1.01e-8 * np.linalg.norm(b)
    ctx.close()


def test_graded_rejects_bad_nodes():
    from paper_2412_05082_b200 import api, _lib
    bad = np.linspace(0, 1, 9)
    bad[3] = bad[2]
    with pytest.raises(_lib.C0ipError) as e:
        api.Context(2, 2, 3, nodes=[bad, None])
    assert e.value.status == _lib.ERR_ARG
