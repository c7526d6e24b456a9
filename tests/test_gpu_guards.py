"""Out-of-bounds and read-only guards for every device entry point (stand-in for compute-sanitizer
memcheck, which is closed on this GPU pool).

The C ABI takes bare device pointers (include/c0ip.h), so a kernel that indexes past a vector writes
into whatever lies next to it.  Each vector here is a view into one larger allocation with GUARD
sentinel elements on both sides; after the call every guard must be bit-identical and every input
the ABI declares read-only (b, the coarse vector of prolongate_add, ...) must be unchanged.  Sizes
reach the fused tile kernels (2D N >= 8, 3D N >= 8) with boundary and interior tiles, every degree.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GUARD = 4096
DEV = "cuda:0"


class Guarded:
    """n-element vector between two GUARD-element sentinel regions of one allocation."""

    def __init__(self, n, dtype, values=None, seed=0):
        self.n = n
        self.buf = torch.empty(n + 2 * GUARD, dtype=dtype, device=DEV)
        g = torch.Generator(device="cpu").manual_seed(seed)
        sent = torch.rand(2 * GUARD, generator=g, dtype=torch.float64).to(dtype) * 1e30 + 7.0
        self.buf[:GUARD] = sent[:GUARD].to(DEV)
        self.buf[GUARD + n:] = sent[GUARD:].to(DEV)
        self.t = self.buf[GUARD:GUARD + n]
        if values is not None:
            self.t.copy_(values)
        self.ref_guard = torch.cat([self.buf[:GUARD], self.buf[GUARD + n:]]).clone()

    def guards_intact(self):
        now = torch.cat([self.buf[:GUARD], self.buf[GUARD + self.n:]])
        it = torch.int64 if now.dtype == torch.float64 else torch.int32
        return bool(torch.equal(now.view(it), self.ref_guard.view(it)))     # bitwise


def rand(n, dtype, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.rand(n, generator=g, dtype=torch.float64) * 2 - 1).to(dtype).to(DEV)


CASES = [(2, k, 12) for k in range(2, 8)] + [(2, 4, 9)] + [(3, k, 9) for k in range(2, 6)]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("d,k,N", CASES)
def test_fused_ops_stay_in_bounds(d, k, N, dtype):
    from paper_2412_05082_b200 import api
    ctx = api.Context(d, k, 3, cells_override=N)
    n = ctx.n_dofs(3)
    x, b, y = Guarded(n, dtype, rand(n, dtype, 1), 11), Guarded(n, dtype, rand(n, dtype, 2), 12), Guarded(n, dtype, None, 13)
    b0 = b.t.clone()
    ctx.apply(3, x.t, y.t)
    ctx.residual(3, b.t, x.t, y.t)
    om = 0.25 if d == 2 else 0.1
    for sm in ("avs_atomic", "avs_det", "avs_colored"):
        ctx.smooth(3, sm, 1, om, b.t, x.t)
    for rev in (False, True):
        ctx.smooth(3, "mvs", 1, 0.8, b.t, x.t, reverse=rev)
    torch.cuda.synchronize()
    assert x.guards_intact() and b.guards_intact() and y.guards_intact()
    assert torch.equal(b.t, b0), "b is read-only"
    assert torch.isfinite(x.t).all()
    ctx.close()


@pytest.mark.parametrize("d,k,L", [(2, 2, 5), (2, 4, 4), (2, 7, 3), (3, 2, 4), (3, 4, 3)])
def test_transfers_and_solvers_stay_in_bounds(d, k, L):
    from paper_2412_05082_b200 import api
    ctx = api.Context(d, k, L)
    nf, nc = ctx.n_dofs(L), ctx.n_dofs(L - 1)
    f, c = Guarded(nf, torch.float64, rand(nf, torch.float64, 3), 21), Guarded(nc, torch.float64, None, 22)
    ctx.restrict(L, f.t, c.t)
    c0 = c.t.clone()
    ctx.prolongate_add(L, c.t, f.t)
    torch.cuda.synchronize()
    assert f.guards_intact() and c.guards_intact()
    assert torch.equal(c.t, c0), "prolongate_add reads the coarse vector only"
    b = Guarded(nf, torch.float64, ctx.rhs(L), 23)
    xs = Guarded(nf, torch.float64, torch.zeros(nf, dtype=torch.float64, device=DEV), 24)
    b0 = b.t.clone()
    om = 0.25 if d == 2 else 0.1
    _, rep, _ = ctx.pcg(api.MG("avs", 2, om), b.t, xs.t, max_iter=40)
    _, rep2, _ = ctx.gmres(api.MG("mvs", 1, 0.8 if d == 2 else 0.7, symmetric=False), b.t,
                           torch.zeros_like(b.t), max_iter=40, restart=10)
    z = Guarded(nf, torch.float64, None, 25)
    ctx.vcycle(api.MG("mvs", 1, 0.8, cycle_dtype=torch.float32), b.t, z.t)
    torch.cuda.synchronize()
    assert b.guards_intact() and xs.guards_intact() and z.guards_intact()
    assert torch.equal(b.t, b0), "the right-hand side is read-only"
    assert rep["converged"] and rep2["converged"]
    ctx.close()
