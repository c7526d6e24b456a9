"""Distributed slab path on the GPU: two ranks on cuda:0 with gloo (ghost rows staged through host
memory), against the single-domain library and the oracle.  One process per rank (torch.multiprocessing)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(fn, world, *args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=600)
        out[r] = res
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        if isinstance(out[r], str):
            raise AssertionError(f"rank {r}: {out[r]}")
    return out


def _entry(fn, rank, world, port, q, *args):
    import traceback
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        q.put((rank, globals()[fn](rank, world, *args)))
    except Exception:
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _mvs_step(rank, world, d, k, N, omega):
    import torch
    from paper_2412_05082_b200 import api
    from paper_2412_05082_b200.dist import partition, exchange
    from c0ip_inputs import random_xb
    L = 3
    ctx = api.Context(d, k, L, cells_override=N)
    n = k * N - 1
    row = n ** (d - 1)
    x, b = random_xb(k, d, N)
    s = partition(N, k, world, 4 * k - 2)[rank]
    rows = slice(s.row0, s.row0 + s.lrows)
    xw = torch.tensor(x.reshape(-1, row)[rows].ravel(), device="cuda:0")
    bw = torch.tensor(b.reshape(-1, row)[rows].ravel(), device="cuda:0")
    rw = torch.empty_like(xw)
    for c in range(2 ** (d + 1)):
        exchange(xw, s, row)
        ctx.slab_mvs_color(L, omega, c, s.row0, s.lrows, s.own_lo, s.own_hi, bw, xw, rw)
    own = xw.view(-1, row)[s.own_local].cpu().numpy()
    ctx.close()
    return (s.own_lo, s.own_hi, own)


@pytest.mark.parametrize("d,k,N,omega", [(2, 3, 32, 0.8), (2, 4, 24, 0.8), (2, 6, 16, 0.8), (3, 2, 16, 0.7),
                                         (3, 4, 12, 0.7)])
def test_slab_mvs_step_bitwise_equals_single_domain(d, k, N, omega):
    """Colours in lockstep across 2 ranks, one ghost exchange per colour: the gathered MVS step equals the
    single-domain step bitwise (same kernels, identical inputs on the straddling patches)."""
    from paper_2412_05082_b200 import api
    from c0ip_inputs import random_xb
    out = _run("_mvs_step", 2, d, k, N, omega)
    ctx = api.Context(d, k, 3, cells_override=N)
    x, b = random_xb(k, d, N)
    xt = torch.tensor(x, device="cuda:0")
    ctx.smooth(3, "mvs", 1, omega, torch.tensor(b, device="cuda:0"), xt)
    full = xt.cpu().numpy().reshape(-1, (k * N - 1) ** (d - 1))
    ctx.close()
    for r, (lo, hi, own) in out.items():
        assert np.array_equal(own, full[lo - 1: hi - 1]), r


def _pcg(rank, world, d, k, L, kind, steps, omega, solver="cg"):
    import torch
    from paper_2412_05082_b200 import api
    from paper_2412_05082_b200.dist import DistMG, DistPCG, DistGMRES
    ctx = api.Context(d, k, L)
    b = ctx.rhs(L)
    mg = DistMG(ctx, kind, steps, omega, symmetric=(solver == "cg"))
    lev = mg.levels[L]
    s = lev.slab
    bw = b.view(-1, lev.row)[s.row0: s.row0 + s.lrows].reshape(-1).clone()
    x, n, hist = (DistPCG(mg) if solver == "cg" else DistGMRES(mg)).solve(bw)
    own = lev.owned(x).cpu().numpy()
    res = (s.own_lo, s.own_hi, own, n, hist, sorted(mg.levels), mg.exchanges)
    ctx.close()
    return res


@pytest.mark.parametrize("d,k,L,kind,steps,omega", [(2, 2, 5, "avs", 2, 0.25), (2, 4, 5, "mvs", 1, 0.8),
                                                    (3, 2, 4, "avs", 2, 0.1)])
def test_distributed_pcg_matches_oracle(d, k, L, kind, steps, omega):
    """MG-PCG on 2 slabs (distributed levels + agglomerated coarse cycle, all-reduced dots): the iteration count
    within 1 of the oracle's PCG with the same cycle, the gathered solution at the tolerance of the FP64 solve."""
    from oracle.multigrid import Hierarchy, pcg, precondition
    from oracle.operator import paper_rhs
    from oracle.discretization import default_sigma
    out = _run("_pcg", 2, d, k, L, kind, steps, omega)
    s = default_sigma(k)
    h = Hierarchy(k, d, L, s)
    bo = paper_rhs(k, d, 2 ** L, s)
    xo, no, ho = pcg(h.A[L], bo, lambda r: precondition(h, r, kind, steps, omega))
    row = (k * 2 ** L - 1) ** (d - 1)
    xg = np.zeros_like(xo).reshape(-1, row)
    for r, (lo, hi, own, n, hist, levels, nx) in out.items():
        assert abs(n - no) <= 1, (r, n, no, levels)
        xg[lo - 1: hi - 1] = own.reshape(-1, row)
        assert len(levels) >= 2                       # at least two distributed levels
    xg = xg.ravel()
    assert np.linalg.norm(xg - xo) <= 1e-6 * np.linalg.norm(xo)
    assert np.linalg.norm(bo - h.A[L] @ xg) <= 1.05e-8 * np.linalg.norm(bo)


def _avs_overlap(rank, world, d, k, N, omega):
    import torch
    from paper_2412_05082_b200 import api
    from paper_2412_05082_b200.dist import partition, exchange, avs_step_overlapped
    from c0ip_inputs import random_xb
    ctx = api.Context(d, k, 3, cells_override=N)
    n = k * N - 1
    row = n ** (d - 1)
    x, b = random_xb(k, d, N)
    s = partition(N, k, world, 4 * k - 2)[rank]
    rows = slice(s.row0, s.row0 + s.lrows)
    xw = torch.tensor(x.reshape(-1, row)[rows].ravel(), device="cuda:0")
    bw = torch.tensor(b.reshape(-1, row)[rows].ravel(), device="cuda:0")
    rw = torch.empty_like(xw)
    x2 = xw.clone()
    avs_step_overlapped(ctx, 3, omega, s, row, bw, xw, rw)
    exchange(x2, s, row)
    ctx.slab_avs_step(3, omega, s.row0, s.lrows, s.own_lo, s.own_hi, bw, x2, torch.empty_like(x2))
    own, ref = xw.view(-1, row)[s.own_local].cpu().numpy(), x2.view(-1, row)[s.own_local].cpu().numpy()
    ctx.close()
    return bool(np.array_equal(own, ref))


@pytest.mark.parametrize("d,k,N,omega", [(2, 4, 32, 0.25), (2, 3, 40, 0.25), (3, 2, 16, 0.1), (3, 3, 16, 0.1)])
def test_overlapped_avs_step_equals_slab_step(d, k, N, omega):
    """Residual of the interior rows during the halo exchange, boundary strips after it, then c0ip_slab_fdm:
    bitwise the same owned rows as c0ip_slab_avs_step."""
    out = _run("_avs_overlap", 2, d, k, N, omega)
    assert all(out.values()), out


@pytest.mark.parametrize("d,k,L,omega", [(2, 4, 5, 0.8), (3, 2, 4, 0.7)])
def test_distributed_gmres_mvs_matches_oracle(d, k, L, omega):
    """The paper's MVS protocol on 2 slabs: FGMRES around the same-order (nonsymmetric) MVS V-cycle with colours in
    lockstep; iteration count within 1 of the oracle's FGMRES, gathered solution at the tolerance."""
    from oracle.multigrid import Hierarchy, gmres, precondition
    from oracle.operator import paper_rhs
    from oracle.discretization import default_sigma
    out = _run("_pcg", 2, d, k, L, "mvs", 1, omega, "gmres")
    s = default_sigma(k)
    h = Hierarchy(k, d, L, s)
    bo = paper_rhs(k, d, 2 ** L, s)
    xo, no, ho = gmres(h.A[L], bo, lambda r: precondition(h, r, "mvs", 1, omega, symmetric=False))
    row = (k * 2 ** L - 1) ** (d - 1)
    xg = np.zeros_like(xo).reshape(-1, row)
    for r, (lo, hi, own, n, hist, levels, nx) in out.items():
        assert abs(n - no) <= 1, (r, n, no)
        xg[lo - 1: hi - 1] = own.reshape(-1, row)
    xg = xg.ravel()
    floor = 32 * 2.2e-16 * np.linalg.norm(abs(h.A[L]) @ np.abs(xg))        # SURVEY.md F9 rounding floor
    assert np.linalg.norm(bo - h.A[L] @ xg) <= 1.05e-8 * np.linalg.norm(bo) + floor
