"""Multi-process (gloo, world_size 2, CPU) tests of the slab decomposition host logic:
partition coverage and the ghost-row exchange that precedes every slab smoothing step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_05082_b200.dist import partition, exchange_ghosts


@pytest.mark.parametrize("N,k,R", [(16, 2, 2), (64, 4, 4), (585, 7, 8), (33, 3, 3)])
def test_partition_covers_rows_once(N, k, R):
    g = 4 * k - 2
    slabs = partition(N, k, R, g)
    owned = np.concatenate([np.arange(s.own_lo, s.own_hi) for s in slabs])
    assert np.array_equal(owned, np.arange(1, k * N))
    for s in slabs:
        assert s.win_lo == max(1, s.own_lo - g) and s.win_hi == min(k * N, s.own_hi + g)
        assert s.own_lo % k == 0 or s.own_lo == 1          # cuts at cell boundaries (vertex rows)


def test_partition_rejects_thin_slabs():
    with pytest.raises(ValueError):
        partition(8, 4, 8, 14)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, N, k, row_len, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = k * N - 1
        glob = torch.arange(n * row_len, dtype=torch.float64)           # global rows, row-major
        s = partition(N, k, world, 4 * k - 2)[rank]
        x = glob.view(n, row_len)[s.win_lo - 1:s.win_hi - 1].clone().reshape(-1)
        xv = x.view(-1, row_len)
        xv[: s.own_lo - s.win_lo] = -1.0                                 # poison ghosts
        xv[s.own_hi - s.win_lo:] = -1.0
        got = exchange_ghosts(x, s, row_len)
        ok = torch.equal(x, glob.view(n, row_len)[s.win_lo - 1:s.win_hi - 1].reshape(-1))
        q.put((rank, ok, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,k", [(16, 2), (12, 3)])
def test_ghost_exchange_gloo_world2(N, k):
    world, row_len = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, k, row_len, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    g = 4 * k - 2
    assert all(got == g * row_len * 8 for _, _, got in res)
