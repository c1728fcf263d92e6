"""NEXT-4 comparator: the 1.5D A-stationary SpMM, run in real gloo worlds on CPU.

Each rank's Y tile must equal rows [B_i, B_{i+1}) of a dense brute-force A X (fp64; numpy dense
product, independent of the comparator's sparse pieces), for p = 2 (c = 1: the 1D case, 2 rounds),
p = 4 (c = 2: one round, all-reduce over the grid row) and p = 8 (c = 2, 2 rounds).  The
ledger must add up to P:322's beta term nk/c + nkc/p (within the ring all-reduce factor).
"""
import os

import numpy as np
import pytest

import datagen
from comparators.one_five_d import grid_c, ledger, tile_bounds


def test_grid_c():
    # c = floor(sqrt(p)), lowered so that c^2 | p (P:320's p/c^2 rounds)
    assert [grid_c(p) for p in (1, 2, 3, 4, 6, 8, 9, 16, 18)] == [1, 1, 1, 2, 1, 2, 3, 4, 3]


@pytest.mark.parametrize("p", [2, 4, 8])
def test_ledger_totals(p):
    n, k, es = 1000, 16, 8
    c = grid_c(p)
    L = [ledger(n, k, es, p, c, r) for r in range(p)]
    q = p // c
    B = tile_bounds(n, q)
    for r, l in enumerate(L):
        i, j = divmod(r, c)
        col_rows = B[(j + 1) * (q // c)] - B[j * (q // c)]   # the n/c rows of column block j
        own = (B[i + 1] - B[i]) if j * (q // c) <= i < (j + 1) * (q // c) else 0
        assert l["bcast_recv_bytes"] == (col_rows - own) * k * es
        # received bytes never exceed P:322's beta term
        assert l["bcast_recv_bytes"] + l["allreduce_bytes"] <= l["predicted_beta_bytes"] + k * es * c


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from comparators.one_five_d import OneFiveD
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = datagen.make_graph("RMAT(9,6,3)")
        rng = np.random.default_rng(7)
        X = rng.standard_normal((g.n, 8))
        Ad = np.zeros((g.n, g.n))
        rows = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
        np.add.at(Ad, (rows, g.col), g.val)
        Yref = Ad @ X
        op = OneFiveD(g.n, g.row_ptr, g.col, g.val, 8, torch.float64, rank, world, torch.device("cpu"))
        r0, r1 = op.row_range
        Y = op.step(torch.from_numpy(X[r0:r1].copy())).numpy()
        err = float(np.abs(Y - Yref[r0:r1]).max() / max(1.0, np.abs(Yref).max()))
        q.put((rank, "ok" if err < 1e-12 else f"err {err}", op.c, op.rounds))
    except Exception as e:  # report, do not hang the other ranks' queue reads
        q.put((rank, f"exc {e!r}", 0, 0))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_one_five_d_gloo(world):
    import multiprocessing as mp
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
    c = grid_c(world)
    assert all(r[2] == c and r[3] == world // c // c for r in res), res
