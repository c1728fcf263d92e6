"""Distributed routing (host logic of the NCCL path) checked on CPU.

Every rank computes its own part of the schedule from the same decomposition (dist.cpp::dist_schedule);
NCCL send/recv pairs only match if, for every level and every pair (a, b), the rows a sends to b
equal the rows b expects from a (forward exchange of X rows, Alg. 2; reverse exchange of
results going home).  Also: the pi_0 row ranges partition [0, n), the local work
partitions every level's entries (Eq. (1)), heads are owned exactly once, level-0 zero rows are
exactly the entry-less rows.  Checked in one process for several world sizes and in a real
2-process gloo world (torch.distributed) exchanging the schedules.
"""
import os

import numpy as np
import pytest

import datagen
import paper_2402_19364_b200 as ab


def _dec(spec="RMAT(12,8,1)", b=64, band="block", homes=1):
    g = datagen.make_graph(spec)
    return g, ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b, band=band, homes=homes)


def check_schedules(g, D, scheds, strict=False):
    G = len(scheds)
    assert scheds[0]["lo"] == 0 and scheds[-1]["hi"] == g.n
    for a in range(G - 1):
        assert scheds[a]["hi"] == scheds[a + 1]["lo"]
    nl = D.info()["levels"]
    for i in range(nl):
        li = D.level_info(i)
        perm, rp, col, val = D.export_level(i)
        for a in range(G):
            for bb in range(G):
                sa, sb = scheds[a]["levels"][i], scheds[bb]["levels"][i]
                assert sa["send"][bb] == sb["recv"][a], (i, a, bb)
                assert sa["out"][bb] == sb["in"][a], (i, a, bb)
        assert sum(s["levels"][i]["entries"] for s in scheds) == li["nnz"]
        assert sum(s["levels"][i]["heads"] for s in scheds) == li["head"]
        if i > 0:
            # every level-i vertex outside the head is fetched exactly once (strict band: at least once,
            # plus the rows within b of a rank's tile range that its body rows read), every non-empty
            # body row goes home once
            fetched = sum(int(s["levels"][i]["recv"].sum()) for s in scheds)
            if strict:
                assert fetched >= li["n_i"] - li["head"]
            else:
                assert fetched == li["n_i"] - li["head"]
            nonempty = int((np.diff(rp)[li["head"]:] > 0).sum())
            assert sum(int(s["levels"][i]["out"].sum()) for s in scheds) == nonempty
    perm0, rp0, col0, _ = D.export_level(0)
    h0 = D.level_info(0)["head"]
    n0 = D.level_info(0)["n_i"]
    assert sum(s["levels"][0]["zero_rows"] for s in scheds) == int((np.diff(rp0)[h0:] == 0).sum())
    # level 0: a rank receives exactly the distinct non-head columns outside its pi_0 range that its
    # body rows read (none for the block band: a tile never leaves its rank), each from that column's home
    for a, s in enumerate(scheds):
        lo, hi = s["lo"], s["hi"]
        need = set()
        for p in range(max(h0, lo), min(hi, n0)):
            for q in col0[rp0[p]:rp0[p + 1]]:
                if q >= h0 and not lo <= q < hi:
                    need.add(int(q))
        if not strict:
            assert not need
        homes = np.zeros(len(scheds), np.int64)
        for q in need:
            homes[[t for t, z in enumerate(scheds) if z["lo"] <= q < z["hi"]][0]] += 1
        assert np.array_equal(s["levels"][0]["recv"], homes), (a, s["levels"][0]["recv"], homes)


@pytest.mark.parametrize("G", [1, 2, 3, 5, 8])
def test_schedule_consistency_single_process(G):
    g, D = _dec()
    check_schedules(g, D, [D.dist_schedule(G, r) for r in range(G)])


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("spec,b", [("RMAT(12,8,1)", 64), ("GRID(48,2)", 32), ("PATH(2000,3)", 16)])
def test_schedule_strict_band(G, spec, b):
    g, D = _dec(spec, b, band="strict")
    check_schedules(g, D, [D.dist_schedule(G, r) for r in range(G)], strict=True)


@pytest.mark.parametrize("G", [2, 3, 4, 8])
@pytest.mark.parametrize("band", ["block", "strict"])
def test_schedule_home_aware(G, band):
    """R25: a decomposition made for G homes uses its home ranges as the pi_0 split and gives rank g
    the tiles of home g's trees; schedules for another rank count fall back to the cost split."""
    g, D = _dec("RMAT(13,8,2)", 128, band=band, homes=G)
    sc = [D.dist_schedule(G, r) for r in range(G)]
    check_schedules(g, D, sc, strict=band == "strict")
    los = D.homes(-1)[1]
    assert [s["lo"] for s in sc] == list(los[:-1]) and sc[-1]["hi"] == los[-1]
    other = 2 if G != 2 else 3
    check_schedules(g, D, [D.dist_schedule(other, r) for r in range(other)], strict=band == "strict")


def test_schedule_more_ranks_than_tiles():
    g, D = _dec("RMAT(8,4,1)", 128)
    check_schedules(g, D, [D.dist_schedule(6, r) for r in range(6)])


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, D = _dec("GRID(48,2)", 64)
    s = D.dist_schedule(world, rank)
    mine = [s]
    allv = [None] * world
    dist.all_gather_object(allv, mine[0])
    try:
        check_schedules(g, D, allv)
        q.put((rank, "ok"))
    except AssertionError as e:
        q.put((rank, f"fail {e}"))
    dist.destroy_process_group()


def test_schedule_gloo_world2():
    import multiprocessing as mp
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
