"""The GPU LA-Decompose (arrow_decompose_gpu) against the host decomposer.

The host decomposer is itself pinned bit-exact to the oracle (test_boundary.py) and to the survey's
golden hashes (A.10); the GPU one must produce the identical decomposition -- same levels, heads,
permutations, canonical CSRs and values -- on every input, both bands, every seed, with and
without the level cap.  The large golden instances (configs G and R) are checked against A.10
directly and timed against the host decomposer (printed, not asserted).
"""
import json
import os
import time

import numpy as np
import pytest

import datagen
import oracle
import paper_2402_19364_b200 as ab
from paper_2402_19364_b200.arrow import FLAG_GPU_DECOMPOSE, ArrowError

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "a10_golden.json")))


def _same(Dg, Dh):
    assert Dg.info() == Dh.info()
    for i in range(Dh.info()["levels"]):
        assert Dg.level_info(i) == Dh.level_info(i), i
        for a, b in zip(Dg.export_level(i), Dh.export_level(i)):
            assert np.array_equal(a.view(np.int64) if a.dtype == np.float64 else a,
                                  b.view(np.int64) if b.dtype == np.float64 else b), i
    assert Dg.sha256() == Dh.sha256()


SPECS = [("RMAT(10,8,1)", 64), ("RMAT(12,4,1)", 256), ("GRID(40,2)", 32), ("PATH(300,3)", 4), ("TREE(500,2)", 8),
         ("WEB(11,3)", 64), ("RMAT(9,8,7)", 3), ("STAR(20)", 2), ("CYCLE(50)", 2), ("PATH(2,1)", 2),
         ("RMAT(11,8,5)", 2), ("RMAT(13,8,2)", 4096), ("RMAT(14,16,3)", 128), ("GRID(200,1)", 64)]


@pytest.mark.parametrize("spec,b", SPECS)
@pytest.mark.parametrize("band", ["block", "strict"])
def test_gpu_decomposer_matches_host(spec, b, band):
    g = datagen.make_graph(spec)
    Dh = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b, band=band)
    Dg = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b, band=band, device="cuda")
    _same(Dg, Dh)


@pytest.mark.parametrize("spec,b", [("RMAT(10,8,1)", 64), ("PATH(1000,1)", 4), ("GRID(64,1)", 64)])
def test_gpu_decomposer_matches_oracle(spec, b):
    g = datagen.make_graph(spec)
    Dg = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b, device="cuda")
    assert Dg.sha256() == oracle.decomposition_sha256(oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b))


@pytest.mark.parametrize("seed", [1, 7, 12345, 2**63 + 5])
def test_gpu_decomposer_seeds(seed):
    g = datagen.rmat(11, 6, seed % 1000)
    Dh = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 32, seed=seed)
    Dg = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 32, seed=seed, device="cuda")
    _same(Dg, Dh)


@pytest.mark.parametrize("spec,b", [("RMAT(12,8,1)", 64), ("GRID(100,1)", 32), ("RMAT(14,8,2)", 256), ("PATH(500,1)", 8)])
@pytest.mark.parametrize("homes", [2, 3, 4, 8])
@pytest.mark.parametrize("band,hl", [("block", 1), ("strict", 1), ("block", 3)])
def test_gpu_decomposer_homes(spec, b, homes, band, hl):
    """R25 (home-set-aware levels >= 1) on the GPU: the same decomposition, home ranges and starts."""
    g = datagen.make_graph(spec)
    Dh = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b, band=band, homes=homes, home_levels=hl)
    Dg = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b, band=band, homes=homes, home_levels=hl, device="cuda")
    _same(Dg, Dh)
    assert np.array_equal(Dg.homes(-1)[1], Dh.homes(-1)[1]) and Dg.home_levels() == hl
    for i in range(1, min(hl, Dh.info()["levels"] - 1) + 1):
        assert np.array_equal(Dg.homes(i)[1], Dh.homes(i)[1])


def test_gpu_decomposer_level_cap_residual():
    g = datagen.rmat(10, 8, 1)
    with pytest.raises(ArrowError) as e:
        ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, levels=2, device="cuda")
    assert e.value.code == "ARROW_E_LEVELS"
    Dh = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, levels=2, keep_residual=True)
    Dg = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, levels=2, keep_residual=True, device="cuda")
    _same(Dg, Dh)
    for a, b in zip(Dg.export_residual(), Dh.export_residual()):
        assert np.array_equal(a, b)


def test_gpu_decomposer_degenerate():
    # no entries; isolated vertices only; a single self-loop-free edge
    D = ab.Decomposition(5, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0), 2, device="cuda")
    assert D.info()["levels"] == 0
    rp = np.array([0, 1, 2, 2, 2], np.int64)
    col = np.array([1, 0], np.int32)
    Dh = ab.Decomposition(4, rp, col, np.ones(2), 2)
    Dg = ab.Decomposition(4, rp, col, np.ones(2), 2, device="cuda")
    _same(Dg, Dh)
    with pytest.raises(ArrowError):
        ab.Decomposition(4, rp, col, np.ones(2), 1, device="cuda")
    # the symmetry check runs on the device: (0, 2) without (2, 0)
    with pytest.raises(ArrowError) as e:
        ab.Decomposition(3, np.array([0, 2, 3, 3], np.int64), np.array([1, 2, 0], np.int32), np.ones(3), 2,
                         device="cuda")
    assert e.value.code == "ARROW_E_NOT_SYMMETRIC"


@pytest.mark.parametrize("inst", GOLD["instances"], ids=lambda g: g["graph"])
def test_gpu_decomposer_golden(inst):
    g = datagen.make_graph(inst["graph"])
    t0 = time.perf_counter()
    Dg = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, inst["b"], device="cuda")
    tg = time.perf_counter() - t0
    assert Dg.sha256() == inst["sha_dec"]
    if inst.get("large"):
        assert [Dg.level_info(i)["n_i"] for i in range(Dg.info()["levels"])] == inst["n_i"]
        t0 = time.perf_counter()
        ab.Decomposition(g.n, g.row_ptr, g.col, g.val, inst["b"])
        th = time.perf_counter() - t0
        print(f"\n[decompose] {inst['graph']} b={inst['b']}: host {th:.3f} s, GPU {tg:.3f} s "
              f"(x{th / tg:.2f}, host threads {os.cpu_count()})")


def test_plan_with_gpu_decompose_flag():
    import torch
    g = datagen.make_graph("RMAT(12,8,1)")
    X = torch.randn(g.n, 16, device="cuda", dtype=torch.float32)
    Ph = ab.Plan(g.n, g.row_ptr, g.col, g.val.astype(np.float32), 128)
    Pg = ab.Plan(g.n, g.row_ptr, g.col, g.val.astype(np.float32), 128, flags=FLAG_GPU_DECOMPOSE)
    for i in range(Ph.info()["levels"]):
        for a, b in zip(Pg.export_level(i), Ph.export_level(i)):
            assert np.array_equal(a, b)
    Yh, Yg = Ph.spmm(X), Pg.spmm(X)
    torch.cuda.synchronize()
    assert torch.allclose(Yh, Yg, rtol=1e-5, atol=1e-5)
