"""The C-ABI library (CPU-side checks; no GPU compute).

* libarrow_b200.so loads and exports every function include/arrow.h declares.
* The host decomposer behind arrow_plan_create (arrow_decompose) reproduces the oracle's
  decomposition bit-exactly (north_star: "Structure and indexing results must match the
  oracle bit-exact") and the survey's golden hashes.
* Error paths of §8(b): bad CSR, asymmetric pattern, b < 2, level cap, NULLs, save/load.
* Without a CUDA device, plan creation fails loudly (no CPU fallback).
"""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import datagen
import oracle
import paper_2402_19364_b200 as ab
from paper_2402_19364_b200.arrow import ArrowError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "a10_golden.json")))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "arrow.h")).read()
    declared = set(re.findall(r"^\s*(?:arrow_status|const char \*|int32_t)\s*\*?\s*(arrow_\w+)\s*\(", hdr, re.M))
    assert declared == set(ab.SYMBOLS), declared ^ set(ab.SYMBOLS)
    L = ab.lib()
    for s in declared:
        assert hasattr(L, s), s
    assert L.arrow_abi_version() == 1
    for i, name in enumerate(ab.STATUS):
        assert L.arrow_status_string(i).decode() == name


def _oracle_dec(g, b, levels=0):
    return oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, levels=levels)


@pytest.mark.parametrize("spec,b", [("RMAT(10,8,1)", 64), ("RMAT(12,4,1)", 256), ("GRID(40,2)", 32),
                                    ("PATH(300,3)", 4), ("TREE(500,2)", 8), ("WEB(11,3)", 64),
                                    ("RMAT(9,8,7)", 3), ("STAR(20)", 2), ("CYCLE(50)", 2), ("PATH(2,1)", 2),
                                    ("RMAT(11,8,5)", 2), ("RMAT(13,8,2)", 4096)])
def test_decomposer_bit_exact_vs_oracle(spec, b):
    g = datagen.make_graph(spec)
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b)
    ref = _oracle_dec(g, b)
    assert D.info()["levels"] == ref.order
    for i, lv in enumerate(ref.levels):
        perm, rp, col, val = D.export_level(i)
        assert np.array_equal(perm, lv.perm) and np.array_equal(rp, lv.row_ptr)
        assert np.array_equal(col, lv.col) and np.array_equal(val.view(np.int64), lv.val.view(np.int64))
        li = D.level_info(i)
        assert (li["n_i"], li["head"], li["nnz"]) == (lv.n_i, lv.head, lv.nnz)
    assert D.sha256() == oracle.decomposition_sha256(ref)


@pytest.mark.parametrize("seed", [1, 7, 12345])
def test_decomposer_seeds(seed):
    g = datagen.rmat(11, 6, seed)
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 32, seed=seed)
    ref = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, 32, seed=seed)
    assert D.sha256() == oracle.decomposition_sha256(ref)


@pytest.mark.parametrize("inst", [g for g in GOLD["instances"] if not g.get("large")], ids=lambda g: g["graph"])
def test_decomposer_golden(inst):
    g = datagen.make_graph(inst["graph"])
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, inst["b"])
    assert D.sha256() == inst["sha_dec"]


@pytest.mark.slow
@pytest.mark.parametrize("inst", [g for g in GOLD["instances"] if g.get("large")], ids=lambda g: g["graph"])
def test_decomposer_golden_large(inst):
    g = datagen.make_graph(inst["graph"])
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, inst["b"])
    assert [D.level_info(i)["n_i"] for i in range(D.info()["levels"])] == inst["n_i"]
    assert D.sha256() == inst["sha_dec"]


def test_level_cap_and_residual():
    g = datagen.rmat(10, 8, 1)
    with pytest.raises(ArrowError) as e:
        ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, levels=2)
    assert e.value.code == "ARROW_E_LEVELS"
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 16, levels=2, keep_residual=True)
    ref = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, 16, levels=2)
    assert D.info()["levels"] == 2
    u, v, a = D.export_residual()
    ru, rv, ra = ref.residual
    o = np.lexsort((rv, ru))
    assert np.array_equal(u, ru[o]) and np.array_equal(v, rv[o]) and np.array_equal(a, ra[o])


def test_save_load_roundtrip(tmp_path):
    g = datagen.rmat(11, 8, 3)
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 64, levels=3, keep_residual=True)
    p = str(tmp_path / "dec.bin")
    D.save(p)
    E = ab.Decomposition.load(p)
    assert E.info() == D.info() and E.sha256() == D.sha256()
    assert all(np.array_equal(a, b) for a, b in zip(E.export_residual(), D.export_residual()))
    raw = bytearray(open(p, "rb").read())
    raw[100] ^= 0xFF
    open(p, "wb").write(bytes(raw))
    with pytest.raises(ArrowError):
        ab.Decomposition.load(p)
    with pytest.raises(ArrowError):
        ab.Decomposition.load(str(tmp_path / "missing.bin"))


def test_error_paths():
    g = datagen.path(10, None)
    with pytest.raises(ArrowError) as e:
        ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 1)
    assert e.value.code == "ARROW_E_INVALID_ARG"
    with pytest.raises(ArrowError) as e:
        ab.Decomposition(g.n, g.row_ptr, g.col, g.val, 4, levels=-1)
    assert e.value.code == "ARROW_E_INVALID_ARG"
    # asymmetric pattern
    rp = np.array([0, 1, 1], np.int64)
    with pytest.raises(ArrowError) as e:
        ab.Decomposition(2, rp, np.array([1], np.int32), np.ones(1), 2)
    assert e.value.code == "ARROW_E_NOT_SYMMETRIC"
    # unsorted / duplicate / out-of-range columns, bad row_ptr
    bad = [
        (np.array([0, 2, 4], np.int64), np.array([1, 0, 0, 1], np.int32)),   # unsorted row 0
        (np.array([0, 2, 3], np.int64), np.array([1, 1, 0], np.int32)),      # duplicate
        (np.array([0, 1, 2], np.int64), np.array([5, 0], np.int32)),         # out of range
        (np.array([1, 1, 2], np.int64), np.array([1, 0], np.int32)),         # row_ptr[0] != 0
    ]
    for rp, col in bad:
        with pytest.raises(ArrowError) as e:
            ab.Decomposition(2, rp, col, np.ones(len(col)), 2)
        assert e.value.code == "ARROW_E_BAD_CSR"
    # NULL output pointer / NULL A
    L = ab.lib()
    assert L.arrow_decompose(None, 2, 0, 4, 0, None) == 1
    assert L.arrow_plan_info(None, None) == 1
    assert L.arrow_plan_destroy(None) == 0
    # empty matrix -> order 0
    D = ab.Decomposition(5, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0), 2)
    assert D.info()["levels"] == 0
    # self-loops are accepted (R21) and captured
    rp = np.array([0, 2, 4, 5], np.int64)
    col = np.array([0, 1, 0, 1, 2], np.int32)
    D = ab.Decomposition(3, rp, col, np.ones(5), 2)
    assert sum(D.level_info(i)["nnz"] for i in range(D.info()["levels"])) == 5


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    g = datagen.rmat(8, 4, 1)
    with pytest.raises(ArrowError) as e:
        ab.Plan(g.n, g.row_ptr, g.col, g.val, 16)
    assert e.value.code == "ARROW_E_CUDA"
