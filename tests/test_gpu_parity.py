"""GPU parity: arrow_spmm (sm_100a kernels, via the C ABI) against the oracle O1.

Bars (BASELINE.json north_star):
  * fp64: bitwise equal to O1 on dyadic data (every partial sum is exact, so any summation
    order and the L2 atomics of the head slices give the exact result), and golden sha256(Y);
  * fp32: ||Y - Y_O1||_F / ||Y_O1||_F <= 1e-4, plus an element-wise bound
    |Y - Y_O1| <= 1e-5 * (|A| |X|)  (fp32 accumulation of <= 1e5 nonnegative terms).
Sizes span several tiles and windows with ragged tails; k covers odd widths and every
vector/lane configuration; plus empty, n <= b, star, level-capped residual, permuted order,
host-buffer entry point, and the full configs G and R at the bench's launch configuration
(R on sampled rows).
"""
import hashlib
import json
import os

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2402_19364_b200 as ab  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = {g["graph"]: g for g in json.load(open(os.path.join(ROOT, "tests", "golden", "a10_golden.json")))["instances"]}
FP32_FRO = 1e-4
FP32_ELEM = 1e-5


def run(plan, X):
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    Y = plan.spmm(Xd)
    torch.cuda.synchronize()
    return Y.cpu().numpy()


def absbound(g, X):
    """|A| |X| row-wise (the scale of each output element)."""
    return oracle.spmm(g.n, g.row_ptr, g.col, np.abs(g.val), np.abs(X).astype(np.float64))


def check_fp32(g, Y, X):
    ref = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X)
    Y = Y.astype(np.float64)
    den = np.linalg.norm(ref)
    fro = np.linalg.norm(Y - ref) / den if den > 0 else np.linalg.norm(Y)
    assert fro <= FP32_FRO, fro
    assert np.all(np.abs(Y - ref) <= FP32_ELEM * absbound(g, X) + 1e-30)
    return fro


@pytest.mark.parametrize("spec,b,k", [("RMAT(12,4,1)", 256, 16), ("PATH(1000,1)", 4, 8), ("GRID(64,1)", 64, 8),
                                      ("RMAT(16,8,1)", 256, 8), ("GRID(256,1)", 256, 8), ("PATH(10,1)", 2, 1)])
def test_fp64_golden_bitwise(spec, b, k):
    g = datagen.make_graph(spec)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, b, dtype="f64")
    X = datagen.make_x(g.n, k)
    Y = run(plan, X)
    assert np.array_equal(Y, oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))
    assert hashlib.sha256(Y.astype("<f8").tobytes()).hexdigest() == GOLD[spec]["sha_y"]
    assert plan.sha256() == GOLD[spec]["sha_dec"]


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 8, 12, 16, 31, 32, 33, 64, 96, 128, 130, 256, 260])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_k_sweep(k, dtype):
    g = datagen.rmat(11, 8, 3)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 64, dtype=dtype, window_rows=128, head_chunk=7)
    X = datagen.make_x(g.n, k, dtype=np.float64 if dtype == "f64" else np.float32)
    Y = run(plan, X)
    if dtype == "f64":
        assert np.array_equal(Y, oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))
    else:
        check_fp32(g, Y, X)


@pytest.mark.parametrize("window_rows,head_chunk", [(0, 0), (1, 1), (300, 3), (1 << 20, 1 << 20)])
def test_layout_options(window_rows, head_chunk):
    g = datagen.rmat(12, 8, 2)
    X = datagen.make_x(g.n, 32)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 100, dtype="f64", window_rows=window_rows, head_chunk=head_chunk)
    assert np.array_equal(run(plan, X), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))


def test_random_values_fp64_tolerance():
    """Non-dyadic random values: fp64 within 1e-12 (north_star)."""
    g = datagen.rmat(12, 8, 4)
    rng = np.random.default_rng(0)
    S = g.to_scipy()
    S.data = rng.standard_normal(S.nnz)
    S = (S + S.T).tocsr()
    S.sort_indices()
    X = rng.standard_normal((g.n, 24))
    plan = ab.Plan(g.n, S.indptr, S.indices, S.data, 128, dtype="f64")
    Y = run(plan, X)
    ref = oracle.spmm(g.n, S.indptr, S.indices, S.data, X)
    assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) <= 1e-12
    # asymmetric VALUES with a symmetric pattern are allowed (R21)
    S2 = g.to_scipy()
    S2.data = rng.standard_normal(S2.nnz)
    plan2 = ab.Plan(g.n, S2.indptr, S2.indices, S2.data, 128, dtype="f64")
    ref2 = oracle.spmm(g.n, S2.indptr, S2.indices, S2.data, X)
    assert np.linalg.norm(run(plan2, X) - ref2) / np.linalg.norm(ref2) <= 1e-12


@pytest.mark.parametrize("spec,b", [("STAR(50)", 2), ("RMAT(6,4,1)", 1000), ("CYCLE(9)", 2), ("TREE(3000,5)", 8),
                                    ("WEB(12,2)", 64), ("PATH(2,1)", 2)])
def test_degenerate_and_shapes(spec, b):
    g = datagen.make_graph(spec)
    X = datagen.make_x(g.n, 8)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, b, dtype="f64")
    assert np.array_equal(run(plan, X), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))


def test_empty_matrix_zeroes_y():
    plan = ab.Plan(7, np.zeros(8, np.int64), np.zeros(0, np.int32), np.zeros(0), 2, dtype="f64")
    Y = torch.full((7, 3), 5.0, dtype=torch.float64, device="cuda")
    plan.spmm(torch.ones((7, 3), dtype=torch.float64, device="cuda"), Y)
    torch.cuda.synchronize()
    assert torch.all(Y == 0)


def test_residual_level_and_permuted_order():
    g = datagen.rmat(12, 8, 1)
    X = datagen.make_x(g.n, 16)
    ref = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 32, levels=2, residual="csr", dtype="f64")
    assert plan.info()["residual_nnz"] > 0
    assert np.array_equal(run(plan, X), ref)
    # pi_0 order: X and Y rows permuted by perm_0 (row p <-> vertex perm_0[p])
    pp = ab.Plan(g.n, g.row_ptr, g.col, g.val, 32, dtype="f64", order="permuted")
    perm0 = pp.export_level(0)[0]
    Yp = run(pp, X[perm0])
    assert np.array_equal(Yp, ref[perm0])


def test_host_entry_point_and_repeat():
    g = datagen.rmat(12, 8, 5)
    X = datagen.make_x(g.n, 32, dtype=np.float32)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 256, dtype="f32")
    Yh = plan.spmm_host(X)
    Yd = run(plan, X)
    # fp32 head-row partials are added atomically (order not fixed), so two calls agree to rounding
    np.testing.assert_allclose(Yh, Yd, rtol=1e-5, atol=1e-5)
    check_fp32(g, Yh, X)
    check_fp32(g, Yd, X)
    # repeated calls are deterministic in fp64 and k may change between calls
    p64 = ab.Plan(g.n, g.row_ptr, g.col, g.val, 256, dtype="f64")
    for k in (8, 64, 8):
        X = datagen.make_x(g.n, k)
        assert np.array_equal(run(p64, X), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))


def test_host_batch_pipelined():
    """arrow_spmm_host_batch: every item equals O1 bitwise (fp64, dyadic), with pinned and pageable
    host buffers, an odd count (both slots reused), then k changing; fp32 within 1e-4."""
    g = datagen.rmat(12, 8, 5)
    p64 = ab.Plan(g.n, g.row_ptr, g.col, g.val, 256, dtype="f64")
    for k, pinned in ((16, True), (16, False), (40, True)):
        Xs = [datagen.make_x(g.n, k, s_x=100 + c) for c in range(5)]
        if pinned:
            Xs = [torch.from_numpy(X).pin_memory().numpy() for X in Xs]
            Ys = [torch.empty((g.n, k), dtype=torch.float64).pin_memory().numpy() for _ in Xs]
        else:
            Ys = None
        Ys = p64.spmm_host_batch(Xs, Ys)
        for X, Y in zip(Xs, Ys):
            assert np.array_equal(Y, oracle.spmm(g.n, g.row_ptr, g.col, g.val, X))
    p32 = ab.Plan(g.n, g.row_ptr, g.col, g.val, 256, dtype="f32")
    Xs = [datagen.make_x(g.n, 128, s_x=7 + c, dtype=np.float32) for c in range(3)]
    for X, Y in zip(Xs, p32.spmm_host_batch(Xs)):
        check_fp32(g, Y, X)
    assert p32.spmm_host_batch([]) == []
    with pytest.raises(ValueError):
        p32.spmm_host_batch([Xs[0], Xs[0][:, :64]])


def test_profiling_counters():
    g = datagen.rmat(12, 8, 5)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 256, dtype="f32")
    X = torch.from_numpy(datagen.make_x(g.n, 128, dtype=np.float32)).cuda()
    plan.set_profiling(True)
    for _ in range(3):
        plan.spmm(X)
    kt = plan.kernel_times()
    L = plan.info()["levels"]
    assert kt["calls"] == 3 and 3 <= kt["segments"]["launches"] <= 3 * L and kt["segments"]["ms"] > 0


def test_errors_on_device():
    g = datagen.rmat(10, 8, 5)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 64, dtype="f32")
    X = torch.zeros((g.n, 8), dtype=torch.float32, device="cuda")
    with pytest.raises(ab.ArrowError) as e:
        plan.spmm_ptr(X.data_ptr(), X.data_ptr(), 8, 0)   # aliasing
    assert e.value.code == "ARROW_E_INVALID_ARG"
    with pytest.raises(ab.ArrowError):
        plan.spmm_ptr(0, X.data_ptr(), 8, 0)
    with pytest.raises(ValueError):
        plan.spmm(X.double())


def test_config_G_full():
    """Config G (GRID(1024), b=4096, k=32, fp32) in full, element by element."""
    inst = GOLD["GRID(1024,1)"]
    g = datagen.make_graph(inst["graph"])
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, inst["b"], dtype="f32")
    assert plan.sha256() == inst["sha_dec"]
    X = datagen.make_x(g.n, 32, dtype=np.float32)
    check_fp32(g, run(plan, X), X)
    p64 = ab.Plan(g.n, g.row_ptr, g.col, g.val, inst["b"], dtype="f64")
    Y64 = run(p64, datagen.make_x(g.n, 32))
    assert hashlib.sha256(Y64.astype("<f8").tobytes()).hexdigest() == inst["sha_y"]


@pytest.mark.slow
def test_config_R_sampled():
    """Config R (RMAT(22,8,1), b=16384, k=128, fp32) at the bench's launch configuration; the
    oracle checks sampled output rows (all head vertices of every level + random rows), plus
    the golden structure hash and fp64 golden sha256(Y) at k=128."""
    inst = GOLD["RMAT(22,8,1)"]
    g = datagen.make_graph(inst["graph"])
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, inst["b"], dtype="f32")
    info = plan.info()
    assert info["levels"] == inst["levels"]
    assert [plan.level_info(i)["n_i"] for i in range(info["levels"])] == inst["n_i"]
    X = datagen.make_x(g.n, 128, dtype=np.float32)
    Xd = torch.from_numpy(X).cuda()
    Y = plan.spmm(Xd)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    heads = np.concatenate([plan.export_level(i)[0][:plan.level_info(i)["head"]] for i in range(info["levels"])])
    rows = np.unique(np.concatenate([heads, rng.integers(0, g.n, 20000)]))
    Ys = Y[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64)
    ref = oracle.spmm_rows(g.row_ptr, g.col, g.val, X, rows)
    assert np.linalg.norm(Ys - ref) / np.linalg.norm(ref) <= FP32_FRO
    S = g.to_scipy()
    bound = (abs(S)[rows] @ np.abs(X.astype(np.float64)))
    assert np.all(np.abs(Ys - ref) <= FP32_ELEM * bound + 1e-30)
    del Xd, Y
    p64 = ab.Plan(g.n, g.row_ptr, g.col, g.val, inst["b"], dtype="f64")
    Y64 = p64.spmm(torch.from_numpy(datagen.make_x(g.n, 128)).cuda())
    torch.cuda.synchronize()
    assert hashlib.sha256(Y64.cpu().numpy().astype("<f8").tobytes()).hexdigest() == inst["sha_y"]


def test_graph_replay_on_a_stream():
    """On a non-default stream a single-GPU call is captured once into a CUDA graph and replayed;
    new X contents, a new Y buffer and a new k must all give the oracle's result (fp64, bitwise)."""
    g = datagen.rmat(12, 8, 6)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 128, dtype="f64")
    s = torch.cuda.Stream()
    for k, reps in ((16, 3), (8, 2), (16, 2)):
        Y = torch.empty((g.n, k), dtype=torch.float64, device="cuda")
        Xd = torch.empty((g.n, k), dtype=torch.float64, device="cuda")
        for r in range(reps):
            X = datagen.make_x(g.n, k, s_x=10 + r)
            Xd.copy_(torch.from_numpy(X))
            torch.cuda.synchronize()
            plan.spmm(Xd, Y, stream=s)
            s.synchronize()
            assert np.array_equal(Y.cpu().numpy(), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X)), (k, r)


@pytest.mark.parametrize("order,flags", [("original", 0), ("permuted", 0), ("original", 2)])
def test_iterate_relu(order, flags):
    """NEXT-1: X_{t+1} = relu(A X_t) with the activation fused into K-A, against the oracle applied
    step by step (fp64; one iteration is exact on dyadic data, more within 1e-12); flags = 2: the
    deterministic mode, whose head partials land after the last level (activation after K-C)."""
    g = datagen.rmat(13, 8, 7)
    rng = np.random.default_rng(5)
    # signed values so that ReLU is not the identity: a(u,v) -> +-a(u,v), symmetric
    S = g.to_scipy().tocoo()
    sign = np.where(((S.row.astype(np.int64) * 1315423911 + S.col) ^ (S.col.astype(np.int64) * 1315423911 + S.row)) & 4, -1.0, 1.0)
    S.data = S.data * sign
    S = S.tocsr()
    S.sort_indices()
    plan = ab.Plan(g.n, S.indptr, S.indices, S.data, 128, dtype="f64", order=order, flags=flags)
    perm0 = plan.export_level(0)[0] if order == "permuted" else np.arange(g.n)
    k = 16
    X0 = datagen.make_x(g.n, k) - 0.5
    for iters, exact in ((1, True), (2, False), (4, False)):
        ref = X0.copy()
        for _ in range(iters):
            ref = np.maximum(oracle.spmm(g.n, S.indptr, S.indices, S.data, ref), 0.0)
        Xd = torch.from_numpy(np.ascontiguousarray(X0[perm0])).cuda()
        out = plan.spmm_iterate(Xd, iters, "relu")
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        want = ref[perm0]
        if exact:
            assert np.array_equal(got, want), (iters, np.abs(got - want).max())
        else:
            assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12
    # identity activation == repeated arrow_spmm
    Xd = torch.from_numpy(np.ascontiguousarray(X0[perm0])).cuda()
    out = plan.spmm_iterate(Xd, 1, "none")
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.spmm(g.n, S.indptr, S.indices, S.data, X0)[perm0])


@pytest.mark.parametrize("spec,b,k", [("RMAT(12,4,1)", 256, 16), ("GRID(256,1)", 256, 8), ("RMAT(16,8,1)", 256, 128),
                                      ("PATH(1000,1)", 4, 3), ("WEB(12,2)", 64, 32), ("RMAT(14,8,3)", 1000, 33)])
@pytest.mark.parametrize("order", ["original", "permuted"])
def test_strict_band_parity(spec, b, k, order):
    """NEXT-2: plans built with the strict band (|p-q| <= b, P:253 / Fig. 3).  Structure bit-exact
    against the oracle's strict decomposition; fp64 Y bitwise equal to O1 on dyadic data; fp32
    within the north-star tolerance."""
    g = datagen.make_graph(spec)
    ref = oracle.la_decompose(g.n, g.row_ptr, g.col, g.val, b, band="strict")
    p64 = ab.Plan(g.n, g.row_ptr, g.col, g.val, b, dtype="f64", band="strict", order=order)
    assert p64.sha256() == oracle.decomposition_sha256(ref)
    X = datagen.make_x(g.n, k)
    perm0 = ref.levels[0].perm if order == "permuted" else np.arange(g.n)
    Y = run(p64, X[perm0])
    Yo = oracle.spmm(g.n, g.row_ptr, g.col, g.val, X)
    assert np.array_equal(Y, Yo[perm0])
    p32 = ab.Plan(g.n, g.row_ptr, g.col, g.val, b, dtype="f32", band="strict", order=order)
    X32 = X.astype(np.float32)
    Y32 = run(p32, X32[perm0])
    out = np.empty_like(Y32)
    out[perm0] = Y32
    check_fp32(g, out, X32)


# ---------------------------------------------------------------- offsets beyond 32 bits, config W
_BIG = {}


def _big_decomposition(spec, b):
    if (spec, b) not in _BIG:
        _BIG.clear()
        g = datagen.make_graph(spec)
        _BIG[(spec, b)] = (g, ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b))
    return _BIG[(spec, b)]


def _sampled_check(g, plan, X, dtype, extra_rows=()):
    """Run the plan on X and compare sampled rows (random, the last 2000 -- the largest X/Y byte
    offsets --, every level's head vertices, extra_rows) with O1: fp64 bitwise (dyadic data),
    fp32 within the Frobenius and element-wise bounds."""
    Xd = torch.from_numpy(X).cuda()
    Y = plan.spmm(Xd)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    lv = plan.info()["levels"]
    heads = np.concatenate([plan.export_level(i)[0][:plan.level_info(i)["head"]] for i in range(lv)])
    rows = np.unique(np.concatenate([heads, rng.integers(0, g.n, 20000), np.arange(max(0, g.n - 2000), g.n),
                                     np.asarray(extra_rows, np.int64)])).astype(np.int64)
    Ys = Y[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.float64)
    del Xd, Y
    torch.cuda.empty_cache()
    ref = oracle.spmm_rows(g.row_ptr, g.col, g.val, X, rows)
    if dtype == "f64":
        assert np.array_equal(Ys, ref)
        return
    assert np.linalg.norm(Ys - ref) / np.linalg.norm(ref) <= FP32_FRO
    bound = oracle.spmm_rows(g.row_ptr, g.col, np.abs(g.val), np.abs(X).astype(np.float64), rows)
    assert np.all(np.abs(Ys - ref) <= FP32_ELEM * bound + 1e-30)


@pytest.mark.slow
@pytest.mark.parametrize("spec,b,k,dtype", [("RMAT(23,8,1)", 32768, 256, "f32"),   # full-warp rows, 2 slabs
                                            ("RMAT(23,8,1)", 32768, 128, "f64"),   # fp64 full-warp rows
                                            ("PATH(33554432,1)", 4096, 64, "f32")])  # 8-byte-lane rows
def test_offsets_beyond_4GiB(spec, b, k, dtype):
    """X and Y of 8 GiB each (n k s > 2^32): every gather, store and read-modify-write address above
    4 GiB must be formed in 64 bits.  Sampled rows include the last 2000 rows (largest offsets)."""
    g, dec = _big_decomposition(spec, b)
    assert g.n * k * (8 if dtype == "f64" else 4) > 2 ** 32
    plan = ab.Plan(decomposition=dec, dtype=dtype)
    X = datagen.make_x(g.n, k, dtype=np.float64 if dtype == "f64" else np.float32)
    _sampled_check(g, plan, X, dtype)
    plan.close()


@pytest.mark.slow
def test_config_W_sampled():
    """Config W (web-like WEB(24,1): 168 M nnz, b = 65536, 5 levels, k = 32 fp32) at the bench's
    launch configuration, on sampled rows (the short-row kernel k_segsmall), plus fp64 bitwise."""
    g, dec = _big_decomposition("WEB(24,1)", 65536)
    for dtype in ("f32", "f64"):
        plan = ab.Plan(decomposition=dec, dtype=dtype)
        X = datagen.make_x(g.n, 32, dtype=np.float64 if dtype == "f64" else np.float32)
        _sampled_check(g, plan, X, dtype)
        plan.close()
    _BIG.clear()


def test_capture_inside_torch_cuda_graph():
    """a caller that captures arrow_spmm into its own CUDA graph (torch.cuda.graph) gets the
    kernels in that graph (the library skips its internal graph while the stream is capturing);
    arrow_plan_reserve sizes every workspace first.  Replays with new X contents match O1 bitwise."""
    g = datagen.rmat(12, 8, 7)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 128, dtype="f64")
    k = 16
    plan.reserve(k)
    X = torch.from_numpy(datagen.make_x(g.n, k, s_x=21)).cuda()
    Y = torch.empty_like(X)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    plan.spmm(X, Y, stream=s)  # warm-up outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        plan.spmm(X, Y, stream=s)
    for r in range(3):
        Xh = datagen.make_x(g.n, k, s_x=30 + r)
        X.copy_(torch.from_numpy(Xh))
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(Y.cpu().numpy(), oracle.spmm(g.n, g.row_ptr, g.col, g.val, Xh)), r


@pytest.mark.parametrize("k", [128, 32, 8])
def test_deterministic_flag_bitwise_repeatable(k):
    """ARROW_FLAG_DETERMINISTIC (S2/S3 without atomics: per-(head row, window) partial slots added in
    a fixed order by K-C): fp32 results are bitwise identical call to call and within the fp32
    bounds of O1; fp64 equals O1 bitwise on dyadic data; the k = 8/32 short-row kernels too."""
    g = datagen.rmat(13, 8, 5)
    X = datagen.make_x(g.n, k, dtype=np.float32)
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, 256, dtype="f32", flags=ab.arrow.FLAG_DETERMINISTIC,
                   window_rows=1024)
    Y1, Y2 = run(plan, X), run(plan, X)
    assert np.array_equal(Y1.view(np.uint32), Y2.view(np.uint32))
    check_fp32(g, Y1, X)
    p64 = ab.Plan(g.n, g.row_ptr, g.col, g.val, 256, dtype="f64", flags=ab.arrow.FLAG_DETERMINISTIC)
    X64 = datagen.make_x(g.n, k)
    assert np.array_equal(run(p64, X64), oracle.spmm(g.n, g.row_ptr, g.col, g.val, X64))
