#!/usr/bin/env python
"""Benchmark of the arrow-decomposition SpMM hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config R] [--k 128] [--dtype f32]
    python bench.py --impl reference ...        # the oracle (O1, CPU) on the same workload

Metric (BASELINE.json): "SpMM GFLOP/s and HBM-roofline % at 1/2/4/8 B200 (k=32,128)".
A step = one arrow_spmm(plan, X, Y, k) = every §8(a) row (head stage, body rows + head
slices, head epilogue, per level) over the whole synthetic input; FLOP = 2 nnz k.
Workload at N=1: config R = RMAT(22,8,1) (65.2M nnz), b = 16384, k = 128, fp32 -- the
configuration BASELINE.json's target is quoted on.  X and Y are 2 GiB each (> L2), so
consecutive steps need no L2 flush.  Timing: CUDA events on the launching stream, W warm-up
steps, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

CONFIGS = {
    "T": dict(graph="RMAT(12,4,1)", b=256, k=16, dtype="f64"),
    "G": dict(graph="GRID(1024,1)", b=4096, k=32, dtype="f32"),
    "R": dict(graph="RMAT(22,8,1)", b=16384, k=128, dtype="f32"),
    "S20": dict(graph="RMAT(20,8,1)", b=4096, k=128, dtype="f32"),
    "S21": dict(graph="RMAT(21,8,1)", b=8192, k=128, dtype="f32"),
    "S23": dict(graph="RMAT(23,8,1)", b=32768, k=128, dtype="f32"),
    "S24": dict(graph="RMAT(24,8,1)", b=65536, k=128, dtype="f32"),
    "W": dict(graph="WEB(24,1)", b=65536, k=32, dtype="f32"),
}
METRIC = "SpMM GFLOP/s and HBM-roofline % at 1/2/4/8 B200 (k=32,128)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def load_traffic(config, k, dtype):
    """ncu-measured DRAM bytes per step of the dominant kernel, from a committed summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t.get(f"{config}:k{k}:{dtype}")
    except Exception:
        return None


class ClockSampler:
    """NVML clocks + throttle reasons sampled every 20 ms while running."""

    def __init__(self, dev_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for name, bit in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.02)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": sorted(self.reasons)}


def make_inputs(cfg, k, dtype):
    g = datagen.make_graph(cfg["graph"])
    X = datagen.make_x(g.n, k, dtype=np.float64 if dtype == "f64" else np.float32)
    return g, X


def cpu_oracle_baseline(g, X, k, budget_s=12.0, max_reps=10):
    """O1 (oracle/spmm_ref.c, fp64, OpenMP over rows) on the host cores: full SpMMs repeated
    until ~budget_s of CPU work (bounded sample of the same workload)."""
    import oracle
    threads = len(os.sched_getaffinity(0))
    oracle.spmm(g.n, g.row_ptr, g.col, g.val, X, nthreads=threads)  # warm-up (page-in)
    times = []
    t_all = time.perf_counter()
    while len(times) < max_reps and (time.perf_counter() - t_all) < budget_s:
        t0 = time.perf_counter()
        oracle.spmm(g.n, g.row_ptr, g.col, g.val, X, nthreads=threads)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    gflops = 2.0 * g.nnz * k / t / 1e9
    # one core (SURVEY §8 acceptance 5): O1 on every 16th output row, one thread, ~5 s of work
    rows = np.arange(0, g.n, 16, dtype=np.int64)
    nnz_s = int((g.row_ptr[rows + 1] - g.row_ptr[rows]).sum())
    t1s = []
    t_all = time.perf_counter()
    while len(t1s) < 5 and (time.perf_counter() - t_all) < 5.0:
        t0 = time.perf_counter()
        oracle.spmm_rows(g.row_ptr, g.col, g.val, X, rows, nthreads=1)
        t1s.append(time.perf_counter() - t0)
    t1 = statistics.median(t1s)
    return {"value": round(gflops, 3), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
            "sample": f"{len(times)} full SpMMs Y=AX of the same A and X in fp64 (median {t:.3f} s each, "
                      f"1 warm-up), oracle/spmm_ref.c with OpenMP over rows",
            "one_core": {"value": round(2.0 * nnz_s * k / t1 / 1e9, 3), "unit": "GFLOP/s", "cores": 1,
                         "sample": f"every 16th output row ({len(rows)} rows, {nnz_s} entries), "
                                   f"median of {len(t1s)}: {t1:.3f} s"}}


def cusparse_baseline(g, Xd, k, flop, stream, reps=10):
    """Library comparator (SURVEY §8 acceptance 5): the same Y = A X with cuSPARSE CSR SpMM through
    torch.sparse.mm on the same device-resident X, timed with CUDA events like our own step."""
    import torch
    try:
        dev = Xd.device
        A = torch.sparse_csr_tensor(torch.from_numpy(g.row_ptr.astype(np.int64)).to(dev),
                                    torch.from_numpy(g.col.astype(np.int64)).to(dev),
                                    torch.from_numpy(g.val.astype(np.float32 if Xd.dtype == torch.float32 else np.float64)).to(dev),
                                    size=(g.n, g.n))
        with torch.cuda.stream(stream):
            for _ in range(3):
                Y = torch.sparse.mm(A, Xd)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                Y = torch.sparse.mm(A, Xd)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        del A, Y
        torch.cuda.empty_cache()
        return {"impl": "cuSPARSE CSR SpMM via torch.sparse.mm (same X, device-resident)", "ms_per_step": round(ms, 4),
                "value": round(flop / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "steps": reps}
    except Exception as e:  # a comparator, not the product: report why it did not run
        return {"impl": "cuSPARSE via torch.sparse.mm", "unavailable": str(e)[:200]}


def one_d_baseline(g, X, k, dtype, world, rank, dev, flop, steps=10):
    """SURVEY §8(e) comparator: 1D-row SpMM -- rank r owns rows [n r/G, n (r+1)/G) of A and X,
    all-gathers X over NCCL and multiplies its row block with cuSPARSE (torch.sparse.mm).
    Device-timed like our step (barrier + CUDA events, max over ranks)."""
    import torch
    import torch.distributed as dist
    try:
        n = g.n
        lo, hi = n * rank // world, n * (rank + 1) // world
        rp = g.row_ptr[lo:hi + 1].astype(np.int64)
        npdt = np.float64 if dtype == "f64" else np.float32
        A = torch.sparse_csr_tensor(torch.from_numpy(rp - rp[0]).to(dev),
                                    torch.from_numpy(g.col[rp[0]:rp[-1]].astype(np.int64)).to(dev),
                                    torch.from_numpy(g.val[rp[0]:rp[-1]].astype(npdt)).to(dev), size=(hi - lo, n))
        # equal-sized shards for all_gather_into_tensor: pad the row count to ceil(n / G)
        per = (n + world - 1) // world
        Xl = torch.zeros((per, k), dtype=torch.float64 if dtype == "f64" else torch.float32, device=dev)
        Xl[:hi - lo] = torch.from_numpy(np.ascontiguousarray(X[lo:hi])).to(dev)
        Xf = torch.empty((per * world, k), dtype=Xl.dtype, device=dev)

        def step():
            dist.all_gather_into_tensor(Xf, Xl)
            # rows of rank r sit at [r*per, r*per + (its rows)); with n % G == 0 this is X itself
            return torch.sparse.mm(A, Xf[:n] if n % world == 0 else torch.cat([Xf[r * per:r * per + (n * (r + 1) // world - n * r // world)] for r in range(world)]))

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        del A, Xl, Xf
        torch.cuda.empty_cache()
        return {"impl": "1D-row: NCCL all_gather of X + cuSPARSE row-block SpMM (torch.sparse.mm)",
                "ms_per_step": round(ms, 4), "value": round(flop / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                "allgather_bytes_per_gpu": int((world - 1) * per * k * (8 if dtype == "f64" else 4))}
    except Exception as e:
        return {"impl": "1D-row baseline", "unavailable": str(e)[:200]}


def one_five_d_baseline(g, X, k, dtype, world, rank, dev, flop, steps=10):
    """NEXT-4 comparator: the paper's 1.5D A-stationary SpMM with c = floor(sqrt(p))
     -- NCCL broadcasts along grid columns, cuSPARSE local products, an all-reduce of the
    Y tile (comparators/one_five_d.py).  Device-timed like our step (barrier + CUDA events, max over
    ranks); the ledger is the bytes a rank receives per step vs P:322's beta term."""
    import torch
    import torch.distributed as dist
    try:
        from comparators.one_five_d import OneFiveD
        tdt = torch.float64 if dtype == "f64" else torch.float32
        op = OneFiveD(g.n, g.row_ptr, g.col, g.val, k, tdt, rank, world, dev)
        r0, r1 = op.row_range
        Xt = torch.from_numpy(np.ascontiguousarray(X[r0:r1])).to(dev)
        for _ in range(3):
            op.step(Xt)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            op.step(Xt)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        led = op.ledger(8 if dtype == "f64" else 4)
        mx = torch.tensor([led["bcast_recv_bytes"] + led["allreduce_bytes"]], dtype=torch.float64, device=dev)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        del op, Xt
        torch.cuda.empty_cache()
        return {"impl": f"1.5D A-stationary (c={led['c']}, {led['rounds']} round(s)): NCCL broadcast + cuSPARSE + all-reduce",
                "ms_per_step": round(ms, 4), "value": round(flop / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                "recv_bytes_per_gpu_max": int(mx.item()), "predicted_beta_bytes": led["predicted_beta_bytes"]}
    except Exception as e:
        return {"impl": "1.5D A-stationary baseline", "unavailable": str(e)[:200]}


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle as it stands, on this arm's config and metric (rank 0 only)."""
    if rank != 0:
        return
    k, dtype = args.k or cfg["k"], args.dtype or cfg["dtype"]
    g, X = make_inputs(cfg, k, dtype)
    import oracle
    # every host core this process may use: torchrun sets OMP_NUM_THREADS=1 for each rank, which
    # would time the oracle on one core when the driver launches the reference arm with N > 1
    threads = len(os.sched_getaffinity(0))
    oracle.spmm(g.n, g.row_ptr, g.col, g.val, X, nthreads=threads)  # page-in
    times = []
    for _ in range(args.warmup):
        oracle.spmm(g.n, g.row_ptr, g.col, g.val, X, nthreads=threads)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.spmm(g.n, g.row_ptr, g.col, g.val, X, nthreads=threads)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    flop = 2.0 * g.nnz * k
    val = flop / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config {args.config}: {cfg['graph']} b={cfg['b']} k={k}", "n": g.n, "nnz": g.nnz,
                   "k": k, "b": cfg["b"]},
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
                         "sample": f"each step = one full fp64 SpMM of the workload on the host (oracle/spmm_ref.c)"},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="R", choices=sorted(CONFIGS))
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--dtype", default="", choices=["", "f32", "f64"])
    ap.add_argument("--impl", default="arrow", choices=["arrow", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--order", default="original", choices=["original", "permuted"],
                    help="X/Y row order: original vertex ids, or pi_0 order (R18; forced when distributed)")
    ap.add_argument("--iterate", type=int, default=10, help="iterations of the fused-ReLU iterate timing (0: skip)")
    ap.add_argument("--no-lib-baseline", action="store_true", help="skip the cuSPARSE (torch.sparse) comparator")
    ap.add_argument("--band", default="block", choices=["block", "strict"],
                    help="LA-Decompose step 3 band: block-diagonal tiles (R3) or strict |p-q| <= b (NEXT-2)")
    ap.add_argument("--transport", default="auto", choices=["auto", "p2p", "nccl"],
                    help="distributed plans: peer memory over NVLink (p2p) or NCCL broadcast/send/recv/reduce")
    ap.add_argument("--window-rows", type=int, default=0)
    ap.add_argument("--head-chunk", type=int, default=0)
    ap.add_argument("--batch-segments", type=int, default=0)
    ap.add_argument("--flags", type=int, default=0, help="arrow_options.flags (ARROW_FLAG_*)")
    ap.add_argument("--home-aware", action=argparse.BooleanOptionalAction, default=True,
                    help="N > 1: decompose with home-set-aware levels >= 1 for the N ranks (R25; default on)")
    ap.add_argument("--home-levels", type=int, default=0,
                    help="--home-aware: levels 1..L use same-home forests (0 = the library default for N ranks)")
    ap.add_argument("--gpu-decompose", action=argparse.BooleanOptionalAction, default=True,
                    help="decompose on the GPU (N = 1: the plan's own decomposition; N > 1: rank 0's; default on)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2402_19364_b200 as ab

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    k, dtype = args.k or cfg["k"], args.dtype or cfg["dtype"]
    es = 8 if dtype == "f64" else 4
    g, X = make_inputs(cfg, k, dtype)
    # tile window of the layout (profiles/r02/win/, S2/): the library default for 512-byte rows (level 0
    # 65,536 rows, levels >= 1 16,384); for shorter rows up to ~8 MB of X rows but at most n/64 rows
    # (config R k=32: 65,536 rows, -4.7 %; RMAT scale 20 was 14-19 % slower with 65,536)
    n_cfg = g.n
    window_rows = args.window_rows or (0 if k * es >= 512 else
                                       min(16384 * min(4, 512 // (k * es)), max(16384, n_cfg // 64)))

    comm = None
    if world > 1:
        uid = [ab.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ab.Comm(world, rank, uid[0])
    dec = None
    decompose_s = [None]
    if world > 1:
        # one decomposition for the node (on rank 0's GPU by default, home-aware for the N ranks): rank 0
        # computes and checkpoints it, the others load it (arrow_decomposition_save/load)
        import tempfile
        path = [os.path.join(tempfile.mkdtemp(prefix="arrow_bench_"), "A.dec") if rank == 0 else None]
        dist.broadcast_object_list(path, src=0)
        if rank == 0:
            t0 = time.perf_counter()
            dec = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, cfg["b"], band=args.band,
                                   homes=world if args.home_aware else 1, home_levels=args.home_levels,
                                   device="cuda" if args.gpu_decompose else "cpu")
            decompose_s[0] = time.perf_counter() - t0
            dec.save(path[0])
        dist.barrier()
        if rank != 0:
            dec = ab.Decomposition.load(path[0])
        dist.barrier()
        if rank == 0:
            os.remove(path[0])
            os.rmdir(os.path.dirname(path[0]))
    home_levels_used = dec.home_levels() if dec is not None else 0
    plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, cfg["b"], dtype=dtype, comm=comm, decomposition=dec,
                   order=("permuted" if comm is not None else args.order),
                   window_rows=window_rows, head_chunk=args.head_chunk, batch_segments=args.batch_segments,
                   band=args.band, transport=args.transport,
                   flags=args.flags | (ab.arrow.FLAG_GPU_DECOMPOSE if (args.gpu_decompose and dec is None) else 0))
    info = plan.info()
    lo, hi = plan.local_begin, plan.local_end
    if comm is not None or args.order == "permuted":
        perm0 = plan.export_level(0)[0]
        Xl = X[perm0[lo:hi]]
    else:
        Xl = X
    plan.reserve(k)
    stream = torch.cuda.Stream(dev)
    Xd = torch.from_numpy(np.ascontiguousarray(Xl)).to(dev)
    Yd = torch.empty_like(Xd)
    torch.cuda.synchronize()

    def step():
        plan.spmm_ptr(Xd.data_ptr(), Yd.data_ptr(), k, stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    # second timed pass with per-kernel CUDA events (plan profiling) for the kernel breakdown and the
    # K-A roofline; kept separate so that the event records do not inflate the step time above
    if world > 1:
        dist.barrier()
    plan.set_profiling(True)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof_step_ms = p0.elapsed_time(p1) / args.steps
    kt = plan.kernel_times()
    plan.set_profiling(False)
    clk = clocks.stop()
    t_tensor = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_tensor, op=dist.ReduceOp.MAX)
    ms_per_step = float(t_tensor.item()) / args.steps

    flop = 2.0 * g.nnz * k
    gflops = flop / (ms_per_step * 1e-3) / 1e9
    b_alg = plan.bytes_alg(k)

    # dominant kernel (K-A segment stream): algorithmic bytes of its launches per step
    s = es
    ka_bytes = 0
    ka_launches = 0
    for i in range(info["levels"] + (1 if info["residual_nnz"] else 0)):
        li = plan.level_info(i)
        y_rows = (li["rows"] - li["head"]) if i == 0 else 2 * (li["n_i"] - li["head"])
        ka_bytes += li["nnz"] * (s + 4) + (li["rows"] + 1) * 8 + li["rows"] * 4 + li["n_i"] * k * s + y_rows * k * s
        ka_launches += 1
    # K-A's share of the step, measured with per-kernel CUDA events in the profiled pass (graph replay
    # off), applied to the graph-replayed timed step: the kernel's time can never exceed the step's
    ka_share = min(1.0, (kt["segments"]["ms"] / max(1, kt["calls"])) / prof_step_ms)
    ka_ms_per_step = ka_share * ms_per_step
    peak, peak_src = load_peaks()
    # distributed: each rank runs ~1/G of every level's entries and rows (cost-balanced split), so its
    # K-A launches move ~ka_bytes / G; the fraction is that per-rank share over the per-rank K-A time
    ka_bytes = ka_bytes // world
    achieved = ka_bytes / (ka_ms_per_step * 1e-3) / 1e9
    step_share = ka_share

    # e2e: the same call with HOST buffers (H2D of X, D2H of Y inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        Xh = torch.from_numpy(np.ascontiguousarray(Xl)).pin_memory()
        Yh = torch.empty_like(Xh).pin_memory()
        Xh_np, Yh_np = Xh.numpy(), Yh.numpy()
        plan.spmm_host(Xh_np, Yh_np, stream.cuda_stream)  # warm (allocates staging)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            plan.spmm_host(Xh_np, Yh_np, stream.cuda_stream)
        te = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": round(flop / float(te.item()) / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(Xl.nbytes) * world, "d2h_bytes_per_step": int(Xl.nbytes) * world,
               "ms_per_step": round(float(te.item()) * 1e3, 3),
               "mode": "arrow_spmm_host per step (H2D, kernels, D2H, sync)"}
        # the batched host entry: H2D of step c+1 and D2H of step c-1 overlap the kernels of c
        # (arrow_spmm_host_batch; collective for N > 1); every step still copies its X in and its Y out
        Yh2 = torch.empty_like(Xh).pin_memory().numpy()
        nb = max(args.e2e_steps, 4)
        Xs, Ys = [Xh_np] * nb, [Yh_np if c % 2 == 0 else Yh2 for c in range(nb)]
        plan.spmm_host_batch(Xs[:2], Ys[:2], stream.cuda_stream)  # warm (allocates the slots)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        plan.spmm_host_batch(Xs, Ys, stream.cuda_stream)
        tbt = torch.tensor([(time.perf_counter() - t0) / nb], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tbt, op=dist.ReduceOp.MAX)
        tb = float(tbt.item())
        e2e.update({"value": round(flop / tb / 1e9, 3), "ms_per_step": round(tb * 1e3, 3),
                    "mode": f"arrow_spmm_host_batch of {nb} steps (copies pipelined with the kernels)",
                    "sequential": {"value": e2e["value"], "ms_per_step": e2e["ms_per_step"],
                                   "mode": e2e["mode"]}})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_baseline(g, X, k)
    # NEXT-1: iterated X_{t+1} = relu(A X_t) with the activation fused into K-A (same plan, same X)
    it = None
    if world == 1 and args.iterate > 0:
        Xi = Xd.clone()
        Yi = torch.empty_like(Xd)
        with torch.cuda.stream(stream):
            plan.spmm_iterate(Xi, 2, "relu", Yi, stream=stream)
            i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            Xi.copy_(Xd)
            i0.record(stream)
            plan.spmm_iterate(Xi, args.iterate, "relu", Yi, stream=stream)
            i1.record(stream)
        torch.cuda.synchronize()
        ms_it = i0.elapsed_time(i1) / args.iterate
        it = {"activation": "relu", "iters": args.iterate, "ms_per_iter": round(ms_it, 4),
              "value": round(flop / (ms_it * 1e-3) / 1e9, 3), "unit": "GFLOP/s"}
        del Xi, Yi
    # alpha-beta ledger: the rows this rank actually exchanges (plan-time
    # routes) against the survey's prediction 2 (sum_{i>=1} n_i - h_i) k s (G-1)/G^2 + sum_i h_i k s
    nvl = None
    if world > 1 and dec is not None:
        sch = dec.dist_schedule(world, rank)
        f_send = sum(int(l["send"].sum() - l["send"][rank]) for l in sch["levels"][1:])
        f_recv = sum(int(l["recv"].sum() - l["recv"][rank]) for l in sch["levels"][1:])
        r_send = sum(int(l["out"].sum() - l["out"][rank]) for l in sch["levels"][1:])
        r_recv = sum(int(l["in"].sum() - l["in"][rank]) for l in sch["levels"][1:])
        heads = sum(dec.level_info(i)["head"] for i in range(dec.info()["levels"]))
        body1 = sum(dec.level_info(i)["n_i"] - dec.level_info(i)["head"] for i in range(1, dec.info()["levels"]))
        row_b = k * es
        mine = torch.tensor([max(f_send + r_send, f_recv + r_recv) * row_b + heads * row_b], dtype=torch.float64, device=dev)
        dist.all_reduce(mine, op=dist.ReduceOp.MAX)
        pred = 2 * body1 * row_b * (world - 1) / world ** 2 + heads * row_b
        nvl = {"rows_fwd_send": f_send, "rows_fwd_recv": f_recv, "rows_rev_send": r_send, "rows_rev_recv": r_recv,
               "bytes_per_gpu_per_direction_max": int(mine.item()), "bytes_predicted_per_gpu_per_direction": int(pred),
               "t_bound_ms_at_900GBs": round(float(mine.item()) / 900e9 * 1e3, 4),
               "note": "rank-0 row counts; bytes = max over ranks of (forward + reverse rows) x k x s + head blocks"}
    oned = oned15 = None
    if world > 1 and not args.no_lib_baseline:
        oned = one_d_baseline(g, X, k, dtype, world, rank, dev, flop)
        oned15 = one_five_d_baseline(g, X, k, dtype, world, rank, dev, flop)
    lib = None
    if rank == 0 and world == 1 and not args.no_lib_baseline:
        lib = cusparse_baseline(g, Xd, k, flop, stream)

    if rank == 0:
        # ncu DRAM bytes of the single-GPU K-A launches (profiles/traffic.json); none measured for N > 1
        traffic = load_traffic(args.config, k, dtype) if (args.band == "block" and world == 1) else None
        line = {
            "metric": METRIC, "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": f"config {args.config}: {cfg['graph']} b={cfg['b']} k={k}",
                       "n": g.n, "nnz": g.nnz, "k": k, "b": cfg["b"], "levels": info["levels"],
                       "sum_n_i": info["sum_rows"], "parallelism": f"arrow tiles over {world} GPU(s)",
                       "band": args.band,
                       "window_rows": window_rows or ("default: level 0 65536, levels >= 1 16384" if world == 1 else 16384),
                       "arrangement": ("home-aware (R25) for %d ranks, levels 1..%d" % (world, home_levels_used))
                                      if (args.home_aware and world > 1)
                                      else "random spanning forest, smallest-first (R6-R12)",
                       "order": "permuted (pi_0)" if (comm is not None or args.order == "permuted") else "original",
                       "l2": "inputs larger than L2 (X, Y %.2f GiB each), no flush" % (Xl.nbytes / 2**30)},
            # whole-job algorithmic bytes over the step against the N GPUs' aggregate HBM bandwidth
            "hbm_roofline": {"bytes_alg_per_step": b_alg, "achieved_GBs": round(b_alg / (ms_per_step * 1e-3) / 1e9, 1),
                             "frac_of_measured": round(b_alg / (ms_per_step * 1e-3) / 1e9 / (peak * world), 4),
                             "frac_of_8TBs": round(b_alg / (ms_per_step * 1e-3) / (8e12 * world), 4),
                             "gpus": world},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "K-A (k_ka for full-warp rows, k_segsmall for short rows, else k_segments)",
                         "timing": "K-A share of the step from per-kernel CUDA events (profiled pass) x the "
                                   "graph-replayed step time (timed pass)",
                         "bytes_per_step": ka_bytes, "launches_per_step": ka_launches,
                         "ms_per_step": round(ka_ms_per_step, 4), "share_of_step": round(step_share, 4),
                         "peak_source": peak_src},
            "kernel_ms_per_step": {kname: round(kt[kname]["ms"] / max(1, kt["calls"]), 4)
                                   for kname in ("head_stage", "segments", "head_epilogue", "comm")},
            "per_launch_ms": kt["launch_ms"],
            "gpu_launches": int(sum(kt[kname]["launches"] for kname in ("head_stage", "segments", "head_epilogue"))),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "library_baseline": lib if world == 1 else oned,
            "baseline_1_5d": oned15,
            "iterate": it,
            "nvlink": nvl,
            "create_seconds": round(info["create_seconds"], 2),
        }
        if decompose_s[0] is not None:
            line["decompose_seconds"] = round(decompose_s[0], 3)
        print(json.dumps(line), flush=True)
    plan.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
