#!/usr/bin/env python
"""Config S: Kronecker/R-MAT scales 20..24 x k in {8, 32, 128}, fp32, 1 GPU.

One process per scale list; per scale the graph and its decomposition are built once, then one plan
per k is timed like bench.py (CUDA events on a dedicated stream, graph replay, W warm-up steps).
Every line carries the HBM roofline on B_alg (measured peak) and a bounded CPU-oracle sample.
    python profiles/r02/sweep_s.py --scales 20,21,22,23,24 --ks 8,32,128 > gpurun_out/r02/S/s.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scales", default="20,21,22,23,24")
    ap.add_argument("--ks", default="8,32,128")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=4.0)
    args = ap.parse_args()
    import torch
    import paper_2402_19364_b200 as ab
    dev = torch.device("cuda", 0)
    peak, peak_src = bench.load_peaks()
    for scale in [int(x) for x in args.scales.split(",")]:
        t0 = time.time()
        g = datagen.make_graph(f"RMAT({scale},8,1)")
        b = (1 << scale) // 256
        dec = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, b)
        t_dec = time.time() - t0
        for k in [int(x) for x in args.ks.split(",")]:
            # the bench's window choice: library default at 512-byte rows, ~8 MB of rows below
            win = 0 if k * 4 >= 512 else min(16384 * min(4, 512 // (k * 4)), max(16384, g.n // 64))
            plan = ab.Plan(decomposition=dec, dtype="f32", window_rows=win)
            X = datagen.make_x(g.n, k, dtype=np.float32)
            Xd = torch.from_numpy(X).to(dev)
            Yd = torch.empty_like(Xd)
            st = torch.cuda.Stream(dev)
            for _ in range(args.warmup):
                plan.spmm_ptr(Xd.data_ptr(), Yd.data_ptr(), k, st.cuda_stream)
            torch.cuda.synchronize()
            clocks = bench.ClockSampler(0)
            clocks.start()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.steps):
                plan.spmm_ptr(Xd.data_ptr(), Yd.data_ptr(), k, st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            clk = clocks.stop()
            ms = e0.elapsed_time(e1) / args.steps
            flop = 2.0 * g.nnz * k
            balg = plan.bytes_alg(k)
            cpu = bench.cpu_oracle_baseline(g, X, k, budget_s=args.cpu_budget, max_reps=3)
            info = plan.info()
            line = {"metric": bench.METRIC, "config": {"workload": f"config S: RMAT({scale},8,1) b={b} k={k}",
                                                        "n": g.n, "nnz": g.nnz, "k": k, "b": b,
                                                        "levels": info["levels"], "sum_n_i": info["sum_rows"]},
                    "dtype": "f32", "value": round(flop / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                    "ms_per_step": round(ms, 4), "steps": args.steps, "warmup": args.warmup,
                    "roofline": {"bound": "hbm", "bytes_alg_per_step": balg,
                                 "achieved": round(balg / (ms * 1e-3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                                 "frac": round(balg / (ms * 1e-3) / 1e9 / peak, 4), "peak_source": peak_src},
                    "cpu_baseline": {k2: cpu[k2] for k2 in ("value", "unit", "cores", "kind", "sample")},
                    "clocks": clk, "decompose_s": round(t_dec, 1)}
            print(json.dumps(line), flush=True)
            plan.close()
            del Xd, Yd
            torch.cuda.empty_cache()
        dec.close()


if __name__ == "__main__":
    main()
