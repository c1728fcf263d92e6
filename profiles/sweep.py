"""Layout/scheduling sweep on one GPU: decompose once, build plans with different options,
time arrow_spmm with CUDA events (per-kernel times via the library's profiling events).

    python profiles/sweep.py --config R --variants "w=65536,bs=32,hc=256;w=16384,bs=8"
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import datagen  # noqa: E402
import paper_2402_19364_b200 as ab  # noqa: E402


def parse(v):
    d = {}
    for kv in v.split(","):
        if kv.strip():
            k, x = kv.split("=")
            d[k.strip()] = int(x)
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="R")
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--dtype", default="")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--variants", default="")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    k, dtype = args.k or cfg["k"], args.dtype or cfg["dtype"]
    t0 = time.time()
    g = datagen.make_graph(cfg["graph"])
    X = datagen.make_x(g.n, k, dtype=np.float64 if dtype == "f64" else np.float32)
    D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, cfg["b"])
    print(f"# gen+decompose {time.time() - t0:.1f}s", flush=True)
    Xd = torch.from_numpy(X).cuda()
    Yd = torch.empty_like(Xd)
    st = torch.cuda.Stream()
    for v in args.variants.split(";"):
        ka = None
        if ":" in v:
            ka, v = v.split(":", 1)
        os.environ["ARROW_KA"] = ka or "seg"
        o = parse(v)
        for key, env in (("ta", "ARROW_TAIL_ATOMIC"), ("sbs", "ARROW_SEG_BS")):
            if key in o:
                os.environ[env] = str(o[key])
        plan = ab.Plan(decomposition=D, dtype=dtype, window_rows=o.get("w", 0), head_chunk=o.get("hc", 0),
                       batch_segments=o.get("bs", 0))
        for _ in range(3):
            plan.spmm_ptr(Xd.data_ptr(), Yd.data_ptr(), k, st.cuda_stream)
        torch.cuda.synchronize()
        plan.set_profiling(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            plan.spmm_ptr(Xd.data_ptr(), Yd.data_ptr(), k, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        kt = plan.kernel_times()
        balg = plan.bytes_alg(k)
        print(json.dumps({"variant": v, "ms": round(ms, 4), "GBs_alg": round(balg / ms / 1e6, 1),
                          "gflops": round(2 * g.nnz * k / ms / 1e6, 1),
                          "segments_ms": round(kt["segments"]["ms"] / kt["calls"], 4),
                          "zero_ms": round(kt["head_stage"]["ms"] / kt["calls"], 4),
                          "launch_ms": kt["launch_ms"]}), flush=True)
        plan.close()


if __name__ == "__main__":
    main()
