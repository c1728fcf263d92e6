"""Time LA-Decompose host vs GPU (arrow_decompose_ex / arrow_decompose_gpu) on the survey's configs.
ARROW_DECOMPOSE_TRACE=1 prints the per-phase split on stderr.  Usage: python profiles/r02/gd_time.py [spec:b ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("ARROW_DECOMPOSE_TRACE", "1")
import datagen
import paper_2402_19364_b200 as ab

specs = sys.argv[1:] or ["GRID(1024,1):4096", "RMAT(22,8,1):16384", "RMAT(24,8,1):65536"]
import torch
torch.zeros(1, device="cuda")  # context up front
for sb in specs:
    spec, b = sb.rsplit(":", 1)
    g = datagen.make_graph(spec)
    row = {"graph": spec, "b": int(b), "n": g.n, "nnz": int(g.row_ptr[-1])}
    for dev in ("cuda", "cuda", "cpu"):
        t0 = time.perf_counter()
        D = ab.Decomposition(g.n, g.row_ptr, g.col, g.val, int(b), device=dev)
        row[dev] = round(time.perf_counter() - t0, 3)
        row["levels"] = D.info()["levels"]
        if dev == "cpu":
            row["same"] = D.sha256() == sha
        else:
            sha = D.sha256()
        del D
    print(row, flush=True)
