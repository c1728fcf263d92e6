"""Worker for the multi-GPU parity test: one process per GPU, NCCL comm from arrow_comm_*; each rank
computes its pi_0 row shard of Y = A X and checks it against the oracle O1 rows (fp64: bitwise on
dyadic data; fp32: 1e-4 Frobenius and the element-wise bound |Y - Y_O1| <= 1e-5 (|A| |X|) of
tests/test_gpu_parity.py).  The transport comes from ARROW_TEST_TRANSPORT (auto | p2p | nccl, passed as
options.transport).  Run under torchrun or spawned by tests/test_gpu_dist.py."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (graph, b, widths used in successive calls, dtype): the width changes between calls re-allocate
# (and, for the P2P transport, re-share) the workspaces; every call uses a fresh X
CASES = [("RMAT(12,8,1)", 64, (16, 16, 16), "f64"), ("RMAT(14,8,2)", 256, (128, 128, 128), "f32"),
         ("RMAT(13,8,4)", 128, (64, 128, 64), "f64"), ("RMAT(13,8,5)", 512, (32, 64, 32), "f32"),
         ("GRID(128,1)", 256, (32, 32), "f64"), ("TREE(5000,3)", 16, (8, 8), "f64"),
         ("RMAT(10,4,3)", 1024, (4, 4), "f64"), ("PATH(3000,1)", 8, (3, 5), "f64"),
         # strict band (|p - q| <= b): level-0 and level->=1 rows read X rows of the neighbouring ranks
         ("RMAT(13,8,4)", 128, (64, 16), "f64", "strict"), ("GRID(128,1)", 256, (32,), "f32", "strict"),
         ("PATH(3000,1)", 8, (3,), "f64", "strict"), ("RMAT(12,8,1)", 32, (8,), "f64", "strict"),
         # home-set-aware levels >= 1 for this world size (R25, ARROW_FLAG_HOME_AWARE)
         ("RMAT(13,8,4)", 128, (64, 16), "f64", "block", "homes"), ("RMAT(14,8,2)", 256, (128,), "f32", "block", "homes"),
         ("GRID(128,1)", 256, (32,), "f64", "strict", "homes")]


def run(rank, world, port):
    import torch
    import torch.distributed as dist
    import datagen
    import oracle
    import paper_2402_19364_b200 as ab
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(port))
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = [ab.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = ab.Comm(world, rank, uid[0])
    fails = []
    transport = os.environ.get("ARROW_TEST_TRANSPORT", "auto")
    for spec, b, ks, dtype, *extra in CASES:
        g = datagen.make_graph(spec)
        band = extra[0] if extra else "block"
        flags = ab.arrow.FLAG_HOME_AWARE if "homes" in extra else 0
        plan = ab.Plan(g.n, g.row_ptr, g.col, g.val, b, dtype=dtype, comm=comm, transport=transport,
                       band=band, flags=flags)
        lo, hi = plan.local_begin, plan.local_end
        perm0 = plan.export_level(0)[0]
        rows = perm0[lo:hi]
        for rep, k in enumerate(ks):
            X = datagen.make_x(g.n, k, s_x=3 + rep, dtype=np.float64 if dtype == "f64" else np.float32)
            Xl = torch.from_numpy(np.ascontiguousarray(X[rows])).cuda()
            Y = plan.spmm(Xl)
            torch.cuda.synchronize()
            Y = Y.cpu().numpy().astype(np.float64)
            ref = oracle.spmm_rows(g.row_ptr, g.col, g.val, X, rows)
            if dtype == "f64":
                ok = np.array_equal(Y, ref)
            else:
                den = np.linalg.norm(ref)
                scale = oracle.spmm_rows(g.row_ptr, g.col, np.abs(g.val), np.abs(X).astype(np.float64), rows)
                ok = ((np.linalg.norm(Y - ref) / den if den > 0 else np.linalg.norm(Y)) <= 1e-4 and
                      bool(np.all(np.abs(Y - ref) <= 1e-5 * scale + 1e-30)))
            if not ok:
                fails.append(f"{spec} b={b} {extra} k={k} call {rep} {dtype} rank {rank}: max err {np.abs(Y - ref).max()}")
        if spec == "RMAT(12,8,1)" and b == 64:
            # the batched host-buffer entry (collective): two items, copies pipelined with the kernels
            Xs = [datagen.make_x(g.n, 16, s_x=11 + c) for c in range(3)]
            Ys = plan.spmm_host_batch([np.ascontiguousarray(X[rows]) for X in Xs])
            for c, (X, Yb) in enumerate(zip(Xs, Ys)):
                if not np.array_equal(Yb, oracle.spmm_rows(g.row_ptr, g.col, g.val, X, rows)):
                    fails.append(f"{spec} host batch item {c} rank {rank}")
        plan.close()
    comm.close()
    dist.destroy_process_group()
    return fails


if __name__ == "__main__":
    r = int(os.environ.get("RANK", "0"))
    w = int(os.environ.get("WORLD_SIZE", "1"))
    f = run(r, w, 29511)
    print("DIST_OK" if not f else "DIST_FAIL " + "; ".join(f), flush=True)
    sys.exit(0 if not f else 1)
