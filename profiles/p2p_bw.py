"""Peer-to-peer bandwidth probe (copy engines and SM stores) between the GPUs of one box.

Usage (GPU box, >= 2 GPUs): python profiles/p2p_bw.py
Prints GB/s for: one copy 0->1; 0->all peers concurrently; all-to-all concurrently (every GPU
sending to every peer); the same copies while GPU 0 runs a bandwidth-heavy kernel.
"""
import torch

MB = 1 << 20


def timed(fn, devs, reps=5):
    for _ in range(2):
        fn()
    for d in devs:
        torch.cuda.synchronize(d)
    st = {d: torch.cuda.Event(enable_timing=True) for d in devs}
    en = {d: torch.cuda.Event(enable_timing=True) for d in devs}
    import time
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    for d in devs:
        torch.cuda.synchronize(d)
    return (time.perf_counter() - t0) / reps


def main():
    G = torch.cuda.device_count()
    print("gpus", G)
    for a in range(G):
        for b in range(G):
            if a != b and not torch.cuda.can_device_access_peer(a, b):
                print("no peer access", a, b)
    nbytes = 256 * MB
    src = [torch.empty(nbytes // 4, dtype=torch.float32, device=f"cuda:{d}").fill_(1) for d in range(G)]
    dst = {(a, b): torch.empty(nbytes // 4, dtype=torch.float32, device=f"cuda:{b}") for a in range(G) for b in range(G) if a != b}
    streams = {(a, b): torch.cuda.Stream(device=a) for a in range(G) for b in range(G) if a != b}

    def copies(pairs):
        def run():
            for (a, b) in pairs:
                with torch.cuda.stream(streams[(a, b)]):
                    dst[(a, b)].copy_(src[a], non_blocking=True)
        return run

    devs = list(range(G))
    t = timed(copies([(0, 1)]), devs)
    print(f"0->1 single copy: {nbytes / t / 1e9:.1f} GB/s")
    pairs = [(0, b) for b in range(1, G)]
    t = timed(copies(pairs), devs)
    print(f"0->all ({G-1} peers) concurrent: {len(pairs) * nbytes / t / 1e9:.1f} GB/s out of GPU 0")
    pairs = [(a, b) for a in range(G) for b in range(G) if a != b]
    t = timed(copies(pairs), devs)
    print(f"all-to-all concurrent: {len(pairs) * nbytes / G / t / 1e9:.1f} GB/s out of each GPU")
    # with a bandwidth-heavy kernel on every GPU (large copy within HBM)
    big = [torch.empty(1 << 30, dtype=torch.uint8, device=f"cuda:{d}") for d in range(G)]
    big2 = [torch.empty(1 << 30, dtype=torch.uint8, device=f"cuda:{d}") for d in range(G)]
    hs = [torch.cuda.Stream(device=d) for d in range(G)]

    def loaded():
        for d in range(G):
            with torch.cuda.stream(hs[d]):
                for _ in range(3):
                    big2[d].copy_(big[d], non_blocking=True)
        copies(pairs)()
    t = timed(loaded, devs)
    print(f"all-to-all concurrent with local HBM copies running: ~{len(pairs) * nbytes / G / t / 1e9:.1f} GB/s out of each GPU (lower bound)")


if __name__ == "__main__":
    main()
