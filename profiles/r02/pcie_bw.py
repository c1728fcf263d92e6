"""PCIe copy probe (one B200): host<->device bandwidth of pinned 2 GiB buffers, one copy vs the same
bytes split over 2/4 streams (copy engines), each direction alone and both at once (what
arrow_spmm_host_batch overlaps).  Prints one JSON line per case (GB/s per direction)."""
import json
import torch

GB = 2 ** 30
n = 2 * GB
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]


def run(h2d, d2h, parts, reps=5):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        for s in streams[:2 * parts]:
            s.wait_event(e0)
        c = n // parts
        for p in range(parts):
            if h2d:
                with torch.cuda.stream(streams[p]):
                    d_in[p * c:(p + 1) * c].copy_(h_in[p * c:(p + 1) * c], non_blocking=True)
            if d2h:
                with torch.cuda.stream(streams[parts + p]):
                    h_out[p * c:(p + 1) * c].copy_(d_out[p * c:(p + 1) * c], non_blocking=True)
        for s in streams[:2 * parts]:
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3
        best = t if best is None else min(best, t)
    return n / best / 1e9


for h2d, d2h in ((True, False), (False, True), (True, True)):
    for parts in (1, 2, 4):
        print(json.dumps({"h2d": h2d, "d2h": d2h, "streams_per_direction": parts,
                          "GBps_per_direction": round(run(h2d, d2h, parts), 2)}), flush=True)
