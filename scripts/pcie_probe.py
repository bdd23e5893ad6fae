"""Diagnostic: raw pinned-host <-> device copy rates vs concurrent streams
(what bounds bench.py's e2e host-buffer number)."""
import time

import torch

MiB = 1 << 20
sz = 256 * MiB
nb = 8
host = [torch.empty(sz, dtype=torch.uint8).pin_memory() for _ in range(nb)]
dev = [torch.empty(sz, dtype=torch.uint8, device="cuda") for _ in range(nb)]


def run(h2d_streams, d2h_streams, reps=2):
    ss = [torch.cuda.Stream() for _ in range(h2d_streams + d2h_streams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                for k in range(i, nb, len(ss)) if False else range(nb // max(1, len(ss))):
                    j = (i * 7 + k) % nb
                    if i < h2d_streams:
                        dev[j].copy_(host[j], non_blocking=True)
                    else:
                        host[j].copy_(dev[j], non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    moved = reps * len(ss) * (nb // max(1, len(ss))) * sz
    return moved / t / 1e9


for h, d in ((1, 0), (2, 0), (4, 0), (0, 1), (0, 2), (0, 4), (1, 1), (2, 2), (4, 4)):
    print(f"h2d streams {h} d2h streams {d}: {run(h, d):6.1f} GB/s total", flush=True)
