"""Diagnostic: small-message latency of each AllReduce kernel with and without
an L2 flush between calls (8 co-resident ranks, CUDA-graph timed)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import time_coll
    from paper_2504_09014_b200 import _lib, make_world
    n = int(os.environ.get("RANKS", "8"))
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    algos = os.environ.get("ALGOS", "1pa,2pa_ll,1pa_hb,2pa").split(",")
    for nb in [int(x) for x in os.environ.get("SIZES", "1024,16384,65536,262144").split(",")]:
        count = nb // 2
        send = [torch.randn(count, device=dev).to(torch.bfloat16) for _ in range(n)]
        recv = [torch.empty_like(s) for s in send]
        row = []
        for a in algos:
            tf = time_coll(w, "allreduce", send, recv, count, "bf16", _lib.ALGOS[a], 50, 3, flush)
            tw = time_coll(w, "allreduce", send, recv, count, "bf16", _lib.ALGOS[a], 50, 3, None)
            row.append(f"{a}: flushed {tf * 1e6:6.2f} warm {tw * 1e6:6.2f}")
        print(f"{nb:>8} B  " + " | ".join(row), flush=True)
    w.close()


if __name__ == "__main__":
    main()
