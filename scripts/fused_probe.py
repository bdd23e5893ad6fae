"""Diagnostic: K13 fused AllReduce + residual + RMSNorm latency at C5 shapes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import time_graph
    from paper_2504_09014_b200 import allreduce_add_rmsnorm, make_world
    n, hidden = 8, 8192
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    row = []
    for b in (1, 4, 8, 16, 32, 64, 256):
        xs = [torch.randn(b, hidden, device=dev).to(torch.bfloat16) for _ in range(n)]
        rs = [torch.randn(b, hidden, device=dev).to(torch.bfloat16) for _ in range(n)]
        ys = [torch.empty_like(x) for x in xs]
        wt = torch.ones(hidden, device=dev, dtype=torch.bfloat16)
        algo = os.environ.get("ALGO") or None
        t = time_graph(dev, lambda: allreduce_add_rmsnorm(w, xs, rs, wt, norm_out=ys, algo=algo), 20, 3, flush)
        row.append(f"b={b}: {t * 1e6:6.2f} us")
    print("K13 " + " | ".join(row), flush=True)
    w.close()


if __name__ == "__main__":
    main()
