"""Diagnostic: graph-timed latency of chosen AllReduce algorithms over sizes on
8 co-resident ranks (L2 flushed).  Usage: algo_sweep.py ALGO[,ALGO..] [dtype]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2504_09014_b200 import _lib, make_world
    algos = sys.argv[1].split(",")
    dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
    es = {"f32": 4, "bf16": 2, "f16": 2, "i32": 4}[dtype]
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16, "i32": torch.int32}[dtype]
    n = 8
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for nb in [int(x) for x in os.environ.get("SIZES", ",".join(str(1 << k) for k in range(10, 23, 2))).split(",")]:
        c = nb // es
        xs = [torch.randn(c, device=dev).to(tdt) for _ in range(n)]
        ys = [torch.empty_like(x) for x in xs]
        row = [f"{nb:9d}"]
        for a in algos:
            t = bench.time_coll(w, "allreduce", xs, ys, c, dtype, _lib.ALGOS[a], 20, 3, flush)
            row.append(f"{a}={t * 1e6:8.2f}us")
        print("  ".join(row), flush=True)


if __name__ == "__main__":
    main()
