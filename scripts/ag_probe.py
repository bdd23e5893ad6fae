"""Direct AllGather (K6) latency / HBM rate, 8 co-resident ranks, bf16,
CUDA-graph timed (inputs > L2 or L2 flushed).  CF_AG_BULK=0 selects the
register kernel, default the TMA bulk-copy kernel (shards >= 1 MiB)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import time_coll
    from paper_2504_09014_b200 import _lib, make_world
    n = 8
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for nb in (16 << 20, 64 << 20, 256 << 20, 1 << 30):
        shard = nb // 2 // n
        xs = [torch.randn(shard, device=dev).to(torch.bfloat16) for _ in range(n)]
        ys = [torch.empty(shard * n, device=dev, dtype=torch.bfloat16) for _ in range(n)]
        t = time_coll(w, "allgather", xs, ys, shard, "bf16", _lib.ALGOS["allpairs_ag"], 10, 3,
                      flush if nb < 64 << 20 else None)
        hbm = (nb + n * nb) / t / 1e9   # every shard read once + every output written once
        print(f"AG out {nb >> 20:5d} MiB  {t * 1e6:8.1f} us  {hbm:7.0f} GB/s HBM "
              f"({hbm / 6559.7:.1%} of peak)  bulk={os.environ.get('CF_AG_BULK', '1')}")
        for y in ys[:2]:
            assert torch.equal(y.view(n, shard), torch.stack(xs)), "AllGather result differs"
    w.close()


if __name__ == "__main__":
    main()
