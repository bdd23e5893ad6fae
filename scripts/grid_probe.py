"""Diagnostic: K3 two-shot at 256 MiB / 16 MiB per rank vs the per-rank CTA cap."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import time_coll
    from paper_2504_09014_b200 import _lib, make_world
    n = 8
    for mb in [int(x) for x in os.environ.get("CAPS", "0,18,37").split(",")]:
        w = make_world(1, n, devices=[0] * n, max_blocks=mb)
        dev = w.device(0)
        row = []
        for nb in [int(x) << 20 for x in os.environ.get("MIB", "16,256").split(",")]:
            cnt = nb // 2
            send = [torch.randn(cnt, device=dev).to(torch.bfloat16) for _ in range(n)]
            recv = [torch.empty_like(s) for s in send]
            t = time_coll(w, "allreduce", send, recv, cnt, "bf16", _lib.ALGOS["2pa"], 10, 3, None)
            row.append(f"2pa {nb >> 20} MiB {t * 1e6:8.1f} us")
            t = time_coll(w, "allgather", [s[:cnt // n] for s in send], recv, cnt // n, "bf16",
                          _lib.ALGOS["allpairs_ag"], 10, 3, None)
            row.append(f"ag {nb >> 20} MiB {t * 1e6:8.1f} us")
            del send, recv
        print(f"max_blocks={mb:3d}: " + " | ".join(row), flush=True)
        w.close()


if __name__ == "__main__":
    main()
