"""A/B of the fused K13 CTA size (CF_K13_THREADS, read at every launch) at the
C5 consumer shapes, 8 co-resident ranks, through bench.run_fused (CUDA graphs,
L2 flushed)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2504_09014_b200 import make_world
    w = make_world(1, 8, devices=[0] * 8)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=w.device(0))
    for rep in range(2):
        for th in os.environ.get("THREADS", "default,256,512").split(","):
            if th == "default":
                os.environ.pop("CF_K13_THREADS", None)
            else:
                os.environ["CF_K13_THREADS"] = th
            rows = bench.run_fused(w, flush)["rows"]
            print(f"threads={th:7s} " + "  ".join(f"b={r['batch']}:{r['fused_us']}" for r in rows), flush=True)
    w.close()


if __name__ == "__main__":
    main()
