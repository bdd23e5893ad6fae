"""Diagnostic: C5 plan latencies (reference-lowered 2pa / 1pa plans scaled to
[b, 8192] bf16, K10) on 8 co-resident ranks, CUDA-graph timed, L2 flushed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import time_plan
    from paper_2504_09014_b200 import Runtime, make_world, parse_plan
    from paper_2504_09014_b200.plan import scale_plan
    n = 8
    w = make_world(1, n, devices=[0] * n, threads=int(os.environ.get("THREADS", "0")))
    dev = w.device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for pname in os.environ.get("PLANS", "2pa_memory_n8_e64,2pa_ll_n8_e64,1pa_n8_e64").split(","):
        with open(os.path.join(ROOT, "tests", "golden", "plans", pname + ".json"), "rb") as f:
            base = parse_plan(f.read())
        row = []
        for b in (1, 4, 16, 64, 256):
            rt = Runtime(scale_plan(base, 128 * b), w, dtype="bf16")
            xs = [torch.randn(rt.in_elems, device=dev).to(torch.bfloat16) for _ in range(n)]
            ys = [torch.empty(rt.out_elems, device=dev, dtype=torch.bfloat16) for _ in range(n)]
            t = time_plan(rt, xs, ys, 20, 3, flush)
            row.append(f"b={b}: {t * 1e6:6.2f} us")
            rt.close()
        print(f"{pname:<20} " + " | ".join(row), flush=True)
    w.close()


if __name__ == "__main__":
    main()
