"""C5 (Llama-70B TP decode AllReduce [b, 8192] bf16, 8 co-resident ranks, L2
flushed between timed calls): the DSL plans on K10 next to the hand kernel
of the same algorithm, for A/B runs of libcf builds (CF_LIB_PATH)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2504_09014_b200 import Runtime, _lib, make_world, parse_plan
    from paper_2504_09014_b200.plan import scale_plan
    n = 8
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hand = {"2pa_memory": "2pa", "2pa_ll": "2pa_ll", "1pa": "1pa"}
    print(f"lib={os.path.basename(os.path.dirname(_lib.LIB_PATH))}/{os.path.basename(_lib.LIB_PATH)}")
    for pname in ("2pa_memory", "2pa_ll", "1pa"):
        with open(os.path.join(ROOT, "tests", "golden", "plans", pname + "_n8_e64.json"), "rb") as f:
            base = parse_plan(f.read())
        for b in [int(x) for x in os.environ.get("BATCH", "1,16,64,256").split(",")]:
            plan = scale_plan(base, 128 * b)
            rt = Runtime(plan, w, dtype="bf16")
            xs = [torch.randn(rt.in_elems, device=dev).to(torch.bfloat16) for _ in range(n)]
            ys = [torch.empty(rt.out_elems, device=dev, dtype=torch.bfloat16) for _ in range(n)]
            tp = bench.time_plan(rt, xs, ys, 20, 3, flush)
            th = bench.time_coll(w, "allreduce", xs, ys, rt.in_elems, "bf16", _lib.ALGOS[hand[pname]], 20, 3, flush)
            print(f"{pname:11s} b={b:3d}  plan {tp * 1e6:7.2f} us  hand {th * 1e6:7.2f} us  "
                  f"ratio {tp / th:5.2f}  K={rt.K if hasattr(rt, 'K') else '?'} ops={rt.n_device_ops}")
            rt.close()


if __name__ == "__main__":
    main()
