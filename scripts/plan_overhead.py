"""Fixed cost of the plan interpreter: time trivial plans on 8 co-resident
ranks (diagnostic; CUDA-graph timing like bench.py)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2504_09014_b200 import Runtime, _lib, make_world
    from paper_2504_09014_b200.algorithms import build_2pa
    from paper_2504_09014_b200.lowering import LoweringParams, ProgramGraph, lower
    n = 8
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)

    def graph_sync(elems):
        g = ProgramGraph("sync", "custom", LoweringParams(n, elems))
        g.buffer("in", "input", "all", elems)
        g.buffer("out", "output", "all", elems)
        for r in range(n):
            g.tb_sync(r)
        return g

    def graph_copy(elems):
        g = ProgramGraph("copy", "custom", LoweringParams(n, elems))
        g.buffer("in", "input", "all", elems)
        g.buffer("out", "output", "all", elems)
        for r in range(n):
            g.copy(r, dst=("out", 0, elems), src=("in", 0, elems))
        return g

    cases = [("sync", graph_sync(8192)), ("copy16k", graph_copy(8192)),
             ("2pa_b1", build_2pa(LoweringParams(n, 8192, "bf16"), "memory")),
             ("2pa_b64", build_2pa(LoweringParams(n, 8192 * 64, "bf16"), "memory"))]
    from paper_2504_09014_b200 import parse_plan
    from paper_2504_09014_b200.plan import scale_plan
    with open(os.path.join(ROOT, "tests/golden/plans/1pa_n8_e64.json"), "rb") as f:
        p1 = parse_plan(f.read())
    cases += [("1pa_b1", scale_plan(p1, 128)), ("1pa_b64", scale_plan(p1, 8192))]
    for name, g in cases:
        plan = g if not isinstance(g, ProgramGraph) else lower(g, LoweringParams(n, g.params.elems, "bf16"))
        rt = Runtime(plan, w, dtype="bf16")
        xs = [torch.randn(rt.in_elems, device=dev).to(torch.bfloat16) for _ in range(n)]
        ys = [torch.empty(rt.out_elems, device=dev, dtype=torch.bfloat16) for _ in range(n)]
        t_warm = bench.time_plan(rt, xs, ys, 50, 3, None)
        print(f"{name:10s} device_ops={rt.n_device_ops:3d}  {t_warm * 1e6:7.2f} us (L2 warm)")
        rt.close()
    # the hand-written kernels on the same sizes, for comparison
    for elems in (8192, 8192 * 64):
        xs = [torch.randn(elems, device=dev).to(torch.bfloat16) for _ in range(n)]
        ys = [torch.empty(elems, device=dev, dtype=torch.bfloat16) for _ in range(n)]
        for algo in ("2pa", "1pa_hb"):
            t = bench.time_coll(w, "allreduce", xs, ys, elems, "bf16", _lib.ALGOS[algo], 50, 3, None)
            print(f"hand {algo:6s} {elems * 2:8d} B  {t * 1e6:7.2f} us (L2 warm)")


if __name__ == "__main__":
    main()
