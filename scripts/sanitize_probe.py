"""Every libcf kernel once at ragged sizes (4 co-resident ranks), for
compute-sanitizer memcheck: `compute-sanitizer --tool memcheck python
scripts/sanitize_probe.py` (diagnostic)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]


def main():
    import numpy as np
    import torch
    from inputs import gen_inputs
    from oracle import oracle
    from paper_2504_09014_b200 import (Runtime, allreduce_add_rmsnorm, collective, make_world, parse_plan)
    from paper_2504_09014_b200.plan import scale_plan
    n = 4
    w = make_world(1, n, devices=[0] * n, use_multicast="emulate", nvls_bytes=16 << 10, spin_timeout_ms=60000)
    bad = 0
    for elems in (5, 1001, 4099, 4096, 6000):
        for dtype in ("f32", "bf16"):
            ins = gen_inputs(n, elems, dtype, "normal", elems)
            for algo, var in (("1pa", ""), ("1pa_hb", ""), ("2pa", "memory"), ("2pa", "ll"), ("2pa", "port"),
                              ("switch_2pa", ""), ("2pr", "")):
                got = collective("allreduce", ins, w, dtype=dtype, algo=algo, variant=var)
                want = oracle.allreduce(ins, {"1pa_hb": "1pa"}.get(algo, algo), dtype)
                if algo != "2pa" or var != "port" or dtype == "f32":
                    bad += sum(not np.array_equal(g.view(np.uint8), x.view(np.uint8)) for g, x in zip(got, want))
            for algo in ("ring_rs", "rs_direct"):
                collective("reducescatter", ins, w, dtype=dtype, algo=algo)
            for algo in ("allpairs_ag", "ring_ag"):
                collective("allgather", ins, w, dtype=dtype, algo=algo)
    xs = [torch.randn(3, 256, device="cuda") for _ in range(n)]
    rs = [torch.randn(3, 256, device="cuda") for _ in range(n)]
    for algo in ("1pa_hb", "2pa"):
        allreduce_add_rmsnorm(w, xs, rs, torch.ones(256, device="cuda"), algo=algo)
    with open(os.path.join(ROOT, "tests", "golden", "plans", "1pa_n4_e8.json"), "rb") as f:
        rt = Runtime(scale_plan(parse_plan(f.read()), 3), w, dtype="f32")
    rt.execute(gen_inputs(n, rt.in_elems, "f32", "normal", 1))
    rt.close()
    w.synchronize()
    w.check_device_error()
    print("sanitize probe done, mismatches:", bad)
    w.close()


if __name__ == "__main__":
    main()
