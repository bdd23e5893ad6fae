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
                              ("switch_2pa", ""), ("2pr", ""), ("2pr", "ring")):
                got = collective("allreduce", ins, w, dtype=dtype, algo=algo, variant=var)
                want = oracle.allreduce(ins, {"1pa_hb": "1pa", "2pa_ll": "2pa"}.get(algo, algo), dtype)
                if algo != "2pa" or var != "port" or dtype == "f32":
                    bad += sum(not np.array_equal(g.view(np.uint8), x.view(np.uint8)) for g, x in zip(got, want))
            for algo, var in (("ring_rs", ""), ("ring_rs", "ring"), ("rs_direct", "")):
                collective("reducescatter", ins, w, dtype=dtype, algo=algo, variant=var)
            for algo, var in (("allpairs_ag", ""), ("ring_ag", ""), ("ring_ag", "ring")):
                collective("allgather", ins, w, dtype=dtype, algo=algo, variant=var)
    # K6 bulk (TMA) AllGather: a whole-16-byte shard of >= 4 MiB
    sh = [torch.randn((4 << 20) // 4 + 4, device="cuda") for _ in range(n)]
    got = collective("allgather", sh, w)
    bad += sum(not torch.equal(g, torch.cat(sh)) for g in got)
    # K5 in place on symmetric buffers (emulated switch)
    w.symmetric_heap(8 << 20)
    xs = w.alloc_symmetric(4099, torch.float32)
    for r, x in enumerate(xs):
        x.copy_(torch.full((4099,), float(r + 1), device="cuda"))
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200 import _lib
    C.run("allreduce", xs, xs, 4099, "f32", _lib.ALGOS["switch_2pa"], w)
    w.synchronize()
    bad += sum(not torch.all(x == float(n * (n + 1) // 2)).item() for x in xs)
    # K13: one-shot, and two-shot with rows >= n (phase 1 over every CTA, all-CTA barrier)
    for rows in (3, 9):
        xs = [torch.randn(rows, 256, device="cuda") for _ in range(n)]
        rs = [torch.randn(rows, 256, device="cuda") for _ in range(n)]
        for algo in ("1pa_hb", "2pa"):
            allreduce_add_rmsnorm(w, xs, rs, torch.ones(256, device="cuda"), algo=algo)
    # K10: LL plans at a small scale (batched packet items over every thread)
    # and larger ones (fused reads, the 2pa_ll reduce broadcast from registers,
    # the 1pa scatter / read-reduce streamed), HB plan
    for name, scale in (("1pa_n4_e8", 3), ("2pa_ll_n4_e8", 3), ("1pa_n4_e8", 4096), ("2pa_ll_n4_e8", 4096),
                        ("1pa_n4_e8", 65536 + 8), ("2pa_memory_n4_e8", 1000)):
        with open(os.path.join(ROOT, "tests", "golden", "plans", name + ".json"), "rb") as f:
            rt = Runtime(scale_plan(parse_plan(f.read()), scale), w, dtype="f32")
        ins = gen_inputs(n, rt.in_elems, "f32", "normal", scale)
        res = rt.execute(ins)
        rt.execute(ins)   # second call: the host-resolved binding
        rt.close()
        want = oracle.allreduce(ins, "1pa" if name.startswith("1pa") else "2pa", "f32")
        outs = res.outputs if hasattr(res, "outputs") else res
        bad += sum(not np.array_equal(np.asarray(g).view(np.uint8), x.view(np.uint8)) for g, x in zip(outs, want))
    w.synchronize()
    w.check_device_error()
    print("sanitize probe done, mismatches:", bad)
    w.close()


if __name__ == "__main__":
    main()
