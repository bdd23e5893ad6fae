"""Diagnostic: the 2pa *port* variant (PortChannel puts served by the host
proxy's copy-engine DMA, run as a lowered DSL plan on K10) vs the 2pa memory
kernel (K3), 8 co-resident ranks, bf16.  Eager calls timed with CUDA events
(the proxy is a host thread: a CUDA graph replays the device side only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200 import make_world
    n = 8
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)
    for nb in [int(x) for x in os.environ.get("SIZES", "1048576,16777216,268435456,1073741824").split(",")]:
        cnt = nb // 2
        rt = C._plan_runtime(w, "allreduce", "2pa", "port", C._padded(cnt, n), "bf16")
        xs = [torch.randn(rt.in_elems, device=dev).to(torch.bfloat16) for _ in range(n)]
        ys = [torch.empty(rt.out_elems, device=dev, dtype=torch.bfloat16) for _ in range(n)]

        def timed(fn, iters=5):
            for _ in range(2):
                fn()
            w.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                fn()
            e1.record()
            w.synchronize()
            return e0.elapsed_time(e1) / 1e3 / iters

        tp = timed(lambda: rt.run_raw(xs, ys))
        rt.check_device_error()
        from paper_2504_09014_b200 import _lib
        tm = timed(lambda: C.run("allreduce", xs, ys, rt.in_elems, "bf16", _lib.ALGOS["2pa"], w))
        bus = lambda t: nb / t / 1e9 * 2 * (n - 1) / n   # noqa: E731
        print(f"{nb >> 20:6d} MiB  port {tp * 1e6:9.1f} us ({bus(tp):6.1f} GB/s busbw)   "
              f"memory {tm * 1e6:9.1f} us ({bus(tm):6.1f} GB/s)", flush=True)
    w.close()


if __name__ == "__main__":
    main()
