"""Small driver for ncu: a few launches of one collective configuration with 8
co-resident ranks on cuda:0 (no timing, no sweep).

    python scripts/profile_kernels.py --algo 2pa --bytes 268435456 --dtype bf16 --iters 3
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="2pa")
    ap.add_argument("--kind", default="allreduce")
    ap.add_argument("--bytes", type=int, default=256 << 20)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--plan", default="")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--emulate-nvls", action="store_true",
                    help="world with the emulated switch (switch_2pa runs the K5 NVLS kernel)")
    args = ap.parse_args()
    import torch
    from paper_2504_09014_b200 import _lib, make_world
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200.dtypes import ELEM_SIZE, torch_dtype
    n = args.ranks
    w = make_world(1, n, devices=[0] * n, use_multicast="emulate" if args.emulate_nvls else True)
    dev = w.device(0)
    count = args.bytes // ELEM_SIZE[args.dtype]
    tdt = torch_dtype(args.dtype)
    if args.plan:
        from paper_2504_09014_b200 import Runtime, parse_plan
        from paper_2504_09014_b200.plan import scale_plan
        with open(args.plan, "rb") as f:
            plan = scale_plan(parse_plan(f.read()), args.scale)
        rt = Runtime(plan, w, dtype=args.dtype)
        send = [torch.randn(rt.in_elems, device=dev).to(tdt) for _ in range(n)]
        recv = [torch.empty(rt.out_elems, device=dev, dtype=tdt) for _ in range(n)]
        for _ in range(args.iters):
            rt.run_raw(send, recv)
    elif args.kind == "fused":
        # K13: AllReduce + residual + RMSNorm on [rows, 8192]
        from paper_2504_09014_b200 import allreduce_add_rmsnorm
        hidden = 8192
        rows = max(1, args.bytes // (hidden * ELEM_SIZE[args.dtype]))
        xs = [torch.randn(rows, hidden, device=dev).to(tdt) for _ in range(n)]
        rs = [torch.randn(rows, hidden, device=dev).to(tdt) for _ in range(n)]
        ys = [torch.empty_like(x) for x in xs]
        wt = torch.ones(hidden, device=dev, dtype=tdt)
        algo = None if args.algo == "auto" else args.algo
        for _ in range(args.iters):
            allreduce_add_rmsnorm(w, xs, rs, wt, algo=algo, norm_out=ys)
    else:
        if args.kind == "allgather":
            send = [torch.randn(count // n, device=dev).to(tdt) for _ in range(n)]
            recv = [torch.empty(count, device=dev, dtype=tdt) for _ in range(n)]
            cnt = count // n
        elif args.kind == "reducescatter":
            send = [torch.randn(count, device=dev).to(tdt) for _ in range(n)]
            recv = [torch.empty(count // n, device=dev, dtype=tdt) for _ in range(n)]
            cnt = count // n
        else:
            send = [torch.randn(count, device=dev).to(tdt) for _ in range(n)]
            recv = [torch.empty_like(s) for s in send]
            cnt = count
        for _ in range(args.iters):
            C.run(args.kind, send, recv, cnt, args.dtype, _lib.ALGOS[args.algo], w)
    torch.cuda.synchronize(dev)
    w.check_device_error()
    print("done")


if __name__ == "__main__":
    main()
