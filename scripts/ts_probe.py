"""Diagnostic (needs libcf built with `make EXTRA=-DCF_TS`): per-phase device
timestamps (ns after kernel entry) of the LL kernels and the C5 plans, printed
by thread 0 of the first CTA of every rank / program."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2504_09014_b200 import Runtime, _lib, make_world, parse_plan  # noqa: E402
from paper_2504_09014_b200 import collectives as C  # noqa: E402
from paper_2504_09014_b200.plan import scale_plan  # noqa: E402

n = 8
w = make_world(1, n, devices=[0] * n)
dev = w.device(0)
for nb in [int(x) for x in os.environ.get("SIZES", "1024,16384").split(",")]:
    count = nb // 2
    send = [torch.randn(count, device=dev).to(torch.bfloat16) for _ in range(n)]
    recv = [torch.empty_like(s) for s in send]
    for a in os.environ.get("ALGOS", "1pa,2pa_ll").split(","):
        if not a:
            continue
        for it in range(4):
            print(f"--- {a} {nb} iter {it}", flush=True)
            C.run("allreduce", send, recv, count, "bf16", _lib.ALGOS[a], w)
            torch.cuda.synchronize(dev)
for pname in [p for p in os.environ.get("PLANS", "").split(",") if p]:
    base = parse_plan(open(os.path.join(ROOT, "tests", "golden", "plans", pname + ".json"), "rb").read())
    for b in [int(x) for x in os.environ.get("BATCH", "1,64").split(",")]:
        rt = Runtime(scale_plan(base, 128 * b), w, dtype="bf16")
        xs = [torch.randn(rt.in_elems, device=dev).to(torch.bfloat16) for _ in range(n)]
        ys = [torch.empty(rt.out_elems, device=dev, dtype=torch.bfloat16) for _ in range(n)]
        for it in range(4):
            print(f"--- plan {pname} b={b} iter {it}", flush=True)
            rt.run_raw(xs, ys)
            torch.cuda.synchronize(dev)
        rt.close()
w.close()
