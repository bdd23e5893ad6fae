"""Diagnostic (needs libcf built with EXTRA=-DCF_TS): per-phase device timestamps
of the LL kernels, printed by thread 0 of CTA 0 of every rank."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2504_09014_b200 import _lib, make_world
from paper_2504_09014_b200 import collectives as C
n = 8
w = make_world(1, n, devices=[0] * n)
dev = w.device(0)
for nb in (1024, 16384):
    count = nb // 2
    send = [torch.randn(count, device=dev).to(torch.bfloat16) for _ in range(n)]
    recv = [torch.empty_like(s) for s in send]
    for a in ("1pa", "2pa_ll"):
        for it in range(4):
            print(f"--- {a} {nb} iter {it}", flush=True)
            C.run("allreduce", send, recv, count, "bf16", _lib.ALGOS[a], w)
            torch.cuda.synchronize(dev)
w.close()
