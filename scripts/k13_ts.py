"""Diagnostic (needs `make EXTRA=-DCF_TS`): K13 per-phase stamps (entry,
phase 1 done, mid handshake done, each finished row, end) at C5 shapes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2504_09014_b200 import allreduce_add_rmsnorm, make_world  # noqa: E402

n, hidden = 8, 8192
w = make_world(1, n, devices=[0] * n)
dev = w.device(0)
for b in [int(x) for x in os.environ.get("BATCH", "16,64").split(",")]:
    xs = [torch.randn(b, hidden, device=dev).to(torch.bfloat16) for _ in range(n)]
    rs = [torch.randn(b, hidden, device=dev).to(torch.bfloat16) for _ in range(n)]
    ys = [torch.empty_like(x) for x in xs]
    wt = torch.ones(hidden, device=dev, dtype=torch.bfloat16)
    for it in range(3):
        print(f"--- k13 b={b} algo={os.environ.get('ALGO', '2pa')} iter {it}", flush=True)
        allreduce_add_rmsnorm(w, xs, rs, wt, norm_out=ys, algo=os.environ.get("ALGO", "2pa"))
        torch.cuda.synchronize(dev)
w.close()
