"""One ring ReduceScatter (or 2PR) configuration, a few calls (ncu target)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2504_09014_b200 import _lib, make_world  # noqa: E402
from paper_2504_09014_b200 import collectives as C  # noqa: E402

algo, nb = sys.argv[1], int(sys.argv[2])
n = 8
w = make_world(1, n, devices=[0] * n)
cnt = nb // 2
send = [torch.randn(cnt, device="cuda").to(torch.bfloat16) for _ in range(n)]
if algo == "ring_rs":
    out = [torch.empty(cnt // n, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
    for _ in range(3):
        C.run("reducescatter", send, out, cnt // n, "bf16", _lib.ALGOS[algo], w)
else:
    out = [torch.empty_like(s) for s in send]
    for _ in range(3):
        C.run("allreduce", send, out, cnt, "bf16", _lib.ALGOS[algo], w)
torch.cuda.synchronize()
print("ok")
