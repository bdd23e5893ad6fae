"""Run one hand-kernel AllReduce configuration a few times (ncu target)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2504_09014_b200 import _lib, make_world  # noqa: E402
from paper_2504_09014_b200 import collectives as C  # noqa: E402

algo, elems = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = 8
w = make_world(1, n, devices=[0] * n)
xs = [torch.randn(elems, device="cuda").to(torch.bfloat16) for _ in range(n)]
ys = [torch.empty_like(x) for x in xs]
for _ in range(reps):
    C.run("allreduce", xs, ys, elems, "bf16", _lib.ALGOS[algo], w)
torch.cuda.synchronize()
print("ok")
