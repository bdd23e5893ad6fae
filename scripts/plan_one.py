"""Run one C5 plan configuration a few times (ncu target): plan name, batch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2504_09014_b200 import Runtime, make_world, parse_plan  # noqa: E402
from paper_2504_09014_b200.plan import scale_plan  # noqa: E402

pname, b = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n = 8
w = make_world(1, n, devices=[0] * n)
with open(os.path.join(ROOT, "tests", "golden", "plans", pname + "_n8_e64.json"), "rb") as f:
    plan = scale_plan(parse_plan(f.read()), 128 * b)
rt = Runtime(plan, w, dtype="bf16")
xs = [torch.randn(rt.in_elems, device="cuda").to(torch.bfloat16) for _ in range(n)]
ys = [torch.empty(rt.out_elems, device="cuda", dtype=torch.bfloat16) for _ in range(n)]
for _ in range(reps):
    rt.run_raw(xs, ys)
torch.cuda.synchronize()
rt.check_device_error()
print("ok")
