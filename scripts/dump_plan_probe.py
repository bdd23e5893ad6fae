"""Load plans with CF_PLAN_DUMP=1 (libcf prints each compiled device program)."""
import os
import sys
sys.path.insert(0, os.getcwd())
from paper_2504_09014_b200 import Runtime, make_world, parse_plan  # noqa: E402
from paper_2504_09014_b200.plan import scale_plan  # noqa: E402

w = make_world(1, 8, devices=[0] * 8)
for name in os.environ.get("PLANS", "2pa_ll_n8_e64").split(","):
    for scale in [int(x) for x in os.environ.get("SCALES", "128").split(",")]:
        base = parse_plan(open(f"tests/golden/plans/{name}.json", "rb").read())
        rt = Runtime(scale_plan(base, scale), w, dtype="bf16")
        rt.close()
