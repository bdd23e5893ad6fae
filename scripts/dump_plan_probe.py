import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2504_09014_b200 import Runtime, make_world, parse_plan
from paper_2504_09014_b200.plan import scale_plan
w = make_world(1, 8, devices=[0] * 8)
for p in ("1pa_n8_e64", "2pa_memory_n8_e64"):
    base = parse_plan(open(f"tests/golden/plans/{p}.json", "rb").read())
    rt = Runtime(scale_plan(base, 128), w, dtype="bf16")
    print("K", getattr(rt, "K", None), "ops", rt.n_device_ops, flush=True)
    rt.close()
