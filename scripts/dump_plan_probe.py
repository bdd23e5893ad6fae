import os, sys
sys.path.insert(0, os.getcwd())
from paper_2504_09014_b200 import Runtime, make_world, parse_plan
from paper_2504_09014_b200.plan import scale_plan
w = make_world(1, 8, devices=[0] * 8)
base = parse_plan(open("tests/golden/plans/2pa_ll_n8_e64.json", "rb").read())
rt = Runtime(scale_plan(base, 128), w, dtype="bf16")
rt.close()
