import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests/golden")
import numpy as np
from inputs import gen_inputs
from oracle import oracle
from paper_2504_09014_b200 import collective, make_world
bad = 0
for trial in range(int(os.environ.get("TRIALS", "20"))):
    for n in (2, 4, 8):
        w = make_world(1, n, devices=[0] * n, use_multicast="emulate", nvls_bytes=64 << 10, spin_timeout_ms=5000)
        for dtype in ("i32", "f32", "bf16"):
            dist = {"f32": "wide", "i32": "int"}.get(dtype, "normal")
            for elems in (4096, 16384 + 3, 200001):
                ins = gen_inputs(n, elems, dtype, dist, 31 * n + elems % 17)
                want = oracle.allreduce(ins, "switch_2pa", dtype)
                for rep in range(2):
                    got = collective("allreduce", ins, w, dtype=dtype, algo="switch_2pa")
                    for r in range(n):
                        g, wt = got[r].view(np.uint8).reshape(len(got[r]), -1), want[r].view(np.uint8).reshape(len(want[r]), -1)
                        diff = np.nonzero(np.any(g != wt, axis=1))[0]
                        if len(diff):
                            bad += 1
                            print(f"trial {trial} n={n} {dtype} elems={elems} rep={rep} rank={r}: {len(diff)} bad elems, first {diff[:8]}, last {diff[-4:]}", flush=True)
        w.close()
print("bad", bad)
