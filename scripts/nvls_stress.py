"""Diagnostic: the emulated-switch NVLS kernel (K5 control path) in the same
sequence as tests/test_gpu_collectives.py::test_nvls_kernel_control_path_emulated,
repeated; on a mismatch prints which elements / pieces are wrong and how."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np  # noqa: E402
from inputs import gen_inputs  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2504_09014_b200 import collective, make_world  # noqa: E402

bad = 0
for trial in range(int(os.environ.get("TRIALS", "20"))):
    for n in (2, 4, 8):
        for dtype in ("f32", "bf16", "f16", "i32"):
            w = make_world(1, n, devices=[0] * n, use_multicast="emulate", nvls_bytes=64 << 10,
                           spin_timeout_ms=5000)
            dist = {"f32": "wide", "i32": "int"}.get(dtype, "normal")
            for elems in (1, 7, 4096, 16384 + 3, 200001):
                ins = gen_inputs(n, elems, dtype, dist, 31 * n + elems % 17)
                want = oracle.allreduce(ins, "switch_2pa", dtype)
                for rep in range(2):
                    got = collective("allreduce", ins, w, dtype=dtype, algo="switch_2pa")
                    for r in range(n):
                        g = got[r].view(np.uint8).reshape(len(got[r]), -1)
                        wt = want[r].view(np.uint8).reshape(len(want[r]), -1)
                        diff = np.nonzero(np.any(g != wt, axis=1))[0]
                        if len(diff):
                            bad += 1
                            es = g.shape[1]
                            vec = diff * es // 16
                            print(f"trial {trial} n={n} {dtype} elems={elems} rep={rep} rank={r}: {len(diff)} bad, "
                                  f"elems {diff[:6]}..{diff[-3:]} vectors {np.unique(vec)[:8]} pieces "
                                  f"{np.unique(vec // 4096)} got {got[r][diff[:3]]} want {want[r][diff[:3]]}",
                                  flush=True)
            try:
                w.check_device_error()
            except Exception as e:
                print("device error", n, dtype, e, flush=True)
            w.close()
print("bad", bad)
