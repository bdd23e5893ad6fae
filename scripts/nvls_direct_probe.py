"""NVLS AllReduce (emulated switch, 8 co-resident ranks, bf16): the staging
kernel (K5, unregistered tensors: copy-in / reduce+broadcast / copy-out) vs
the in-place kernel on symmetric buffers (K5 direct).  Prints device times;
run under ncu for the per-kernel DRAM bytes (expected drop: 4 S per rank)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_09014_b200 import _lib, make_world  # noqa: E402
from paper_2504_09014_b200 import collectives as C  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64 << 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n = 8
w = make_world(1, n, devices=[0] * n, use_multicast="emulate", nvls_bytes=S)
w.symmetric_heap(2 * S + (4 << 20))
cnt = S // 2
plain_x = [torch.randn(cnt, device="cuda").to(torch.bfloat16) for _ in range(n)]
plain_y = [torch.empty_like(x) for x in plain_x]
sx = w.alloc_symmetric(cnt, torch.bfloat16)
sy = w.alloc_symmetric(cnt, torch.bfloat16)
for a, b in zip(sx, plain_x):
    a.copy_(b)
aid = _lib.ALGOS["switch_2pa"]
for name, xs, ys in (("staging", plain_x, plain_y), ("direct", sx, sy)):
    C.run("allreduce", xs, ys, cnt, "bf16", aid, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        C.run("allreduce", xs, ys, cnt, "bf16", aid, w)
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    print(f"{name}: {t * 1e6:.1f} us per call, {S >> 20} MiB per rank, "
          f"{2 * n * S / t / 1e9:.0f} GB/s of 2nS (in read once + out written once)")
for a, b in zip(sy, plain_y):
    assert torch.equal(a, b), "direct and staging results differ"
w.check_device_error()
print("direct == staging: ok")
