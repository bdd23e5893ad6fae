"""Diagnostic: host-buffer AllReduce pipeline depth vs e2e time, raw PCIe copy rates."""
import sys, os, time
sys.path.insert(0, ".")
import torch
from paper_2504_09014_b200 import make_world, collective
w = make_world(1, 8, devices=[0]*8)
n = 8; count = (256 << 20) // 2
host_in = [torch.randn(count).to(torch.bfloat16).pin_memory() for _ in range(n)]
host_out = [torch.empty_like(h).pin_memory() for h in host_in]
for pcs in (1, 4, 8, 16, 32):
    os.environ["CF_HOST_PIECES"] = str(pcs)
    ts = []
    for it in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        collective("allreduce", host_in, w, algo="2pa", outputs=host_out)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(pcs, [round(t*1e3, 1) for t in ts])
# raw copy rates
a = host_in[0]; d = torch.empty(count, dtype=torch.bfloat16, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(a, non_blocking=True)), ("d2h", lambda: host_out[0].copy_(d, non_blocking=True))):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(8): fn()
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(name, round(8 * 256 / 1024 / t, 1), "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1):
    for _ in range(8): d.copy_(a, non_blocking=True)
d2 = torch.empty_like(d)
with torch.cuda.stream(s2):
    for _ in range(8): host_out[1].copy_(d2, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter() - t0
print("duplex", round(2 * 8 * 256 / 1024 / t, 1), "GB/s total")
