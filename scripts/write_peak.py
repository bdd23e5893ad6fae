"""Write-only and copy HBM rates on this B200 (torch memset / copy, CUDA
events, best of 10): the roofline of the write-dominated AllGather."""
import torch

x = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
y = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
for name, fn, nbytes in (("memset (write only)", lambda: x.zero_(), 2 << 30),
                         ("copy (read + write)", lambda: y.copy_(x), 4 << 30)):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    print(f"{name}: {nbytes / best / 1e9:.0f} GB/s")
