"""Diagnostic: AllGather / ReduceScatter rows of the bench sweep and 2pr at 64 MiB."""
import sys; sys.path.insert(0, ".")
import torch, bench
from paper_2504_09014_b200 import make_world
w = make_world(1, 8, devices=[0]*8)
dev = w.device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
maxe = (256 << 20) // 2
send = [torch.randn(maxe, device=dev).to(torch.bfloat16) for _ in range(8)]
recv = [torch.empty_like(s) for s in send]
r = bench.run_ag_rs(w, flush, send, recv)
for row in r["rows"]: print(row)
r = bench.time_coll(w, "allreduce", send[:8], recv, (64<<20)//2, "bf16", 5, 5, 3, None)
print("2pr 64MiB", r*1e6)
