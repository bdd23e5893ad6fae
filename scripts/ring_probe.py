"""Diagnostic: ring / direct ReduceScatter, AllGather and 2PR latency at a few
sizes (8 co-resident ranks, bf16, CUDA-graph timed, inputs > L2 or flushed)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import algo_id, time_coll
    from paper_2504_09014_b200 import _lib, make_world
    n = 8
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for nb in [int(x) for x in os.environ.get("SIZES", "1048576,16777216,268435456").split(",")]:
        cnt = nb // 2
        send = [torch.randn(cnt, device=dev).to(torch.bfloat16) for _ in range(n)]
        rs_out = [torch.empty(cnt // n, device=dev, dtype=torch.bfloat16) for _ in range(n)]
        ar_out = [torch.empty_like(s) for s in send]
        ag_in = [s[:cnt // n] for s in send]
        fl = flush if nb < 64 << 20 else None
        it = 20 if nb <= 16 << 20 else 5
        row = []
        for kind, algo, ins, outs, c in (("reducescatter", "ring_rs+ring", send, rs_out, cnt // n),
                                         ("reducescatter", "rs_direct", send, rs_out, cnt // n),
                                         ("allgather", "ring_ag+ring", ag_in, ar_out, cnt // n),
                                         ("allreduce", "2pr+ring", send, ar_out, cnt),
                                         ("allreduce", "2pa", send, ar_out, cnt)):
            t = time_coll(w, kind, ins, outs, c, "bf16", algo_id(algo), it, 3, fl)
            row.append(f"{algo} {t * 1e6:8.1f}")
        print(f"{nb:>10} B  " + " | ".join(row), flush=True)
    w.close()


if __name__ == "__main__":
    main()
