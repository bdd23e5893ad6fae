"""Multi-process bootstrap over gloo (CPU, world_size 2): the handle exchange
the one-process-per-GPU communicator relies on."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2504_09014_b200.comm import all_gather_bytes
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    blob = bytes([rank] * 7 + [255 - rank]) * 32          # 256-byte handle-sized blob
    got = all_gather_bytes(blob, None)
    q.put((rank, got))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_all_gather_bytes_rank_order(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([r] * 7 + [255 - r]) * 32 for r in range(world)]
    for r in range(world):
        assert res[r] == want
