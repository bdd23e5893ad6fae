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


def _fd_worker(rank, world, port, q, path):
    import os
    import torch.distributed as dist
    from paper_2504_09014_b200.comm import share_fd
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    fd = os.open(path, os.O_RDONLY) if rank == 0 else None
    got = share_fd(fd, rank, world)
    q.put((rank, os.pread(got, 64, 0)))
    os.close(got)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_share_fd_passes_descriptor(world, tmp_path):
    """The NVLS setup's fd hand-off (rank 0's multicast handle -> every rank,
    SCM_RIGHTS over a Unix socket whose path travels through the bootstrap)."""
    path = tmp_path / "payload"
    path.write_bytes(b"commforge multicast handle")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fd_worker, args=(r, world, port, q, str(path))) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(v == b"commforge multicast handle" for v in res.values())


def _max_worker(rank, world, port, q):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import gather_max_over_ranks
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    rows = [{"bytes": 1 << 20, "cf_graph_s": 1e-5 * (rank + 1), "nccl_graph_s": 3e-5 / (rank + 1),
             "nccl_sym_graph_s": 2.5e-5 + 1e-6 * rank},
            {"bytes": 1 << 20, "kind": "allgather", "cf_graph_s": 2e-5 * (world - rank)},
            {"bytes": 16384, "plan": "2pa_memory", "batch": 1, "cf_plan_graph_s": 5e-6 + 1e-6 * rank}]
    q.put((rank, gather_max_over_ranks(1.0 + rank, 10.0 - rank, rows, world)))
    dist.destroy_process_group()


def test_bench_times_are_max_over_ranks():
    """bench.py --gpus N: every time is the max over ranks (gloo, world 2),
    busbw uses the collective's bus factor."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_max_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]
    t, te, sweep = res[0]
    assert (t, te) == (2.0, 10.0)
    assert sweep[0]["cf_graph"]["us"] == 20.0 and sweep[0]["nccl_graph"]["us"] == 30.0
    # the better NCCL buffer mode is the bar (max over ranks first)
    assert sweep[0]["nccl_sym_graph"]["us"] == 26.0 and sweep[0]["nccl_best_us"] == 26.0
    assert sweep[0]["cf_vs_nccl_best"] == 1.3
    # AllReduce: 2 (n-1)/n; AllGather: (n-1)/n
    assert sweep[0]["cf_graph"]["busbw"] == round((1 << 20) / 2e-5 * 1.0 / 1e9, 2)
    assert sweep[1]["kind"] == "allgather" and sweep[1]["cf_graph"]["us"] == 40.0
    assert sweep[1]["cf_graph"]["busbw"] == round((1 << 20) / 4e-5 * 0.5 / 1e9, 2)
    assert sweep[2]["plan"] == "2pa_memory" and sweep[2]["cf_plan_graph"]["us"] == 6.0


def _fd_all_worker(rank, world, port, q, base):
    import os
    import torch.distributed as dist
    from paper_2504_09014_b200.comm import share_fd
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    mine = os.open(f"{base}.{rank}", os.O_RDONLY)
    seen = {}
    for src in range(world):   # the symmetric-heap exchange: every rank's fd to every rank
        got = share_fd(mine if src == rank else None, rank, world, src=src)
        seen[src] = os.pread(got, 64, 0)
        if src != rank:
            os.close(got)
    os.close(mine)
    q.put((rank, seen))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_share_fd_all_to_all(world, tmp_path):
    """Communicator.setup_symmetric's heap exchange: every rank's descriptor
    reaches every other rank (share_fd with src = each rank in turn)."""
    base = tmp_path / "heap"
    for r in range(world):
        (tmp_path / f"heap.{r}").write_bytes(f"heap of rank {r}".encode())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fd_all_worker, args=(r, world, port, q, str(base))) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r] == {s: f"heap of rank {s}".encode() for s in range(world)}
