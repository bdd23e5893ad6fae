"""The bench's NCCL comparison baseline (scripts/nccl_ctypes.py) on real
hardware: the ctypes bindings bench.py --gpus N uses on the driver's 8-GPU
box (ncclCommInitRank, ncclMemAlloc + ncclCommWindowRegister, the three
collectives, CUDA-graph capture), exercised here as a one-rank communicator
so that a binding mistake shows up on a 1-GPU lease instead of as a missing
comparison in the scaling run.  Test infrastructure only: the product never
loads NCCL."""

import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class _Raw:
    """A raw device allocation seen by torch (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3}


def _nccl():
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    from nccl_ctypes import Nccl
    return Nccl


def test_nccl_ctypes_one_rank_graph_and_symmetric_window():
    import torch
    Nccl = _nccl()
    assert Nccl.version() >= 22800
    torch.cuda.set_device(0)
    nc = Nccl(1, 0, Nccl.unique_id())
    try:
        n = 1 << 16
        x = torch.randn(n, device="cuda").to(torch.bfloat16)
        y = torch.empty_like(x)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                nc.all_reduce(x.data_ptr(), y.data_ptr(), n, "bf16", s.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(x, y)   # one rank: the sum is the input
        cur = torch.cuda.current_stream().cuda_stream
        ag, rs = torch.empty_like(x), torch.empty_like(x)
        nc.all_gather(x.data_ptr(), ag.data_ptr(), n, "bf16", cur)
        nc.reduce_scatter(x.data_ptr(), rs.data_ptr(), n, "bf16", cur)
        torch.cuda.synchronize()
        assert torch.equal(ag, x) and torch.equal(rs, x)
        # symmetric windows (the bench's second NCCL mode)
        sp, rp = nc.mem_alloc(2 * n), nc.mem_alloc(2 * n)
        nc.register_symmetric(sp, 2 * n)
        nc.register_symmetric(rp, 2 * n)
        st = torch.as_tensor(_Raw(sp, n), device="cuda")
        rt = torch.as_tensor(_Raw(rp, n), device="cuda")
        st.copy_(x.view(torch.int16))
        nc.all_reduce(sp, rp, n, "bf16", cur)
        torch.cuda.synchronize()
        assert torch.equal(rt, x.view(torch.int16))
    finally:
        nc.close()
