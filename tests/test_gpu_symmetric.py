"""Symmetric heap (cfSymHeapCreate / cfMemAlloc) and the in-place NVLS
AllReduce on it (K5 direct: multimem.ld_reduce from the send buffer,
multimem.st into the recv buffer, no staging copies), plus the SwitchChannel
device handle for user kernels.

On 1-GPU boxes the switch is EMULATED (mode 2: the same kernel and schedule,
the two multimem instructions replaced by per-member unicast loads / stores
in the reference switch order 0 + x_0 + ... + x_{n-1}), so results are
bit-exact to the oracle's switch_2pa.  With real multicast (mode 1, >= 2 GPUs:
the tests at the bottom skip below that) the switch's summation order is
unspecified: SURVEY §8(c) tolerance |y - y_ref| <= 2^-8 |y_ref| (bf16),
2^-11 (f16), plus (n-1) 2^-24 sum|x_i|; i32 exact."""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp
from inputs import gen_inputs
from oracle import oracle

pytestmark = pytest.mark.gpu

HEAP = 64 << 20
DT = {"f32": "float32", "bf16": "bfloat16", "f16": "float16", "i32": "int32"}


def _tdt(dt):
    import torch
    return getattr(torch, DT[dt])


def _fill(t, arr, dt):
    import torch
    src = torch.from_numpy(arr.view(np.int16) if dt == "bf16" else arr)
    t.copy_(src.view(t.dtype) if dt == "bf16" else src)


def _host(t, dt):
    import torch
    return t.view(torch.int16).cpu().numpy().view(np.uint16) if dt == "bf16" else t.cpu().numpy()


def _world(n, **kw):
    from paper_2504_09014_b200 import make_world
    w = make_world(1, n, devices=[0] * n, use_multicast="emulate", spin_timeout_ms=5000, **kw)
    assert w.symmetric_heap(HEAP) == 2
    return w


def _run(w, n, elems, dt, seed, in_place=False, algo="switch_2pa"):
    from paper_2504_09014_b200 import collectives as C
    ins = gen_inputs(n, elems, dt, "normal" if dt in ("bf16", "f16") else ("int" if dt == "i32" else "wide"), seed)
    xs = w.alloc_symmetric(elems, _tdt(dt))
    ys = xs if in_place else w.alloc_symmetric(elems, _tdt(dt))
    for r in range(n):
        _fill(xs[r], ins[r], dt)
    C.run("allreduce", xs, ys, elems, dt, __import__("paper_2504_09014_b200")._lib.ALGOS[algo], w)
    w.synchronize()
    w.check_device_error()
    got = [_host(y, dt) for y in ys]
    w.free_symmetric(xs)
    if not in_place:
        w.free_symmetric(ys)
    return ins, got


@pytest.mark.parametrize("dt", ["bf16", "f32", "f16", "i32"])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_switch_in_place_on_symmetric_buffers_matches_oracle(n, dt):
    w = _world(n)
    for elems in (8 * 4096, 4099, 3, 1 << 18):
        ins, got = _run(w, n, elems, dt, 31 + elems)
        want = oracle.allreduce(ins, "switch_2pa", dt)
        for r in range(n):
            assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), (elems, r)
    w.close()


def test_switch_symmetric_in_place_send_equals_recv():
    n = 8
    w = _world(n)
    ins, got = _run(w, n, 8 * 1000 + 5, "bf16", 5, in_place=True)
    want = oracle.allreduce(ins, "switch_2pa", "bf16")
    for r in range(n):
        assert np.array_equal(got[r], want[r]), r
    w.close()


def test_switch_symmetric_split_launch_handshakes(monkeypatch):
    """One launch per rank on its own stream (CF_SPLIT_GROUPS=1): the entry and
    exit handshakes of the in-place kernel run."""
    monkeypatch.setenv("CF_SPLIT_GROUPS", "1")
    n = 4
    w = _world(n)
    for rep in range(3):
        ins, got = _run(w, n, 4 * 65536 + 9, "f32", 70 + rep)
        want = oracle.allreduce(ins, "switch_2pa", "f32")
        for r in range(n):
            assert np.array_equal(got[r].view(np.uint32), want[r].view(np.uint32)), (rep, r)
    w.close()


def test_hb_algorithms_and_graph_replay_on_symmetric_buffers():
    """Symmetric buffers are ordinary buffers for every other algorithm, and
    the in-place NVLS kernel replays from a CUDA graph (epochs advance)."""
    import torch
    from paper_2504_09014_b200 import _lib
    from paper_2504_09014_b200 import collectives as C
    n, elems = 8, 8 * 2048
    w = _world(n)
    for algo, oname in (("2pa", "2pa"), ("1pa", "1pa"), ("1pa_hb", "1pa")):
        ins, got = _run(w, n, elems, "f32", 3, algo=algo)
        want = oracle.allreduce(ins, oname, "f32")
        for r in range(n):
            assert np.array_equal(got[r].view(np.uint32), want[r].view(np.uint32)), (algo, r)
    xs = w.alloc_symmetric(elems, torch.float32)
    ys = w.alloc_symmetric(elems, torch.float32)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        C.run("allreduce", xs, ys, elems, "f32", _lib.ALGOS["switch_2pa"], w)
    for rep in range(3):
        ins = gen_inputs(n, elems, "f32", "uniform", 90 + rep)
        for r in range(n):
            _fill(xs[r], ins[r], "f32")
        g.replay()
        torch.cuda.synchronize()
        want = oracle.allreduce(ins, "switch_2pa", "f32")
        for r in range(n):
            assert np.array_equal(_host(ys[r], "f32").view(np.uint32), want[r].view(np.uint32)), (rep, r)
    w.check_device_error()
    w.close()


def test_symmetric_allocator_offsets_and_errors():
    import torch
    from paper_2504_09014_b200.errors import BadSizeError, ConfigError, OutOfBoundsError
    w = _world(2)
    a = w.alloc_symmetric(1000, torch.float32)
    b = w.alloc_symmetric(10, torch.bfloat16)
    base = [ctypes.c_void_p() for _ in range(2)]
    bases = (ctypes.c_void_p * 2)()
    nbytes, mode = ctypes.c_size_t(), ctypes.c_int()
    from paper_2504_09014_b200 import _lib
    _lib.check(_lib.lib().cfSymHeapInfo(w.comm, 0, bases, ctypes.byref(nbytes), ctypes.byref(mode)))
    assert mode.value == 2 and nbytes.value >= HEAP
    for r in range(2):   # same offsets on every rank
        _lib.check(_lib.lib().cfSymHeapInfo(w.comm, r, bases, None, None))
        base[r] = bases[r]
    offs = [[t.data_ptr() - base[r] for r, t in enumerate(ts)] for ts in (a, b)]
    assert offs[0][0] == offs[0][1] and offs[1][0] == offs[1][1] and offs[1][0] >= 4000
    w.free_symmetric(a)
    c = w.alloc_symmetric(100, torch.float32)      # first fit reuses the freed range
    assert c[0].data_ptr() == a[0].data_ptr()
    with pytest.raises(BadSizeError):
        w.alloc_symmetric(HEAP, torch.float32)
    with pytest.raises(OutOfBoundsError):
        w.free_symmetric([torch.empty(4, device="cuda")])
    with pytest.raises(ConfigError):
        w.symmetric_heap(HEAP)
    w.close()


def test_switch_channel_device_from_user_kernel():
    """cf::SwitchChannelDevice (reduce / broadcast / reduce_broadcast over heap
    offsets) from a user kernel, emulated switch: rank r reduces chunk r of
    every member's heap range and broadcasts it (an NVLS AllReduce written
    against the Primitive API)."""
    import torch
    lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "kernels", "libcf_channels_test.so"))
    n, elems = 4, 4 * 1024
    w = _world(n)
    xs = w.alloc_symmetric(elems, torch.float32)
    ys = w.alloc_symmetric(elems, torch.float32)
    ins = gen_inputs(n, elems, "f32", "uniform", 12)
    for r in range(n):
        _fill(xs[r], ins[r], "f32")
    bases = (ctypes.c_void_p * n)()
    _lib = __import__("paper_2504_09014_b200")._lib
    _lib.check(_lib.lib().cfSymHeapInfo(w.comm, 0, bases, None, None))
    off_in, off_out = xs[0].data_ptr() - bases[0], ys[0].data_ptr() - bases[0]
    handles = b"".join(w.switch_channel(r) for r in range(n))
    rc = lib.cftest_switch_allreduce(handles, n, ctypes.c_size_t(off_in), ctypes.c_size_t(off_out),
                                     ctypes.c_size_t(elems * 4))
    assert rc == 0
    want = oracle.allreduce(ins, "switch_2pa", "f32")
    for r in range(n):
        assert np.array_equal(_host(ys[r], "f32").view(np.uint32), want[r].view(np.uint32)), r
    w.close()


# ------------------------------------------------------------------ one process per rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _mp_worker(rank, world, port, q, mode, dev_of_rank):
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path[:0] = [root, os.path.join(root, "tests", "golden")]
        import torch
        import torch.distributed as dist
        from inputs import gen_inputs
        from paper_2504_09014_b200.comm import Communicator
        dev = dev_of_rank(rank)
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        comm = Communicator(device=dev, spin_timeout_ms=60000)
        got_mode = comm.setup_symmetric(HEAP, mode=mode)
        out = {"mode": got_mode}
        for dt in ("bf16", "f32"):
            for elems in (world * 4096, 4099):
                ins = gen_inputs(world, elems, dt, "normal" if dt == "bf16" else "uniform", 40 + elems)
                x = comm.alloc_symmetric(elems, _tdt(dt))
                y = comm.alloc_symmetric(elems, _tdt(dt))
                _fill(x, ins[rank], dt)
                for algo in ("switch_2pa", "2pa", "1pa_hb"):
                    comm.all_reduce(x, y, algo=algo)     # no registration: symmetric
                    torch.cuda.synchronize()
                    out[(dt, elems, algo)] = _host(y, dt).copy()
                ag = comm.alloc_symmetric(world * elems, _tdt(dt))
                comm.all_gather(x, ag, algo="allpairs_ag")
                torch.cuda.synchronize()
                out[(dt, elems, "ag")] = _host(ag, dt).copy()
                for t in (x, y, ag):
                    comm.free_symmetric(t)
        comm.check_device_error()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, out))
    except Exception as e:  # surface the failure to the parent
        import traceback
        q.put((rank, f"{type(e).__name__}: {e}\n{traceback.format_exc()}"))


def _run_mp(world, mode, dev_of_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, q, mode, dev_of_rank)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    return res


def _dev0(rank):
    return 0


def _dev_rank(rank):
    return rank


def _check_mp(res, world, exact_switch):
    for dt in ("bf16", "f32"):
        for elems in (world * 4096, 4099):
            ins = gen_inputs(world, elems, dt, "normal" if dt == "bf16" else "uniform", 40 + elems)
            for r in range(world):
                for algo, oname in (("2pa", "2pa"), ("1pa_hb", "1pa")):
                    want = oracle.allreduce(ins, oname, dt)[r]
                    assert np.array_equal(res[r][(dt, elems, algo)].view(np.uint8), want.view(np.uint8)), \
                        (dt, elems, algo, r)
                assert np.array_equal(res[r][(dt, elems, "ag")], oracle.allgather(ins)[r])
                want = oracle.allreduce(ins, "switch_2pa", dt)[r]
                got = res[r][(dt, elems, "switch_2pa")]
                if exact_switch:
                    assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (dt, elems, r)
                else:
                    _within_switch_tolerance(got, want, ins, dt)


def _f32(a, dt):
    return (a.astype(np.uint32) << 16).view(np.float32) if dt == "bf16" else a.astype(np.float32)


def _within_switch_tolerance(got, want, ins, dt):
    n = len(ins)
    g, w = _f32(got, dt), _f32(want, dt)
    sabs = np.sum([np.abs(_f32(a, dt)) for a in ins], axis=0)
    rel = 2.0 ** -8 if dt == "bf16" else (2.0 ** -11 if dt == "f16" else 0.0)
    tol = rel * np.abs(w) + (n - 1) * 2.0 ** -24 * sabs
    assert np.all(np.abs(g - w) <= tol), float(np.max(np.abs(g - w) - tol))


def test_two_processes_one_gpu_symmetric_heap_emulated_switch():
    """Heaps exchanged as POSIX fds (SCM_RIGHTS), peers mapped; switch_2pa in
    place (emulated switch: exact), 2pa / 1pa_hb / AllGather on symmetric
    buffers without any registration."""
    res = _run_mp(2, "emulate", _dev0)
    assert all(res[r]["mode"] == 2 for r in range(2))
    _check_mp(res, 2, exact_switch=True)


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.skipif("_ngpus() < 2", reason="NVLS multicast needs >= 2 GPUs (runs on the driver's 8-GPU box)")
def test_nvls_multicast_one_process_per_gpu():
    """REAL multimem.ld_reduce / multimem.st: one process per GPU, heaps bound
    to one multicast object; tolerance per SURVEY §8(c) (switch order
    unspecified)."""
    n = min(_ngpus(), 8)
    res = _run_mp(n, "auto", _dev_rank)
    if any(res[r]["mode"] != 1 for r in range(n)):
        pytest.skip("the box advertises multicast but the object did not build (no fabric / IMEX)")
    _check_mp(res, n, exact_switch=False)


@pytest.mark.skipif("_ngpus() < 2", reason="NVLS multicast needs >= 2 GPUs (runs on the driver's 8-GPU box)")
def test_nvls_multicast_in_process_world():
    import torch
    from paper_2504_09014_b200 import _lib, make_world
    from paper_2504_09014_b200 import collectives as C
    n = min(_ngpus(), 8)
    w = make_world(1, n, devices=list(range(n)), spin_timeout_ms=10000)
    try:
        from paper_2504_09014_b200.errors import CommforgeError
        try:
            mode = w.symmetric_heap(HEAP, mode=1 if w.multicast_supported() else 0)
        except CommforgeError as e:   # the driver refused the multicast object (no fabric manager / IMEX)
            pytest.skip(f"no multicast object on this box: {e}")
        if mode != 1:
            pytest.skip("no multicast object on this box")
        for dt in ("bf16", "f32", "i32"):
            elems = n * 65536 + 3
            ins = gen_inputs(n, elems, dt, {"bf16": "normal", "f32": "uniform", "i32": "int"}[dt], 8)
            xs = w.alloc_symmetric(elems, _tdt(dt))
            ys = w.alloc_symmetric(elems, _tdt(dt))
            for r in range(n):
                _fill(xs[r], ins[r], dt)
            C.run("allreduce", xs, ys, elems, dt, _lib.ALGOS["switch_2pa"], w)
            w.synchronize()
            w.check_device_error()
            want = oracle.allreduce(ins, "switch_2pa", dt)
            for r in range(n):
                got = _host(ys[r], dt)
                if dt == "i32":
                    assert np.array_equal(got, want[r])
                else:
                    _within_switch_tolerance(got, want[r], ins, dt)
            w.free_symmetric(xs)
            w.free_symmetric(ys)
        torch.cuda.synchronize()
    finally:
        w.close()
