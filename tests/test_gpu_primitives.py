"""The device Primitive API from user kernels (tests/kernels/channels_test.cu):
MemoryChannel put/signal/wait and put_packets/read_packets, PortChannel
put/signal/put_with_signal/flush/wait through the proxy.  Ring pass over
co-resident ranks: rank r sends its buffer to rank r+1."""

import ctypes
import os

import pytest

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(__file__), "kernels", "libcf_channels_test.so")


def _setup(n, nbytes, port=False, tag=3):
    import torch
    from paper_2504_09014_b200 import make_world
    w = make_world(1, n, spin_timeout_ms=4000)
    src = [torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=w.device(r)) for r in range(n)]
    dst = [torch.zeros(nbytes * 12, dtype=torch.uint8, device=w.device(r)) for r in range(n)]
    outs = [torch.zeros(nbytes, dtype=torch.uint8, device=w.device(r)) for r in range(n)]
    make = w.port_channel if port else w.memory_channel
    tx = [make(r, (r + 1) % n, tag, src[r], dst[(r + 1) % n]) for r in range(n)]
    rx = [tx[(r - 1) % n] for r in range(n)]
    return w, src, dst, outs, tx, rx


def _ptrs(ts):
    return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])


@pytest.mark.parametrize("ll", [0, 1])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_memory_channel_ring_pass(n, ll):
    lib = ctypes.CDLL(LIB)
    nbytes = 4096
    w, src, dst, outs, tx, rx = _setup(n, nbytes)
    rc = lib.cftest_mem_ring(b"".join(tx), b"".join(rx), n, ctypes.c_size_t(nbytes), ll, 7,
                             _ptrs(outs), 5)
    assert rc == 0
    w.check_device_error()
    for r in range(n):
        assert bool((outs[r] == src[(r - 1) % n]).all()), r
    w.close()


@pytest.mark.parametrize("n", [2, 4])
def test_port_channel_ring_pass(n):
    lib = ctypes.CDLL(LIB)
    nbytes = 1 << 20
    w, src, dst, outs, tx, rx = _setup(n, nbytes, port=True)
    rc = lib.cftest_port_ring(b"".join(tx), b"".join(rx), n, ctypes.c_size_t(nbytes), _ptrs(outs), 6)
    assert rc == 0
    w.check_device_error()
    for r in range(n):
        assert bool((outs[r] == src[(r - 1) % n]).all()), r
    w.close()


@pytest.mark.parametrize("port", [False, True])
def test_channel_objects_of_the_reference_api(port):
    """channels.MemoryChannel / PortChannel (cf/channels.py:54-330 signatures)
    build the device handles the user kernels run the ring pass on."""
    import torch
    from paper_2504_09014_b200 import make_world
    from paper_2504_09014_b200.channels import HB, MemoryChannel, PortChannel
    lib = ctypes.CDLL(LIB)
    n, nbytes = 4, 1 << 16
    w = make_world(1, n, spin_timeout_ms=4000)
    src = [torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=w.device(r)) for r in range(n)]
    dst = [torch.zeros(nbytes * 12, dtype=torch.uint8, device=w.device(r)) for r in range(n)]
    outs = [torch.zeros(nbytes, dtype=torch.uint8, device=w.device(r)) for r in range(n)]
    if port:
        ch = [PortChannel(w, None, r, (r + 1) % n, src[r], dst[(r + 1) % n], tag=4) for r in range(n)]
    else:
        ch = [MemoryChannel(w, None, HB, r, (r + 1) % n, src[r], dst[(r + 1) % n], tag=4) for r in range(n)]
    tx = [c.handle for c in ch]
    rx = [tx[(r - 1) % n] for r in range(n)]
    if port:
        rc = lib.cftest_port_ring(b"".join(tx), b"".join(rx), n, ctypes.c_size_t(nbytes), _ptrs(outs), 6)
    else:
        rc = lib.cftest_mem_ring(b"".join(tx), b"".join(rx), n, ctypes.c_size_t(nbytes), 0, 7, _ptrs(outs), 5)
    assert rc == 0
    w.check_device_error()
    for r in range(n):
        assert bool((outs[r] == src[(r - 1) % n]).all()), r
    w.close()


def test_switch_channel_object_handles():
    """channels.SwitchChannel: one cf::SwitchChannelDevice per member over the
    symmetric heap (emulated switch on one GPU)."""
    from paper_2504_09014_b200 import make_world
    from paper_2504_09014_b200.channels import SwitchChannel
    n = 4
    w = make_world(1, n, spin_timeout_ms=4000, use_multicast="emulate")
    w.symmetric_heap(4 << 20)
    sc = SwitchChannel(w, None, range(n))
    assert sorted(sc.handles) == list(range(n))
    assert all(len(h) > 0 for h in sc.handles.values())
    w.close()
