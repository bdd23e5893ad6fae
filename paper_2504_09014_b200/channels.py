"""Channel objects of the reference's Primitive API (``cf/channels.py``) on
B200.

In the reference a channel is a simulator object whose ``put`` / ``signal`` /
``wait`` / ``flush`` / ``put_packets`` / ``read_packets`` run inside simulated
thread-block contexts (``cf/channels.py:54-409``).  On a GPU those operations
run inside CUDA kernels; the host-side object here is what builds the device
handle a kernel calls them on (``device/cf_device.cuh``:
``cf::MemoryChannelDevice``, ``cf::PortChannelDevice``,
``cf::SwitchChannelDevice``), with the reference's constructor signatures.
Regions are CUDA tensors (the reference's region ids name world-owned byte
arrays); ``sched`` -- the simulated scheduler -- is accepted and ignored: real
GPUs schedule themselves.
"""

from __future__ import annotations

from .errors import OutOfBoundsError, TopologyError, WrongProtocolError

LL = "LL"   # cf/channels.py:33-34
HB = "HB"


class MemoryChannel:
    """Directed src_rank -> dst_rank memory-mapped channel, LL or HB
    (cf/channels.py:153-330): zero-copy peer stores / loads, a semaphore in
    the destination's heap, LL16 packets.  ``handle`` is the
    ``cf::MemoryChannelDevice`` bytes for the kernels of both endpoints."""

    def __init__(self, world, sched, protocol: str, src_rank: int, dst_rank: int, src_region=None,
                 dst_region=None, name: str = "mem", tag: int = 0):
        if protocol not in (LL, HB):
            raise WrongProtocolError(f"unknown protocol {protocol!r}")
        if src_region is None or dst_region is None:
            raise OutOfBoundsError("a device channel needs its source and destination tensors")
        self.world, self.protocol, self.name = world, protocol, name
        self.src_rank, self.dst_rank = src_rank, dst_rank
        self.src_region, self.dst_region = src_region, dst_region
        self.handle = world.memory_channel(src_rank, dst_rank, tag, src_region, dst_region)


class PortChannel:
    """Directed src_rank -> dst_rank port-mapped channel (cf/channels.py:54-150):
    puts are requests to libcf's host proxy, which copies with the DMA engine
    and then writes the semaphore; ``flush`` waits for completion.  The request
    ring holds 1024 entries (``capacity`` is accepted and ignored)."""

    def __init__(self, world, sched, src_rank: int, dst_rank: int, src_region=None, dst_region=None,
                 capacity: int | None = None, name: str = "port", tag: int = 0):
        if src_region is None or dst_region is None:
            raise OutOfBoundsError("a device channel needs its source and destination tensors")
        self.world, self.name = world, name
        self.src_rank, self.dst_rank = src_rank, dst_rank
        self.src_region, self.dst_region = src_region, dst_region
        self.handle = world.port_channel(src_rank, dst_rank, tag, src_region, dst_region)


class SwitchChannel:
    """Switch-mapped reduce / broadcast over the same offset of every member's
    symmetric heap (cf/channels.py:333-409): ``multimem.ld_reduce`` /
    ``multimem.st`` on the NVLS multicast object, or the emulated switch.
    ``handles[r]`` is the ``cf::SwitchChannelDevice`` of member rank r.  The
    members are every rank of the world (one multicast object per heap);
    ``multimem`` / ``local`` (the reference's region maps) are accepted and
    ignored -- offsets into the symmetric heap address the data."""

    def __init__(self, world, sched, ranks, multimem=None, local=None, name: str = "switch"):
        ranks = list(ranks)
        if sorted(ranks) != list(range(world.num_ranks)):
            raise TopologyError("a switch channel spans every rank of the world (one multicast object)")
        self.world, self.name, self.ranks = world, name, ranks
        self.handles = {r: world.switch_channel(r) for r in ranks}
