"""Communicator bootstrap: the B200 replacement of the reference's simulated
cluster (``cf/world.py:80-185``, ``make_world``).

A :class:`World` is one process driving every rank (the reference's model:
all ranks live in one process).  Ranks are placed on distinct GPUs when the
box has enough of them, otherwise they are co-resident on one GPU: their CTAs
then run in a single launch and "peer" memory is the same HBM.  Either way the
kernels, the synchronization and the results are identical; only the link
(NVLink vs HBM) differs.

Per rank, libcf allocates a symmetric heap (rank state, semaphore slab, LL
scratch) that replaces the reference's zero-filled ``Region``s and
``Semaphore``s (``cf/world.py:24-51``).  Collective buffers are caller-owned
torch tensors (``cf/executor.py:160-175`` copied arrays in and out; here the
facade does that only for numpy inputs).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

from . import _lib
from .errors import BadSizeError, OutOfBoundsError, TopologyError

INTRA = "intra"
INTER = "inter"
SEED_ENV_VAR = "COMMFORGE_SEED"


@dataclass(frozen=True)
class Topology:
    """cf/world.py:54-77.  One NVSwitch domain: every pair is an intra link."""

    num_nodes: int
    gpus_per_node: int
    intra_kind: str = "switch-attached"

    @property
    def num_ranks(self) -> int:
        return self.num_nodes * self.gpus_per_node

    def node_of(self, rank: int) -> int:
        return rank // self.gpus_per_node

    def link_class(self, a: int, b: int) -> str:
        return INTRA if self.node_of(a) == self.node_of(b) else INTER

    def links(self):
        n = self.num_ranks
        return {(a, b, self.link_class(a, b)) for a in range(n) for b in range(n) if a != b}


class World:
    """In-process communicator over ``num_nodes * gpus_per_node`` ranks."""

    def __init__(self, num_nodes: int = 1, gpus_per_node: int = 1,
                 intra_kind: str = "switch-attached", seed: int = 0, devices=None,
                 ll_max_bytes: int = 0, max_blocks: int = 0, threads: int = 0,
                 spin_timeout_ms: int = 0, use_multicast=True, nvls_bytes: int = 0):
        if num_nodes * gpus_per_node < 1:
            raise BadSizeError("world needs at least one rank")
        if num_nodes != 1:
            raise TopologyError("multi-node worlds are out of scope: one NVSwitch domain "
                                "(the hierarchical 2ph algorithms need an inter-node fabric)")
        env = os.environ.get(SEED_ENV_VAR)
        self.seed = int(env) if env is not None else seed
        self.num_nodes = num_nodes
        self.gpus_per_node = gpus_per_node
        self.intra_kind = intra_kind
        self.topology = Topology(num_nodes, gpus_per_node, intra_kind)
        n = self.num_ranks
        if n > _lib.CF_MAX_RANKS:
            raise BadSizeError(f"at most {_lib.CF_MAX_RANKS} ranks per NVSwitch domain")
        import torch
        if not torch.cuda.is_available():
            raise TopologyError("no CUDA device: the collective path runs only on GPUs")
        if devices is None:
            ndev = torch.cuda.device_count()
            devices = list(range(n)) if ndev >= n else [0] * n
        devices = [int(d) for d in devices]
        if len(devices) != n:
            raise OutOfBoundsError(f"need {n} device ids, got {len(devices)}")
        self.devices = devices
        # NVLS is set up when every rank has its own multicast-capable GPU;
        # use_multicast="emulate" runs switch_2pa's NVLS kernel on unicast
        # staging with per-rank loads / stores in place of multimem (tests)
        mc = 2 if use_multicast == "emulate" else int(bool(use_multicast))
        cfg = _lib.cfConfig(ll_max_bytes, max_blocks, threads, int(spin_timeout_ms) * 1_000_000, mc, nvls_bytes)
        handle = ctypes.c_void_p()
        devs = (ctypes.c_int * n)(*devices)
        _lib.check(_lib.lib().cfCommInitAll(ctypes.byref(handle), n, devs, ctypes.byref(cfg)))
        self._comm = handle
        self.config = cfg

    # -- reference surface -------------------------------------------------

    @property
    def num_ranks(self) -> int:
        return self.num_nodes * self.gpus_per_node

    @property
    def coresident(self) -> bool:
        return len(set(self.devices)) < len(self.devices)

    @property
    def comm(self):
        if self._comm is None:
            raise TopologyError("world is closed")
        return self._comm

    def device(self, rank: int):
        import torch
        return torch.device("cuda", self.devices[rank])

    def streams(self):
        import torch
        if os.environ.get("CF_SPLIT_GROUPS") == "1" and len(set(self.devices)) < self.num_ranks:
            # one launch per rank on a shared device (test mode of libcf's
            # per-device launch path): each rank needs its own stream, ordered
            # after the caller's current stream
            if getattr(self, "_rank_streams", None) is None:
                self._rank_streams = [torch.cuda.Stream(self.device(r)) for r in range(self.num_ranks)]
            for r, st in enumerate(self._rank_streams):
                st.wait_stream(torch.cuda.current_stream(self.device(r)))
            return [st.cuda_stream for st in self._rank_streams]
        return [torch.cuda.current_stream(self.device(r)).cuda_stream for r in range(self.num_ranks)]

    def synchronize(self):
        """Wait for the streams the world's collectives were issued on (not
        the whole device: unrelated streams, e.g. a compute kernel running
        beside the collectives, are not waited for)."""
        import torch
        for d in sorted(set(self.devices)):
            torch.cuda.current_stream(d).synchronize()
        for st in getattr(self, "_rank_streams", None) or ():
            st.synchronize()

    def check_device_error(self):
        """Raise DeadlockError if any device wait of this world timed out."""
        self.synchronize()
        code = ctypes.c_int()
        _lib.check(_lib.lib().cfCommLastDeviceError(self.comm, ctypes.byref(code)))
        if code.value:
            _lib.lib().cfCommClearDeviceError(self.comm)
            from .errors import raise_status
            raise_status(code.value, "device-side wait timed out (peer never signalled)")

    def _channel(self, fn, src, dst, tag, src_buf, dst_buf) -> bytes:
        buf = ctypes.create_string_buffer(256)
        nbytes = ctypes.c_size_t(256)
        _lib.check(fn(self.comm, int(src), int(dst), int(tag), src_buf.data_ptr(), dst_buf.data_ptr(),
                      buf, ctypes.byref(nbytes)))
        return buf.raw[:nbytes.value]

    def memory_channel(self, src: int, dst: int, tag: int, src_buf, dst_buf) -> bytes:
        """Device handle of a MemoryChannel src -> dst (cf/channels.py:153-300) over
        two CUDA tensors, for user kernels (cf::MemoryChannelDevice)."""
        return self._channel(_lib.lib().cfMemoryChannelCreate, src, dst, tag, src_buf, dst_buf)

    def port_channel(self, src: int, dst: int, tag: int, src_buf, dst_buf) -> bytes:
        """Device handle of a PortChannel src -> dst (cf/channels.py:54-150): puts
        are copy-engine DMA issued by libcf's proxy (cf::PortChannelDevice)."""
        return self._channel(_lib.lib().cfPortChannelCreate, src, dst, tag, src_buf, dst_buf)

    def set_cta_budget(self, ctas: int, algo: str | None = None) -> None:
        """CTAs per rank for `algo` (None: every algorithm; "fused": the K13
        kernel; 0 restores the default) -- include/cf.h cfCommSetCtaBudget."""
        aid = -1 if algo is None else (_lib.CF_ALGO_COUNT if algo == "fused" else _lib.ALGOS[algo])
        _lib.check(_lib.lib().cfCommSetCtaBudget(self.comm, aid, int(ctas)))

    def tune(self, kind: str = "allreduce", dtype: str = "bf16", sizes=None, algos=None, iters: int = 10,
             install: bool = True) -> dict:
        """Measure every candidate algorithm at each size (CUDA graphs, L2 not
        flushed) and install the fastest-per-size table for ``algo="auto"``
        (cfCommSetSelection; see tune.py).  Ranks must share one device (the
        co-resident world); returns {"table", "sizes", "times"}."""
        import torch
        from . import collectives as C
        from . import tune as T
        from .dtypes import ELEM_SIZE, torch_dtype
        from .timing import _measure
        if len(set(self.devices)) != 1:
            raise TopologyError("World.tune times ranks that share one GPU; use Communicator.tune per GPU")
        sizes = sorted(sizes or T.DEFAULT_SIZES)
        n, es, tdt = self.num_ranks, ELEM_SIZE[dtype], torch_dtype(dtype)
        ll_max = self.config.ll_max_bytes or (4 << 20)
        per_in = max(sizes) // es if kind == "allreduce" else max(1, max(sizes) // es // n)
        per_out = per_in if kind == "allreduce" else per_in * n
        xs = [torch.randn(per_in, device=self.device(r)).to(tdt) for r in range(n)]
        ys = [torch.empty(per_out, device=self.device(r), dtype=tdt) for r in range(n)]
        names = list(algos or T.CANDIDATES[kind])
        times = {a: [None] * len(sizes) for a in names}
        for i, nb in enumerate(sizes):
            cnt = max(1, nb // es) if kind == "allreduce" else max(1, nb // es // n)
            oc = cnt if kind == "allreduce" else cnt * n
            for a in T.candidates(kind, ll_max, nb, names):
                aid = T.algo_id(a)
                xi, yi = [x[:cnt] for x in xs], [y[:oc] for y in ys]
                try:
                    times[a][i] = _measure(self, lambda: C.run(kind, xi, yi, cnt, dtype, aid, self), iters, 3)
                except BadSizeError:   # beyond this algorithm's capacity (e.g. the LL scratch)
                    pass
        table = T.selection_from_times(sizes, times)
        if install:
            T.install(self.comm, kind, dtype, table)
        return {"table": table, "sizes": sizes, "times": times}

    # -- symmetric heap (cfSymHeapCreate / cfMemAlloc) ----------------------

    def symmetric_heap(self, nbytes: int, mode=None) -> int:
        """Create every rank's symmetric heap of `nbytes` (include/cf.h).
        mode: 1 NVLS multicast, 2 emulated switch, 0 plain; default: the
        world's use_multicast ("emulate" -> 2; multicast built -> 1; else 0).
        Returns the mode in use."""
        if mode is None:
            mode = 2 if self.config.use_multicast == 2 else (1 if self.multicast_supported() else 0)
        _lib.check(_lib.lib().cfSymHeapCreate(self.comm, int(nbytes), int(mode), None))
        self._sym_mode = int(mode)
        return self._sym_mode

    def alloc_symmetric(self, numel: int, dtype) -> list:
        """Collective allocation from the symmetric heap: one tensor per rank,
        all at the same heap offset.  switch_2pa runs in place on them
        (multimem, no staging) and no registration is ever needed."""
        import torch
        es = torch.empty(0, dtype=dtype).element_size()
        ptrs = (ctypes.c_void_p * self.num_ranks)()
        _lib.check(_lib.lib().cfMemAlloc(self.comm, int(numel) * es, ptrs))
        return [_lib.tensor_at(ptrs[r], numel, dtype, self.device(r)) for r in range(self.num_ranks)]

    def free_symmetric(self, tensors) -> None:
        _lib.check(_lib.lib().cfMemFree(self.comm, tensors[0].data_ptr()))

    def switch_channel(self, rank: int) -> bytes:
        """Device handle of the SwitchChannel over the symmetric heaps for
        `rank`'s kernels (cf::SwitchChannelDevice; cf/channels.py:333-409)."""
        buf = ctypes.create_string_buffer(256)
        nbytes = ctypes.c_size_t(256)
        _lib.check(_lib.lib().cfSwitchChannelCreate(self.comm, int(rank), buf, ctypes.byref(nbytes)))
        return buf.raw[:nbytes.value]

    def multicast_supported(self) -> bool:
        v = ctypes.c_int()
        _lib.check(_lib.lib().cfCommMulticastSupported(self.comm, ctypes.byref(v)))
        return bool(v.value)

    def close(self):
        if self._comm is not None:
            _lib.lib().cfCommDestroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __repr__(self):
        return (f"World(ranks={self.num_ranks}, devices={self.devices}, "
                f"coresident={self.coresident})")


def device_multicast_capable(dev: int) -> bool:
    """CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED of a device (NVLS availability)."""
    v = ctypes.c_int()
    _lib.check(_lib.lib().cfDeviceMulticastSupported(int(dev), ctypes.byref(v)))
    return bool(v.value)


def make_world(num_nodes=1, gpus_per_node=1, intra_kind="switch-attached", seed=0, **kw) -> World:
    """cf/world.py:184-185 with the same arguments; extra keywords (devices,
    ll_max_bytes, max_blocks, threads, spin_timeout_ms) tune the communicator."""
    return World(num_nodes, gpus_per_node, intra_kind, seed, **kw)
