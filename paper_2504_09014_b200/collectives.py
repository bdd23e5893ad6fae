"""Collective API: the drop-in replacement of ``cf/collectives.py``.

``collective(kind, inputs, world, ...)`` keeps the reference signature
(``cf/collectives.py:532-573``): per-rank inputs in, per-rank outputs back,
zero-padding to the algorithm's required multiple, AllReduce outputs
truncated, ReduceScatter shards on the padded domain.  The work runs in the
hand-written sm_100a kernels of libcf (no host arithmetic): each GPU algorithm
reproduces its reference algorithm's accumulation order, so i32 and f32
results are bit-identical to the reference's ``collective()``.

Inputs may be numpy arrays (copied to the ranks' devices and back, like the
reference copies into its regions, ``cf/executor.py:160-175``) or CUDA torch
tensors (zero-copy; outputs are returned as tensors on the ranks' devices).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .dtypes import CODES, ELEM_SIZE, NP_DTYPES, from_torch
from .errors import NoAlgoError, ShapeError, TopologyError

ALGO_NAMES = ("ring_rs", "ring_ag", "2pr", "1pa", "2pa", "2ph", "allpairs_ag", "switch_2pa")

KiB = 1024
MiB = 1024 * 1024

# Reference defaults (cf/collectives.py:418) -- used when a Selector carries
# explicit thresholds; the default Selector asks libcf's measured table.
DEFAULT_THRESHOLDS = {"small": 32 * KiB, "large": 64 * MiB, "hier": 1 * MiB}

_COLL = {"allreduce": 0, "allgather": 1, "reducescatter": 2}


@dataclass(frozen=True)
class AlgoDescriptor:
    """cf/collectives.py:421-433."""

    name: str
    protocol: str
    channel_type: str
    min_bytes: int
    max_bytes: int | None
    scope: str
    variant: str = ""

    def covers(self, nbytes: int) -> bool:
        return self.min_bytes <= nbytes and (self.max_bytes is None or nbytes < self.max_bytes)


def default_table(collective: str, thresholds: dict | None = None) -> list[AlgoDescriptor]:
    """The reference's threshold table (cf/collectives.py:436-461), single node."""
    t = {**DEFAULT_THRESHOLDS, **(thresholds or {})}
    if collective == "allreduce":
        return [AlgoDescriptor("1pa", "LL", "memory", 0, t["small"], "single-node"),
                AlgoDescriptor("2pa", "HB", "memory", t["small"], t["large"], "single-node",
                               variant="memory"),
                AlgoDescriptor("2pr", "HB", "port", t["large"], None, "single-node")]
    if collective == "allgather":
        return [AlgoDescriptor("allpairs_ag", "HB", "memory", 0, t["hier"], "single-node"),
                AlgoDescriptor("ring_ag", "HB", "port", t["hier"], None, "single-node")]
    if collective == "reducescatter":
        return [AlgoDescriptor("ring_rs", "HB", "port", 0, None, "single-node")]
    raise NoAlgoError(f"unknown collective {collective!r}")


# libcf algorithm id -> descriptor fields
_DESC = {
    "1pa": ("1pa", "LL", "memory", ""), "1pa_hb": ("1pa_hb", "HB", "memory", ""),
    "2pa": ("2pa", "HB", "memory", "memory"), "2pa_ll": ("2pa", "LL", "memory", "ll"),
    "switch_2pa": ("switch_2pa", "HB", "switch", ""), "2pr": ("2pr", "HB", "port", ""),
    "allpairs_ag": ("allpairs_ag", "HB", "memory", ""), "ring_ag": ("ring_ag", "HB", "port", ""),
    "ring_rs": ("ring_rs", "HB", "port", ""), "rs_direct": ("rs_direct", "HB", "memory", ""),
}


@dataclass
class Selector:
    """cf/collectives.py:464-486.  By default it is the reference's threshold
    table, so ``collective()`` picks the reference's algorithm -- the same
    output shapes (e.g. ring_rs pads ReduceScatter to 2n) and the same
    accumulation order, hence the reference's bits.  ``measured=True`` asks
    libcf's measured crossover table for the world instead (the fastest
    kernel per size; its order may differ from the reference's pick)."""

    thresholds: dict = field(default_factory=dict)
    override: str | None = None
    override_variant: str = ""
    measured: bool = False

    def table(self, collective: str) -> list[AlgoDescriptor]:
        return default_table(collective, self.thresholds)

    def select(self, collective: str, nbytes: int, topology, world=None,
               dtype: str = "f32") -> AlgoDescriptor:
        if topology.num_nodes != 1:
            raise TopologyError("multi-node selection is out of scope (one NVSwitch domain)")
        if self.override:
            for d in self.table(collective):
                if d.name == self.override and (not self.override_variant
                                                or d.variant == self.override_variant):
                    return d
            return AlgoDescriptor(self.override, "HB", "port", 0, None, "single-node",
                                  variant=self.override_variant)
        if self.measured and world is not None:
            algo = ctypes.c_int()
            _lib.check(_lib.lib().cfSelectAlgorithm(world.comm, _COLL[collective], int(nbytes),
                                                    CODES[dtype], ctypes.byref(algo)))
            name, proto, chan, var = _DESC[_lib.ALGO_NAMES[algo.value]]
            return AlgoDescriptor(name, proto, chan, 0, None, "single-node", variant=var)
        for d in self.table(collective):
            if d.covers(nbytes):
                return d
        raise NoAlgoError(f"no algorithm covers {nbytes} bytes for {collective}")


def select_algorithm(collective: str, nbytes: int, topology, selector: Selector | None = None,
                     world=None, dtype: str = "f32") -> AlgoDescriptor:
    return (selector or Selector()).select(collective, nbytes, topology, world=world, dtype=dtype)


def required_multiple(name: str, n: int, gpus_per_node: int = 1) -> int:
    """cf/collectives.py:497-504 (single-node subset plus the new names)."""
    table = {"ring_rs": 2 * n, "2pr": 2 * n, "1pa": 1, "1pa_hb": 1, "2pa": n, "switch_2pa": n,
             "ring_ag": 1, "allpairs_ag": 1, "rs_direct": n}
    if name not in table:
        raise NoAlgoError(f"unknown algorithm {name!r}")
    return table[name]


def _algo_id(kind: str, name: str, variant: str) -> int:
    if name == "2ph":
        raise TopologyError("2ph is the multi-node hierarchical algorithm (out of scope)")
    if name == "2pa":
        key = {"": "2pa", "memory": "2pa", "ll": "2pa_ll", "port": "2pa"}.get(variant)
        if key is None:
            raise NoAlgoError(f"unknown 2pa variant {variant!r}")
    else:
        key = name
    if key not in _lib.ALGOS or key == "auto":
        raise NoAlgoError(f"unknown algorithm {name!r}")
    links = 0
    if key in ("2pr", "ring_rs", "ring_ag"):
        # variant "ring" (extension): the literal ring over point-to-point
        # links; "" runs the same order and padding all-pairs (cf.h
        # CF_ALGO_RING_LINKS) -- identical results
        if variant not in ("", "ring"):
            raise NoAlgoError(f"unknown {key} variant {variant!r}")
        links = _lib.CF_ALGO_RING_LINKS if variant == "ring" else 0
    ok = {"allreduce": {"1pa", "1pa_hb", "2pa", "2pa_ll", "switch_2pa", "2pr"},
          "allgather": {"allpairs_ag", "ring_ag"},
          "reducescatter": {"ring_rs", "rs_direct"}}[kind]
    if key not in ok:
        raise NoAlgoError(f"{name!r} is not a {kind} algorithm")
    return _lib.ALGOS[key] | links


def _padded(elems: int, multiple: int) -> int:
    return elems if elems % multiple == 0 else elems + multiple - elems % multiple


def _to_device(arrays, world, dtype):
    import torch
    out = []
    for r, a in enumerate(arrays):
        a = np.ascontiguousarray(a, NP_DTYPES[dtype])
        t = torch.from_numpy(a.view(np.int16)).view(torch.bfloat16) if dtype == "bf16" \
            else torch.from_numpy(a)
        out.append(t.to(world.device(r)))
    return out


def _to_host(t, dtype):
    import torch
    t = t.detach().cpu()
    if dtype == "bf16":
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def run(kind: str, send, recv, count: int, dtype: str, algo: int, world) -> None:
    """Raw entry: one libcf call on per-rank CUDA tensors (no padding, no copies)."""
    n = world.num_ranks
    sp = _lib.ptr_array([t.data_ptr() for t in send])
    rp = _lib.ptr_array([t.data_ptr() for t in recv])
    st = _lib.ptr_array(world.streams())
    fn = {"allreduce": _lib.lib().cfAllReduce, "allgather": _lib.lib().cfAllGather,
          "reducescatter": _lib.lib().cfReduceScatter}[kind]
    assert len(send) == n and len(recv) == n
    _lib.check(fn(world.comm, sp, rp, int(count), CODES[dtype], int(algo), st))


def _plan_runtime(world, kind, name, var, elems, dtype):
    """Lowered DSL plan of a library algorithm on this world (cached per shape):
    the MSCCL++ DSL path -- builder, native lowering, GPU interpreter (K10)."""
    from .algorithms import build_algo
    from .executor import Runtime
    from .lowering import LoweringParams, lower
    cache = world.__dict__.setdefault("_plan_cache", {})
    key = (kind, name, var, elems, dtype)
    if key not in cache:
        proto = "LL" if name == "1pa" or var == "ll" else "HB"
        params = LoweringParams(world.num_ranks, elems, dtype, proto)
        cache[key] = Runtime(lower(build_algo(name, params, variant=var), params), world)
    return cache[key]


def _run_via_plan(kind, name, var, tensors, elems, dtype, world):
    import torch
    n = world.num_ranks
    if kind == "allgather":
        rt = _plan_runtime(world, kind, name, var, elems, dtype)
        ins = tensors
    else:
        padded = _padded(elems, required_multiple(name, n))
        rt = _plan_runtime(world, kind, name, var, padded, dtype)
        ins = tensors if padded == elems else \
            [torch.cat([t, t.new_zeros(padded - elems)]) for t in tensors]
    outs = [t.new_empty(rt.out_elems) for t in ins]
    rt.run_raw(ins, outs)
    world.synchronize()
    rt.check_device_error()
    return [o[:elems] for o in outs] if kind == "allreduce" else outs


def collective(kind: str, inputs, world, selector: Selector | None = None, dtype: str = "i32",
               algo: str | None = None, variant: str = "", mode: str = "round-robin",
               seed: int | None = None, outputs=None, via_plan: bool = False):
    """Select, run on the GPUs, return per-rank outputs (cf/collectives.py:532-573).

    `mode` and `seed` drive the reference's simulated scheduler; real GPUs
    schedule themselves, so they are accepted and ignored.  `outputs`
    (extension): per-rank host torch tensors to receive the results when the
    inputs are host torch tensors (e.g. pinned buffers reused across calls).
    `via_plan` (extension) runs the algorithm as a lowered DSL plan on the GPU
    interpreter instead of its hand-written kernel; the 2pa "port" variant
    always does (its puts are PortChannel requests served by the proxy's
    copy-engine DMA).  Plan ops round 2-byte types once per op.
    """
    import torch
    if kind not in _COLL:
        raise NoAlgoError(f"unknown collective {kind!r}")
    n = world.num_ranks
    if len(inputs) != n:
        raise ShapeError(f"need {n} inputs, got {len(inputs)}")
    on_gpu = all(isinstance(a, torch.Tensor) and a.is_cuda for a in inputs)
    host_tensors = all(isinstance(a, torch.Tensor) and not a.is_cuda for a in inputs)
    if on_gpu:
        dtype = from_torch(inputs[0].dtype)
        tensors = [a.contiguous().view(-1) for a in inputs]
    elif host_tensors:
        # host torch tensors (pinned for async copies): AllReduce goes through
        # cfAllReduceHost below; the other collectives copy H2D, run, copy D2H
        dtype = from_torch(inputs[0].dtype)
        tensors = [a.reshape(-1) for a in inputs]
        on_gpu = True
    else:
        tensors = None
        arrays = [np.asarray(a) for a in inputs]
        if dtype == "bf16" and arrays[0].dtype != np.uint16:
            raise ShapeError("bf16 numpy inputs are uint16 bit patterns")
        arrays = [np.ascontiguousarray(a, NP_DTYPES[dtype]).reshape(-1) for a in arrays]
    lens = [int(t.numel()) for t in tensors] if on_gpu else [len(a) for a in arrays]
    elems = lens[0]
    if any(e != elems for e in lens):
        raise ShapeError("all ranks must contribute equally-sized inputs")

    sel = selector or Selector()
    if algo:
        name, var = algo, variant
    else:
        nbytes = elems * ELEM_SIZE[dtype] * (n if kind == "allgather" else 1)
        d = sel.select(kind, nbytes, world.topology, world=world, dtype=dtype)
        name, var = d.name, d.variant
    aid = _algo_id(kind, name, var)
    base = _lib.ALGO_NAMES[aid & ~_lib.CF_ALGO_RING_LINKS]
    mult = required_multiple(base if base != "2pa_ll" else "2pa", n)

    if host_tensors and kind == "allreduce" and elems and not (via_plan or (name == "2pa" and var == "port")):
        # host in, host out through libcf's pipelined host path (copies overlap the kernel)
        src = [a.contiguous().view(-1) for a in inputs]
        pin = src[0].is_pinned()
        host = outputs if outputs is not None else \
            [torch.empty(a.shape, dtype=a.dtype, pin_memory=pin) for a in src]
        _lib.check(_lib.lib().cfAllReduceHost(
            world.comm, _lib.ptr_array([a.data_ptr() for a in src]),
            _lib.ptr_array([h.data_ptr() for h in host]), elems, CODES[dtype], aid,
            _lib.ptr_array(world.streams())))
        world.synchronize()
        world.check_device_error()
        return host
    if not on_gpu:
        tensors = _to_device(arrays, world, dtype)
    elif host_tensors:
        tensors = [t.to(world.device(r), non_blocking=True) for r, t in enumerate(tensors)]
    if elems == 0:
        shape = {"allreduce": 0, "allgather": 0, "reducescatter": 0}[kind]
        outs = [t.new_empty(shape) for t in tensors]
        return outs if on_gpu else [_to_host(o, dtype) for o in outs]
    if via_plan or (name == "2pa" and var == "port"):
        outs = _run_via_plan(kind, name, var or ("memory" if name == "2pa" else ""), tensors, elems,
                             dtype, world)
    elif kind == "allreduce":
        recv = [torch.empty_like(t) for t in tensors]
        run(kind, tensors, recv, elems, dtype, aid, world)
        outs = recv
    elif kind == "allgather":
        recv = [t.new_empty(n * elems) for t in tensors]
        run(kind, tensors, recv, elems, dtype, aid, world)
        outs = recv
    else:
        padded = _padded(elems, mult)
        if padded != elems:
            tensors = [torch.cat([t, t.new_zeros(padded - elems)]) for t in tensors]
        recv = [t.new_empty(padded // n) for t in tensors]
        run(kind, tensors, recv, padded // n, dtype, aid, world)
        outs = recv
    if host_tensors:
        pin = inputs[0].is_pinned()
        host = outputs if outputs is not None else \
            [torch.empty(o.shape, dtype=o.dtype, pin_memory=pin) for o in outs]
        for h, o in zip(host, outs):
            h.copy_(o, non_blocking=pin)
        world.synchronize()
        world.check_device_error()
        return host
    world.synchronize()
    world.check_device_error()
    return outs if on_gpu else [_to_host(o, dtype) for o in outs]


# The reference defines the algorithm builders in this module
# (cf/collectives.py:30-270); they live in algorithms.py here.
from .algorithms import (build_1pa, build_2pa, build_2pr, build_algo, build_allpairs_ag,  # noqa: E402,F401
                         build_ring_ag, build_ring_rs, build_switch_2pa)
