"""Measured replacement of the reference's benchmark API (cf/timing.py).

The reference times plans on an alpha-beta discrete-event model
(``CostParams``, ``simulate_timed``; cf/timing.py:36-300) -- simulation
tooling that real B200s replace with measurement.  What
carries over is the API a user benchmarks with: ``algobw`` (the same
definition, cf/timing.py:54-58), ``run_benchmark`` / ``BenchRow`` /
``rows_to_csv`` (cf/timing.py:304-358) -- here every latency is measured on
the world's GPUs: the collective captured ``iters`` times in one CUDA graph,
replayed, timed with CUDA events on the replay stream (best of ``reps``).
``CostParams`` is accepted for signature compatibility and ignored.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field

from .errors import BadSizeError, BadTimeError

# cf/timing.py:313-314 (single node); 1pa_hb is this package's extra one-shot
SINGLE_NODE_VARIANTS = [("1pa", ""), ("2pa", "ll"), ("2pa", "memory"), ("2pa", "port"),
                        ("switch_2pa", ""), ("2pr", ""), ("1pa_hb", "")]
_OTHER = {"allgather": [("allpairs_ag", ""), ("ring_ag", "")],
          "reducescatter": [("rs_direct", ""), ("ring_rs", "")]}


@dataclass
class LinkParams:
    """cf/timing.py:26-33: an alpha-beta link (seconds, bytes / second)."""
    alpha: float
    beta: float

    def __post_init__(self):
        if self.alpha < 0 or self.beta <= 0:
            raise BadTimeError("alpha must be >= 0 and beta positive")


@dataclass
class CostParams:
    """The reference's cost-model parameters (cf/timing.py:36-45), kept for
    signature compatibility: ``transfer_time`` evaluates them; the benchmark
    API ignores them (its latencies are measured)."""
    intra: LinkParams = field(default_factory=lambda: LinkParams(829e-9, 397.5e9))
    inter: LinkParams = field(default_factory=lambda: LinkParams(4.89e-6, 48.94e9))
    tb_sync: float = 200e-9
    sem_op: float = 100e-9
    proxy_hop: float = 500e-9

    def link(self, link_class: str) -> LinkParams:
        from .world import INTRA
        return self.intra if link_class == INTRA else self.inter


def transfer_time(link_class: str, nbytes: int, p: CostParams) -> float:
    """The alpha-beta transfer time of the reference's model (cf/timing.py:48-51)."""
    lp = p.link(link_class)
    return lp.alpha + nbytes / lp.beta


@dataclass(frozen=True)
class TimedEvent:
    """cf/timing.py:61-68."""
    ctx: str
    label: str
    start: float
    end: float
    link: tuple | None = None
    nbytes: int = 0


@dataclass
class TimedTrace:
    """cf/timing.py:71-79.  From ``simulate_timed`` here: one event per
    (rank, program) spanning the measured execution, no per-op events."""
    events: list
    makespan: float

    def link_bytes(self, link_class: str | None = None) -> int:
        return sum(e.nbytes for e in self.events
                   if e.link is not None and (link_class is None or e.link[2] == link_class))


def simulate_timed(plan, world, p: CostParams | None = None, dtype: str | None = None, iters: int = 20,
                   reps: int = 3) -> TimedTrace:
    """The reference times a plan on its discrete-event model
    (cf/timing.py:295-298); here the plan runs on the world's GPUs (K10) and
    the makespan is its measured latency (CUDA graph, best of ``reps``);
    ``p`` is ignored."""
    import torch
    from .executor import Runtime
    from .dtypes import torch_dtype
    rt = Runtime(plan, world, dtype=dtype)
    try:
        tdt = torch_dtype(rt.dtype)
        n = world.num_ranks
        xs = [torch.zeros(rt.in_elems, device=world.device(r), dtype=tdt) for r in range(n)]
        ys = [torch.empty(rt.out_elems, device=world.device(r), dtype=tdt) for r in range(n)]
        t = _measure(world, lambda: rt.run_raw(xs, ys), iters, reps)
    finally:
        rt.close()
    events = [TimedEvent(f"r{pr.rank}.tb{pr.tb}", "program", 0.0, t) for pr in plan.programs]
    return TimedTrace(events, t)


@dataclass
class BenchRow:
    """cf/timing.py:304-310."""
    algo: str
    collective: str
    nbytes: int
    latency_us: float
    algobw_gbps: float
    selected: bool


def algobw(nbytes: int, latency: float) -> float:
    """Algorithm bandwidth: message size divided by end-to-end latency
    (cf/timing.py:54-58, same error on a non-positive latency)."""
    if latency <= 0:
        raise BadTimeError(f"latency must be positive, got {latency}")
    return nbytes / latency


def busbw(nbytes: int, latency: float, n: int, collective: str = "allreduce") -> float:
    """nccl-tests bus bandwidth: algbw x 2(n-1)/n (AllReduce) or x (n-1)/n
    (AllGather with nbytes = output, ReduceScatter with nbytes = input)."""
    f = 2 * (n - 1) / n if collective == "allreduce" else (n - 1) / n
    return algobw(nbytes, latency) * f


def _measure(world, fn, iters: int, reps: int) -> float:
    import torch
    dev = world.device(0)
    for _ in range(3):
        fn()
    world.synchronize()
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
    world.synchronize()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.current_stream(dev)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / iters
        best = t if best is None else min(best, t)
    world.check_device_error()
    return best


def timed_latency(name: str, variant: str, nbytes: int, world, p: CostParams | None = None,
                  collective: str = "allreduce", dtype: str = "bf16", iters: int = 20, reps: int = 3) -> float:
    """Measured seconds per call of one algorithm -- the reference's signature
    (cf/timing.py:318-328, which computes the same quantity on its model);
    ``p`` is ignored."""
    import torch
    from . import collectives as C
    from .dtypes import ELEM_SIZE, torch_dtype
    n = world.num_ranks
    es = ELEM_SIZE[dtype]
    tdt = torch_dtype(dtype)
    if collective == "allreduce":
        cnt = max(1, nbytes // es)
        if name == "2pa" and variant == "port":
            cnt = C._padded(cnt, C.required_multiple("2pa", n))
            rt = C._plan_runtime(world, "allreduce", "2pa", "port", cnt, dtype)
            xs = [torch.randn(rt.in_elems, device=world.device(r)).to(tdt) for r in range(n)]
            ys = [torch.empty(rt.out_elems, device=world.device(r), dtype=tdt) for r in range(n)]
            return _measure(world, lambda: rt.run_raw(xs, ys), iters, reps)
        aid = C._algo_id("allreduce", name, variant)
        xs = [torch.randn(cnt, device=world.device(r)).to(tdt) for r in range(n)]
        ys = [torch.empty_like(x) for x in xs]
        return _measure(world, lambda: C.run("allreduce", xs, ys, cnt, dtype, aid, world), iters, reps)
    shard = max(1, nbytes // es // n)
    aid = C._algo_id(collective, name, variant)
    if collective == "allgather":
        xs = [torch.randn(shard, device=world.device(r)).to(tdt) for r in range(n)]
        ys = [torch.empty(shard * n, device=world.device(r), dtype=tdt) for r in range(n)]
    else:
        xs = [torch.randn(shard * n, device=world.device(r)).to(tdt) for r in range(n)]
        ys = [torch.empty(shard, device=world.device(r), dtype=tdt) for r in range(n)]
    return _measure(world, lambda: C.run(collective, xs, ys, shard, dtype, aid, world), iters, reps)


def _key(name: str, variant: str) -> str:
    if name == "2pa":
        return {"ll": "2pa_ll", "port": "2pa_port"}.get(variant, "2pa")
    return name


def run_benchmark(collective: str, sizes: list[int], world, p: CostParams | None = None,
                  selector=None, dtype: str = "bf16", iters: int = 20) -> list[BenchRow]:
    """One row per (algorithm variant, size), measured on the world's GPUs; the
    selector's pick is marked (cf/timing.py:331-349)."""
    from .collectives import Selector
    sel = selector or Selector()
    variants = SINGLE_NODE_VARIANTS if collective == "allreduce" else _OTHER[collective]
    rows = []
    for name, variant in variants:
        for nbytes in sorted(sizes):
            try:
                latency = timed_latency(name, variant, nbytes, world, p, collective, dtype, iters)
            except BadSizeError:   # beyond an LL algorithm's capacity: no row, as no plan
                continue
            pick = sel.select(collective, nbytes, world.topology, world=world, dtype=dtype)
            chosen = _key(name, variant) == _key(pick.name, pick.variant or "")
            rows.append(BenchRow(algo=name if not variant else f"{name}_{variant}", collective=collective,
                                 nbytes=nbytes, latency_us=latency * 1e6,
                                 algobw_gbps=algobw(nbytes, latency) / 1e9, selected=chosen))
    return rows


def rows_to_csv(rows: list[BenchRow]) -> str:
    """cf/timing.py:352-358 (same columns)."""
    out = io.StringIO()
    out.write("algo,collective,bytes,latency_us,algobw_gbps,selected\n")
    for r in rows:
        out.write(f"{r.algo},{r.collective},{r.nbytes},{r.latency_us:.6f},"
                  f"{r.algobw_gbps:.6f},{int(r.selected)}\n")
    return out.getvalue()
