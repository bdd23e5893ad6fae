"""Collective algorithm builders in the DSL (``ProgramGraph``).

Each builder records the data movement of one algorithm of the reference
library (``cf/collectives.py:30-270``) with the same channel declaration order
and instruction order, so ``lower(build_x(params), params)`` yields plans
byte-identical to the reference's.  The plans run on libcf's GPU interpreter;
the hand-written kernels implement the same algorithms directly.
"""

from __future__ import annotations

from .errors import NoAlgoError, ShapeError
from .lowering import BuilderChannel, LoweringParams, ProgramGraph


def _prev(r, n):
    return (r - 1) % n


def build_ring_rs(params: LoweringParams, out_full: bool = False,
                  graph: ProgramGraph | None = None) -> ProgramGraph:
    """Overlapped ring ReduceScatter (cf/collectives.py:30-79).  Step s puts the
    first half of chunk (r - s) to the next rank, reduces the previous arrival's
    second half while it flies, puts the second half and reduces the fresh
    arrival's first half; the last arrival is the rank's own chunk, reduced
    into the zero-initialized output."""
    n, elems = params.num_ranks, params.elems
    if elems % (2 * n):
        raise ShapeError(f"ring ReduceScatter needs elems divisible by {2 * n}")
    cs = elems // n
    h = cs // 2
    g = graph or ProgramGraph("ring_rs", "reducescatter", params)
    g.buffer("input", "input", "all", elems)
    g.buffer("scratch", "scratch", "all", elems)
    if not out_full:
        g.buffer("output", "output", "all", cs)
    if n == 1:
        g.copy(0, dst=("output", 0, cs), src=("input", 0, cs))
        return g
    to_next = [g.port_channel(r, (r + 1) % n) for r in range(n)]
    for r in range(n):
        tx, rx = to_next[r], to_next[_prev(r, n)]
        out_buf, out_off = ("output", r * cs) if out_full else ("output", 0)
        for s in range(n):
            cur = ((r + n - s) % n) * cs          # chunk sent this step
            arr = ((r + n - s - 1) % n) * cs      # chunk arriving this step
            tx.put(dst=("scratch", cur, h), src=("input", cur, h), tb=0)
            tx.signal(tb=0)
            if s > 0:
                g.reduce(r, dst=("input", cur + h, h), src=("scratch", cur + h, h))
            rx.wait(tb=0, arrives=("scratch", arr, h))
            tx.flush(tb=0)
            tx.put(dst=("scratch", cur + h, h), src=("input", cur + h, h), tb=0)
            tx.signal(tb=0)
            if s < n - 1:
                g.reduce(r, dst=("input", arr, h), src=("scratch", arr, h))
            else:
                g.reduce(r, dst=(out_buf, out_off, h), src=("scratch", arr, h))
            rx.wait(tb=0, arrives=("scratch", arr + h, h))
            tx.flush(tb=0)
        g.reduce(r, dst=(out_buf, out_off + h, h), src=("scratch", r * cs + h, h))
    return g


def build_ring_ag(params: LoweringParams) -> ProgramGraph:
    """Ring AllGather (cf/collectives.py:82-104): forward the chunk received
    last step straight into the next rank's output."""
    n, cs = params.num_ranks, params.elems
    g = ProgramGraph("ring_ag", "allgather", params)
    g.buffer("input", "input", "all", cs)
    g.buffer("output", "output", "all", n * cs)
    if n == 1:
        g.copy(0, dst=("output", 0, cs), src=("input", 0, cs))
        return g
    to_next = [g.port_channel(r, (r + 1) % n) for r in range(n)]
    for r in range(n):
        tx, rx = to_next[r], to_next[_prev(r, n)]
        g.copy(r, dst=("output", r * cs, cs), src=("input", 0, cs))
        for t in range(n - 1):
            fwd = ((r + n - t) % n) * cs
            arr = ((r + n - t - 1) % n) * cs
            tx.put(dst=("output", fwd, cs), src=("output", fwd, cs), tb=0)
            tx.signal(tb=0)
            rx.wait(tb=0, arrives=("output", arr, cs))
            tx.flush(tb=0)
    return g


def build_2pr(params: LoweringParams) -> ProgramGraph:
    """Two-phase ring AllReduce (cf/collectives.py:107-136): the ring
    ReduceScatter into the full output, then a ring AllGather of halves on the
    same port channels."""
    n, elems = params.num_ranks, params.elems
    if elems % (2 * n):
        raise ShapeError(f"two-phase ring needs elems divisible by {2 * n}")
    cs = elems // n
    h = cs // 2
    g = ProgramGraph("2pr", "allreduce", params)
    g.buffer("output", "output", "all", elems)
    build_ring_rs(params, out_full=True, graph=g)
    if n == 1:
        return g
    chans = [BuilderChannel(g, d.id, d.type, d.src, d.dst) for d in g.channels]
    for r in range(n):
        tx, rx = chans[r], chans[_prev(r, n)]
        for t in range(n - 1):
            fwd = (r + n - t) % n
            arr = (r + n - t - 1) % n
            for half in (0, 1):
                off = fwd * cs + half * h
                tx.put(dst=("output", off, h), src=("output", off, h), tb=0)
                tx.signal(tb=0)
                rx.wait(tb=0, arrives=("output", arr * cs + half * h, h))
                tx.flush(tb=0)
    return g


def build_1pa(params: LoweringParams) -> ProgramGraph:
    """One-phase all-pairs over LL memory channels (cf/collectives.py:139-162)."""
    n, e = params.num_ranks, params.elems
    g = ProgramGraph("1pa", "allreduce", params)
    g.buffer("input", "input", "all", e)
    g.buffer("output", "output", "all", e)
    g.buffer("llscr", "scratch", "all", 2 * n * e)
    g.buffer("tmp", "scratch", "all", n * e)
    ch = {(r, p): g.memory_channel(r, p) for r in range(n) for p in range(n) if p != r}
    for r in range(n):
        peers = [p for p in range(n) if p != r]
        for p in peers:
            ch[(r, p)].put_packets(dst=("llscr", r * e, e), src=("input", 0, e), tb=0)
        g.copy(r, dst=("output", 0, e), src=("input", 0, e))
        for p in peers:
            ch[(p, r)].read_packets(dst=("tmp", p * e, e), src=("llscr", p * e, e), tb=0)
        for p in peers:
            g.reduce(r, dst=("output", 0, e), src=("tmp", p * e, e))
    return g


def build_2pa(params: LoweringParams, variant: str = "memory") -> ProgramGraph:
    """Two-phase all-pairs AllReduce (cf/collectives.py:165-232); variants
    "memory" (HB pull-reduce + put), "port" (push to slots + reduce + push) and
    "ll" (two packet phases)."""
    n, e = params.num_ranks, params.elems
    if e % n:
        raise ShapeError(f"two-phase all-pairs needs elems divisible by {n}")
    cs = e // n
    g = ProgramGraph(f"2pa_{variant}", "allreduce", params)
    g.buffer("input", "input", "all", e)
    g.buffer("output", "output", "all", e)
    if variant == "ll":
        g.buffer("ph1", "scratch", "all", 2 * e)
        g.buffer("ph2", "scratch", "all", 2 * e)
        g.buffer("tmp", "scratch", "all", e)
    elif variant == "port":
        g.buffer("slots", "scratch", "all", e)
    make = g.port_channel if variant == "port" else g.memory_channel
    ch = {(r, p): make(r, p) for r in range(n) for p in range(n) if p != r}
    for r in range(n):
        peers = [p for p in range(n) if p != r]
        mine = ("output", r * cs, cs)
        if variant == "memory":
            g.copy(r, dst=mine, src=("input", r * cs, cs))
            for p in peers:
                ch[(r, p)].reduce(dst=mine, src=("input", r * cs, cs), tb=0)
            for p in peers:
                ch[(r, p)].put(dst=mine, src=mine, tb=0)
                ch[(r, p)].signal(tb=0)
            for p in peers:
                ch[(p, r)].wait(tb=0, arrives=("output", p * cs, cs))
        elif variant == "port":
            for p in peers:
                ch[(r, p)].put(dst=("slots", r * cs, cs), src=("input", p * cs, cs), tb=0)
                ch[(r, p)].signal(tb=0)
            g.copy(r, dst=mine, src=("input", r * cs, cs))
            for p in peers:
                ch[(p, r)].wait(tb=0, arrives=("slots", p * cs, cs))
            for p in peers:
                g.reduce(r, dst=mine, src=("slots", p * cs, cs))
            for p in peers:
                ch[(r, p)].put(dst=mine, src=mine, tb=0)
                ch[(r, p)].signal(tb=0)
            for p in peers:
                ch[(p, r)].wait(tb=0, arrives=("output", p * cs, cs))
            for p in peers:
                ch[(r, p)].flush(tb=0)
        elif variant == "ll":
            for p in peers:
                ch[(r, p)].put_packets(dst=("ph1", r * cs, cs), src=("input", p * cs, cs), tb=0)
            g.copy(r, dst=mine, src=("input", r * cs, cs))
            for p in peers:
                ch[(p, r)].read_packets(dst=("tmp", p * cs, cs), src=("ph1", p * cs, cs), tb=0)
            for p in peers:
                g.reduce(r, dst=mine, src=("tmp", p * cs, cs))
            for p in peers:
                ch[(r, p)].put_packets(dst=("ph2", r * cs, cs), src=mine, tb=0)
            for p in peers:
                ch[(p, r)].read_packets(dst=("output", p * cs, cs), src=("ph2", p * cs, cs),
                                        tb=0)
        else:
            raise NoAlgoError(f"unknown 2pa variant {variant!r}")
    return g


def build_switch_2pa(params: LoweringParams) -> ProgramGraph:
    """Switch (NVLS) two-phase AllReduce (cf/collectives.py:235-250)."""
    n, e = params.num_ranks, params.elems
    if e % n:
        raise ShapeError(f"switch all-pairs needs elems divisible by {n}")
    cs = e // n
    g = ProgramGraph("switch_2pa", "allreduce", params)
    g.buffer("input", "input", "all", e)
    g.buffer("output", "output", "all", e)
    g.buffer("tmp", "scratch", "all", cs)
    sw = g.switch_channel(list(range(n)))
    for r in range(n):
        sw.reduce(r, dst=("tmp", 0, cs), src=("input", r * cs, cs), tb=0)
        sw.broadcast(r, dst=("output", r * cs, cs), src=("tmp", 0, cs), tb=0)
    return g


def build_allpairs_ag(params: LoweringParams) -> ProgramGraph:
    """All-pairs AllGather over HB memory channels (cf/collectives.py:253-270)."""
    n, cs = params.num_ranks, params.elems
    g = ProgramGraph("allpairs_ag", "allgather", params)
    g.buffer("input", "input", "all", cs)
    g.buffer("output", "output", "all", n * cs)
    ch = {(r, p): g.memory_channel(r, p) for r in range(n) for p in range(n) if p != r}
    for r in range(n):
        peers = [p for p in range(n) if p != r]
        g.copy(r, dst=("output", r * cs, cs), src=("input", 0, cs))
        for p in peers:
            ch[(r, p)].put(dst=("output", r * cs, cs), src=("input", 0, cs), tb=0)
            ch[(r, p)].signal(tb=0)
        for p in peers:
            ch[(p, r)].wait(tb=0, arrives=("output", p * cs, cs))
    return g


def build_algo(name: str, params: LoweringParams, world=None, variant: str = "") -> ProgramGraph:
    """cf/collectives.py:507-525 (single-node algorithms)."""
    table = {"ring_rs": build_ring_rs, "ring_ag": build_ring_ag, "2pr": build_2pr,
             "1pa": build_1pa, "switch_2pa": build_switch_2pa, "allpairs_ag": build_allpairs_ag}
    if name == "2pa":
        return build_2pa(params, variant=variant or "memory")
    if name == "2ph":
        from .errors import TopologyError
        raise TopologyError("2ph is the multi-node hierarchical algorithm (out of scope)")
    if name not in table:
        raise NoAlgoError(f"unknown algorithm {name!r}")
    return table[name](params)
