"""Collective algorithm library as DSL programs (drop-in for the builders of
``cf/collectives.py:30-270``).

The programs themselves are recorded by libcf's native builders
(``cfDslBuild`` in ``csrc/cf_dsl.cpp``) and returned as ``ProgramGraph``
objects, so callers can extend them before ``lower()`` exactly as with the
reference.  Channel creation order and per-stream instruction order follow the
reference, hence ``lower(build_x(params), params)`` is byte-identical to the
reference plan (``tests/golden/plans``).  The hand-written kernels of
``csrc/cf_collectives.cu`` implement the same algorithms directly.
"""

from __future__ import annotations

from .errors import NoAlgoError, TopologyError
from .lowering import LoweringParams, ProgramGraph, native_program

_NATIVE = frozenset(("ring_rs", "ring_ag", "2pr", "1pa", "switch_2pa", "allpairs_ag"))


def _graph(algo: str, params: LoweringParams, variant: str = "") -> ProgramGraph:
    prog = native_program(algo, params, variant)
    g = ProgramGraph(prog["name"], prog["collective"], params)
    g.absorb(prog)
    return g


def build_ring_rs(params: LoweringParams, out_full: bool = False, graph: ProgramGraph | None = None) -> ProgramGraph:
    """Overlapped ring ReduceScatter (cf/collectives.py:30-79), recorded into
    `graph` when given.  `out_full` reduces into the rank's chunk of a
    full-size output the graph already declares (2PR's first phase)."""
    if not out_full:
        prog = native_program("ring_rs", params)
    else:
        # 2PR records exactly this phase first: keep its prefix, up to the
        # first AllGather put (source: the output buffer), minus the output
        # declaration 2PR makes itself
        prog = native_program("2pr", params)
        rows = prog["instrs"]
        cut = next((i for i, row in enumerate(rows) if row[2] == "put" and row[4] and row[4][0] == "output"),
                   len(rows))
        prog = dict(prog, instrs=rows[:cut], buffers=[b for b in prog["buffers"] if b[0] != "output"])
    g = graph if graph is not None else ProgramGraph("ring_rs", "reducescatter", params)
    g.absorb(prog)
    return g


def build_ring_ag(params: LoweringParams) -> ProgramGraph:
    """Ring AllGather forwarding the last arrival (cf/collectives.py:82-104)."""
    return _graph("ring_ag", params)


def build_2pr(params: LoweringParams) -> ProgramGraph:
    """Two-phase ring AllReduce on port channels (cf/collectives.py:107-136)."""
    return _graph("2pr", params)


def build_1pa(params: LoweringParams) -> ProgramGraph:
    """One-phase all-pairs over LL memory channels (cf/collectives.py:139-162)."""
    return _graph("1pa", params)


def build_2pa(params: LoweringParams, variant: str = "memory") -> ProgramGraph:
    """Two-phase all-pairs, variant memory / ll / port (cf/collectives.py:165-232)."""
    return _graph("2pa", params, variant or "memory")


def build_switch_2pa(params: LoweringParams) -> ProgramGraph:
    """NVLS reduce + broadcast per owned chunk (cf/collectives.py:235-250)."""
    return _graph("switch_2pa", params)


def build_allpairs_ag(params: LoweringParams) -> ProgramGraph:
    """All-pairs AllGather over HB memory channels (cf/collectives.py:253-270)."""
    return _graph("allpairs_ag", params)


def build_algo(name: str, params: LoweringParams, world=None, variant: str = "") -> ProgramGraph:
    """cf/collectives.py:510-525 (single-node algorithms)."""
    if name == "2ph":
        raise TopologyError("2ph is the multi-node hierarchical algorithm (out of scope)")
    if name == "2pa":
        return build_2pa(params, variant or "memory")
    if name not in _NATIVE:
        raise NoAlgoError(f"unknown algorithm {name!r}")
    return _graph(name, params)
