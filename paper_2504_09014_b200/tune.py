"""Measured algorithm selection ("measured crossover table per
(collective, dtype, n) from the sweep").

The reference's Selector is a fixed size table (``cf/collectives.py:436-491``).
Here ``World.tune`` / ``Communicator.tune`` time every candidate algorithm at
a ladder of sizes on the live GPUs (CUDA graphs, max over ranks), keep the
fastest per size and install the resulting table in libcf
(``cfCommSetSelection``), identical on every rank, so ``algo="auto"`` follows
what this box measured -- co-resident ranks on one GPU, or NVLink between
GPUs.  On a multicast heap the smallest size from which the in-place NVLS
kernel wins is measured too (``cfCommSetNvlsMinBytes``).
"""

from __future__ import annotations

import ctypes

from . import _lib
from .dtypes import CODES
from .errors import NoAlgoError

KiB, MiB = 1 << 10, 1 << 20
DEFAULT_SIZES = tuple(KiB << (2 * i) for i in range(9))            # 1 KiB .. 64 MiB, x4
CANDIDATES = {"allreduce": ("1pa", "2pa_ll", "2pa", "1pa_hb"),
              "allgather": ("allpairs_ag", "ring_ag+ring")}
_COLL = {"allreduce": 0, "allgather": 1}
_LL = ("1pa", "2pa_ll")


def algo_id(name: str) -> int:
    """libcf id of a candidate name ("2pa_ll", "ring_ag+ring" = literal ring)."""
    base, _, links = name.partition("+")
    if base not in _lib.ALGOS or base == "auto":
        raise NoAlgoError(f"unknown algorithm {name!r}")
    return _lib.ALGOS[base] | (_lib.CF_ALGO_RING_LINKS if links else 0)


def selection_from_times(sizes, times: dict) -> list:
    """[(max_bytes, algo)] from per-size timings ``times[algo][i]`` (seconds,
    None = not run at sizes[i]): the fastest algorithm per size, runs of one
    winner merged; the last entry also covers every larger size."""
    table = []
    for i, nb in enumerate(sorted(sizes)):
        best = min(((t[i], a) for a, t in times.items() if t[i] is not None), default=None)
        if best is None:
            continue
        if table and table[-1][1] == best[1]:
            table[-1] = (nb, best[1])
        else:
            table.append((nb, best[1]))
    return table


def nvls_min_from_times(sizes, nvls: list, best: list):
    """Smallest size from which NVLS beats the best other algorithm at that
    size and at every larger measured size (None: never)."""
    start = None
    for nb, tn, tb in zip(sorted(sizes), nvls, best):
        if tn is not None and tb is not None and tn < tb:
            start = nb if start is None else start
        else:
            start = None
    return start


def install(comm_handle, kind: str, dtype: str, table: list) -> None:
    """cfCommSetSelection with a [(max_bytes, algo name)] table ([] = built-in)."""
    n = len(table)
    mb = (ctypes.c_size_t * max(1, n))(*[int(b) for b, _ in table])
    ids = (ctypes.c_int * max(1, n))(*[algo_id(a) for _, a in table])
    _lib.check(_lib.lib().cfCommSetSelection(comm_handle, _COLL[kind], CODES[dtype], n, mb, ids))


def candidates(kind: str, ll_max_bytes: int, nbytes: int, algos=None):
    for a in (algos or CANDIDATES[kind]):
        if a in _LL and nbytes > ll_max_bytes:
            continue
        yield a


def time_graph(device, fn, iters: int, reps: int = 3, before=None) -> float:
    """Seconds per call of ``fn`` captured ``iters`` times in one CUDA graph,
    best of ``reps`` replays (``before()`` runs ahead of every replay, e.g. a
    bootstrap barrier so that every rank replays together)."""
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize(device)
    s = torch.cuda.Stream(device)
    s.wait_stream(torch.cuda.current_stream(device))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
    torch.cuda.synchronize(device)
    best = None
    for _ in range(reps):
        if before is not None:
            before()
        st = torch.cuda.current_stream(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        e1.synchronize()
        t = e0.elapsed_time(e1) / 1e3 / iters
        best = t if best is None else min(best, t)
    return best
