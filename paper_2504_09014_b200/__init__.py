"""B200-native collective hot path of MSCCL++ (arXiv 2504.09014).

Drop-in for the reference package's API (commforge 0.1.0, ``cf/__init__.py:12-17``):
the collective facade, the selector and the world bootstrap run on
hand-written sm_100a kernels in ``libcf.so`` (C ABI: ``include/cf.h``).
"""

__version__ = "0.1.0"

import os as _os

# The PortChannel proxy (a host thread issuing copy-engine DMA on its own
# stream) must not share a hardware work queue with the caller's stream: with
# CUDA's default 8 connections, a collective kernel waiting for the proxy's
# copy and the next kernel queued behind it on the caller's stream can land
# the copy behind that next kernel -- a deadlock (measured: two back-to-back
# port-channel plan calls time out with 1 or 8 connections, run with 32).  The
# setting is read when the CUDA context is created, so it is applied here,
# before any CUDA use, unless the caller chose a value.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .collectives import AlgoDescriptor, Selector, collective, required_multiple, select_algorithm
from .errors import CommforgeError
from .executor import RunResult, Runtime
from .fused import allreduce_add_rmsnorm
from .lowering import LoweringParams, ProgramGraph, lower
from .plan import ExecutionPlan, parse_plan, serialize_plan, validate_plan
from .timing import (BenchRow, CostParams, algobw, busbw, rows_to_csv, run_benchmark, simulate_timed,
                     transfer_time)
from .world import Topology, World, make_world

SimWorld = World  # the reference's name for the world type (cf/world.py:80)

__all__ = [
    "AlgoDescriptor", "BenchRow", "CommforgeError", "CostParams", "allreduce_add_rmsnorm", "algobw", "busbw",
    "ExecutionPlan", "LoweringParams", "ProgramGraph", "RunResult", "Runtime", "Selector", "SimWorld",
    "Topology", "World", "collective", "lower", "make_world", "parse_plan", "required_multiple",
    "rows_to_csv", "run_benchmark", "select_algorithm", "serialize_plan", "simulate_timed", "transfer_time",
    "validate_plan",
]
