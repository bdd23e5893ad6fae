"""B200-native collective hot path of MSCCL++ (arXiv 2504.09014).

Drop-in for the reference package's API (commforge 0.1.0, ``cf/__init__.py:12-17``):
the collective facade, the selector and the world bootstrap run on
hand-written sm_100a kernels in ``libcf.so`` (C ABI: ``include/cf.h``).
"""

__version__ = "0.1.0"

from .collectives import AlgoDescriptor, Selector, collective, required_multiple, select_algorithm
from .errors import CommforgeError
from .executor import RunResult, Runtime
from .fused import allreduce_add_rmsnorm
from .lowering import LoweringParams, ProgramGraph, lower
from .plan import ExecutionPlan, parse_plan, serialize_plan, validate_plan
from .timing import BenchRow, CostParams, algobw, busbw, rows_to_csv, run_benchmark
from .world import Topology, World, make_world

SimWorld = World  # the reference's name for the world type (cf/world.py:80)

__all__ = [
    "AlgoDescriptor", "BenchRow", "CommforgeError", "CostParams", "allreduce_add_rmsnorm", "algobw", "busbw",
    "ExecutionPlan", "LoweringParams", "ProgramGraph", "RunResult", "Runtime", "Selector", "SimWorld",
    "Topology", "World", "collective", "lower", "make_world", "parse_plan", "required_multiple",
    "rows_to_csv", "run_benchmark", "select_algorithm", "serialize_plan", "validate_plan",
]
