"""Plan runtime: drop-in for ``cf/executor.py`` (``Runtime``, ``RunResult``).

``Runtime(plan, world)`` hands the plan's canonical bytes to libcf's native
loader, which validates it and compiles it to a device op array (K10, see
``csrc/cf_plan.cu``); ``execute(inputs)`` runs every (rank, tb) program on the
GPUs in one launch per device.  The reference interleaves thread blocks with a
simulated scheduler (``cf/executor.py:135-178``); on a GPU the blocks really
run concurrently, so ``mode``/``seed`` are accepted and ignored, ``races`` is
always empty (data races are a compute-sanitizer concern on real hardware)
and ``trace`` lists issue/complete events in per-program order.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .dtypes import CODES, NP_DTYPES, from_torch
from .errors import DeadlockError, RankMismatchError, ShapeError
from .plan import ExecutionPlan, serialize_plan


@dataclass
class RunResult:
    outputs: list
    races: list
    trace: list | None
    steps: int


class Runtime:
    """A plan bound to a world (cf/executor.py:73-93).  Rebinding is allowed."""

    def __init__(self, plan: ExecutionPlan, world, dtype: str | None = None):
        if world.num_ranks != plan.num_ranks:
            raise RankMismatchError(f"plan wants {plan.num_ranks} ranks, world has {world.num_ranks}")
        if not plan.lowered:
            raise ShapeError("cannot execute a pre-lowering document; lower it first")
        self.plan = plan
        self.world = world
        self.dtype = dtype or plan.dtype
        doc = serialize_plan(plan)
        handle = ctypes.c_void_p()
        _lib.check(_lib.lib().cfPlanLoad(world.comm, doc, len(doc),
                                         CODES[dtype] if dtype else -1, ctypes.byref(handle)))
        self._plan = handle
        in_e, out_e = ctypes.c_size_t(), ctypes.c_size_t()
        dt, nprog, nops = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(_lib.lib().cfPlanInfo(handle, ctypes.byref(in_e), ctypes.byref(out_e),
                                         ctypes.byref(dt), ctypes.byref(nprog), ctypes.byref(nops)))
        self.in_elems, self.out_elems = in_e.value, out_e.value
        self.n_programs, self.n_device_ops = nprog.value, nops.value
        self.sched = None

    def execute(self, inputs, mode: str = "round-robin", seed: int | None = None,
                collect_trace: bool = False) -> RunResult:
        import torch
        n = self.plan.num_ranks
        if len(inputs) != n:
            raise ShapeError(f"need {n} input arrays, got {len(inputs)}")
        on_gpu = all(isinstance(a, torch.Tensor) and a.is_cuda for a in inputs)
        npdt = NP_DTYPES[self.dtype]
        if on_gpu:
            if from_torch(inputs[0].dtype) != self.dtype:
                raise ShapeError(f"inputs are {inputs[0].dtype}, plan executes {self.dtype}")
            ins = [a.contiguous().view(-1) for a in inputs]
        else:
            ins = []
            for r, a in enumerate(inputs):
                a = np.ascontiguousarray(np.asarray(a, npdt)).reshape(-1)
                t = torch.from_numpy(a.view(np.int16)).view(torch.bfloat16) if self.dtype == "bf16" \
                    else torch.from_numpy(a)
                ins.append(t.to(self.world.device(r)))
        for r, a in enumerate(ins):
            if a.numel() != self.in_elems:
                raise ShapeError(f"rank {r}: input length {a.numel()} != declared {self.in_elems}")
        outs = [torch.empty(self.out_elems, dtype=ins[0].dtype, device=self.world.device(r))
                for r in range(n)]
        _lib.check(_lib.lib().cfPlanExecute(self._plan, _lib.ptr_array([t.data_ptr() for t in ins]),
                                            _lib.ptr_array([t.data_ptr() for t in outs]),
                                            _lib.ptr_array(self.world.streams())))
        self.world.synchronize()
        code = ctypes.c_int()
        _lib.check(_lib.lib().cfPlanLastDeviceError(self._plan, ctypes.byref(code)))
        if code.value:
            _lib.lib().cfPlanClearDeviceError(self._plan)   # the plan runs again after a reset
            raise DeadlockError(message="plan execution timed out on the device: a wait, packet "
                                        "read or barrier was never satisfied")
        trace = self._static_trace() if collect_trace else None
        if not on_gpu:
            if self.dtype == "bf16":
                outs = [o.cpu().view(torch.int16).numpy().view(np.uint16) for o in outs]
            else:
                outs = [o.cpu().numpy() for o in outs]
        return RunResult(outputs=outs, races=[], trace=trace, steps=0)

    def execute_traced(self, inputs, mode: str = "round-robin", seed: int | None = None) -> RunResult:
        return self.execute(inputs, mode=mode, seed=seed, collect_trace=True)

    def run_raw(self, send, recv) -> None:
        """Enqueue one execution on per-rank CUDA tensors (no checks, no sync)."""
        _lib.check(_lib.lib().cfPlanExecute(self._plan, _lib.ptr_array([t.data_ptr() for t in send]),
                                            _lib.ptr_array([t.data_ptr() for t in recv]),
                                            _lib.ptr_array(self.world.streams())))

    def check_device_error(self):
        """Synchronize and raise DeadlockError if a device wait of this plan timed out."""
        self.world.synchronize()
        code = ctypes.c_int()
        _lib.check(_lib.lib().cfPlanLastDeviceError(self._plan, ctypes.byref(code)))
        if code.value:
            _lib.lib().cfPlanClearDeviceError(self._plan)   # the plan runs again after a reset
            raise DeadlockError(message="plan execution timed out on the device")

    def _static_trace(self):
        ev = []
        for p in sorted(self.plan.programs, key=lambda q: (q.rank, q.tb)):
            for i, op in enumerate(p.ops):
                ev.append(("issue", p.rank, p.tb, i, op.op))
                ev.append(("complete", p.rank, p.tb, i, op.op))
        return ev

    def close(self):
        if getattr(self, "_plan", None) is not None:
            _lib.lib().cfPlanDestroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init(plan: ExecutionPlan, world) -> Runtime:
    return Runtime(plan, world)
