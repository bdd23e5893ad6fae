"""Error taxonomy of the drop-in API.

Same class names and stable ``.code`` strings as the reference
(commforge 0.1.0, ``cf/errors.py:6-93``), so callers that catch
``commforge`` errors by class or by code keep working.  The C ABI returns a
``cfStatus`` per call; ``raise_status`` maps it to these classes.
"""

from __future__ import annotations


class CommforgeError(Exception):
    code = "E_GENERIC"

    def __init__(self, message: str = ""):
        super().__init__(message or self.code)


def _make(name: str, code: str, doc: str = ""):
    cls = type(name, (CommforgeError,), {"code": code, "__doc__": doc or None})
    return cls


BadSizeError = _make("BadSizeError", "E_BAD_SIZE")
NoSemError = _make("NoSemError", "E_NO_SEM")
BadDeltaError = _make("BadDeltaError", "E_BAD_DELTA")
OutOfBoundsError = _make("OutOfBoundsError", "E_OOB")
ProxyDownError = _make("ProxyDownError", "E_PROXY_DOWN")
ZeroFlagError = _make("ZeroFlagError", "E_ZERO_FLAG")
WrongProtocolError = _make("WrongProtocolError", "E_WRONG_PROTOCOL")
BadAlignError = _make("BadAlignError", "E_BAD_ALIGN")
PlanSyntaxError = _make("PlanSyntaxError", "E_SYNTAX")
PlanVersionError = _make("PlanVersionError", "E_VERSION")
PlanRefError = _make("PlanRefError", "E_REF")
ShapeError = _make("ShapeError", "E_SHAPE")
ProtocolError = _make("ProtocolError", "E_PROTOCOL")
RankMismatchError = _make("RankMismatchError", "E_RANK_MISMATCH")
TopologyError = _make("TopologyError", "E_TOPOLOGY")
NoAlgoError = _make("NoAlgoError", "E_NO_ALGO")
BadTimeError = _make("BadTimeError", "E_BAD_TIME")
ConfigError = _make("ConfigError", "E_CONFIG")
CudaError = _make("CudaError", "E_CUDA", "CUDA runtime/driver failure inside libcf (no reference twin).")
InternalError = _make("InternalError", "E_INTERNAL", "libcf invariant violated (no reference twin).")


class DeadlockError(CommforgeError):
    """A device-side wait exceeded the spin timeout (the GPU analogue of the
    reference scheduler's quiescence, cf/sched.py:93-99)."""

    code = "E_DEADLOCK"

    def __init__(self, blocked=None, message: str = ""):
        self.blocked = list(blocked or [])
        names = ", ".join(f"{n} ({r})" for n, r in self.blocked)
        super().__init__(message or f"deadlock: blocked contexts: {names}")


BY_CODE = {cls.code: cls for cls in (
    CommforgeError, BadSizeError, NoSemError, BadDeltaError, OutOfBoundsError, DeadlockError,
    ProxyDownError, ZeroFlagError, WrongProtocolError, BadAlignError, PlanSyntaxError,
    PlanVersionError, PlanRefError, ShapeError, ProtocolError, RankMismatchError, TopologyError,
    NoAlgoError, BadTimeError, ConfigError, CudaError, InternalError)}

# cfStatus numbering of include/cf.h
STATUS_CODES = ["OK", "E_GENERIC", "E_BAD_SIZE", "E_NO_SEM", "E_BAD_DELTA", "E_OOB", "E_DEADLOCK",
                "E_PROXY_DOWN", "E_ZERO_FLAG", "E_WRONG_PROTOCOL", "E_BAD_ALIGN", "E_SYNTAX",
                "E_VERSION", "E_REF", "E_SHAPE", "E_PROTOCOL", "E_RANK_MISMATCH", "E_TOPOLOGY",
                "E_NO_ALGO", "E_BAD_TIME", "E_CONFIG", "E_CUDA", "E_INTERNAL"]


def raise_status(status: int, message: str = "") -> None:
    if status == 0:
        return
    code = STATUS_CODES[status] if 0 <= status < len(STATUS_CODES) else "E_GENERIC"
    cls = BY_CODE.get(code, CommforgeError)
    if cls is DeadlockError:
        raise DeadlockError(message=message or "device wait timed out")
    raise cls(message or code)
