"""ctypes binding of libcf.so (include/cf.h).

The product path has no CPU fallback: if the in-tree extension is missing the
import of any GPU entry point raises, it never silently computes on the host.
"""

from __future__ import annotations

import ctypes
import os

from .errors import raise_status

_HERE = os.path.dirname(os.path.abspath(__file__))
# CF_LIB_PATH: load another in-tree build of libcf (A/B diagnostics)
LIB_PATH = os.environ.get("CF_LIB_PATH") or os.path.join(_HERE, "libcf.so")

CF_MAX_RANKS = 8
CF_MAX_BLOCKS = 1024
CF_HANDLE_BYTES = 256
CF_BUFFER_HANDLE_BYTES = 128

ALGOS = {
    "auto": -1, "1pa": 0, "1pa_hb": 1, "2pa": 2, "2pa_ll": 3, "switch_2pa": 4, "2pr": 5,
    "allpairs_ag": 6, "ring_ag": 7, "ring_rs": 8, "rs_direct": 9,
}
ALGO_NAMES = {v: k for k, v in ALGOS.items()}
CF_ALGO_RING_LINKS = 0x100   # cf.h: OR into 2pr / ring_rs / ring_ag for the literal ring transport
CF_ALGO_COUNT = 10   # cfAlgo count; also the CTA-budget slot of the fused K13 kernel
CF_PLAN_HANDLE_BYTES = 128

# every symbol include/cf.h declares (tests check the .so exports all of them)
EXPORTS = (
    "cfStatusCode", "cfLastErrorMessage", "cfVersion", "cfCommInitAll", "cfCommCreateRank",
    "cfCommGetHandle", "cfCommConnect", "cfCommDestroy", "cfBufferExport", "cfBufferImport",
    "cfBufferRelease", "cfMemoryChannelCreate", "cfPortChannelCreate",
    "cfDeviceMulticastSupported", "cfNvlsCreate", "cfNvlsImport", "cfNvlsBind", "cfNvlsEmulate",
    "cfCommNumRanks",
    "cfCommLocalRanks",
    "cfCommMulticastSupported", "cfCommLastDeviceError", "cfCommClearDeviceError", "cfAllReduce",
    "cfAllGather", "cfReduceScatter", "cfAllReduceHost", "cfAllReduceHostStaged",
    "cfAllReduceAddRMSNorm", "cfSelectAlgorithm", "cfPlanLoad", "cfPlanExecute",
    "cfPlanInfo", "cfPlanLastDeviceError", "cfPlanClearDeviceError", "cfPlanGetHandle", "cfPlanConnect", "cfPlanDestroy",
    "cfDslBuild", "cfDslLower", "cfSymHeapCreate", "cfSymHeapMapPeer", "cfSymHeapMulticast",
    "cfSymHeapInfo", "cfMemAlloc", "cfMemFree", "cfSwitchChannelCreate", "cfCommSetCtaBudget",
    "cfCommSetSelection", "cfCommSetNvlsMinBytes",
)


class cfConfig(ctypes.Structure):
    _fields_ = [("ll_max_bytes", ctypes.c_size_t), ("max_blocks", ctypes.c_int),
                ("threads", ctypes.c_int), ("spin_timeout_ns", ctypes.c_uint64),
                ("use_multicast", ctypes.c_int), ("nvls_bytes", ctypes.c_size_t)]


_lib = None

vp = ctypes.c_void_p
i32 = ctypes.c_int
sz = ctypes.c_size_t
P = ctypes.POINTER

_PROTOS = {
    "cfStatusCode": ([i32], ctypes.c_char_p),
    "cfLastErrorMessage": ([], ctypes.c_char_p),
    "cfVersion": ([], i32),
    "cfCommInitAll": ([P(vp), i32, P(i32), P(cfConfig)], i32),
    "cfCommCreateRank": ([P(vp), i32, i32, i32, P(cfConfig)], i32),
    "cfCommGetHandle": ([vp, vp, P(sz)], i32),
    "cfCommConnect": ([vp, vp, sz], i32),
    "cfCommDestroy": ([vp], i32),
    "cfBufferExport": ([vp, vp, sz, vp], i32),
    "cfBufferImport": ([vp, vp, vp, sz], i32),
    "cfBufferRelease": ([vp, vp], i32),
    "cfDeviceMulticastSupported": ([i32, P(i32)], i32),
    "cfMemoryChannelCreate": ([vp, i32, i32, i32, vp, vp, vp, P(sz)], i32),
    "cfPortChannelCreate": ([vp, i32, i32, i32, vp, vp, vp, P(sz)], i32),
    "cfNvlsCreate": ([vp, P(i32)], i32),
    "cfNvlsImport": ([vp, i32], i32),
    "cfNvlsBind": ([vp], i32),
    "cfNvlsEmulate": ([vp, vp, sz], i32),
    "cfCommNumRanks": ([vp, P(i32)], i32),
    "cfCommLocalRanks": ([vp, P(i32), P(i32)], i32),
    "cfCommMulticastSupported": ([vp, P(i32)], i32),
    "cfCommLastDeviceError": ([vp, P(i32)], i32),
    "cfCommClearDeviceError": ([vp], i32),
    "cfAllReduce": ([vp, P(vp), P(vp), sz, i32, i32, P(vp)], i32),
    "cfAllGather": ([vp, P(vp), P(vp), sz, i32, i32, P(vp)], i32),
    "cfReduceScatter": ([vp, P(vp), P(vp), sz, i32, i32, P(vp)], i32),
    "cfAllReduceHost": ([vp, P(vp), P(vp), sz, i32, i32, P(vp)], i32),
    "cfAllReduceHostStaged": ([vp, P(vp), P(vp), P(vp), P(vp), sz, i32, i32, P(vp)], i32),
    "cfAllReduceAddRMSNorm": ([vp, P(vp), P(vp), P(vp), P(vp), P(vp), sz, sz, ctypes.c_float, i32, i32,
                               P(vp)], i32),
    "cfSelectAlgorithm": ([vp, i32, sz, i32, P(i32)], i32),
    "cfPlanLoad": ([vp, ctypes.c_char_p, sz, i32, P(vp)], i32),
    "cfPlanExecute": ([vp, P(vp), P(vp), P(vp)], i32),
    "cfPlanLastDeviceError": ([vp, P(i32)], i32),
    "cfPlanClearDeviceError": ([vp], i32),
    "cfCommSetCtaBudget": ([vp, i32, i32], i32),
    "cfCommSetSelection": ([vp, i32, i32, i32, P(sz), P(i32)], i32),
    "cfCommSetNvlsMinBytes": ([vp, sz], i32),
    "cfSymHeapCreate": ([vp, sz, i32, P(i32)], i32),
    "cfSymHeapMapPeer": ([vp, i32, i32], i32),
    "cfSymHeapMulticast": ([vp, i32, P(i32)], i32),
    "cfSymHeapInfo": ([vp, i32, P(vp), P(sz), P(i32)], i32),
    "cfMemAlloc": ([vp, sz, P(vp)], i32),
    "cfMemFree": ([vp, vp], i32),
    "cfSwitchChannelCreate": ([vp, i32, vp, P(sz)], i32),
    "cfDslBuild": ([ctypes.c_char_p, ctypes.c_char_p, i32, sz, ctypes.c_char_p, ctypes.c_char_p, vp, sz, P(sz)], i32),
    "cfDslLower": ([ctypes.c_char_p, sz, i32, i32, vp, sz, P(sz)], i32),
    "cfPlanInfo": ([vp, P(sz), P(sz), P(i32), P(i32), P(i32)], i32),
    "cfPlanGetHandle": ([vp, vp, P(sz)], i32),
    "cfPlanConnect": ([vp, vp, sz], i32),
    "cfPlanDestroy": ([vp], i32),
}


def lib():
    """Load libcf.so once (raises if the extension was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libcf.so not built at {LIB_PATH}: run __graft_entry__.build() "
                              "(the product has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _PROTOS.items():
            if not hasattr(L, name):
                continue   # tests/test_abi.py asserts every declared symbol is exported
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise_status(status, lib().cfLastErrorMessage().decode(errors="replace"))


def ptr_array(values):
    arr = (vp * len(values))(*[int(v) if v is not None else None for v in values])
    return arr


class _DevMem:
    """__cuda_array_interface__ view of raw device bytes (no ownership)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def tensor_at(ptr: int, numel: int, dtype, device):
    """A torch tensor over libcf-owned device memory (e.g. a cfMemAlloc
    buffer).  The memory stays libcf's: free it through libcf, not torch."""
    import torch
    es = torch.empty(0, dtype=dtype).element_size()
    raw = torch.as_tensor(_DevMem(ptr, numel * es), device=device)
    return raw.view(dtype)
