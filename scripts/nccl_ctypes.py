"""NCCL through ctypes -- the COMPARISON BASELINE of bench.py, never part of
the product path (paper_2504_09014_b200/ does not import it).

BASELINE.md / SURVEY.md §8(d): NCCL 2.28 runs the same sizes in CUDA-graph
mode in two buffer modes and the better one is the bar:
  1. default buffers (caller's cudaMalloc / torch tensors);
  2. symmetric windows: ncclMemAlloc + ncclCommWindowRegister(...,
     NCCL_WIN_COLL_SYMMETRIC) (nccl.h:58-61, 141, 273), which enables NCCL's
     low-latency symmetric kernels.
The library is the torch-bundled libnccl.so.2 (2.28.x, the one torch itself
loads), falling back to the system one.
"""

from __future__ import annotations

import ctypes
import os

NCCL_WIN_COLL_SYMMETRIC = 0x01
DTYPES = {"i32": 2, "f16": 6, "f32": 7, "bf16": 9}
SUM = 0


def _load():
    cands = []
    try:
        import nvidia.nccl
        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
        cands.append(os.path.join(base, "lib", "libnccl.so.2"))
    except Exception:
        pass
    cands.append("libnccl.so.2")
    err = None
    for c in cands:
        try:
            return ctypes.CDLL(c)
        except OSError as e:
            err = e
    raise OSError(f"libnccl.so.2 not found: {err}")


class NcclError(RuntimeError):
    pass


class UniqueId(ctypes.Structure):
    """ncclUniqueId (nccl.h:38-39): a 128-byte struct passed BY VALUE."""
    _fields_ = [("internal", ctypes.c_char * 128)]


class Nccl:
    """One NCCL communicator (one rank per process)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = _load()
            vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
            L.ncclGetUniqueId.argtypes = [ctypes.c_char_p]
            L.ncclCommInitRank.argtypes = [ctypes.POINTER(vp), i32, UniqueId, i32]
            L.ncclCommDestroy.argtypes = [vp]
            L.ncclMemAlloc.argtypes = [ctypes.POINTER(vp), sz]
            L.ncclMemFree.argtypes = [vp]
            L.ncclCommWindowRegister.argtypes = [vp, vp, sz, ctypes.POINTER(vp), i32]
            L.ncclCommWindowDeregister.argtypes = [vp, vp]
            L.ncclAllReduce.argtypes = [vp, vp, sz, i32, i32, vp, vp]
            L.ncclAllGather.argtypes = [vp, vp, sz, i32, vp, vp]
            L.ncclReduceScatter.argtypes = [vp, vp, sz, i32, i32, vp, vp]
            L.ncclGetVersion.argtypes = [ctypes.POINTER(i32)]
            L.ncclGetErrorString.restype = ctypes.c_char_p
            cls._lib = L
        return cls._lib

    @classmethod
    def version(cls) -> int:
        v = ctypes.c_int()
        cls._check(cls.lib().ncclGetVersion(ctypes.byref(v)))
        return v.value

    @classmethod
    def _check(cls, r):
        if r != 0:
            raise NcclError(f"NCCL error {r}: {cls.lib().ncclGetErrorString(r).decode()}")

    @classmethod
    def unique_id(cls) -> bytes:
        buf = ctypes.create_string_buffer(128)
        cls._check(cls.lib().ncclGetUniqueId(buf))
        return buf.raw

    def __init__(self, nranks: int, rank: int, uid: bytes):
        self.comm = ctypes.c_void_p()
        u = UniqueId.from_buffer_copy(uid)
        self._check(self.lib().ncclCommInitRank(ctypes.byref(self.comm), nranks, u, rank))
        self.nranks, self.rank = nranks, rank
        self._wins = []
        self._mem = []

    def mem_alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        self._check(self.lib().ncclMemAlloc(ctypes.byref(p), nbytes))
        self._mem.append(p.value)
        return p.value

    def register_symmetric(self, ptr: int, nbytes: int):
        """Collective: every rank registers its buffer of the same size."""
        w = ctypes.c_void_p()
        self._check(self.lib().ncclCommWindowRegister(self.comm, ptr, nbytes, ctypes.byref(w),
                                                      NCCL_WIN_COLL_SYMMETRIC))
        self._wins.append(w.value)
        return w.value

    def all_reduce(self, send: int, recv: int, count: int, dtype: str, stream: int):
        self._check(self.lib().ncclAllReduce(send, recv, count, DTYPES[dtype], SUM, self.comm, stream))

    def all_gather(self, send: int, recv: int, sendcount: int, dtype: str, stream: int):
        self._check(self.lib().ncclAllGather(send, recv, sendcount, DTYPES[dtype], self.comm, stream))

    def reduce_scatter(self, send: int, recv: int, recvcount: int, dtype: str, stream: int):
        self._check(self.lib().ncclReduceScatter(send, recv, recvcount, DTYPES[dtype], SUM, self.comm, stream))

    def close(self):
        L = self.lib()
        for w in self._wins:
            L.ncclCommWindowDeregister(self.comm, w)
        self._wins = []
        for p in self._mem:
            L.ncclMemFree(p)
        self._mem = []
        if self.comm:
            L.ncclCommDestroy(self.comm)
            self.comm = ctypes.c_void_p()
