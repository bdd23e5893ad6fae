"""One process per GPU: the multi-process communicator.

The reference runs every rank in one process (``make_world``); a real
8xB200 job runs one process per GPU.  Bootstrap is pluggable: any
``torch.distributed`` process group (gloo or nccl; NCCL is never used for
data) all-gathers the opaque handles libcf exports (``cfCommGetHandle`` for
the symmetric heap, ``cfBufferExport`` for registered tensors).  After that
every collective is a single libcf kernel over NVLink peer memory.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .collectives import _algo_id
from .dtypes import CODES, from_torch
from .errors import BadSizeError, ShapeError


def all_gather_bytes(blob: bytes, group=None) -> list:
    """All-gather one fixed-size byte string per rank (rank order)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(dev)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    return [bytes(o.cpu().numpy().tobytes()) for o in out]


def share_fd(fd, rank: int, nranks: int, group=None, src: int = 0) -> int:
    """Collective: rank `src` passes its file descriptor `fd` to every other
    rank of the group (same host) over a Unix-domain socket with SCM_RIGHTS;
    the socket path travels through the bootstrap group.  Returns the fd valid
    in this process (`src`: its own; others: a new descriptor to close)."""
    import os
    import socket
    import tempfile
    import torch.distributed as dist
    path, srv = None, None
    if rank == src:
        path = os.path.join(tempfile.mkdtemp(prefix="cf_fd_"), "sock")
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(path)
        srv.listen(max(1, nranks))
    box = [path]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, src) if group is not None else src,
                              group=group)
    if rank == src:
        for _ in range(nranks - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"f"], [fd])
            conn.close()
        srv.close()
        dist.barrier(group=group)
        os.unlink(path)
        os.rmdir(os.path.dirname(path))
        return fd
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    cli.connect(box[0])
    _, fds, _, _ = socket.recv_fds(cli, 1, 1)
    cli.close()
    dist.barrier(group=group)
    return fds[0]


class Communicator:
    """This process's rank of an ``nranks``-GPU communicator."""

    def __init__(self, group=None, device=None, ll_max_bytes: int = 0, max_blocks: int = 0,
                 threads: int = 0, spin_timeout_ms: int = 0):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        cfg = _lib.cfConfig(ll_max_bytes, max_blocks, threads, int(spin_timeout_ms) * 1_000_000, 0)
        h = ctypes.c_void_p()
        L = _lib.lib()
        _lib.check(L.cfCommCreateRank(ctypes.byref(h), self.nranks, self.rank, self.device.index,
                                      ctypes.byref(cfg)))
        self._comm = h
        blob = ctypes.create_string_buffer(_lib.CF_HANDLE_BYTES)
        nbytes = ctypes.c_size_t(_lib.CF_HANDLE_BYTES)
        _lib.check(L.cfCommGetHandle(h, blob, ctypes.byref(nbytes)))
        handles = all_gather_bytes(blob.raw, group)
        allh = b"".join(handles)
        _lib.check(L.cfCommConnect(h, allh, _lib.CF_HANDLE_BYTES))
        self._registered = {}
        self._ll_max = int(ll_max_bytes) or (4 << 20)   # libcf's default LL capacity

    @property
    def comm(self):
        return self._comm

    def register(self, tensor) -> None:
        """Collective: every rank registers its corresponding tensor."""
        L = _lib.lib()
        blob = ctypes.create_string_buffer(_lib.CF_BUFFER_HANDLE_BYTES)
        nbytes = tensor.numel() * tensor.element_size()
        _lib.check(L.cfBufferExport(self._comm, tensor.data_ptr(), nbytes, blob))
        allh = b"".join(all_gather_bytes(blob.raw, self.group))
        _lib.check(L.cfBufferImport(self._comm, tensor.data_ptr(), allh, _lib.CF_BUFFER_HANDLE_BYTES))
        self._registered[tensor.data_ptr()] = tensor

    def deregister(self, tensor) -> None:
        _lib.check(_lib.lib().cfBufferRelease(self._comm, tensor.data_ptr()))
        self._registered.pop(tensor.data_ptr(), None)

    def _call(self, fn, send, recv, count, algo, stream):
        import torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        st = _lib.ptr_array([s.cuda_stream])
        _lib.check(fn(self._comm, _lib.ptr_array([send.data_ptr()]), _lib.ptr_array([recv.data_ptr()]),
                      int(count), CODES[from_torch(send.dtype)], int(algo), st))

    def all_reduce(self, send, recv=None, algo: str = "auto", variant: str = "", stream=None):
        import torch
        recv = torch.empty_like(send) if recv is None else recv
        aid = -1 if algo == "auto" else _algo_id("allreduce", algo, variant)
        self._call(_lib.lib().cfAllReduce, send, recv, send.numel(), aid, stream)
        return recv

    def all_gather(self, send, recv=None, algo: str = "auto", stream=None, variant: str = ""):
        recv = send.new_empty(send.numel() * self.nranks) if recv is None else recv
        aid = -1 if algo == "auto" else _algo_id("allgather", algo, variant)
        self._call(_lib.lib().cfAllGather, send, recv, send.numel(), aid, stream)
        return recv

    def reduce_scatter(self, send, recv=None, algo: str = "auto", stream=None, variant: str = ""):
        if send.numel() % self.nranks:
            raise ShapeError("reduce_scatter input must hold nranks equal shards")
        recv = send.new_empty(send.numel() // self.nranks) if recv is None else recv
        aid = -1 if algo == "auto" else _algo_id("reducescatter", algo, variant)
        self._call(_lib.lib().cfReduceScatter, send, recv, recv.numel(), aid, stream)
        return recv

    def all_reduce_host(self, host_send, host_recv=None, algo: str = "auto", variant: str = "", stream=None,
                        sync: bool = True):
        """AllReduce of a HOST tensor (pinned for overlap): the pipelined
        host path (``cfAllReduceHostStaged``) -- windowed H2D copy, K3 and D2H
        copy overlap.  Collective: every rank calls it with the same size.
        Device staging buffers are allocated and registered on first use per
        (size, dtype) and reused.  With ``sync`` (default) the call returns
        once ``host_recv`` holds the result; otherwise it is stream-ordered."""
        import torch
        src = host_send.contiguous().view(-1)
        host_recv = torch.empty(src.shape, dtype=src.dtype, pin_memory=src.is_pinned()) \
            if host_recv is None else host_recv
        key = (src.numel(), src.dtype)
        stage = self.__dict__.setdefault("_stage", {})
        if key not in stage:
            for old in list(stage.values()):   # one staging pair at a time
                for t in old:
                    self.deregister(t)
            stage.clear()
            pair = (torch.empty(src.numel(), dtype=src.dtype, device=self.device),
                    torch.empty(src.numel(), dtype=src.dtype, device=self.device))
            for t in pair:
                self.register(t)
            stage[key] = pair
        ds, dr = stage[key]
        aid = -1 if algo == "auto" else _algo_id("allreduce", algo, variant)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        P = _lib.ptr_array
        _lib.check(_lib.lib().cfAllReduceHostStaged(
            self._comm, P([src.data_ptr()]), P([host_recv.data_ptr()]), P([ds.data_ptr()]), P([dr.data_ptr()]),
            src.numel(), CODES[from_torch(src.dtype)], aid, P([s.cuda_stream])))
        if sync:
            s.synchronize()
        return host_recv

    def all_reduce_add_rmsnorm(self, send, residual, weight, eps: float = 1e-6, algo: str = "auto",
                               resid_out=None, norm_out=None, stream=None):
        """K13 on this rank (see ``fused.allreduce_add_rmsnorm``): returns
        ``(norm_out, resid_out)``; ``resid_out`` defaults to ``residual``
        (updated in place).  The two-shot algorithm writes both outputs from
        the peers, so register them (``register``) before the first call."""
        import torch
        if send.dim() != 2:
            raise ShapeError("all_reduce_add_rmsnorm takes [rows, hidden] tensors")
        resid_out = residual if resid_out is None else resid_out
        norm_out = torch.empty_like(send) if norm_out is None else norm_out
        aid = {"auto": -1, "1pa_hb": _lib.ALGOS["1pa_hb"], "2pa": _lib.ALGOS["2pa"]}.get(algo)
        if aid is None:
            raise ShapeError(f"fused allreduce+rmsnorm runs as 1pa_hb or 2pa, not {algo!r}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        P = _lib.ptr_array
        _lib.check(_lib.lib().cfAllReduceAddRMSNorm(
            self._comm, P([send.data_ptr()]), P([residual.data_ptr()]), P([resid_out.data_ptr()]),
            P([norm_out.data_ptr()]), P([weight.data_ptr()]), send.shape[0], send.shape[1], float(eps),
            CODES[from_torch(send.dtype)], aid, P([s.cuda_stream])))
        return norm_out, resid_out

    def load_plan(self, plan, dtype: str | None = None) -> "RankRuntime":
        """Collective: load an execution plan on this rank (K10, one process per
        GPU) -- every rank loads the same plan, the plan heaps are exchanged
        through the bootstrap.  See ``RankRuntime``."""
        return RankRuntime(self, plan, dtype)

    def setup_nvls(self) -> bool:
        """Collective: build the NVLS multicast object (SwitchChannel).  Rank 0
        creates it and passes its POSIX fd to the other ranks over a Unix
        socket (SCM_RIGHTS, ``share_fd``); every rank then binds and maps its
        memory.  All ranks must share one host.  Returns False on every rank
        when any GPU lacks multicast support or any step fails on any rank
        (every step's outcome is agreed on before the next, so a failure
        never leaves a rank waiting in a collective)."""
        import os
        import torch.distributed as dist
        L = _lib.lib()

        def agree(ok: bool) -> bool:
            flags = [None] * self.nranks
            dist.all_gather_object(flags, bool(ok), group=self.group)
            return all(flags)

        if not agree(self._multicast_capable()):
            return False
        fd = ctypes.c_int(-1)
        if self.rank == 0:
            created = L.cfNvlsCreate(self._comm, ctypes.byref(fd)) == 0
        else:
            created = True
        if not agree(created):
            return False
        got = share_fd(fd.value if self.rank == 0 else None, self.rank, self.nranks, self.group)
        imported = True
        if self.rank != 0:
            imported = L.cfNvlsImport(self._comm, got) == 0
            os.close(got)
        ok = agree(imported)          # every device added before any bind
        if ok:
            ok = agree(L.cfNvlsBind(self._comm) == 0)
        if self.rank == 0:
            os.close(fd.value)
        return ok

    def setup_nvls_emulated(self, staging_bytes: int = 64 << 20) -> None:
        """Collective: the emulated switch (no multicast object): every rank
        registers a staging buffer (input + output halves) and switch_2pa runs
        the NVLS kernel with per-rank loads / stores over the mapped peers'
        staging in place of multimem.  Tests the one-process-per-GPU NVLS
        control path on boxes without multicast."""
        import torch
        staging = torch.zeros(staging_bytes, dtype=torch.uint8, device=self.device)
        self.register(staging)
        _lib.check(_lib.lib().cfNvlsEmulate(self._comm, staging.data_ptr(), staging_bytes))
        self._nvls_staging = staging

    def set_cta_budget(self, ctas: int, algo: str | None = None) -> None:
        """CTAs per rank for `algo` (None: every algorithm; "fused": K13; 0:
        the default, 64 one rank per GPU) -- include/cf.h cfCommSetCtaBudget."""
        aid = -1 if algo is None else (_lib.CF_ALGO_COUNT if algo == "fused" else _lib.ALGOS[algo])
        _lib.check(_lib.lib().cfCommSetCtaBudget(self._comm, aid, int(ctas)))

    def setup_symmetric(self, nbytes: int, mode: str = "auto") -> int:
        """Collective: this rank's symmetric heap (include/cf.h cfSymHeapCreate),
        its POSIX fd sent to every peer (SCM_RIGHTS over Unix sockets) and the
        peers' heaps mapped here; with multicast, the heaps are bound to one
        NVLS object (rank 0 creates it).  mode: "auto" (multicast when every
        GPU supports it and the object builds, else plain), "emulate" (the
        switch as unicast loads / stores: boxes without multicast), "none".
        Returns the mode in use (1 multicast, 2 emulated, 0 plain); every
        rank agrees on it."""
        import os
        import torch.distributed as dist
        L = _lib.lib()

        def agree(ok: bool) -> bool:
            flags = [None] * self.nranks
            dist.all_gather_object(flags, bool(ok), group=self.group)
            return all(flags)

        want = {"emulate": 2, "none": 0}.get(mode, 1)
        if want == 1 and not agree(self._multicast_capable()):
            want = 0
        fd = ctypes.c_int(-1)
        _lib.check(L.cfSymHeapCreate(self._comm, int(nbytes), want, ctypes.byref(fd)))
        for src in range(self.nranks):
            got = share_fd(fd.value if src == self.rank else None, self.rank, self.nranks, self.group, src=src)
            if src != self.rank:
                _lib.check(L.cfSymHeapMapPeer(self._comm, src, got))
                os.close(got)
        os.close(fd.value)
        self._sym_mode = want
        if want == 1:
            mfd = ctypes.c_int(-1)
            ok = agree(L.cfSymHeapMulticast(self._comm, 0, ctypes.byref(mfd)) == 0) if self.rank == 0 else \
                agree(True)
            if ok:
                got = share_fd(mfd.value if self.rank == 0 else None, self.rank, self.nranks, self.group)
                if self.rank != 0:
                    g = ctypes.c_int(got)
                    ok = L.cfSymHeapMulticast(self._comm, 1, ctypes.byref(g)) == 0
                    os.close(got)
                ok = agree(ok)          # every device added before any bind
            if ok:
                ok = agree(L.cfSymHeapMulticast(self._comm, 2, ctypes.byref(mfd)) == 0)
            if self.rank == 0 and mfd.value >= 0:
                os.close(mfd.value)
            if not ok:
                # heap stays usable (HB algorithms); libcf stops using the
                # switch on every rank, so AUTO picks the same kernel everywhere
                _lib.check(L.cfSymHeapMulticast(self._comm, 3, ctypes.byref(mfd)))
                self._sym_mode = 0
        return self._sym_mode

    def tune(self, kind: str = "allreduce", dtype: str = "bf16", sizes=None, algos=None, iters: int = 10,
             install: bool = True, nvls: bool = True, budgets=(32, 64)) -> dict:
        """Collective: time every candidate algorithm at each size on this
        rank's GPU (CUDA graphs, every replay preceded by a bootstrap barrier),
        take the max over ranks, and install the same fastest-per-size table on
        every rank (cfCommSetSelection; see tune.py).  On a multicast heap the
        smallest size from which in-place NVLS wins is measured and installed
        too (cfCommSetNvlsMinBytes).  For AllReduce the two-shot kernel's CTA
        budget is measured at the largest size over ``budgets`` and the
        fastest installed (cfCommSetCtaBudget; budgets above half the SMs give
        up the guarantee that a collective stays resident next to a compute
        kernel holding the other half -- the default candidates stay below).  Buffers come from the
        symmetric heap when there is one, else they are registered for the
        call.  Returns {"table", "sizes", "times", "nvls_min_bytes",
        "cta_budget_2pa"}."""
        import torch
        import torch.distributed as dist
        from . import tune as T
        from .dtypes import ELEM_SIZE, torch_dtype
        L = _lib.lib()
        sizes = sorted(sizes or T.DEFAULT_SIZES)
        n, es, tdt = self.nranks, ELEM_SIZE[dtype], torch_dtype(dtype)
        ll_max = self._ll_max
        sym = getattr(self, "_sym_mode", -1)
        per_in = max(sizes) // es if kind == "allreduce" else max(1, max(sizes) // es // n)
        per_out = per_in if kind == "allreduce" else per_in * n
        if sym >= 0:
            x, y = self.alloc_symmetric(per_in, tdt), self.alloc_symmetric(per_out, tdt)
        else:
            x = torch.empty(per_in, device=self.device, dtype=tdt)
            y = torch.empty(per_out, device=self.device, dtype=tdt)
            self.register(x)
            self.register(y)
        x.copy_(torch.randn(per_in, device=self.device).to(tdt))
        fn = {"allreduce": L.cfAllReduce, "allgather": L.cfAllGather}[kind]
        barrier = lambda: dist.barrier(group=self.group)   # noqa: E731
        # AUTO never picks 1pa_hb one process per GPU (cfAllReduce: the
        # in-place test is not rank-uniform there), so it is not a candidate
        names = [a for a in (algos or T.CANDIDATES[kind]) if a != "1pa_hb"]
        if nvls and kind == "allreduce" and sym == 1:
            names.append("switch_2pa")
        local = torch.full((len(names), len(sizes)), -1.0, dtype=torch.float64)
        for i, nb in enumerate(sizes):
            cnt = max(1, nb // es) if kind == "allreduce" else max(1, nb // es // n)
            oc = cnt if kind == "allreduce" else cnt * n
            for k, a in enumerate(names):
                if a not in T.candidates(kind, ll_max, nb, [a]):
                    continue
                aid = T.algo_id(a)
                xi, yi = x[:cnt], y[:oc]
                try:   # validation errors are raised before any launch, identically on every rank
                    local[k, i] = T.time_graph(self.device, lambda: self._call(fn, xi, yi, cnt, aid, None), iters,
                                               before=barrier)
                except BadSizeError:   # beyond this algorithm's capacity (e.g. the LL scratch)
                    pass
        # CTA budget of the two-shot kernel at the largest size (NVLink saturates
        # well below 148 SMs; the default is 64 per rank)
        bt = torch.full((len(budgets),), -1.0, dtype=torch.float64)
        if kind == "allreduce" and budgets:
            cnt = max(sizes) // es
            aid = _lib.ALGOS["2pa"]
            for k, b in enumerate(budgets):
                self.set_cta_budget(int(b), "2pa")
                bt[k] = T.time_graph(self.device, lambda: self._call(fn, x[:cnt], y[:cnt], cnt, aid, None), iters,
                                     before=barrier)
            self.set_cta_budget(0, "2pa")
        self.check_device_error()
        dist.all_reduce(bt, op=dist.ReduceOp.MAX, group=self.group)
        dist.all_reduce(local, op=dist.ReduceOp.MAX, group=self.group)   # slowest rank, same on all ranks
        times = {a: [None if v < 0 else float(v) for v in local[k].tolist()] for k, a in enumerate(names)}
        nv = times.pop("switch_2pa", None)
        table = T.selection_from_times(sizes, times)
        nvls_min = None
        if nv is not None:
            best = [min((t[i] for t in times.values() if t[i] is not None), default=None) for i in range(len(sizes))]
            nvls_min = T.nvls_min_from_times(sizes, nv, best)
        best_budget = None
        if kind == "allreduce" and budgets:
            best_budget = int(budgets[int(torch.argmin(bt).item())])
        if install:
            T.install(self._comm, kind, dtype, table)
            if best_budget is not None:
                self.set_cta_budget(best_budget, "2pa")
            if nv is not None:
                _lib.check(L.cfCommSetNvlsMinBytes(self._comm, ctypes.c_size_t(nvls_min if nvls_min else
                                                                              (1 << 64) - 1)))
        if sym >= 0:
            self.free_symmetric(x)
            self.free_symmetric(y)
        else:
            self.deregister(x)
            self.deregister(y)
        if nv is not None:
            times["switch_2pa"] = nv
        return {"table": table, "sizes": sizes, "times": times, "nvls_min_bytes": nvls_min,
                "cta_budget_2pa": best_budget,
                "cta_budget_times_us": {int(b): round(float(t) * 1e6, 2) for b, t in zip(budgets, bt.tolist())}}

    def disable_switch(self) -> None:
        """Collective: stop using the NVLS switch on this heap (every rank calls
        it, e.g. after a failed first multimem execution); the heap stays
        usable for the other algorithms."""
        mfd = ctypes.c_int(-1)
        _lib.check(_lib.lib().cfSymHeapMulticast(self._comm, 3, ctypes.byref(mfd)))
        self._sym_mode = 0

    def alloc_symmetric(self, numel: int, dtype):
        """Collective: a tensor at the same offset of every rank's symmetric
        heap (cfMemAlloc) -- collectives on it need no registration, and
        switch_2pa runs in place on it."""
        import torch
        es = torch.empty(0, dtype=dtype).element_size()
        ptr = (ctypes.c_void_p * 1)()
        _lib.check(_lib.lib().cfMemAlloc(self._comm, int(numel) * es, ptr))
        return _lib.tensor_at(ptr[0], numel, dtype, self.device)

    def free_symmetric(self, tensor) -> None:
        _lib.check(_lib.lib().cfMemFree(self._comm, tensor.data_ptr()))

    def _multicast_capable(self) -> bool:
        from .world import device_multicast_capable
        return device_multicast_capable(self.device.index)

    def check_device_error(self):
        import torch
        torch.cuda.current_stream(self.device).synchronize()
        code = ctypes.c_int()
        _lib.check(_lib.lib().cfCommLastDeviceError(self._comm, ctypes.byref(code)))
        if code.value:
            from .errors import raise_status
            raise_status(code.value, "device-side wait timed out")

    def clear_device_error(self):
        """Reset this rank's device error word after a reported timeout
        (cfCommClearDeviceError); epochs and semaphores only grow, so later
        calls start clean once every rank cleared it."""
        _lib.check(_lib.lib().cfCommClearDeviceError(self._comm))

    def close(self):
        if self._comm is not None:
            _lib.lib().cfCommDestroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RankRuntime:
    """This rank's share of a plan in the one-process-per-GPU mode (the
    multi-process counterpart of ``executor.Runtime``, ``cf/executor.py:73-178``).
    ``run(send, recv)`` enqueues one execution of this rank's programs on the
    stream; every rank must call it in the same order.  Plans that read or
    write the peers' input / output need those tensors registered
    (``Communicator.register``) before the first run."""

    def __init__(self, comm: Communicator, plan, dtype: str | None = None):
        from .plan import ExecutionPlan, serialize_plan
        self.comm = comm
        doc = serialize_plan(plan) if isinstance(plan, ExecutionPlan) else \
            (plan.encode() if isinstance(plan, str) else bytes(plan))
        L = _lib.lib()
        h = ctypes.c_void_p()
        _lib.check(L.cfPlanLoad(comm.comm, doc, len(doc), CODES[dtype] if dtype else -1, ctypes.byref(h)))
        self._plan = h
        blob = ctypes.create_string_buffer(_lib.CF_PLAN_HANDLE_BYTES)
        nbytes = ctypes.c_size_t(_lib.CF_PLAN_HANDLE_BYTES)
        _lib.check(L.cfPlanGetHandle(h, blob, ctypes.byref(nbytes)))
        allh = b"".join(all_gather_bytes(blob.raw, comm.group))
        _lib.check(L.cfPlanConnect(h, allh, _lib.CF_PLAN_HANDLE_BYTES))
        in_e, out_e = ctypes.c_size_t(), ctypes.c_size_t()
        dt, nprog, nops = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(L.cfPlanInfo(h, ctypes.byref(in_e), ctypes.byref(out_e), ctypes.byref(dt),
                                ctypes.byref(nprog), ctypes.byref(nops)))
        self.in_elems, self.out_elems = in_e.value, out_e.value
        self.n_device_ops = nops.value

    def run(self, send, recv, stream=None):
        import torch
        if send.numel() != self.in_elems or recv.numel() != self.out_elems:
            raise ShapeError(f"plan wants {self.in_elems} input / {self.out_elems} output elements")
        s = stream if stream is not None else torch.cuda.current_stream(self.comm.device)
        P = _lib.ptr_array
        _lib.check(_lib.lib().cfPlanExecute(self._plan, P([send.data_ptr()]), P([recv.data_ptr()]),
                                            P([s.cuda_stream])))
        return recv

    def check_device_error(self):
        import torch
        from .errors import DeadlockError
        torch.cuda.current_stream(self.comm.device).synchronize()
        code = ctypes.c_int()
        _lib.check(_lib.lib().cfPlanLastDeviceError(self._plan, ctypes.byref(code)))
        if code.value:
            _lib.lib().cfPlanClearDeviceError(self._plan)   # the plan runs again after a reset
            raise DeadlockError(message="plan execution timed out on the device")

    def close(self):
        if getattr(self, "_plan", None) is not None:
            _lib.lib().cfPlanDestroy(self._plan)
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
