"""Stress driver (test infrastructure for tests/test_gpu_stress.py): runs every
hand-written collective family many times with fresh integer payloads against
the oracle, on whichever libcf build CF_LIB_PATH names (the -DCF_STRESS build,
or a -DCF_DROP_FENCE mutation of it), and prints one JSON summary line:
  {"checks": N, "mismatches": [...], "deadlocks": D, "errors": [...]}

  python tests/stress_worker.py inproc <iters>    8 ranks on cuda:0 (CF_SPLIT_GROUPS
                                                   selects per-rank launches)
  python tests/stress_worker.py mp2 <iters>       2 processes sharing cuda:0
"""

from __future__ import annotations

import json
import os
import socket
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]

from inputs import gen_inputs  # noqa: E402
from oracle import oracle  # noqa: E402

AR = [("1pa", "", "1pa"), ("2pa", "ll", "2pa"), ("2pa", "", "2pa"), ("1pa_hb", "", "1pa"),
      ("switch_2pa", "", "switch_2pa"), ("2pr", "ring", "2pr")]   # "ring": the literal ring kernel
SIZES = (4099, 65536 + 24, 8 * 32768)


FAILFAST = bool(os.environ.get("CF_STRESS_FAILFAST"))   # mutation runs: stop at the first failure


class _Stop(Exception):
    pass


def _summary():
    return {"checks": 0, "mismatches": [], "deadlocks": 0, "errors": []}


def _record(out, name, ok):
    out["checks"] += 1
    if not ok:
        out["mismatches"].append(name if len(out["mismatches"]) < 20 else "...")
        if FAILFAST:
            raise _Stop


def _deadlock(out):
    out["deadlocks"] += 1
    if FAILFAST:
        raise _Stop


def run_inproc(iters: int) -> dict:
    from paper_2504_09014_b200 import make_world
    n = 8
    out = _summary()
    w = make_world(1, n, devices=[0] * n, spin_timeout_ms=3000, use_multicast="emulate")
    w.symmetric_heap(64 << 20)
    try:
        _inproc_loop(w, n, iters, out)
    except _Stop:
        pass
    w.close()
    return out


PLANS = (("1pa_n8_e64", 128 * 16), ("2pa_ll_n8_e64", 128 * 4), ("2pa_memory_n8_e64", 128 * 16))


def _plan_runtimes(w):
    """DSL plans on the compiled K10 kernels (the 1pa plan's streamed packet
    pairs, the LL two-shot plan, the single-op HB plan), i32."""
    from paper_2504_09014_b200 import Runtime, parse_plan
    from paper_2504_09014_b200.plan import scale_plan
    rts = []
    for name, factor in PLANS:
        with open(os.path.join(ROOT, "tests", "golden", "plans", name + ".json"), "rb") as f:
            rts.append((name, Runtime(scale_plan(parse_plan(f.read()), factor), w, dtype="i32")))
    return rts


def _check_plans(rts, n, it, out):
    import torch
    from paper_2504_09014_b200.errors import DeadlockError
    for name, rt in rts:
        ins = gen_inputs(n, rt.in_elems, "i32", "int", 13 * it + rt.in_elems)
        xs = [torch.from_numpy(x).cuda() for x in ins]
        ys = [torch.empty(rt.out_elems, dtype=torch.int32, device="cuda") for _ in range(n)]
        try:
            rt.run_raw(xs, ys)
            rt.check_device_error()
            want = np.sum(np.stack(ins), axis=0, dtype=np.int32)   # i32: exact in any order
            _record(out, f"plan:{name}:{it}", all(np.array_equal(ys[r].cpu().numpy(), want) for r in range(n)))
        except DeadlockError:
            _deadlock(out)


def _inproc_loop(w, n, iters, out):
    rts = _plan_runtimes(w)
    try:
        _inproc_iters(w, n, iters, out, rts)
    finally:
        for _, rt in rts:
            rt.close()


def _inproc_iters(w, n, iters, out, rts):
    import torch
    from paper_2504_09014_b200 import collective
    from paper_2504_09014_b200.errors import DeadlockError
    for it in range(iters):
        _check_plans(rts, n, it, out)
        for elems in SIZES:
            ins = gen_inputs(n, elems, "i32", "int", 1000 * it + elems)
            for name, var, oname in AR:
                try:
                    got = collective("allreduce", ins, w, dtype="i32", algo=name, variant=var)
                    want = oracle.allreduce(ins, oname, "i32")
                    _record(out, f"{name}{var}:{elems}:{it}", all(np.array_equal(g, x) for g, x in zip(got, want)))
                except DeadlockError:
                    _deadlock(out)
                except Exception as e:   # noqa: BLE001
                    out["errors"].append(f"{name}: {type(e).__name__}: {e}"[:200])
            # in-place NVLS on symmetric buffers (K5 direct)
            xs = w.alloc_symmetric(elems, torch.int32)
            ys = w.alloc_symmetric(elems, torch.int32)
            for r in range(n):
                xs[r].copy_(torch.from_numpy(ins[r]))
            try:
                from paper_2504_09014_b200 import _lib
                from paper_2504_09014_b200 import collectives as C
                C.run("allreduce", xs, ys, elems, "i32", _lib.ALGOS["switch_2pa"], w)
                w.check_device_error()
                want = oracle.allreduce(ins, "switch_2pa", "i32")
                _record(out, f"switch_direct:{elems}:{it}",
                        all(np.array_equal(ys[r].cpu().numpy(), want[r]) for r in range(n)))
            except DeadlockError:
                _deadlock(out)
            w.free_symmetric(xs)
            w.free_symmetric(ys)
            sh = gen_inputs(n, elems // n + 1, "i32", "bits", 7 * it + elems)
            for algo in ("allpairs_ag", "ring_ag"):
                try:
                    got = collective("allgather", sh, w, dtype="i32", algo=algo,
                                     variant="ring" if algo == "ring_ag" else "")
                    _record(out, f"{algo}:{elems}:{it}",
                            all(np.array_equal(g, x) for g, x in zip(got, oracle.allgather(sh))))
                except DeadlockError:
                    _deadlock(out)
            rs = gen_inputs(n, 2 * n * (elems // (2 * n) + 1), "i32", "int", 11 * it + elems)
            for algo, oname in (("rs_direct", "2pa"), ("ring_rs", "ring_rs")):
                try:
                    got = collective("reducescatter", rs, w, dtype="i32", algo=algo,
                                     variant="ring" if algo == "ring_rs" else "")
                    want = oracle.reducescatter(rs, oname, "i32")
                    _record(out, f"{algo}:{elems}:{it}", all(np.array_equal(g, x) for g, x in zip(got, want)))
                except DeadlockError:
                    _deadlock(out)
        # K13 two-shot (phase 1 over every CTA, all-CTA barrier): integer-valued
        # f32 rows, so the residual output is exact
        from paper_2504_09014_b200 import allreduce_add_rmsnorm
        rows, hidden = 2 * n + 3, 512
        g = torch.Generator().manual_seed(it)
        xs = [torch.randint(-64, 64, (rows, hidden), generator=g).float().cuda() for _ in range(n)]
        res = [torch.randint(-64, 64, (rows, hidden), generator=g).float().cuda() for _ in range(n)]
        try:
            _, ro = allreduce_add_rmsnorm(w, xs, [x.clone() for x in res], torch.ones(hidden, device="cuda"),
                                          algo="2pa")   # resid_out defaults to the residuals, in place
            w.check_device_error()
            h = sum(x for x in xs)
            _record(out, f"k13:{it}", all(torch.equal(ro[r], h + res[r]) for r in range(n)))
        except DeadlockError:
            _deadlock(out)


def _mp_worker(rank, world, port, iters, q):
    try:
        import torch
        import torch.distributed as dist
        from paper_2504_09014_b200.comm import Communicator
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        comm = Communicator(spin_timeout_ms=3000)
        comm.setup_symmetric(64 << 20, mode="emulate")
        out = _summary()
        try:
            _mp_loop(comm, rank, world, iters, out)
        except _Stop:
            pass
        q.put((rank, out))
        comm.close()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, {"checks": 0, "mismatches": [], "deadlocks": 0, "errors": [f"{type(e).__name__}: {e}"[:300]]}))


def _mp_loop(comm, rank, world, iters, out):
    import torch
    from paper_2504_09014_b200.errors import DeadlockError
    for it in range(iters):
        for elems in SIZES:
            ins = gen_inputs(world, elems, "i32", "int", 1000 * it + elems)
            x = comm.alloc_symmetric(elems, torch.int32)
            y = comm.alloc_symmetric(elems, torch.int32)
            x.copy_(torch.from_numpy(ins[rank]))
            for name, var, oname in AR:
                try:
                    y.zero_()
                    comm.all_reduce(x, y, algo=name, variant=var)
                    comm.check_device_error()
                    _record(out, f"{name}{var}:{elems}:{it}",
                            np.array_equal(y.cpu().numpy(), oracle.allreduce(ins, oname, "i32")[rank]))
                except DeadlockError:
                    _deadlock(out)
            ag = comm.alloc_symmetric(world * elems, torch.int32)
            for algo in ("allpairs_ag", "ring_ag"):
                try:
                    comm.all_gather(x, ag, algo=algo, variant="ring" if algo == "ring_ag" else "")
                    comm.check_device_error()
                    _record(out, f"{algo}:{elems}:{it}", np.array_equal(ag.cpu().numpy(),
                                                                        oracle.allgather(ins)[rank]))
                except DeadlockError:
                    _deadlock(out)
            for t in (x, y, ag):
                comm.free_symmetric(t)


def run_mp2(iters: int) -> dict:
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_worker, args=(r, 2, port, iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900)[1] for _ in procs]
    for p in procs:
        p.join(timeout=60)
    out = _summary()
    for r in res:
        out["checks"] += r["checks"]
        out["mismatches"] += r["mismatches"]
        out["deadlocks"] += r["deadlocks"]
        out["errors"] += r["errors"]
    return out


if __name__ == "__main__":
    mode, iters = sys.argv[1], int(sys.argv[2])
    res = run_inproc(iters) if mode == "inproc" else run_mp2(iters)
    print(json.dumps(res))
