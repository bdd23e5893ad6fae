"""One process per rank (the real-deployment mode), two ranks sharing cuda:0:
gloo bootstrap, IPC-mapped symmetric heaps, registered torch buffers, every
collective kernel vs the oracle.  (On an 8-GPU box the same code runs one
rank per GPU over NVLink.)"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu



def _nv(algo):
    """(name, variant): "2pa_ll" = two-shot LL; "<ring algo>+ring" = the literal ring transport."""
    if algo == "2pa_ll":
        return "2pa", "ll"
    name, _, links = algo.partition("+")
    return name, links

def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path[:0] = [root, os.path.join(root, "tests", "golden")]
        import torch
        import torch.distributed as dist
        from inputs import gen_inputs
        from paper_2504_09014_b200.comm import Communicator
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        comm = Communicator(spin_timeout_ms=60000)
        out = {}
        for elems in (1000, 65536 + 8):
            ins = gen_inputs(world, elems, "f32", "wide", 77 + elems)
            send = torch.from_numpy(ins[rank]).cuda()
            recv = torch.empty_like(send)
            comm.register(send)
            comm.register(recv)
            for algo in ("1pa", "2pa", "2pa_ll", "1pa_hb", "2pr", "2pr+ring"):
                name, var = _nv(algo)
                comm.all_reduce(send, recv, algo=name, variant=var)
                torch.cuda.synchronize()
                out[("ar", algo, elems)] = recv.cpu().numpy().copy()
            ag = torch.empty(world * elems, device="cuda", dtype=torch.float32)
            comm.register(ag)
            for algo in ("allpairs_ag", "ring_ag", "ring_ag+ring"):
                ag.zero_()
                comm.all_gather(send, ag, algo=_nv(algo)[0], variant=_nv(algo)[1])
                torch.cuda.synchronize()
                out[("ag", algo, elems)] = ag.cpu().numpy().copy()
            rs_in = torch.from_numpy(np.concatenate([ins[rank]] * world)).cuda()
            rs_out = torch.empty(elems, device="cuda", dtype=torch.float32)
            comm.register(rs_in)
            for algo in ("rs_direct", "ring_rs", "ring_rs+ring"):
                comm.reduce_scatter(rs_in, rs_out, algo=_nv(algo)[0], variant=_nv(algo)[1])
                torch.cuda.synchronize()
                out[("rs", algo, elems)] = rs_out.cpu().numpy().copy()
            for t in (send, recv, ag, rs_in):
                comm.deregister(t)
        # measured selection: tuned on both GPUs' worth of ranks, same table on every rank
        tuned = comm.tune(sizes=[4096, 65536, 1 << 20], iters=3)
        out[("tune",)] = tuned["table"]
        tin = torch.from_numpy(gen_inputs(world, 1 << 18, "f32", "int", 3)[rank]).cuda()
        comm.register(tin)
        tout = torch.empty_like(tin)
        comm.register(tout)
        comm.all_reduce(tin, tout, algo="auto")
        torch.cuda.synchronize()
        out[("tune_auto",)] = tout.cpu().numpy().copy()
        # a table that would pick 1pa_hb, rank 0 in place and rank 1 out of
        # place: AUTO must still launch one kernel on both ranks
        from paper_2504_09014_b200 import tune as T
        T.install(comm._comm, "allreduce", "f32", [(1 << 30, "1pa_hb")])
        mx = tin[:4096].clone()
        comm.register(mx)
        comm.all_reduce(mx, mx if rank == 0 else tout[:4096], algo="auto")
        torch.cuda.synchronize()
        out[("mixed_inplace",)] = (mx if rank == 0 else tout[:4096]).cpu().numpy().copy()
        comm.deregister(mx)
        comm.deregister(tin)
        comm.deregister(tout)
        # pipelined host-buffer AllReduce (windows: >= 32 MiB per rank, ragged)
        he = (40 << 20) // 4 + 3
        hx = torch.from_numpy(gen_inputs(world, he, "f32", "uniform", 9)[rank]).pin_memory()
        out[("host",)] = comm.all_reduce_host(hx, algo="2pa").numpy().copy()
        out[("host_small",)] = comm.all_reduce_host(hx[:1000].clone().pin_memory(), algo="2pa").numpy().copy()
        # K13 fused AllReduce + residual + RMSNorm, both algorithms
        fx = gen_inputs(world, 6 * 1024, "f32", "uniform", 5)
        x = torch.from_numpy(fx[rank]).cuda().view(6, 1024)
        res = torch.from_numpy(gen_inputs(1, 6 * 1024, "f32", "uniform", 6)[0]).cuda().view(6, 1024)
        wt = torch.linspace(0.5, 1.5, 1024, device="cuda")
        for algo in ("1pa_hb", "2pa"):
            ro = torch.empty_like(res)
            y = torch.empty_like(x)
            for t in (x, ro, y):
                comm.register(t)
            comm.all_reduce_add_rmsnorm(x, res, wt, eps=1e-6, algo=algo, resid_out=ro, norm_out=y)
            torch.cuda.synchronize()
            out[("norm", algo)] = (y.cpu().numpy().copy(), ro.cpu().numpy().copy())
            for t in (x, ro, y):
                comm.deregister(t)
        # NVLS kernel (K5) over the emulated switch: several pieces of a small
        # staging half, ragged count, .sys handshakes across the processes
        comm.setup_nvls_emulated(64 << 10)
        ne = 50001
        nx = gen_inputs(world, ne, "f32", "wide", 33)
        ns = torch.from_numpy(nx[rank]).cuda()
        nr = torch.empty_like(ns)
        for _ in range(2):
            comm.all_reduce(ns, nr, algo="switch_2pa")
            torch.cuda.synchronize()
        out[("nvls",)] = nr.cpu().numpy().copy()
        comm.check_device_error()
        comm.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:  # report instead of hanging the parent
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_two_processes_one_gpu_all_collectives():
    from oracle import oracle
    from inputs import gen_inputs
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, err = q.get(timeout=600)
        assert err is None, err
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    for elems in (1000, 65536 + 8):
        ins = gen_inputs(world, elems, "f32", "wide", 77 + elems)
        for algo in ("1pa", "2pa", "2pa_ll", "1pa_hb", "2pr", "2pr+ring"):
            want = oracle.allreduce(ins, {"2pa_ll": "2pa", "1pa_hb": "1pa", "2pr+ring": "2pr"}.get(algo, algo), "f32")
            for r in range(world):
                assert np.array_equal(res[r][("ar", algo, elems)].view(np.uint32),
                                      want[r].view(np.uint32)), (algo, r, elems)
        cat = np.concatenate(ins)
        rs_ins = [np.concatenate([x] * world) for x in ins]
        rs_want = oracle.reducescatter(rs_ins, "direct", "f32")
        rs_ring = oracle.reducescatter(rs_ins, "ring_rs", "f32")
        for r in range(world):
            for algo in ("allpairs_ag", "ring_ag", "ring_ag+ring"):
                assert np.array_equal(res[r][("ag", algo, elems)], cat), (algo, r)
            assert np.array_equal(res[r][("rs", "rs_direct", elems)].view(np.uint32), rs_want[r].view(np.uint32))
            for algo in ("ring_rs", "ring_rs+ring"):
                assert np.array_equal(res[r][("rs", algo, elems)].view(np.uint32), rs_ring[r].view(np.uint32))
    assert res[0][("tune",)] and res[0][("tune",)] == res[1][("tune",)]   # one table on every rank
    tsum = oracle.allreduce(gen_inputs(world, 1 << 18, "f32", "int", 3), "oracle", "f32")
    for r in range(world):
        assert np.array_equal(res[r][("tune_auto",)], tsum[r])
        assert np.array_equal(res[r][("mixed_inplace",)], tsum[r][:4096])
    hins = gen_inputs(world, (40 << 20) // 4 + 3, "f32", "uniform", 9)
    hwant = oracle.allreduce(hins, "2pa", "f32")
    hsmall = oracle.allreduce([x[:1000] for x in hins], "2pa", "f32")
    for r in range(world):
        assert np.array_equal(res[r][("host",)].view(np.uint32), hwant[r].view(np.uint32))
        assert np.array_equal(res[r][("host_small",)].view(np.uint32), hsmall[r].view(np.uint32))
    nwant = oracle.allreduce(gen_inputs(world, 50001, "f32", "wide", 33), "switch_2pa", "f32")
    for r in range(world):
        assert np.array_equal(res[r][("nvls",)].view(np.uint32), nwant[r].view(np.uint32)), ("nvls", r)
    fx = gen_inputs(world, 6 * 1024, "f32", "uniform", 5)
    h = fx[0].astype(np.float32)
    for x in fx[1:]:
        h = (h + x).astype(np.float32)
    ro = (h + gen_inputs(1, 6 * 1024, "f32", "uniform", 6)[0]).astype(np.float32).reshape(6, 1024)
    var = (ro.astype(np.float64) ** 2).mean(-1, keepdims=True)
    y = ro / np.sqrt(var + 1e-6) * np.linspace(0.5, 1.5, 1024)
    for algo in ("1pa_hb", "2pa"):
        for r in range(world):
            got_y, got_ro = res[r][("norm", algo)]
            assert np.array_equal(got_ro.view(np.uint32), ro.view(np.uint32)), (algo, r)
            np.testing.assert_allclose(got_y, y, rtol=1e-5, atol=1e-6)


PLAN_CASES = [("2pa", "memory", 2048, "f32"), ("2pa", "ll", 1024, "f32"), ("1pa", "", 512, "bf16"),
              ("ring_rs", "", 4096, "f32"), ("allpairs_ag", "", 1000, "f32"), ("2pr", "", 4096, "bf16"),
              ("2pa", "port", 4096, "f32"),
              # compiled LL kernel across processes: the 1pa scatter / read-reduce
              # streamed, the 2pa_ll reduce broadcast from registers
              ("1pa", "", 1 << 20, "f32"), ("2pa", "ll", 65536, "bf16")]


def _plan_doc(name, var, elems, dtype, n):
    from paper_2504_09014_b200.algorithms import build_algo
    from paper_2504_09014_b200.lowering import LoweringParams, lower
    from paper_2504_09014_b200.plan import serialize_plan
    proto = "LL" if name == "1pa" or var == "ll" else "HB"
    params = LoweringParams(n, elems, dtype, proto)
    return serialize_plan(lower(build_algo(name, params, variant=var), params))


def _plan_worker(rank, world, port, q):
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path[:0] = [root, os.path.join(root, "tests", "golden")]
        import torch
        import torch.distributed as dist
        from inputs import gen_inputs
        from paper_2504_09014_b200.comm import Communicator
        from paper_2504_09014_b200.dtypes import torch_dtype
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        comm = Communicator(spin_timeout_ms=60000)
        out = {}
        for name, var, elems, dtype in PLAN_CASES:
            rt = comm.load_plan(_plan_doc(name, var, elems, dtype, world), dtype=dtype)
            ins = gen_inputs(world, rt.in_elems, dtype, "normal", 31 + elems)
            x = ins[rank]
            send = (torch.from_numpy(x.view(np.int16)).view(torch.bfloat16) if dtype == "bf16"
                    else torch.from_numpy(x)).cuda()
            recv = torch.empty(rt.out_elems, dtype=torch_dtype(dtype), device="cuda")
            comm.register(send)
            comm.register(recv)
            for _ in range(3):   # repeated executions reuse lanes / flags / barriers
                rt.run(send, recv)
            torch.cuda.synchronize()
            rt.check_device_error()
            got = recv.cpu()
            out[(name, var, elems)] = (got.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16"
                                       else got.numpy()).copy()
            comm.deregister(send)
            comm.deregister(recv)
            rt.close()
        comm.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception:
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_two_processes_one_gpu_plans():
    """K10 in the one-process-per-GPU mode: plan heaps exchanged over the
    bootstrap, peers' I/O through registered buffers, port channels through
    each process's proxy; outputs equal the sequential plan interpreter's."""
    from oracle import oracle
    from inputs import gen_inputs
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, err = q.get(timeout=600)
        assert err is None, err
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    for name, var, elems, dtype in PLAN_CASES:
        doc = _plan_doc(name, var, elems, dtype, world)
        import json
        in_elems = next(b["elems"] for b in json.loads(doc)["buffers"] if b["kind"] == "input")
        ins = gen_inputs(world, in_elems, dtype, "normal", 31 + elems)
        want = oracle.run_plan(doc, ins, dtype=dtype)
        for r in range(world):
            assert np.array_equal(res[r][(name, var, elems)].view(np.uint8), want[r].view(np.uint8)), (name, var, r)


def _worker4(rank, world, port, q):
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path[:0] = [root, os.path.join(root, "tests", "golden")]
        import torch
        import torch.distributed as dist
        from inputs import gen_inputs
        from paper_2504_09014_b200.comm import Communicator
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        comm = Communicator(spin_timeout_ms=120000)
        out = {}
        elems = 4096 + 8
        ins = gen_inputs(world, elems, "bf16", "normal", 41)
        send = torch.from_numpy(ins[rank].view(np.int16)).cuda().view(torch.bfloat16)
        recv = torch.empty_like(send)
        ag = torch.empty(world * elems, device="cuda", dtype=torch.bfloat16)
        for t in (send, recv, ag):
            comm.register(t)
        for algo in ("1pa", "2pa", "2pa_ll", "2pr", "2pr+ring"):
            name, var = _nv(algo)
            comm.all_reduce(send, recv, algo=name, variant=var)
            torch.cuda.synchronize()
            out[("ar", algo)] = recv.view(torch.int16).cpu().numpy().view(np.uint16).copy()
        comm.all_gather(send, ag, algo="allpairs_ag")
        torch.cuda.synchronize()
        out[("ag",)] = ag.view(torch.int16).cpu().numpy().view(np.uint16).copy()
        comm.setup_nvls_emulated(16 << 10)
        comm.all_reduce(send, recv, algo="switch_2pa")
        torch.cuda.synchronize()
        out[("nvls",)] = recv.view(torch.int16).cpu().numpy().view(np.uint16).copy()
        comm.check_device_error()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception as e:   # report to the parent instead of hanging it
        import traceback
        q.put((rank, None, traceback.format_exc()))


def test_four_processes_one_gpu():
    """Four ranks, one process each, sharing cuda:0 (time-sliced contexts):
    the n > 2 peer tables of the multi-process path (registration, handshakes,
    LL slots, ring links, emulated NVLS staging) vs the oracle, bf16."""
    from oracle import oracle
    from inputs import gen_inputs
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker4, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, out, err = q.get(timeout=900)
        assert err is None, err
        res[r] = out
    for p in procs:
        p.join(timeout=60)
    ins = gen_inputs(world, 4096 + 8, "bf16", "normal", 41)
    for algo in ("1pa", "2pa", "2pa_ll", "2pr", "2pr+ring"):
        want = oracle.allreduce(ins, {"2pa_ll": "2pa", "2pr+ring": "2pr"}.get(algo, algo), "bf16")
        for r in range(world):
            assert np.array_equal(res[r][("ar", algo)], want[r]), (algo, r)
    cat = np.concatenate(ins)
    nwant = oracle.allreduce(ins, "switch_2pa", "bf16")
    for r in range(world):
        assert np.array_equal(res[r][("ag",)], cat)
        assert np.array_equal(res[r][("nvls",)], nwant[r])
