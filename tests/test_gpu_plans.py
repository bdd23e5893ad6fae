"""GPU plan executor (K10) vs the reference runtime's outputs (golden digests)
and vs the oracle's sequential plan interpreter.  Needs a B200."""

import hashlib
import json
import os
import time

import numpy as np
import pytest

from inputs import gen_inputs
from oracle import oracle

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
_WORLDS = {}


def world(n):
    from paper_2504_09014_b200 import make_world
    if n not in _WORLDS:
        _WORLDS[n] = make_world(1, n, spin_timeout_ms=4000)
    return _WORLDS[n]


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def _load(name):
    with open(os.path.join(GOLD, "plans", name + ".json"), "rb") as f:
        return f.read()


def _runs():
    with open(os.path.join(GOLD, "plan_runs.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("run", _runs(), ids=lambda r: f"{r['plan']}-{r['dtype']}")
def test_plan_matches_reference_runtime_bits(run):
    from paper_2504_09014_b200 import Runtime, parse_plan
    doc = _load(run["plan"])
    plan = parse_plan(doc.replace(b'"dtype":"i32"', f'"dtype":"{run["dtype"]}"'.encode()))
    ins = gen_inputs(plan.num_ranks, run["in_elems"], run["dtype"], run["dist"], run["seed"])
    rt = Runtime(plan, world(plan.num_ranks))
    for _ in range(3):   # repeated executions reuse buffers, lanes and flags
        res = rt.execute(ins)
        assert [_digest(o) for o in res.outputs] == run["digests"]
    rt.close()


def test_reference_golden_ring_rs_plan():
    from paper_2504_09014_b200 import Runtime, parse_plan
    with open(os.path.join(GOLD, "frontend", "ring_rs_n4e8_lowered.json"), "rb") as f:
        plan = parse_plan(f.read())
    ins = [np.full(8, r + 1, np.int32) for r in range(4)]
    res = Runtime(plan, world(4)).execute(ins)
    for r in range(4):
        assert (res.outputs[r] == 10).all()   # reference test_executor.py:67-74


def _scaled(doc: bytes, factor: int, dtype: str) -> bytes:
    """Scale every element count / offset of a size-homogeneous library plan."""
    d = json.loads(doc)
    d["dtype"] = "f32"
    for b in d["buffers"]:
        b["elems"] *= factor
    for p in d["programs"]:
        for o in p["ops"]:
            for k in ("src", "dst", "src2", "arrives"):
                if k in o:
                    o[k] = [o[k][0], o[k][1] * factor, o[k][2] * factor]
    return json.dumps(d, sort_keys=True, separators=(",", ":")).encode()


@pytest.mark.parametrize("name,factor", [("2pa_memory_n8_e64", 128), ("1pa_n8_e64", 128),
                                         ("1pa_n8_e64", 128 * 64), ("1pa_n8_e64", 128 * 37 + 8),
                                         ("2pa_ll_n8_e64", 128 * 16),
                                         ("2pa_memory_n8_e64", 128 * 64),
                                         ("2pa_memory_n8_e64_i2", 512),
                                         ("switch_2pa_n8_e64", 1024), ("allpairs_ag_n8_e64", 256)])
@pytest.mark.parametrize("dtype", ["bf16", "f16", "f32"])
def test_c5_shaped_plans_vs_oracle(name, factor, dtype):
    """C5: Llama-70B TP decode AllReduce [b, 8192] through lowered reference plans."""
    from paper_2504_09014_b200 import Runtime, parse_plan
    doc = _scaled(_load(name), factor, dtype)
    plan = parse_plan(doc)
    in_elems = next(b.elems for b in plan.buffers if b.kind == "input")
    ins = gen_inputs(8, in_elems, dtype, "normal", factor, scale=0.02)
    rt = Runtime(plan, world(8), dtype=dtype)
    got = rt.execute(ins).outputs
    want = oracle.run_plan(doc, ins, dtype=dtype)
    for r in range(8):
        assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), r
    rt.close()


def _collective_cases():
    with open(os.path.join(GOLD, "collectives.json")) as f:
        return [c for c in json.load(f) if c["algo"] and c["n"] in (2, 8) and c["elems"] <= 64]


@pytest.mark.parametrize("case", _collective_cases(),
                         ids=lambda c: f"{c['kind']}-{c['algo']}{c['variant']}-n{c['n']}-e{c['elems']}-"
                                       f"{c['dtype']}-{c['dist']}")
def test_dsl_path_matches_reference_bits(case):
    """The MSCCL++ DSL path end to end: native builder + lowering -> plan ->
    GPU interpreter (port channels through the proxy), reference bits."""
    from paper_2504_09014_b200 import collective
    ins = gen_inputs(case["n"], case["elems"], case["dtype"], case["dist"], case["seed"])
    outs = collective(case["kind"], ins, world(case["n"]), dtype=case["dtype"], algo=case["algo"],
                      variant=case["variant"], via_plan=True)
    assert [_digest(o) for o in outs] == case["digests"]


@pytest.mark.parametrize("algo,var", [("2pa", "port"), ("2pr", ""), ("ring_rs", "")])
def test_port_channel_plans_at_size(algo, var):
    """PortChannel DMA at a few MiB: proxy FIFO wrap-around (> 1024 requests
    over the runs), flush, signal-after-put ordering."""
    from paper_2504_09014_b200 import collective
    n = 8
    kind = "reducescatter" if algo == "ring_rs" else "allreduce"
    ins = gen_inputs(n, 1 << 20, "f32", "wide", 5)
    for _ in range(3):
        got = collective(kind, ins, world(n), dtype="f32", algo=algo, variant=var, via_plan=True)
    want = (oracle.reducescatter(ins, "ring_rs", "f32") if kind == "reducescatter"
            else oracle.allreduce(ins, algo, "f32"))
    for r in range(n):
        assert np.array_equal(got[r].view(np.uint32), want[r].view(np.uint32)), r


def test_port_plan_back_to_back_calls_do_not_deadlock():
    """Four port-channel plan calls queued back to back (no host sync): the
    proxy's copies must not queue behind the next plan kernel on a shared
    hardware queue (the package raises CUDA_DEVICE_MAX_CONNECTIONS before the
    context exists; with CUDA's default 8 the second call timed out)."""
    import os
    import torch
    from paper_2504_09014_b200 import collectives as C
    assert int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8")) >= 32
    n = 8
    w = world(n)
    ins = gen_inputs(n, 1 << 18, "f32", "int", 8)
    rt = C._plan_runtime(w, "allreduce", "2pa", "port", 1 << 18, "f32")
    xs = [torch.from_numpy(x).to(w.device(r)) for r, x in enumerate(ins)]
    ys = [torch.empty_like(x) for x in xs]
    for _ in range(4):
        rt.run_raw(xs, ys)
    w.synchronize()
    rt.check_device_error()
    want = oracle.allreduce(ins, "2pa", "f32")
    for r in range(n):
        assert np.array_equal(ys[r].cpu().numpy(), want[r]), r


def test_wait_without_signal_raises_deadlock():
    """reference test_executor.py:77-89, as a device spin timeout."""
    from paper_2504_09014_b200 import Runtime, make_world
    from paper_2504_09014_b200.errors import DeadlockError
    from paper_2504_09014_b200.plan import (BufferDecl, ChannelDecl, ExecutionPlan, PlanOp,
                                            ThreadBlockProgram)
    plan = ExecutionPlan(1, "stuck", "custom", "HB", "i32", 2,
                         [BufferDecl("in", "input", "all", 4), BufferDecl("out", "output", "all", 4)],
                         [ChannelDecl("c0", "memory", src=0, dst=1)],
                         [ThreadBlockProgram(1, 0, (PlanOp("wait", chan="c0"),))])
    w = make_world(1, 2, spin_timeout_ms=300)
    rt = Runtime(plan, w)
    with pytest.raises(DeadlockError):
        rt.execute([np.zeros(4, np.int32)] * 2)
    # the report resets the plan (cfPlanClearDeviceError): the error word is
    # clear, and the next execution really spins for its timeout again
    # instead of short-circuiting on a stale error word
    rt.check_device_error()
    t0 = time.perf_counter()
    with pytest.raises(DeadlockError):
        rt.execute([np.zeros(4, np.int32)] * 2)
    assert time.perf_counter() - t0 >= 0.25
    rt.close()
    w.close()


def test_runtime_rejects_bad_plans():
    from paper_2504_09014_b200 import Runtime, parse_plan
    from paper_2504_09014_b200.errors import RankMismatchError, ShapeError
    plan = parse_plan(_load("2pa_memory_n4_e8"))
    with pytest.raises(RankMismatchError):
        Runtime(plan, world(2))
    with open(os.path.join(GOLD, "frontend", "frontend_1pa_n4e8.json"), "rb") as f:
        pre = parse_plan(f.read())
    with pytest.raises(ShapeError):
        Runtime(pre, world(4))
    rt = Runtime(plan, world(4))
    with pytest.raises(ShapeError):
        rt.execute([np.zeros(7, np.int32)] * 4)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("algo,var", [("2pa", "port"), ("2pa", "memory"), ("2pa", "ll"), ("1pa", ""),
                                      ("2pr", ""), ("switch_2pa", "")])
def test_dsl_path_low_precision_vs_plan_oracle(algo, var, dtype):
    """2-byte types through the DSL path: the plan's buffers have the 2-byte
    type, so every reduce op rounds; the GPU interpreter's bytes equal the
    oracle's sequential plan interpreter on the same lowered plan."""
    from paper_2504_09014_b200 import collective, serialize_plan
    from paper_2504_09014_b200.algorithms import build_algo
    from paper_2504_09014_b200.lowering import LoweringParams, lower
    n, elems = 8, 8 * 96
    ins = gen_inputs(n, elems, dtype, "normal", 91)
    got = collective("allreduce", ins, world(n), dtype=dtype, algo=algo, variant=var, via_plan=True)
    proto = "LL" if algo == "1pa" or var == "ll" else "HB"
    params = LoweringParams(n, elems, dtype, proto)
    doc = serialize_plan(lower(build_algo(algo, params, variant=var), params))
    want = oracle.run_plan(doc, ins, dtype=dtype)
    for r in range(n):
        assert np.array_equal(got[r].view(np.uint8), want[r][:elems].view(np.uint8)), r


@pytest.mark.parametrize("factor", [128 * 4, 128 * 64, 128 * 37 + 8])
def test_1pa_plan_streamed_pairs_in_place(factor, monkeypatch):
    """The compiled LL kernel streams the 1pa plan's packet scatter with its
    read-reduce (a thread reduces unit u one iteration after putting it).
    Streamed and op-by-op runs give the oracle's bits, out of place and in
    place (output = input: a thread only overwrites units it already put),
    on consecutive calls (alternating LL flag epochs)."""
    import torch
    from paper_2504_09014_b200 import Runtime, parse_plan
    doc = _scaled(_load("1pa_n8_e64"), factor, "f32")
    plan = parse_plan(doc)
    e = next(b.elems for b in plan.buffers if b.kind == "input")
    for stream in ("1", "0"):
        monkeypatch.setenv("CF_PLAN_LL_STREAM", stream)
        rt = Runtime(plan, world(8), dtype="f32")
        for it in range(3):
            ins = gen_inputs(8, e, "f32", "normal", factor + it, scale=0.02)
            want = oracle.run_plan(doc, ins, dtype="f32")
            xs = [torch.from_numpy(x).cuda() for x in ins]
            ys = [torch.empty_like(x) for x in xs]
            rt.run_raw(xs, ys)
            rt.check_device_error()
            for r in range(8):
                assert np.array_equal(ys[r].cpu().numpy().view(np.uint32), want[r].view(np.uint32)), (stream, it, r)
            rt.run_raw(xs, xs)   # in place
            rt.check_device_error()
            for r in range(8):
                assert np.array_equal(xs[r].cpu().numpy().view(np.uint32), want[r].view(np.uint32)), (stream, it, r)
        rt.close()
