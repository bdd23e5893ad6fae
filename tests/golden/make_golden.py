"""Generate golden vectors by running the REFERENCE (commforge 0.1.0) on the CPU.

Run here (the dev container, where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It writes small fixtures next to this file; the tests (CPU and GPU) only read
the fixtures, never /root/reference.  Inputs are regenerated from the seeds
recorded in each case by `gen_inputs` (tests/golden/inputs.py), so fixtures
carry only outputs: sha256 digests of every rank's output bytes, plus full
arrays for the small cases.

Fixtures
  collectives.json   reference `collective()` outputs per (kind, algo, variant,
                     n, elems, dtype, dist, seed)       cf/collectives.py:532-573
  plans/*.json       reference `lower(build_algo(...))` canonical plan bytes
                     cf/lowering.py:629-648, cf/plan.py:136-156
  plan_runs.json     reference `Runtime.execute` output digests on those plans
                     cf/executor.py:135-178
  ll_packets.json    reference MemoryChannel.put_ll byte layout  cf/channels.py:244-280
  frontend/*.json    the reference's TS-frontend golden documents (data), used
                     as pre-lowering inputs       pkg/tests/golden/frontend_*.json
  ag_bf16.json       bf16 AllGather through the reference: each rank's bf16
                     shard (random 16-bit patterns, NaNs included) viewed as
                     i32 words -- odd counts padded by one uint16 per shard,
                     stripped afterwards -- and gathered by collective("allgather",
                     algo=allpairs_ag | ring_ag)      cf/collectives.py:253-270, 82-104
                     (`python tests/golden/make_golden.py --ag-bf16` regenerates
                     only this file)
  lowp.json          f16 / bf16 AllReduce anchored on the reference: the
                     reference has 4-byte types only (cf/dtypes.py:7-8), so each
                     case runs the reference's f32 path on the exactly-upcast
                     inputs (its order, f32 adds) and rounds the result once to
                     the 2-byte type (RNE) -- the semantics the kernels
                     implement (`--lowp` regenerates only this file)
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, HERE)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True

from inputs import ag_bf16_shards, gen_inputs  # noqa: E402

from commforge import collective, make_world  # noqa: E402
from commforge.channels import LL, MemoryChannel  # noqa: E402
from commforge.collectives import build_algo  # noqa: E402
from commforge.executor import Runtime  # noqa: E402
from commforge.lowering import LoweringParams, lower  # noqa: E402
from commforge.plan import parse_plan, serialize_plan  # noqa: E402
from commforge.sched import Scheduler  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


AR = [("1pa", ""), ("2pa", "memory"), ("2pa", "ll"), ("2pa", "port"),
      ("switch_2pa", ""), ("2pr", "")]


def collectives_cases():
    cases = []
    for n in (2, 4, 8):
        sizes = [1, 7, 64, 3 * n + 1, 2 * n, 256]
        for elems in sizes:
            for dtype, dist in (("i32", "int"), ("f32", "uniform"), ("f32", "wide")):
                seed = 1000 * n + 10 * elems + {"int": 0, "uniform": 1, "wide": 2}[dist]
                for algo, var in AR:
                    cases.append(("allreduce", algo, var, n, elems, dtype, dist, seed))
                cases.append(("reducescatter", "ring_rs", "", n, elems, dtype, dist, seed))
            seed = 1000 * n + 10 * elems + 7
            for algo in ("allpairs_ag", "ring_ag"):
                cases.append(("allgather", algo, "", n, elems, "i32", "bits", seed))
    # the facade's automatic selection at a few sizes (cf/collectives.py:550-556)
    for n, elems in ((8, 16), (8, 8192), (4, 4096)):
        cases.append(("allreduce", "", "", n, elems, "i32", "int", 77 + elems))
    # default selection with f32 (order-sensitive) on both sides of the 32 KiB
    # crossover, default ReduceScatter (ring_rs: 2n padding, ring order) and
    # default AllGather on both sides of the 1 MiB crossover
    for n, elems in ((8, 16), (8, 8193), (4, 8192), (4, 8191)):
        cases.append(("allreduce", "", "", n, elems, "f32", "uniform", 91 + elems))
    for n, elems in ((4, 12), (8, 24), (8, 100), (2, 7), (4, 1026)):
        cases.append(("reducescatter", "", "", n, elems, "f32", "uniform", 93 + elems))
        cases.append(("reducescatter", "", "", n, elems, "i32", "int", 95 + elems))
    for n, elems in ((8, 5), (4, 65536), (2, 131072)):
        cases.append(("allgather", "", "", n, elems, "i32", "bits", 97 + elems))
    return cases


# default selection under explicit thresholds: the reference's Selector with a
# small `large` so 2pr (ring order) is picked at test sizes (cf/collectives.py:464-486)
SEL_THRESHOLDS = {"small": 64, "large": 1024}


def selector_cases():
    cases = []
    for n, elems in ((4, 8), (4, 100), (8, 512), (8, 1000)):
        cases.append(("allreduce", "", "", n, elems, "f32", "uniform", 101 + elems))
    return cases


def make_collectives():
    out = []
    for kind, algo, var, n, elems, dtype, dist, seed in collectives_cases():
        ins = gen_inputs(n, elems, dtype, dist, seed)
        w = make_world(1, n, seed=7)
        res = collective(kind, ins, w, dtype=dtype, algo=algo or None, variant=var)
        case = {"kind": kind, "algo": algo, "variant": var, "n": n, "elems": elems,
                "dtype": dtype, "dist": dist, "seed": seed,
                "out_len": [int(len(o)) for o in res],
                "digests": [digest(o) for o in res]}
        if elems <= 16:
            case["outputs"] = [np.asarray(o).view(np.uint32).tolist() for o in res]
        out.append(case)
    from commforge.collectives import Selector
    for kind, algo, var, n, elems, dtype, dist, seed in selector_cases():
        ins = gen_inputs(n, elems, dtype, dist, seed)
        w = make_world(1, n, seed=7)
        res = collective(kind, ins, w, dtype=dtype, selector=Selector(thresholds=dict(SEL_THRESHOLDS)))
        out.append({"kind": kind, "algo": "", "variant": "", "n": n, "elems": elems, "dtype": dtype,
                    "dist": dist, "seed": seed, "thresholds": SEL_THRESHOLDS,
                    "out_len": [int(len(o)) for o in res], "digests": [digest(o) for o in res]})
    with open(os.path.join(HERE, "collectives.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"collectives.json: {len(out)} cases")


PLAN_CASES = [
    # (algo, variant, n, elems, instances, protocol)
    ("1pa", "", 4, 8, 1, "LL"), ("1pa", "", 8, 64, 1, "LL"),
    ("2pa", "memory", 4, 8, 1, "HB"), ("2pa", "memory", 8, 64, 1, "HB"),
    ("2pa", "memory", 8, 64, 2, "HB"), ("2pa", "ll", 4, 8, 1, "LL"),
    ("2pa", "port", 4, 8, 1, "HB"), ("switch_2pa", "", 8, 64, 1, "HB"),
    ("allpairs_ag", "", 8, 64, 1, "HB"), ("ring_ag", "", 4, 8, 1, "HB"),
    ("ring_rs", "", 4, 8, 1, "HB"), ("2pr", "", 4, 16, 1, "HB"),
    ("2pa", "memory", 8, 8192, 1, "HB"), ("1pa", "", 8, 8192, 1, "LL"),
    ("ring_rs", "", 2, 8, 1, "HB"), ("2pr", "", 8, 32, 1, "HB"), ("2pr", "", 4, 32, 2, "HB"),
    ("ring_ag", "", 8, 16, 1, "HB"), ("2pa", "ll", 8, 64, 1, "LL"), ("2pa", "ll", 4, 16, 2, "LL"),
    ("2pa", "port", 8, 64, 1, "HB"), ("1pa", "", 2, 8, 1, "LL"), ("1pa", "", 4, 16, 2, "LL"),
    ("switch_2pa", "", 4, 16, 2, "HB"), ("allpairs_ag", "", 4, 8, 2, "HB"),
    ("ring_rs", "", 4, 32, 2, "HB"),
]


def plan_name(algo, var, n, elems, inst):
    v = f"_{var}" if var else ""
    i = f"_i{inst}" if inst > 1 else ""
    return f"{algo}{v}_n{n}_e{elems}{i}"


def make_plans():
    pdir = os.path.join(HERE, "plans")
    os.makedirs(pdir, exist_ok=True)
    runs = []
    for algo, var, n, elems, inst, proto in PLAN_CASES:
        params = LoweringParams(n, elems, "i32", proto, instances=inst)
        w = make_world(1, n)
        plan = lower(build_algo(algo, params, w, variant=var), params)
        doc = serialize_plan(plan)
        name = plan_name(algo, var, n, elems, inst)
        with open(os.path.join(pdir, name + ".json"), "wb") as f:
            f.write(doc)
        in_elems = next(b.elems for b in plan.buffers if b.kind == "input")
        for dtype, dist in (("i32", "int"), ("f32", "wide")):
            if elems > 1024 and dtype == "i32":
                continue
            p2 = parse_plan(doc.replace(b'"dtype":"i32"', f'"dtype":"{dtype}"'.encode()))
            seed = 31 * n + elems + (1 if dtype == "f32" else 0)
            ins = gen_inputs(n, in_elems, dtype, dist, seed)
            res = Runtime(p2, make_world(1, n)).execute(ins)
            runs.append({"plan": name, "dtype": dtype, "dist": dist, "seed": seed,
                         "in_elems": in_elems, "digests": [digest(o) for o in res.outputs]})
    with open(os.path.join(HERE, "plan_runs.json"), "w") as f:
        json.dump(runs, f, indent=0, sort_keys=True)
    print(f"plans: {len(PLAN_CASES)}, plan_runs.json: {len(runs)} runs")


def make_ll():
    """Byte layout written by MemoryChannel.put_ll for a 16-byte payload."""
    kats = []
    for size, flag in ((4, 7), (16, 9), (24, 0x01020304)):
        w = make_world(1, 2, seed=0)
        sched = Scheduler(w)
        src = w.alloc_region(0, size)
        dst = w.alloc_region(1, 2 * size)
        payload = (np.arange(size, dtype=np.uint32) * 37 + 11).astype(np.uint8)
        w.write(src, 0, payload)
        ch = MemoryChannel(w, sched, LL, 0, 1, src, dst)

        def sender(ctx, ch=ch, size=size, flag=flag):
            yield from ch.put_ll(0, 0, size, flag, ctx)

        sched.spawn("tx", sender)
        sched.run()
        kats.append({"payload": payload.tolist(), "flag": flag,
                     "packets": w.read(dst, 0, 2 * size).tolist()})
    with open(os.path.join(HERE, "ll_packets.json"), "w") as f:
        json.dump(kats, f, indent=0)
    print(f"ll_packets.json: {len(kats)} KATs")


def copy_frontend():
    from commforge.lowering import graph_from_plan
    fdir = os.path.join(HERE, "frontend")
    os.makedirs(fdir, exist_ok=True)
    src = "/root/reference/pkg/tests/golden"
    for name in sorted(os.listdir(src)):
        if name.endswith(".json"):
            shutil.copyfile(os.path.join(src, name), os.path.join(fdir, name))
    # the reference's lowering of the TS-frontend documents (pre-lowering -> plan)
    for name in ("frontend_1pa_n4e8", "frontend_ringrs_n4e8"):
        with open(os.path.join(src, name + ".json"), "rb") as f:
            plan = lower(graph_from_plan(parse_plan(f.read())))
        with open(os.path.join(fdir, name + "_lowered.json"), "wb") as f:
            f.write(serialize_plan(plan))
    print("frontend goldens copied")


def make_ag_bf16():
    cases = []
    for n in (2, 4, 8):
        for cnt in (2, 7, 64, 4097):
            seed = 500 * n + cnt
            shards = ag_bf16_shards(n, cnt, seed)
            pad = cnt % 2
            words = [np.concatenate([s_, np.zeros(pad, np.uint16)]).view(np.int32) for s_ in shards]
            for algo in ("allpairs_ag", "ring_ag"):
                world = make_world(1, n, "switch-attached", 0)
                outs = collective("allgather", words, world, dtype="i32", algo=algo)
                got = []
                for o in outs:
                    half = np.asarray(o).view(np.uint16).reshape(n, cnt + pad)[:, :cnt]
                    got.append(half.reshape(-1))
                cat = np.concatenate(shards)
                assert all(np.array_equal(g, cat) for g in got), (n, cnt, algo)
                cases.append({"n": n, "count": cnt, "seed": seed, "algo": algo,
                              "digests": [digest(g) for g in got]})
    with open(os.path.join(HERE, "ag_bf16.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print(f"ag_bf16: {len(cases)} cases")


def _round16(x: np.ndarray, dtype: str) -> np.ndarray:
    """f32 -> f16 / bf16 bit patterns, round to nearest even (finite inputs)."""
    x = np.ascontiguousarray(x, np.float32)
    if dtype == "f16":
        return x.astype(np.float16).view(np.uint16)
    u = x.view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _up32(a: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "f16":
        return np.asarray(a, np.float16).astype(np.float32)
    return (np.asarray(a, np.uint16).astype(np.uint32) << 16).view(np.float32)


def make_lowp():
    cases = []
    for n in (2, 4, 8):
        for elems in (7, 64, 3 * n + 1, 512):
            for dtype in ("f16", "bf16"):
                seed = 700 * n + elems + (1 if dtype == "bf16" else 0)
                ins = gen_inputs(n, elems, dtype, "normal", seed)
                up = [_up32(a, dtype) for a in ins]
                for algo, var in AR:
                    world = make_world(1, n, "switch-attached", 0)
                    outs = collective("allreduce", up, world, dtype="f32", algo=algo, variant=var)
                    cases.append({"n": n, "elems": elems, "dtype": dtype, "seed": seed, "algo": algo,
                                  "variant": var,
                                  "digests": [digest(_round16(np.asarray(o), dtype)) for o in outs]})
    with open(os.path.join(HERE, "lowp.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print(f"lowp: {len(cases)} cases")


if __name__ == "__main__":
    if "--lowp" in sys.argv:
        make_lowp()
        sys.exit(0)
    if "--collectives" in sys.argv:
        make_collectives()
        sys.exit(0)
    if "--ag-bf16" in sys.argv:
        make_ag_bf16()
        sys.exit(0)
    make_ag_bf16()
    make_lowp()
    make_ll()
    make_plans()
    make_collectives()
    copy_frontend()
