"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

from inputs import gen_inputs
from oracle import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def _cases():
    with open(os.path.join(GOLD, "collectives.json")) as f:
        return json.load(f)


def _auto_algo(kind, n, elems, thresholds=None):
    # cf/collectives.py:418-461 single-node defaults, bytes = elems*4*(n if AG)
    t = {"small": 32 * 1024, "large": 64 << 20, **(thresholds or {})}
    nbytes = elems * 4 * (n if kind == "allgather" else 1)
    if kind == "allreduce":
        return "1pa" if nbytes < t["small"] else ("2pa" if nbytes < t["large"] else "2pr")
    if kind == "allgather":
        return "allpairs_ag" if nbytes < 1 << 20 else "ring_ag"
    return "ring_rs"


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['kind']}-{c['algo'] or 'auto'}"
                         f"{c['variant']}-n{c['n']}-e{c['elems']}-{c['dtype']}-{c['dist']}")
def test_oracle_matches_reference_collective(case):
    ins = gen_inputs(case["n"], case["elems"], case["dtype"], case["dist"], case["seed"])
    algo = case["algo"] or _auto_algo(case["kind"], case["n"], case["elems"], case.get("thresholds"))
    if case["kind"] == "allreduce":
        outs = oracle.allreduce(ins, algo, case["dtype"])
    elif case["kind"] == "reducescatter":
        outs = oracle.reducescatter(ins, algo, case["dtype"])
    else:
        outs = oracle.allgather(ins)
    assert [len(o) for o in outs] == case["out_len"]
    assert [_digest(o) for o in outs] == case["digests"]


def test_oracle_ascending_equals_numpy_sum():
    ins = gen_inputs(8, 4096, "f32", "wide", 5)
    want = np.sum(np.stack(ins), axis=0)
    for o in oracle.allreduce(ins, "oracle", "f32"):
        assert np.array_equal(o.view(np.uint32), want.view(np.uint32))


def _runs():
    with open(os.path.join(GOLD, "plan_runs.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("run", _runs(), ids=lambda r: f"{r['plan']}-{r['dtype']}")
def test_oracle_plan_interpreter_matches_reference_runtime(run):
    with open(os.path.join(GOLD, "plans", run["plan"] + ".json"), "rb") as f:
        doc = f.read()
    n = json.loads(doc)["num_ranks"]
    ins = gen_inputs(n, run["in_elems"], run["dtype"], run["dist"], run["seed"])
    outs = oracle.run_plan(doc, ins, dtype=run["dtype"])
    assert [_digest(o) for o in outs] == run["digests"]


def test_ll_packet_layout_matches_reference():
    with open(os.path.join(GOLD, "ll_packets.json")) as f:
        kats = json.load(f)
    for k in kats:
        payload = np.array(k["payload"], np.uint8)
        pk = oracle.ll_pack(payload, k["flag"])
        assert pk.tolist() == k["packets"]
        data, bad = oracle.ll_unpack(pk, k["flag"])
        assert bad == 0 and data.tolist() == k["payload"]
        _, bad = oracle.ll_unpack(pk, k["flag"] + 1)   # stale generation never accepted
        assert bad == len(payload) // 4


def test_ll_zero_flag_and_alignment_rejected():
    with pytest.raises(ValueError, match="E_ZERO_FLAG"):
        oracle.ll_pack(np.zeros(4, np.uint8), 0)
    with pytest.raises(ValueError, match="E_BAD_ALIGN"):
        oracle.ll_pack(np.zeros(6, np.uint8), 1)


def test_f16_rounding_matches_numpy():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 10.0 ** rng.integers(-9, 6, 20000),
                        np.array([65504, 65519.99, 65520, 1e-8, 2.9802322e-08, 5.96e-8, -0.0, np.inf, -np.inf],
                                 np.float32)]).astype(np.float32)
    lib = oracle.lib()
    got = np.array([lib.cfo_f32_to_f16(float(v)) for v in x], np.uint16)
    assert np.array_equal(got, x.astype(np.float16).view(np.uint16))


def test_bf16_rounding_matches_torch():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(50000) * 10.0 ** rng.integers(-30, 30, 50000)).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(oracle.bf16_from_f32(x), want)
    lib = oracle.lib()
    got = np.array([lib.cfo_f32_to_bf16(float(v)) for v in x[:5000]], np.uint16)
    assert np.array_equal(got, want[:5000])


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_half_reduce_is_f32_accumulate_round_once(dtype):
    ins = gen_inputs(8, 1000, dtype, "normal", 3)
    to32 = (lambda a: a.astype(np.float32)) if dtype == "f16" else oracle.bf16_to_f32
    acc = to32(ins[0]).copy()
    for a in ins[1:]:
        acc = (acc + to32(a)).astype(np.float32)
    want = acc.astype(np.float16) if dtype == "f16" else oracle.bf16_from_f32(acc)
    got = oracle.reduce_ordered(dtype, ins, list(range(8)))
    assert np.array_equal(got.view(np.uint16), want.view(np.uint16))


def test_threaded_reduce_matches_single_thread():
    ins = gen_inputs(8, 1 << 18, "f32", "wide", 9)
    a = oracle.reduce_ordered("f32", ins, list(range(8)), nthreads=1)
    b = oracle.reduce_ordered("f32", ins, list(range(8)), nthreads=0)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_oracle_bf16_allgather_matches_reference():
    """bf16 AllGather digests produced by the reference itself (i32 view of
    the 16-bit shards, tests/golden/make_golden.py --ag-bf16) pin the oracle."""
    import hashlib
    from inputs import ag_bf16_shards
    with open(os.path.join(GOLD, "ag_bf16.json")) as f:
        cases = json.load(f)
    assert len(cases) == 24
    for c in cases:
        shards = ag_bf16_shards(c["n"], c["count"], c["seed"])
        for r, o in enumerate(oracle.allgather(shards)):
            assert hashlib.sha256(np.ascontiguousarray(o).view(np.uint8).tobytes()).hexdigest() == \
                c["digests"][r], (c["n"], c["count"], c["algo"], r)


def _lowp_cases():
    with open(os.path.join(GOLD, "lowp.json")) as f:
        return json.load(f)


def test_oracle_lowp_allreduce_matches_reference_f32_path():
    """f16 / bf16 AllReduce: the oracle equals the reference's own f32 path on
    the exactly-upcast inputs, rounded once (tests/golden/make_golden.py --lowp)
    -- the 2-byte semantics anchored on reference outputs, every algorithm."""
    import hashlib
    cases = _lowp_cases()
    assert len(cases) == 144
    for c in cases:
        ins = gen_inputs(c["n"], c["elems"], c["dtype"], "normal", c["seed"])
        name = {"2pa": "2pa"}.get(c["algo"], c["algo"])
        outs = oracle.allreduce(ins, name, c["dtype"])
        got = [hashlib.sha256(np.ascontiguousarray(o).view(np.uint8).tobytes()).hexdigest() for o in outs]
        assert got == c["digests"], (c["n"], c["elems"], c["dtype"], c["algo"], c["variant"])
