"""Plan IR / wire format / validator (CPU).  Mirrors the reference's
tests/test_plan.py coverage on the drop-in module."""

import json
import os

import pytest

from paper_2504_09014_b200.errors import PlanRefError, PlanSyntaxError, PlanVersionError
from paper_2504_09014_b200.plan import (BufferDecl, ChannelDecl, ExecutionPlan, PlanOp,
                                        ThreadBlockProgram, parse_plan, serialize_plan,
                                        validate_plan)

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_plans():
    d = os.path.join(GOLD, "plans")
    return sorted(os.path.join(d, f) for f in os.listdir(d))


@pytest.mark.parametrize("path", _golden_plans(), ids=os.path.basename)
def test_reference_plans_roundtrip_byte_identical(path):
    with open(path, "rb") as f:
        doc = f.read()
    plan = parse_plan(doc)
    assert serialize_plan(plan) == doc
    assert [d for d in validate_plan(plan) if d.severity == "error"] == []


def test_frontend_documents_parse_as_prelowering():
    for name in ("frontend_1pa_n4e8.json", "frontend_ringrs_n4e8.json"):
        with open(os.path.join(GOLD, "frontend", name), "rb") as f:
            doc = f.read()
        plan = parse_plan(doc)
        assert plan.lowered is False
        assert serialize_plan(plan) == json.dumps(json.loads(doc), sort_keys=True,
                                                  separators=(",", ":")).encode()


def copy_plan():
    return ExecutionPlan(
        version=1, name="copy2", collective="custom", protocol="HB", dtype="i32", num_ranks=2,
        buffers=[BufferDecl("in", "input", "all", 4), BufferDecl("out", "output", "all", 4)],
        channels=[ChannelDecl("c0", "memory", src=0, dst=1)],
        programs=[ThreadBlockProgram(0, 0, (PlanOp("put", chan="c0", src=("in", 0, 4),
                                                   dst=("out", 0, 4)),
                                            PlanOp("signal", chan="c0"))),
                  ThreadBlockProgram(1, 0, (PlanOp("wait", chan="c0"),))])


def test_copy_plan_golden_bytes():
    with open(os.path.join(GOLD, "frontend", "copy_plan.json"), "rb") as f:
        assert serialize_plan(copy_plan()) == f.read().strip()


@pytest.mark.parametrize("mutate,exc", [
    (lambda d: d.pop("name"), PlanSyntaxError),
    (lambda d: d.update(extra=1), PlanSyntaxError),
    (lambda d: d.update(version=2), PlanVersionError),
    (lambda d: d.update(protocol="XX"), PlanSyntaxError),
    (lambda d: d.update(num_ranks=0), PlanSyntaxError),
    (lambda d: d["programs"][0]["ops"].append({"op": "jump"}), PlanSyntaxError),
    (lambda d: d["programs"][0]["ops"].append({"op": "signal", "chan": "nope"}), PlanRefError),
    (lambda d: d["programs"][0]["ops"][0].update(src=["ghost", 0, 4]), PlanRefError),
    (lambda d: d["programs"][0]["ops"][0].update(src=["in", "0", 4]), PlanSyntaxError),
    (lambda d: d["buffers"].append(dict(d["buffers"][0])), PlanRefError),
])
def test_parse_errors_use_reference_classes(mutate, exc):
    doc = json.loads(serialize_plan(copy_plan()))
    mutate(doc)
    with pytest.raises(exc):
        parse_plan(json.dumps(doc).encode())


def test_invalid_json():
    with pytest.raises(PlanSyntaxError):
        parse_plan(b"{not json")


def _codes(plan):
    return sorted({(d.severity, d.code) for d in validate_plan(plan)})


def test_validator_diagnostics():
    p = copy_plan()
    assert _codes(p) == []
    bad = ExecutionPlan(1, "bad", "custom", "HB", "i32", 2,
                        [BufferDecl("in", "input", "all", 4), BufferDecl("out", "output", 0, 4)],
                        [ChannelDecl("c0", "memory", src=0, dst=0)],
                        [ThreadBlockProgram(1, 0, (PlanOp("put", chan="c0", src=("in", 0, 8),
                                                          dst=("out", 0, 4)),
                                                   PlanOp("wait", chan="c0")))])
    codes = _codes(bad)
    assert ("error", "channel-loop") in codes
    assert ("error", "bounds") in codes
    assert ("error", "op-rank") in codes
    assert ("warning", "sync-imbalance") in codes


def test_flag_reuse_detected():
    p = ExecutionPlan(1, "ll", "custom", "LL", "i32", 2,
                      [BufferDecl("in", "input", "all", 4), BufferDecl("out", "output", "all", 4),
                       BufferDecl("scr", "scratch", "all", 16)],
                      [ChannelDecl("m0", "memory", src=0, dst=1, protocol="LL")],
                      [ThreadBlockProgram(0, 0, (
                          PlanOp("put_packets", chan="m0", src=("in", 0, 4), dst=("scr", 0, 4), flag=1),
                          PlanOp("put_packets", chan="m0", src=("in", 0, 4), dst=("scr", 2, 4), flag=1)))])
    assert ("error", "flag-reuse") in _codes(p)


def test_timing_api_matches_reference_definitions():
    """algobw / rows_to_csv keep cf/timing.py:54-58, 352-358 (same values,
    same CSV columns, same error code on a non-positive latency)."""
    import paper_2504_09014_b200 as cf
    from paper_2504_09014_b200.errors import BadTimeError
    assert cf.algobw(1 << 20, 1e-3) == (1 << 20) / 1e-3
    assert cf.busbw(1 << 20, 1e-3, 8) == cf.algobw(1 << 20, 1e-3) * 2 * 7 / 8
    assert cf.busbw(1 << 20, 1e-3, 8, "allgather") == cf.algobw(1 << 20, 1e-3) * 7 / 8
    with pytest.raises(BadTimeError):
        cf.algobw(10, 0.0)
    csv = cf.rows_to_csv([cf.BenchRow("2pa_memory", "allreduce", 4096, 3.25, 1.26, True)])
    assert csv == "algo,collective,bytes,latency_us,algobw_gbps,selected\n" \
                  "2pa_memory,allreduce,4096,3.250000,1.260000,1\n"
