"""Collectives beside a compute kernel that holds half of the SMs (the C5
consumer scenario: a GEMM on another stream).  Every handshake kernel waits
on CTA partners; a grid larger than the free SMs could wait on a partner that
is never scheduled.  The CTA budget (cfCommSetCtaBudget; default 64 per rank
one rank per GPU, i.e. under half of B200's 148 SMs) keeps every launch fully
resident on the free half.  Here 8 ranks share one GPU, with one launch per
rank (CF_SPLIT_GROUPS=1: the per-device launch path, CTA-pair handshakes on)
and in the single co-resident launch; the spin kernel holds 74 SMs (one CTA
per SM via its shared-memory request) for the whole run."""

import ctypes
import os

import numpy as np
import pytest
from inputs import gen_inputs
from oracle import oracle

pytestmark = pytest.mark.gpu

LIB = os.path.join(os.path.dirname(__file__), "kernels", "libcf_channels_test.so")


def _check(got, want):
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).view(np.uint8), np.asarray(w).view(np.uint8))


@pytest.mark.parametrize("split", ["0", "1"])
def test_collectives_complete_while_half_the_sms_are_held(split, monkeypatch):
    import torch
    from paper_2504_09014_b200 import allreduce_add_rmsnorm, collective, make_world
    monkeypatch.setenv("CF_SPLIT_GROUPS", split)
    lib = ctypes.CDLL(LIB)
    n = 8
    w = make_world(1, n, devices=[0] * n, spin_timeout_ms=8000, use_multicast="emulate")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    hold = sms // 2
    # budget: 8 ranks x 8 CTAs of 512 threads fit twice over on the free SMs
    w.set_cta_budget(8)

    def body():
        for elems, algos in ((4099, ("1pa", "2pa", "1pa_hb", "switch_2pa")), ((8 << 20) // 4 + 5, ("2pa",)),
                             (8 * 1000, ("2pa_ll",))):
            ins = gen_inputs(n, elems, "f32", "uniform", elems)
            for algo in algos:
                name, var = ("2pa", "ll") if algo == "2pa_ll" else (algo, "")
                got = collective("allreduce", ins, w, dtype="f32", algo=name, variant=var)
                _check(got, oracle.allreduce(ins, {"2pa_ll": "2pa", "1pa_hb": "1pa"}.get(algo, algo), "f32"))
        sh = gen_inputs(n, 3000, "i32", "bits", 4)
        for algo in ("allpairs_ag", "ring_ag"):
            _check(collective("allgather", sh, w, dtype="i32", algo=algo, variant="ring" if algo == "ring_ag" else ""),
                   oracle.allgather(sh))
        rs = gen_inputs(n, n * 2048, "f32", "uniform", 5)
        _check(collective("reducescatter", rs, w, dtype="f32", algo="ring_rs", variant="ring"),
               oracle.reducescatter(rs, "ring_rs", "f32"))
        xs = [torch.randn(64, 1024, device="cuda") for _ in range(n)]
        res = [torch.randn(64, 1024, device="cuda") for _ in range(n)]
        y, ro = allreduce_add_rmsnorm(w, xs, [r.clone() for r in res], torch.ones(1024, device="cuda"),
                                      algo="2pa")
        w.synchronize()
        h = sum(x.double() for x in xs)
        assert torch.allclose(ro[3].double(), h + res[3].double(), atol=1e-4)
        w.check_device_error()

    # once without the hold: CUDA loads modules lazily, and loading one while
    # another kernel spins waits for the whole context -- a deployment runs
    # warmed-up kernels, so the test does too
    body()
    assert lib.cftest_spin_start(hold, 200 * 1024) == 0
    try:
        body()
    finally:
        rc = lib.cftest_spin_stop()
        w.close()
    assert rc == 0, "the SM-holding kernel timed out: the collectives did not complete beside it"
