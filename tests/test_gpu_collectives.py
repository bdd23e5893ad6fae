"""GPU parity: libcf collectives vs the reference's own outputs (golden digests
from tests/golden/make_golden.py) and vs the CPU oracle.  Needs a B200."""

import hashlib
import json
import os

import numpy as np
import pytest

from inputs import gen_inputs
from oracle import oracle

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
_WORLDS = {}


def world(n, **kw):
    from paper_2504_09014_b200 import make_world
    key = (n, tuple(sorted(kw.items())))
    if key not in _WORLDS:
        _WORLDS[key] = make_world(1, n, spin_timeout_ms=5000, **kw)
    return _WORLDS[key]


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def _cases():
    with open(os.path.join(GOLD, "collectives.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['kind']}-{c['algo'] or 'default'}{c['variant']}"
                         f"-n{c['n']}-e{c['elems']}-{c['dtype']}-{c['dist']}{'-sel' if 'thresholds' in c else ''}")
def test_gpu_matches_reference_bits(case):
    """Every reference algorithm on the GPU returns the reference's exact bits;
    so does the facade's default selection (algo=None: the reference's
    threshold table, also with explicit Selector thresholds)."""
    from paper_2504_09014_b200 import Selector, collective
    ins = gen_inputs(case["n"], case["elems"], case["dtype"], case["dist"], case["seed"])
    sel = Selector(thresholds=dict(case["thresholds"])) if "thresholds" in case else None
    outs = collective(case["kind"], ins, world(case["n"]), dtype=case["dtype"], selector=sel,
                      algo=case["algo"] or None, variant=case["variant"])
    assert [len(o) for o in outs] == case["out_len"]
    assert [_digest(o) for o in outs] == case["digests"]


_RING = [c for c in _cases() if c["algo"] in ("2pr", "ring_rs", "ring_ag")]


@pytest.mark.parametrize("case", _RING, ids=lambda c: f"{c['kind']}-{c['algo']}-ring-n{c['n']}-e{c['elems']}-"
                         f"{c['dtype']}-{c['dist']}")
def test_literal_ring_matches_reference_bits(case):
    """The reference's ring algorithms on the literal ring transport
    (variant "ring": K9 / K12 / K7) return the reference's digests too --
    the default all-pairs transport is pinned by
    test_gpu_matches_reference_bits."""
    from paper_2504_09014_b200 import collective
    ins = gen_inputs(case["n"], case["elems"], case["dtype"], case["dist"], case["seed"])
    outs = collective(case["kind"], ins, world(case["n"]), dtype=case["dtype"], algo=case["algo"], variant="ring")
    assert [len(o) for o in outs] == case["out_len"]
    assert [_digest(o) for o in outs] == case["digests"]


def _aid(name):
    """libcf algorithm id; "+ring" = the literal ring transport (CF_ALGO_RING_LINKS)."""
    from paper_2504_09014_b200 import _lib
    base, _, links = name.partition("+")
    return _lib.ALGOS[base] | (_lib.CF_ALGO_RING_LINKS if links else 0)


ALGOS = [("1pa", ""), ("1pa_hb", ""), ("2pa", "memory"), ("2pa", "ll"), ("switch_2pa", ""),
         ("2pr", ""), ("2pr", "ring")]
_ORACLE_NAME = {"1pa_hb": "1pa"}


@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16", "i32"])
@pytest.mark.parametrize("elems", [1, 3, 8, 1000, 4097, 65536 + 24, 262144])
def test_allreduce_vs_oracle(n, dtype, elems):
    from paper_2504_09014_b200 import collective
    dist = {"f32": "wide", "i32": "int"}.get(dtype, "normal")
    ins = gen_inputs(n, elems, dtype, dist, 100 * n + elems % 97)
    for algo, var in ALGOS:
        got = collective("allreduce", ins, world(n), dtype=dtype, algo=algo, variant=var)
        want = oracle.allreduce(ins, _ORACLE_NAME.get(algo, algo), dtype)
        for r in range(n):
            assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), (algo, var, r)


@pytest.mark.parametrize("n,dtype,elems", [(8, "bf16", 32 * 1000), (8, "bf16", 1 << 20), (8, "bf16", (1 << 21) - 32),
                                          (8, "f32", (1 << 20) - 16), (4, "bf16", 3 << 18), (2, "f32", 1 << 19)])
def test_ll_twoshot_multi_round(n, dtype, elems):
    """K4's grid path (chunk bounds on the 8-byte grid) at sizes where every
    thread runs several rounds of kLL2U units, the last one partial: same bits
    as the oracle's two-shot order, twice (parity halves alternate)."""
    from paper_2504_09014_b200 import collective
    ins = gen_inputs(n, elems, dtype, "normal", 77 + elems % 101)
    want = oracle.allreduce(ins, "2pa", dtype)
    for rep in range(2):
        got = collective("allreduce", ins, world(n), dtype=dtype, algo="2pa", variant="ll")
        for r in range(n):
            assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), (rep, r)


@pytest.mark.parametrize("n", [3, 5, 6, 7])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_odd_rank_counts_vs_oracle(n, dtype):
    """Rank counts that are not powers of two (kernels templated on 2/4/8
    slots run n < slots; chunking pads to n or 2n): every AllReduce algorithm,
    both ReduceScatters and both AllGathers, bit-exact to the oracle."""
    from paper_2504_09014_b200 import collective
    dist = {"f32": "wide", "i32": "int"}.get(dtype, "normal")
    for elems in (1, 37, 4096 + 5, 70001):
        ins = gen_inputs(n, elems, dtype, dist, 1000 + 10 * n + elems % 7)
        for algo, var in ALGOS:
            got = collective("allreduce", ins, world(n), dtype=dtype, algo=algo, variant=var)
            want = oracle.allreduce(ins, _ORACLE_NAME.get(algo, algo), dtype)
            for r in range(n):
                assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), (elems, algo, var, r)
        for algo, var in (("ring_rs", ""), ("ring_rs", "ring"), ("rs_direct", "")):
            got = collective("reducescatter", ins, world(n), dtype=dtype, algo=algo, variant=var)
            want = oracle.reducescatter(ins, "ring_rs" if algo == "ring_rs" else "direct", dtype)
            for r in range(n):
                assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), (elems, algo, r)
        for algo, var in (("allpairs_ag", ""), ("ring_ag", ""), ("ring_ag", "ring")):
            got = collective("allgather", ins, world(n), dtype=dtype, algo=algo, variant=var)
            for g, wnt in zip(got, oracle.allgather(ins)):
                assert np.array_equal(g.view(np.uint8), wnt.view(np.uint8)), (elems, algo)
    world(n).check_device_error()


@pytest.mark.parametrize("n", [2, 8])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("elems", [5, 4096, 100003])
def test_reducescatter_allgather_vs_oracle(n, dtype, elems):
    from paper_2504_09014_b200 import collective
    dist = "wide" if dtype == "f32" else "normal"
    ins = gen_inputs(n, elems, dtype, dist, 7 * n + elems % 13)
    for algo, var in (("ring_rs", ""), ("ring_rs", "ring"), ("rs_direct", "")):
        got = collective("reducescatter", ins, world(n), dtype=dtype, algo=algo, variant=var)
        want = oracle.reducescatter(ins, "ring_rs" if algo == "ring_rs" else "direct", dtype)
        for r in range(n):
            assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), (algo, r)
    for algo, var in (("allpairs_ag", ""), ("ring_ag", ""), ("ring_ag", "ring")):
        got = collective("allgather", ins, world(n), dtype=dtype, algo=algo, variant=var)
        for g, wnt in zip(got, oracle.allgather(ins)):
            assert np.array_equal(g.view(np.uint8), wnt.view(np.uint8)), algo


def test_allgather_bf16_nan_patterns_bit_exact():
    """C2: random 16-bit patterns including NaNs move bit-exactly."""
    from paper_2504_09014_b200 import collective
    rng = np.random.default_rng(5)
    for n in (2, 4, 8):
        for cnt in (1, 7, 64, 4096, 1 << 18):
            shards = [rng.integers(0, 1 << 16, cnt, dtype=np.uint32).astype(np.uint16)
                      for _ in range(n)]
            got = collective("allgather", shards, world(n), dtype="bf16", algo="allpairs_ag")
            cat = np.concatenate(shards)
            for g in got:
                assert np.array_equal(g, cat)


def test_repeated_calls_reuse_scratch_and_semaphores():
    """Epoch flags / monotonic semaphores across many back-to-back calls of
    mixed algorithms and sizes (scratch is never zeroed between calls)."""
    import torch
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200 import _lib
    n = 8
    w = world(n)
    rng = np.random.default_rng(3)
    for it in range(60):
        elems = int(rng.choice([1, 33, 1024, 8192, 70000]))
        algo = ["1pa", "2pa", "2pa_ll", "1pa_hb", "2pr", "2pr+ring"][it % 6]
        vals = [torch.full((elems,), float(r + it), device=w.device(r)) for r in range(n)]
        outs = [torch.empty_like(v) for v in vals]
        C.run("allreduce", vals, outs, elems, "f32", _aid(algo), w)
        w.synchronize()
        want = float(sum(r + it for r in range(n)))
        for o in outs:
            assert torch.all(o == want).item(), (it, algo, elems)
    w.check_device_error()


@pytest.mark.parametrize("elems", [4096, 300000, 1 << 20])
def test_allreduce_in_place_vs_oracle(elems):
    """send == recv: every in-place-capable AllReduce kernel (the 2PR AllGather
    phase stores straight into the next rank's buffer, which is also its
    input) returns the oracle's bits."""
    import torch
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200 import _lib
    n = 8
    w = world(n)
    ins = gen_inputs(n, elems, "bf16", "normal", 900 + elems % 89)
    for algo in ("2pa", "2pr", "2pr+ring", "1pa", "2pa_ll"):
        if algo in ("1pa", "2pa_ll") and elems > (1 << 18):
            continue
        want = oracle.allreduce(ins, {"2pa_ll": "2pa", "2pr+ring": "2pr"}.get(algo, algo), "bf16")
        for rep in range(2):   # twice: the second call reuses slots / flags
            bufs = [torch.from_numpy(x.view(np.int16)).to(w.device(r)).view(torch.bfloat16)
                    for r, x in enumerate(ins)]
            C.run("allreduce", bufs, bufs, elems, "bf16", _aid(algo), w)
            w.synchronize()
            for r in range(n):
                got = bufs[r].view(torch.int16).cpu().numpy().view(np.uint16)
                assert np.array_equal(got, want[r]), (algo, rep, r)
    w.check_device_error()


def test_large_allreduce_property():
    """Size-independent check at a large size: integer-valued bf16 sums are exact."""
    import torch
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200 import _lib
    n = 8
    w = world(n)
    elems = 64 << 20   # 128 MiB per rank
    send = [torch.randint(-8, 8, (elems,), device=w.device(r), dtype=torch.int32)
            .to(torch.bfloat16) for r in range(n)]
    want = sum(s.float() for s in send)
    for algo in ("2pa", "switch_2pa", "2pr", "2pr+ring"):
        recv = [torch.empty_like(s) for s in send]
        C.run("allreduce", send, recv, elems, "bf16", _aid(algo), w)
        w.synchronize()
        for o in recv:
            assert torch.equal(o.float(), want), algo
    w.check_device_error()


def test_maximum_size_allreduce_and_allgather():
    """BASELINE's largest sweep point, 1 GiB per rank x 8 co-resident ranks
    (16 GiB resident): integer-valued bf16 two-shot sums are exact and equal
    on every rank; the 8 GiB AllGather output is bit-exact (sampled)."""
    import torch
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200 import _lib
    n = 8
    w = world(n)
    elems = 512 << 20   # 1 GiB of bf16 per rank
    send = [torch.randint(-8, 8, (elems,), device=w.device(r), dtype=torch.int8).to(torch.bfloat16)
            for r in range(n)]
    recv = [torch.empty_like(s) for s in send]
    C.run("allreduce", send, recv, elems, "bf16", _lib.ALGOS["2pa"], w)
    w.synchronize()
    want = torch.zeros(elems, device=w.device(0))
    for s_ in send:
        want += s_.float()
    for o in recv:
        assert torch.equal(o.float(), want)
    del recv, want
    shard = elems // n
    out = [torch.empty(elems, device=w.device(r), dtype=torch.bfloat16) for r in range(n)]
    C.run("allgather", [s_[:shard] for s_ in send], out, shard, "bf16", _lib.ALGOS["allpairs_ag"], w)
    w.synchronize()
    idx = torch.randint(0, elems, (1 << 20,), device=w.device(0))
    cat = torch.cat([s_[:shard] for s_ in send])
    for o in out:
        assert torch.equal(o[idx].view(torch.int16), cat[idx].view(torch.int16))
    w.check_device_error()


def test_ll_capacity_boundary():
    """LL algorithms accept exactly ll_max_bytes per rank and reject one
    element more with E_BAD_SIZE (the scratch is sized for it)."""
    from paper_2504_09014_b200 import collective
    from paper_2504_09014_b200.errors import BadSizeError
    n, cap = 4, 1 << 16
    w = world(n, ll_max_bytes=cap)
    ins = gen_inputs(n, cap // 4, "f32", "int", 71)
    for algo, var in (("1pa", ""), ("2pa", "ll")):
        got = collective("allreduce", ins, w, dtype="f32", algo=algo, variant=var)
        want = oracle.allreduce(ins, "1pa" if algo == "1pa" else "2pa", "f32")
        for r in range(n):
            assert np.array_equal(got[r], want[r]), (algo, r)
        with pytest.raises(BadSizeError):
            collective("allreduce", gen_inputs(n, cap // 4 + 1, "f32", "int", 72), w, dtype="f32",
                       algo=algo, variant=var)


def test_errors_map_to_reference_codes():
    import torch
    from paper_2504_09014_b200 import collective, collectives as C, _lib
    from paper_2504_09014_b200.errors import BadAlignError, BadSizeError, NoAlgoError, ShapeError
    w = world(2, ll_max_bytes=1 << 16)
    big = [np.ones(1 << 15, np.float32) for _ in range(2)]
    with pytest.raises(BadSizeError):
        collective("allreduce", big, w, dtype="f32", algo="1pa")
    with pytest.raises(NoAlgoError):
        collective("allreduce", big, w, dtype="f32", algo="ring_ag")
    with pytest.raises(ShapeError):
        collective("allreduce", big[:1], w, dtype="f32")
    t = [torch.zeros(64, device=w.device(r)) for r in range(2)]
    with pytest.raises(BadAlignError):
        C.run("allreduce", [x[1:] for x in t], [x[1:] for x in t], 8, "f32", _lib.ALGOS["2pa"], w)


def test_nvls_multicast_path_single_rank():
    """K5 plumbing on one GPU: multicast object, unicast+multicast mappings,
    multimem.ld_reduce / multimem.st (a 1-member group returns its input),
    staging in pieces larger than the NVLS half."""
    from paper_2504_09014_b200 import collective, make_world
    from paper_2504_09014_b200.world import device_multicast_capable
    if not device_multicast_capable(0):
        pytest.skip("cuda:0 reports no multicast (NVLS) support")
    w = make_world(1, 1, devices=[0], nvls_bytes=1 << 20)
    if not w.multicast_supported():
        pytest.skip("multicast advertised but the object could not be built on this box")
    try:
        for dtype in ("f32", "bf16", "f16", "i32"):
            dist = {"f32": "wide", "i32": "int"}.get(dtype, "normal")
            for elems in (5, 4096, 3 * (1 << 20) + 3):
                x = gen_inputs(1, elems, dtype, dist, elems)
                got = collective("allreduce", x, w, dtype=dtype, algo="switch_2pa")
                assert np.array_equal(got[0].view(np.uint8), x[0].view(np.uint8)), (dtype, elems)
    finally:
        w.close()


@pytest.mark.parametrize("n", [2, 3, 4, 6, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16", "i32"])
def test_nvls_kernel_control_path_emulated(n, dtype):
    """K5's fused kernel (copy-in, switch reduce / broadcast, copy-out, in
    pieces of the staging half, CTA-pair handshakes) with the two multimem
    instructions emulated by per-rank loads / stores: bit-exact to the
    reference switch order 0 + x_0 + ... + x_{n-1}, including messages of
    several pieces, ragged counts and repeated calls."""
    from paper_2504_09014_b200 import collective, make_world
    w = make_world(1, n, devices=[0] * n, use_multicast="emulate", nvls_bytes=64 << 10,
                   spin_timeout_ms=5000)
    try:
        assert not w.multicast_supported()
        dist = {"f32": "wide", "i32": "int"}.get(dtype, "normal")
        for elems in (1, 7, 4096, 16384 + 3, 200001):
            ins = gen_inputs(n, elems, dtype, dist, 31 * n + elems % 17)
            want = oracle.allreduce(ins, "switch_2pa", dtype)
            for rep in range(2):
                got = collective("allreduce", ins, w, dtype=dtype, algo="switch_2pa")
                for r in range(n):
                    g = got[r].view(np.uint8).reshape(elems, -1)
                    bad = np.nonzero(np.any(g != want[r].view(np.uint8).reshape(elems, -1), axis=1))[0]
                    assert not len(bad), (elems, rep, r, len(bad), bad[:4], bad[-2:], got[r][bad[:3]],
                                          want[r][bad[:3]], [x[bad[:3]] for x in ins])
        w.check_device_error()
    finally:
        w.close()


def test_coresident_world_has_no_multicast():
    assert not world(8).multicast_supported()


@pytest.mark.parametrize("dtype,elems", [("f32", (48 << 20) // 4 + 5), ("bf16", (64 << 20) // 2 + 24),
                                         ("bf16", 1000), ("i32", 4096 + 3)])
def test_host_buffer_allreduce_matches_device_path(dtype, elems):
    """cfAllReduceHost (pinned host tensors through collective()): the
    pipelined windows (>= 32 MiB per rank, ragged chunks) give the same bits
    as the device-buffer kernel, and the small path equals it too."""
    import torch
    from paper_2504_09014_b200 import collective
    from paper_2504_09014_b200.dtypes import torch_dtype
    w = world(8)
    g = torch.Generator().manual_seed(elems)
    host = [(torch.randn(elems, generator=g) * 4).to(torch_dtype(dtype)) if dtype != "i32"
            else torch.randint(-1000, 1000, (elems,), generator=g, dtype=torch.int32) for _ in range(8)]
    host = [h.pin_memory() for h in host]
    got = collective("allreduce", host, w, algo="2pa")
    dev = collective("allreduce", [h.cuda() for h in host], w, algo="2pa")
    for r in range(8):
        assert not got[r].is_cuda
        assert torch.equal(got[r].view(torch.int16 if dtype == "bf16" else got[r].dtype),
                           dev[r].cpu().view(torch.int16 if dtype == "bf16" else dev[r].dtype)), r
    # pageable host tensors take the same path (synchronous copies)
    got2 = collective("allreduce", [h.clone() for h in host[:8]], w, algo="2pa")
    assert all(torch.equal(a, b) for a, b in zip(got, got2))


def test_cuda_graph_replay_advances_epochs():
    """Every kernel family captured ONCE in a CUDA graph and replayed: inputs
    change on every replay (produced inside the graph from a device step
    counter), so a kernel that failed to advance its device epoch would pair
    new LL flags / semaphores with stale ones and return an older replay's
    sums.  f32 integer values: every reduction order is exact."""
    import torch
    from paper_2504_09014_b200 import Runtime, _lib, parse_plan
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200.plan import scale_plan
    n, cnt = 8, 40960 + 24
    w = world(n)
    dev = w.device(0)
    g = torch.Generator(device=dev).manual_seed(77)
    base = [torch.randint(-1000, 1001, (cnt,), device=dev, generator=g).float() for _ in range(n)]
    step = torch.zeros((), device=dev)
    xs = [torch.empty(cnt, device=dev) for _ in range(n)]
    algos = ["1pa", "2pa_ll", "2pa", "1pa_hb", "2pr"]
    outs = {a: [torch.empty(cnt, device=dev) for _ in range(n)] for a in algos}
    rs_out = [torch.empty(cnt // n, device=dev) for _ in range(n)]
    ag_out = [torch.empty(cnt, device=dev) for _ in range(n)]
    plans = {}
    for name in ("2pa_memory_n8_e64", "1pa_n8_e64"):
        with open(os.path.join(GOLD, "plans", name + ".json"), "rb") as f:
            rt = Runtime(scale_plan(parse_plan(f.read()), 640), w, dtype="f32")
        plans[name] = (rt, [torch.empty(rt.out_elems, device=dev) for _ in range(n)])

    def body():
        step.add_(1)
        for r in range(n):
            torch.add(base[r], step * (r + 1), out=xs[r])
        for a in algos:
            C.run("allreduce", xs, outs[a], cnt, "f32", _lib.ALGOS[a], w)
        C.run("reducescatter", xs, rs_out, cnt // n, "f32", _lib.ALGOS["rs_direct"], w)
        C.run("allgather", [x[:cnt // n] for x in xs], ag_out, cnt // n, "f32", _lib.ALGOS["allpairs_ag"], w)
        for rt, ys in plans.values():
            rt.run_raw([x[:rt.in_elems] for x in xs], ys)

    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        body()   # warm-up outside the graph (epoch 1 of every kernel)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(graph, stream=s):
            body()
    torch.cuda.synchronize(dev)
    total_base = torch.stack(base).sum(0)
    for rep in range(6):
        graph.replay()
        torch.cuda.synchronize(dev)
        k = float(step.item())
        assert k == rep + 2
        want = total_base + k * sum(r + 1 for r in range(n))
        for a in algos:
            for r in range(n):
                assert torch.equal(outs[a][r], want), (rep, a, r)
        for r in range(n):
            assert torch.equal(rs_out[r], want[r * (cnt // n):(r + 1) * (cnt // n)]), (rep, "rs", r)
            assert torch.equal(ag_out[r], torch.cat([xs[q][:cnt // n] for q in range(n)])), (rep, "ag", r)
        for name, (rt, ys) in plans.items():
            for r in range(n):
                assert torch.equal(ys[r], want[:rt.out_elems]), (rep, name, r)
    w.check_device_error()
    for rt, _ in plans.values():
        rt.check_device_error()
        rt.close()


def test_one_launch_per_rank_path(monkeypatch):
    """CF_SPLIT_GROUPS=1: ranks that share cuda:0 are launched one kernel per
    rank on their own streams -- the in-process multi-GPU path (per-device
    launches, .sys handshakes, no single-launch shortcuts) of
    make_world(1, 8) on an 8-GPU box, exercised on one GPU.  Every hand
    kernel, K13 and two DSL plans vs the oracle."""
    import torch
    from paper_2504_09014_b200 import Runtime, allreduce_add_rmsnorm, collective, make_world, parse_plan
    from paper_2504_09014_b200.plan import scale_plan
    monkeypatch.setenv("CF_SPLIT_GROUPS", "1")
    n = 4
    w = make_world(1, n, devices=[0] * n, spin_timeout_ms=10000, use_multicast="emulate",
                   nvls_bytes=64 << 10)
    try:
        # host tensors: the pipelined H2D / kernel / D2H path (windows of >= 32 MiB per rank)
        hins = gen_inputs(n, (36 << 20) // 4 + 5, "f32", "uniform", 64)
        got = collective("allreduce", [torch.from_numpy(x).pin_memory() for x in hins], w, dtype="f32",
                         algo="2pa")
        want = oracle.allreduce(hins, "2pa", "f32")
        for r in range(n):
            assert np.array_equal(got[r].numpy().view(np.uint32), want[r].view(np.uint32)), ("host", r)
        for elems, dtype in ((5000, "f32"), (70001, "bf16")):
            dist = "wide" if dtype == "f32" else "normal"
            ins = gen_inputs(n, elems, dtype, dist, 500 + elems % 11)
            for algo, var in ALGOS:
                got = collective("allreduce", ins, w, dtype=dtype, algo=algo, variant=var)
                want = oracle.allreduce(ins, _ORACLE_NAME.get(algo, algo), dtype)
                for r in range(n):
                    assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), (algo, var, r)
            assert len(w._rank_streams) == n   # the per-rank launch path is the one that ran
            for algo, var in (("ring_rs", ""), ("ring_rs", "ring"), ("rs_direct", "")):
                got = collective("reducescatter", ins, w, dtype=dtype, algo=algo, variant=var)
                want = oracle.reducescatter(ins, "ring_rs" if algo == "ring_rs" else "direct", dtype)
                for r in range(n):
                    assert np.array_equal(got[r].view(np.uint8), want[r].view(np.uint8)), (algo, r)
            for algo, var in (("allpairs_ag", ""), ("ring_ag", ""), ("ring_ag", "ring")):
                got = collective("allgather", ins, w, dtype=dtype, algo=algo, variant=var)
                for g, wnt in zip(got, oracle.allgather(ins)):
                    assert np.array_equal(g.view(np.uint8), wnt.view(np.uint8)), algo
        # K13, both algorithms (residual output is the oracle sum + residual, bit for bit)
        xs = gen_inputs(n, 8 * 512, "f32", "uniform", 61)
        res = gen_inputs(1, 8 * 512, "f32", "uniform", 62)[0]
        h = oracle.allreduce(xs, "oracle", "f32")[0]
        for algo in ("1pa_hb", "2pa"):
            xt = [torch.from_numpy(x).cuda().view(8, 512) for x in xs]
            rt = [torch.from_numpy(res).cuda().view(8, 512) for _ in range(n)]
            allreduce_add_rmsnorm(w, xt, rt, torch.ones(512, device="cuda"), eps=1e-6, algo=algo)
            w.synchronize()
            for r in range(n):
                assert np.array_equal(rt[r].cpu().numpy().reshape(-1).view(np.uint32),
                                      (h + res).astype(np.float32).view(np.uint32)), (algo, r)
        # DSL plans (HB and LL) through K10
        for name in ("2pa_memory_n4_e8", "1pa_n4_e8"):
            with open(os.path.join(GOLD, "plans", name + ".json"), "rb") as f:
                plan = scale_plan(parse_plan(f.read()), 512)
            rt_ = Runtime(plan, w, dtype="f32")
            pins = gen_inputs(n, rt_.in_elems, "f32", "int", 63)
            outs = rt_.execute(pins).outputs
            want = oracle.allreduce(pins, "oracle", "f32")
            for r in range(n):
                assert np.array_equal(outs[r][:len(want[r])], want[r]), (name, r)
            rt_.close()
        w.check_device_error()
    finally:
        w.close()


def test_bf16_allgather_matches_reference_digests():
    """libcf's bf16 AllGather (both algorithms) returns the bytes the reference
    itself produced for the same shards (tests/golden/ag_bf16.json)."""
    from inputs import ag_bf16_shards
    from paper_2504_09014_b200 import collective
    with open(os.path.join(GOLD, "ag_bf16.json")) as f:
        cases = json.load(f)
    for c in cases:
        shards = ag_bf16_shards(c["n"], c["count"], c["seed"])
        got = collective("allgather", shards, world(c["n"]), dtype="bf16", algo=c["algo"])
        assert [_digest(g) for g in got] == c["digests"], (c["n"], c["count"], c["algo"])


def test_lowp_allreduce_matches_reference_f32_path():
    """f16 / bf16 AllReduce on the GPU (every hand-kernel algorithm) returns
    the bytes of the reference's f32 path on the upcast inputs rounded once to
    the 2-byte type (tests/golden/lowp.json).  The 2pa *port* variant runs as
    a DSL plan whose intermediate buffers have the 2-byte type, so it rounds
    per plan op (checked against the oracle's plan interpreter in
    test_gpu_plans) and is not part of this round-once table."""
    from paper_2504_09014_b200 import collective
    with open(os.path.join(GOLD, "lowp.json")) as f:
        cases = [c for c in json.load(f) if c["variant"] != "port"]
    assert len(cases) == 120
    for c in cases:
        ins = gen_inputs(c["n"], c["elems"], c["dtype"], "normal", c["seed"])
        got = collective("allreduce", ins, world(c["n"]), dtype=c["dtype"], algo=c["algo"], variant=c["variant"])
        assert [_digest(g) for g in got] == c["digests"], (c["n"], c["elems"], c["dtype"], c["algo"], c["variant"])


def test_run_benchmark_measured_rows():
    """run_benchmark (cf/timing.py:331-349) on real GPUs: one measured row per
    (variant, size), LL variants skipped above their capacity, exactly one
    row per size marked as the selector's pick."""
    from paper_2504_09014_b200 import rows_to_csv, run_benchmark
    w = world(4, ll_max_bytes=1 << 16)
    sizes = [4096, 1 << 20]
    rows = run_benchmark("allreduce", sizes, w, iters=5)
    algos = {(r.algo, r.nbytes) for r in rows}
    assert ("1pa", 4096) in algos and ("1pa", 1 << 20) not in algos   # LL capacity
    assert ("2pa_port", 1 << 20) in algos and ("2pr", 1 << 20) in algos
    for nb in sizes:
        assert sum(r.selected for r in rows if r.nbytes == nb) == 1, nb
    assert all(r.latency_us > 0 and r.algobw_gbps > 0 for r in rows)
    ag = run_benchmark("allgather", [1 << 16], w, iters=5)
    assert [r.algo for r in ag] == ["allpairs_ag", "ring_ag"] and sum(r.selected for r in ag) == 1
    assert rows_to_csv(rows).count("\n") == len(rows) + 1


def test_simulate_timed_measures_a_plan():
    """simulate_timed (cf/timing.py:295-298) runs the plan on the GPUs: the
    makespan is a measured latency, one event per program."""
    from paper_2504_09014_b200 import CostParams, parse_plan, simulate_timed
    with open(os.path.join(GOLD, "plans", "2pa_memory_n8_e64.json"), "rb") as f:
        plan = parse_plan(f.read())
    tr = simulate_timed(plan, world(8), CostParams(), iters=5)
    assert 0 < tr.makespan < 1e-3
    assert len(tr.events) == len(plan.programs) and tr.link_bytes() == 0


def test_host_buffer_allreduce_every_algorithm():
    """Host tensors through collective() for every AllReduce algorithm and the
    selector's pick: same bits as the device-buffer call (the host path copies
    around the same kernels; only 2pa pipelines windows)."""
    import torch
    from paper_2504_09014_b200 import collective
    w = world(8)
    for elems in (5000, (3 << 20) + 7):
        g = torch.Generator().manual_seed(elems)
        host = [(torch.randn(elems, generator=g) * 4).to(torch.bfloat16).pin_memory() for _ in range(8)]
        for algo, var in ALGOS + [(None, "")]:
            if (algo == "1pa" or var == "ll") and elems * 2 > (4 << 20):   # LL capacity
                continue
            got = collective("allreduce", host, w, dtype="bf16", algo=algo, variant=var)
            dev = collective("allreduce", [h.cuda() for h in host], w, dtype="bf16", algo=algo, variant=var)
            for r in range(8):
                assert not got[r].is_cuda
                assert torch.equal(got[r].view(torch.int16), dev[r].cpu().view(torch.int16)), (elems, algo, var, r)


def test_tune_installs_measured_selection():
    """World.tune times every AllReduce candidate per size on the GPU, installs
    the fastest-per-size table (cfCommSetSelection), AUTO and
    Selector(measured=True) follow it, results stay exact; an empty table
    restores the built-in one."""
    import ctypes
    from paper_2504_09014_b200 import Selector, _lib, collective
    from paper_2504_09014_b200 import tune as T
    from paper_2504_09014_b200.collectives import _COLL, _algo_id
    from paper_2504_09014_b200.dtypes import CODES
    n = 8
    w = world(n)
    sizes = [4096, 65536, 1 << 20, 4 << 20]

    def pick(nb):
        algo = ctypes.c_int()
        _lib.check(_lib.lib().cfSelectAlgorithm(w.comm, _COLL["allreduce"], nb, CODES["bf16"],
                                                ctypes.byref(algo)))
        return algo.value

    try:
        res = w.tune(sizes=sizes, iters=5)
        table = res["table"]
        assert table and table[-1][0] == sizes[-1]
        for i, nb in enumerate(sizes):   # the installed pick is the fastest measured at that size
            best = min((t[i], a) for a, t in res["times"].items() if t[i] is not None)[1]
            assert pick(nb) == T.algo_id(best), (nb, best)
            d = Selector(measured=True).select("allreduce", nb, w.topology, world=w, dtype="bf16")
            assert _algo_id("allreduce", d.name, d.variant) == pick(nb)
        rng = np.random.default_rng(3)
        for nb in sizes:   # AUTO on the tuned bf16 table: integer-valued sums are exact
            ins = [(rng.integers(-8, 8, nb // 2).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
                   for _ in range(n)]
            got = collective("allreduce", ins, w, dtype="bf16", selector=Selector(measured=True))
            want = oracle.allreduce(ins, "oracle", "bf16")
            for g, x in zip(got, want):
                assert np.array_equal(g, x), nb
    finally:
        T.install(w.comm, "allreduce", "bf16", [])
    assert pick(4096) == _lib.ALGOS["1pa_hb"]   # the built-in co-resident table again
