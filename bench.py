"""Benchmark of the collective hot path (BASELINE.json metric: AllReduce busbw
GB/s & latency vs message size, % of NVLink peak).

N=1 (default): the 8-rank AllReduce runs with all 8 ranks co-resident on one
B200 (the reference's own setting is 8 simulated ranks in one process, C1).
Every "peer" access is then HBM instead of NVLink, so the roofline of the
dominant kernel is the measured HBM copy bandwidth.  Headline workload: C4
shape, bf16 two-shot, 256 MiB per rank; the sweep adds latency/busbw from 1 KiB
to 1 GiB for the selected algorithm and the C1 config (fp32 1 MiB one-shot LL).

N>1 (torchrun): one rank per GPU over NVLink (one-process-per-GPU mode).

--impl reference: the reference's CPU path for the same workload, i.e. the
oracle port (oracle/, C + pthreads, every host core) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30
N_SIM = 8                      # simulated ranks at N=1
HEAD_BYTES = 256 * MiB         # per-rank message of the headline line
HEAD_DTYPE = "bf16"
METRIC = "AllReduce busbw GB/s & latency vs msg size at 8xB200 (vs NCCL, % of 900 GB/s)"


def busbw(nbytes, seconds, n):
    return nbytes / seconds * 2 * (n - 1) / n / 1e9


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi style clock/throttle sampling during the timed region (NVML)."""

    def __init__(self, dev=0, period=0.002):
        self.dev, self.period = dev, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._nv = pynvml
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._nv = None
        return self

    def _run(self):
        nv = self._nv
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join(timeout=1)

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU arms

def bench_inputs(n, elems, seed):
    """Per-rank bf16 inputs of the headline workload as uint16 patterns: finite
    values of both signs with magnitudes in [2^-31, 2^32) (fast to generate at
    256 MiB per rank; the CPU step's cost does not depend on the values)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        b = rng.integers(0, 1 << 16, elems, dtype=np.uint16)
        out.append((b & np.uint16(0x80FF)) | np.uint16(0x3000) | ((b >> np.uint16(1)) & np.uint16(0x0F00)))
    return out


def cpu_reference_steps(ins, dtype, algo, steps, budget_s=None):
    """Time `steps` full steps of the reference algorithm on the host: the
    oracle port (oracle/, C + pthreads over every host core) over every
    rank's whole message -- the reference computes every rank's output of the
    AllReduce (cf/executor.py:135-178), so one step is the whole job."""
    from oracle import oracle
    ts = []
    t_end = None if budget_s is None else time.perf_counter() + budget_s
    for _ in range(steps):
        t0 = time.perf_counter()
        oracle.allreduce(ins, algo, dtype, nthreads=0)
        ts.append(time.perf_counter() - t0)
        if t_end is not None and time.perf_counter() > t_end:
            break
    return ts


def cpu_baseline(n, full_elems, dtype, algo, budget_s=15.0):
    """The reference's CPU path on the SAME workload (n ranks x full_elems),
    a bounded number of steps (about budget_s of CPU work)."""
    from oracle import oracle
    es = 2 if dtype in ("bf16", "f16") else 4
    ins = bench_inputs(n, full_elems, 77)
    cpu_reference_steps(ins, dtype, algo, 1)            # warm-up (page faults)
    times = cpu_reference_steps(ins, dtype, algo, 20, budget_s)
    t = float(np.median(times))
    return {"value": round(busbw(full_elems * es, t, n), 4), "unit": "GB/s",
            "cores": oracle.max_threads(), "kind": "port",
            "sample": f"{len(times)} full steps of the {n}-rank {dtype} AllReduce ({algo} order), "
                      f"{full_elems * es // MiB} MiB per rank (the bench workload itself); "
                      f"median {t * 1e3:.1f} ms/step"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle
    es = 2
    full = HEAD_BYTES // es
    # the cf arm's rank count: 8 simulated ranks at N=1, one rank per GPU at N>1
    nr = args.gpus if args.gpus > 1 else N_SIM
    ins = bench_inputs(nr, full, 78)
    cpu_reference_steps(ins, HEAD_DTYPE, "2pa", max(1, args.warmup))
    ts = cpu_reference_steps(ins, HEAD_DTYPE, "2pa", args.steps)
    t = float(np.mean(ts))
    # the cf arm's definition: at N>1 the aggregate over the N ranks' GPUs
    # (N x busbw of the same-sized job), at N=1 the one GPU's busbw
    v = busbw(HEAD_BYTES, t, nr) * (args.gpus if args.gpus > 1 else 1)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": HEAD_DTYPE, "data": "synthetic",
            "config": {"workload": f"AllReduce {HEAD_DTYPE} {nr} ranks, {HEAD_BYTES // MiB} MiB "
                                   "per rank (C4 shape), two-shot (2pa) order",
                       "sample_bytes_per_rank": HEAD_BYTES, "same_config": True},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": oracle.max_threads(),
                             "kind": "port",
                             "sample": f"the full workload every step: {nr} x {HEAD_BYTES // MiB} MiB "
                                       "(oracle/ C port of the reference arithmetic, pthreads)"},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- GPU arm

def time_graph(dev, fn, iters, warmup, flush=None, reps=3):
    """Device time per call of `fn`: `iters` calls captured in one CUDA graph
    (no host launch overhead), replayed `reps` times (best), CUDA events on the
    replay stream.  With `flush`, each call is preceded by an L2 flush (memset
    of a buffer larger than L2) and the time of a flush-only graph is
    subtracted."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)

    def capture(with_fn):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(iters):
                    if flush is not None:
                        flush.zero_()
                    if with_fn:
                        fn()
        torch.cuda.synchronize(dev)
        return g

    def replay(g):
        g.replay()
        torch.cuda.synchronize(dev)
        best = None
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            st = torch.cuda.current_stream(dev)
            e0.record(st)
            g.replay()
            e1.record(st)
            e1.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best = t if best is None else min(best, t)
        return best

    t = replay(capture(True))
    if flush is not None:
        t -= replay(capture(False))
    return max(t, 0.0) / iters


def time_coll(world, kind, send, recv, count, dtype, algo, iters, warmup, flush=None, reps=3):
    """time_graph of one libcf collective call on every rank."""
    from paper_2504_09014_b200 import collectives as C
    t = time_graph(world.device(0), lambda: C.run(kind, send, recv, count, dtype, algo, world),
                   iters, warmup, flush, reps)
    world.check_device_error()
    return t



def algo_id(name):
    """libcf algorithm id; "<ring algo>+ring" = the literal ring transport (cf.h CF_ALGO_RING_LINKS)."""
    from paper_2504_09014_b200 import _lib
    base, _, links = name.partition("+")
    return _lib.ALGOS[base] | (_lib.CF_ALGO_RING_LINKS if links else 0)

def time_plan(rt, send, recv, iters, warmup, flush, reps=3):
    """time_graph of one plan execution (K10) on every rank."""
    t = time_graph(rt.world.device(0), lambda: rt.run_raw(send, recv), iters, warmup, flush, reps)
    rt.check_device_error()
    return t


def run_ag_rs(w, flush, send, recv):
    """C2-style AllGather (output bytes S_out) and ReduceScatter (input bytes S)
    in bf16 on 8 co-resident ranks, every algorithm; busbw = algbw (n-1)/n."""
    from paper_2504_09014_b200 import _lib
    n = w.num_ranks
    rows = []
    for nb in [KiB << (2 * i) for i in range(11)]:   # 1 KiB .. 1 GiB (C2's sweep), x4
        row = {"bytes": nb}
        shard = nb // 2 // n
        if shard == 0:
            continue
        iters = 20 if nb <= 16 * MiB else 5
        fl = flush if nb < 64 * MiB else None
        for name in ("allpairs_ag", "ring_ag", "ring_ag+ring"):
            t = time_coll(w, "allgather", [s[:shard] for s in send], [r[:shard * n] for r in recv], shard,
                          "bf16", algo_id(name), iters, 3, fl)
            row["ag_" + name] = {"us": round(t * 1e6, 2), "busbw": round(nb / t / 1e9 * (n - 1) / n, 2)}
        for name in ("rs_direct", "ring_rs", "ring_rs+ring"):
            t = time_coll(w, "reducescatter", [s[:shard * n] for s in send], [r[:shard] for r in recv], shard,
                          "bf16", algo_id(name), iters, 3, fl)
            row["rs_" + name] = {"us": round(t * 1e6, 2), "busbw": round(nb / t / 1e9 * (n - 1) / n, 2)}
        rows.append(row)
    return {"config": "C2/RS: AllGather (S = output bytes) and ReduceScatter (S = input bytes), bf16, "
                      "8 co-resident ranks; ring_ag / ring_rs = the reference's ring algorithms (same bytes / "
                      "ring accumulation order) on the all-pairs transport, '+ring' = the literal ring kernels",
            "rows": rows}


def run_fused(w, flush):
    """K13 vs the unfused composition (AllReduce, then one batched residual add
    and one batched RMSNorm over all ranks' rows) at the C5 shapes."""
    import torch
    import torch.nn.functional as F
    from paper_2504_09014_b200 import _lib, allreduce_add_rmsnorm
    from paper_2504_09014_b200 import collectives as C
    n, dev, hidden = w.num_ranks, w.device(0), 8192
    rows = []
    for b in (1, 4, 16, 64, 256):
        X = torch.randn(n, b, hidden, device=dev).to(torch.bfloat16)
        R = torch.randn(n, b, hidden, device=dev).to(torch.bfloat16)
        H, RO, Y = torch.empty_like(X), torch.empty_like(X), torch.empty_like(X)
        wt = torch.ones(hidden, device=dev, dtype=torch.bfloat16)
        xs, rs, ros, ys = list(X), list(R), list(RO), list(Y)
        hs = list(H)

        def fused():
            allreduce_add_rmsnorm(w, xs, rs, wt, eps=1e-6, resid_out=ros, norm_out=ys)

        def unfused():
            C.run("allreduce", xs, hs, b * hidden, "bf16", _lib.ALGOS["auto"], w)
            torch.add(H, R, out=RO)
            F.rms_norm(RO, (hidden,), wt, 1e-6)

        tf = time_graph(dev, fused, 20, 3, flush)
        tu = time_graph(dev, unfused, 20, 3, flush)
        w.check_device_error()
        rows.append({"batch": b, "bytes": b * hidden * 2, "fused_us": round(tf * 1e6, 2),
                     "unfused_us": round(tu * 1e6, 2), "speedup": round(tu / tf, 2) if tf else None})
    return {"config": "C5 consumer: AllReduce + residual add + RMSNorm [b, 8192] bf16, fused K13 vs "
                      "libcf AllReduce + torch add + torch rms_norm (batched over ranks), 8 co-resident ranks",
            "rows": rows}


def run_gpu_arm(args):
    import torch
    from paper_2504_09014_b200 import _lib, make_world
    from paper_2504_09014_b200 import collectives as C
    from paper_2504_09014_b200.dtypes import torch_dtype

    if args.gpus > 1 or os.environ.get("CF_BENCH_MULTI"):
        # CF_BENCH_MULTI=1 with --gpus 1: the one-process-per-GPU code path
        # (and its NCCL arms) as a single rank -- a path check on 1-GPU boxes
        return run_multi_gpu(args)
    n = N_SIM
    w = make_world(1, n, devices=[0] * n)
    dev = w.device(0)
    es = 2
    count = HEAD_BYTES // es
    tdt = torch_dtype(HEAD_DTYPE)
    gen = torch.Generator(device=dev)
    send = []
    for r in range(n):
        gen.manual_seed(20250409 + 4000 + r)
        send.append(torch.randn(count, device=dev, dtype=torch.float32, generator=gen).to(tdt))
    recv = [torch.empty_like(s) for s in send]
    algo_name = C.select_algorithm("allreduce", HEAD_BYTES, w.topology, selector=C.Selector(measured=True),
                                   world=w, dtype=HEAD_DTYPE)
    algo = _lib.ALGOS["2pa_ll" if algo_name.variant == "ll" else algo_name.name]
    # parity spot check of the headline config (vs the size-independent property:
    # every rank holds identical bits, and a sampled slice equals the oracle)
    C.run("allreduce", send, recv, count, HEAD_DTYPE, algo, w)
    w.synchronize()
    for r in range(1, n):
        assert torch.equal(recv[0], recv[r]), "ranks disagree"
    from oracle import oracle
    sl = slice(count // 3, count // 3 + 4096)
    host = [s[sl].view(torch.int16).cpu().numpy().view(np.uint16) for s in send]
    # 2pa order: chunk owner first; the slice lies in chunk count//3 // cs
    cs = -(-count // n)
    lead = (count // 3) // cs
    assert ((count // 3 + 4096 - 1) // cs) == lead
    want = oracle.reduce_ordered("bf16", host, [lead] + [p for p in range(n) if p != lead])
    got = recv[0][sl].view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(got, want), "headline parity spot check failed"

    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        C.run("allreduce", send, recv, count, HEAD_DTYPE, algo, w)
    w.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize(dev)
        t_start = time.perf_counter()
        for a, b in ev:
            a.record(stream)
            C.run("allreduce", send, recv, count, HEAD_DTYPE, algo, w)
            b.record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t_start
    w.check_device_error()
    per = [a.elapsed_time(b) / 1e3 for a, b in ev]
    t = float(np.sum(per)) / args.steps
    value = busbw(HEAD_BYTES, t, n)
    hbm, peak_kind = load_peaks()
    alg_bytes = 2 * n * HEAD_BYTES                 # every rank's input read once + output written once
    achieved = alg_bytes / t / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": None,
                "peak_kind": peak_kind, "kernel": "pull_reduce_kernel<bf16,8> (K3 two-shot)",
                "algorithmic_bytes_per_launch": alg_bytes}
    prof = os.path.join(ROOT, "profiles", "headline_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            roofline["traffic"] = json.load(f).get("dram_bytes_per_launch")

    # e2e: pinned host inputs -> public collective() -> pinned host outputs
    host_in = [s.cpu().pin_memory() for s in send]
    host_out = [torch.empty_like(h).pin_memory() for h in host_in]
    e2e_times = []
    for it in range(max(2, min(args.steps, 5)) + 1):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        outs = C.collective("allreduce", host_in, w, algo="2pa", outputs=host_out)
        torch.cuda.synchronize(dev)
        if it > 0:
            e2e_times.append(time.perf_counter() - t0)
    te = float(np.mean(e2e_times))
    e2e = {"value": round(busbw(HEAD_BYTES, te, n), 3), "unit": "GB/s",
           "h2d_bytes_per_step": n * HEAD_BYTES, "d2h_bytes_per_step": n * HEAD_BYTES,
           "ms_per_step": round(te * 1e3, 3), "api": "collective('allreduce', pinned host tensors)"}
    del outs

    sweep = []
    tuned = None
    if not args.no_sweep:
        # measured selection on this box (World.tune): AUTO rows of the sweep follow it
        tr = w.tune(kind="allreduce", dtype="bf16", iters=10)
        tuned = {"table": [[int(b), a] for b, a in tr["table"]],
                 "note": "fastest AllReduce per size, CUDA graphs on this box (World.tune -> cfCommSetSelection); "
                         "the sweep's 'auto' rows use it"}
        sweep = run_sweep(w, args)
    cpu = cpu_baseline(n, count, HEAD_DTYPE, "2pa")
    line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": HEAD_DTYPE,
            "data": "synthetic",
            "config": {"workload": f"AllReduce {HEAD_DTYPE}, {n} ranks co-resident on one B200 "
                                   f"(simulated ranks as in C1), {HEAD_BYTES // MiB} MiB per rank (C4 shape)",
                       "ranks": n, "ranks_per_gpu": n, "bytes_per_rank": HEAD_BYTES,
                       "algo": _lib.ALGO_NAMES[algo], "parallelism": "8 ranks / 1 GPU",
                       "l2": "inputs larger than L2 (8 x 256 MiB)"},
            "latency_us": round(t * 1e6, 2), "algbw_gbs": round(HEAD_BYTES / t / 1e9, 2),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps, "clocks": clk.summary(),
            "wall_s_timed": round(wall, 4), "tuned_selection": tuned, "sweep": sweep}
    print(json.dumps(line))
    w.close()
    return 0


def run_sweep(w, args):
    """Latency / busbw per size for the selector's pick and each algorithm
    (8 co-resident ranks), L2 flushed between timed iterations below 64 MiB."""
    import torch
    from paper_2504_09014_b200 import _lib
    from paper_2504_09014_b200 import collectives as C
    n = w.num_ranks
    dev = w.device(0)
    out = []
    flush = torch.empty(256 * MiB, dtype=torch.uint8, device=dev)
    sizes = [1 * KiB << (2 * i) for i in range(0, 11)]  # 1 KiB .. 1 GiB, x4
    big = max(sizes)
    maxe = big // 2
    send = [torch.randn(maxe, device=dev).to(torch.bfloat16) for _ in range(n)]
    recv = [torch.empty_like(s) for s in send]
    ll_max = w.config.ll_max_bytes or 4 * MiB
    for nb in sizes:
        count = nb // 2
        row = {"bytes": nb}
        for name in ("auto", "1pa", "2pa_ll", "2pa", "1pa_hb", "2pr", "2pr+ring"):
            if name in ("1pa", "2pa_ll") and nb > ll_max:
                continue
            if name == "1pa_hb" and nb > 64 * MiB:
                continue
            aid = algo_id(name)
            iters = 20 if nb <= 16 * MiB else 5
            t = time_coll(w, "allreduce", [s[:count] for s in send], [r[:count] for r in recv],
                          count, "bf16", aid, iters, 3, flush if nb < 64 * MiB else None)
            row[name] = {"us": round(t * 1e6, 2), "busbw": round(busbw(nb, t, n), 2)}
        out.append(row)
    # C5: Llama-70B TP-decode AllReduce [b, 8192] bf16 through lowered reference
    # plans (tests/golden/plans, generated by the reference's lower()), K10.
    from paper_2504_09014_b200 import Runtime, parse_plan
    from paper_2504_09014_b200.plan import scale_plan
    c5 = []
    for pname in ("2pa_memory_n8_e64", "2pa_ll_n8_e64", "1pa_n8_e64"):
        with open(os.path.join(ROOT, "tests", "golden", "plans", pname + ".json"), "rb") as f:
            base = parse_plan(f.read())
        for b in (1, 4, 16, 64, 256):
            plan = scale_plan(base, 128 * b)
            rt = Runtime(plan, w, dtype="bf16")
            xs = [torch.randn(rt.in_elems, device=dev).to(torch.bfloat16) * 0.02 for _ in range(n)]
            ys = [torch.empty(rt.out_elems, device=dev, dtype=torch.bfloat16) for _ in range(n)]
            t = time_plan(rt, xs, ys, 20, 3, flush)
            nb = rt.in_elems * 2
            c5.append({"plan": pname.split("_n8")[0], "batch": b, "bytes": nb,
                       "us": round(t * 1e6, 2), "busbw": round(busbw(nb, t, n), 2),
                       "device_ops": rt.n_device_ops})
            rt.close()
    out.append({"config": "C5 Llama-70B TP decode AllReduce via DSL plans (K10), bf16, "
                          "8 co-resident ranks", "rows": c5})
    out.append(run_fused(w, flush))
    out.append(run_ag_rs(w, flush, send, recv))
    # C3: fp16 small-message AllReduce, LL one-shot vs the selector's pick
    c3 = []
    for nb in (KiB, 4 * KiB, 16 * KiB, 64 * KiB, 256 * KiB, MiB):
        cnt = nb // 2
        xs = [s_[:cnt].view(torch.float16) for s_ in send]
        ys = [r_[:cnt].view(torch.float16) for r_ in recv]
        row = {"bytes": nb}
        for name in ("1pa", "auto"):
            t = time_coll(w, "allreduce", xs, ys, cnt, "f16", _lib.ALGOS[name], 20, 3, flush)
            row[name] = {"us": round(t * 1e6, 2), "busbw": round(busbw(nb, t, n), 2)}
        c3.append(row)
    out.append({"config": "C3 AllReduce fp16 1 KiB-1 MiB, LL one-shot (1pa) and the selector's pick, "
                          "8 co-resident ranks", "rows": c3})
    # C1: fp32 1 MiB one-shot LL (8 simulated ranks)
    c1 = [torch.randn(MiB // 4, device=dev) for _ in range(n)]
    c1o = [torch.empty_like(x) for x in c1]
    t = time_coll(w, "allreduce", c1, c1o, MiB // 4, "f32", _lib.ALGOS["1pa"], 50, 5, flush)
    out.append({"config": "C1 AllReduce fp32 1 MiB one-shot LL, 8 co-resident ranks",
                "us": round(t * 1e6, 2), "busbw": round(busbw(MiB, t, n), 2)})
    return out


def nccl_setup(dev, rank, world):
    """NCCL 2.28 through ctypes (scripts/nccl_ctypes.py): the comparison
    baseline only.  Returns (Nccl, None) or (None, reason).  Ranks sharing
    one GPU (CF_BENCH_ONE_GPU) cannot run NCCL (duplicate GPU)."""
    import torch.distributed as dist
    if os.environ.get("CF_BENCH_ONE_GPU"):
        return None, "ranks share cuda:0 (CF_BENCH_ONE_GPU): NCCL needs one GPU per rank"
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"   # no version banner on stdout: one JSON line only
    try:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from nccl_ctypes import Nccl
        uid = [Nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        nc = Nccl(world, rank, uid[0])
        return nc, None
    except Exception as e:   # comparison only: report, never fail the bench
        return None, f"{type(e).__name__}: {e}"[:200]


def multi_parity(comm, dev, rank, world, nvls, sym_mode=-1):
    """Before timing: libcf's NVLink results against the CPU oracle, bit for
    bit (bf16, ragged size, seeded inputs regenerated on every rank): 1pa,
    2pa_ll, 2pa, direct and ring AllGather, both ReduceScatters, and NVLS
    (switch order is unspecified: SURVEY §8(c) tolerance).  Returns
    {check: ok} agreed over ranks (all ranks must pass)."""
    import torch
    import torch.distributed as dist
    from oracle import oracle
    from inputs import gen_inputs
    from paper_2504_09014_b200.dtypes import torch_dtype

    def dev_t(a):
        return torch.from_numpy(a.view(np.int16)).to(dev).view(torch_dtype("bf16"))

    def host(t):
        return t.view(torch.int16).cpu().numpy().view(np.uint16)

    res = {}
    elems = 8 * 4099 + 3     # ragged: chunk bounds off the vector grid
    ins = gen_inputs(world, elems, "bf16", "normal", 20250409 + 7)
    x = dev_t(ins[rank])
    y = torch.empty_like(x)
    comm.register(x)
    comm.register(y)
    algos = [("1pa", "1pa"), ("2pa_ll", "2pa"), ("2pa", "2pa"), ("2pr", "2pr")]
    for name, oname in algos:
        try:
            y.zero_()
            if name == "2pa_ll":
                comm.all_reduce(x, y, algo="2pa", variant="ll")
            else:
                comm.all_reduce(x, y, algo=name)
            torch.cuda.synchronize(dev)
            comm.check_device_error()
            res["allreduce_" + name] = bool(np.array_equal(host(y), oracle.allreduce(ins, oname, "bf16")[rank]))
        except Exception as e:
            res["allreduce_" + name] = f"{type(e).__name__}: {e}"[:160]
    comm.deregister(x)
    comm.deregister(y)
    if sym_mode >= 0:
        # symmetric buffers (no registration): two-shot, and switch_2pa in
        # place -- exact in the reference switch order when emulated, SURVEY
        # §8(c) tolerance with a real multicast object (order unspecified)
        xs = comm.alloc_symmetric(elems, torch_dtype("bf16"))
        ys = comm.alloc_symmetric(elems, torch_dtype("bf16"))
        xs.copy_(x)
        for name in ("2pa",) + (("switch_2pa",) if nvls else ()):
            key = f"allreduce_{name}_symmetric"
            try:
                ys.zero_()
                comm.all_reduce(xs, ys, algo=name)
                torch.cuda.synchronize(dev)
                comm.check_device_error()
                want = oracle.allreduce(ins, name, "bf16")[rank]
                if name == "2pa" or sym_mode == 2:
                    res[key] = bool(np.array_equal(host(ys), want))
                else:
                    w32 = (want.astype(np.uint32) << 16).view(np.float32)
                    g32 = (host(ys).astype(np.uint32) << 16).view(np.float32)
                    sabs = np.sum([np.abs((a.astype(np.uint32) << 16).view(np.float32)) for a in ins], axis=0)
                    tol = 2.0 ** -8 * np.abs(w32) + (world - 1) * 2.0 ** -24 * sabs
                    res[key] = bool(np.all(np.abs(g32 - w32) <= tol))
            except Exception as e:
                res[key] = f"{type(e).__name__}: {e}"[:160]
                comm.clear_device_error()
        comm.free_symmetric(xs)
        comm.free_symmetric(ys)
    # AllGather (bit-exact data movement, random 16-bit patterns incl. NaNs)
    shard = 4099
    sh = [a[:shard] for a in gen_inputs(world, shard, "bf16", "normal", 20250409 + 8)]
    xs = dev_t(sh[rank])
    ys = torch.empty(shard * world, device=dev, dtype=xs.dtype)
    comm.register(xs)
    comm.register(ys)
    for name in ("allpairs_ag", "ring_ag", "ring_ag+ring"):
        try:
            ys.zero_()
            comm.all_gather(xs, ys, algo=name.split("+")[0], variant="ring" if "+" in name else "")
            torch.cuda.synchronize(dev)
            res["allgather_" + name] = bool(np.array_equal(host(ys), oracle.allgather(sh)[rank]))
        except Exception as e:
            res["allgather_" + name] = f"{type(e).__name__}: {e}"[:160]
    comm.deregister(xs)
    comm.deregister(ys)
    # ReduceScatter (reference orders: rs_direct = owner first, ring_rs = ring order)
    shard = 4100   # n * shard divides 2n: ring_rs needs no padding
    rin = gen_inputs(world, shard * world, "bf16", "normal", 20250409 + 9)
    xr = dev_t(rin[rank])
    yr = torch.empty(shard, device=dev, dtype=xr.dtype)
    comm.register(xr)
    comm.register(yr)
    for name in ("rs_direct", "ring_rs", "ring_rs+ring"):
        try:
            comm.reduce_scatter(xr, yr, algo=name.split("+")[0], variant="ring" if "+" in name else "")
            torch.cuda.synchronize(dev)
            want = oracle.reducescatter(rin, "2pa" if name == "rs_direct" else "ring_rs", "bf16")[rank]
            res["reducescatter_" + name] = bool(np.array_equal(host(yr), want[:shard]))
        except Exception as e:
            res["reducescatter_" + name] = f"{type(e).__name__}: {e}"[:160]
    comm.deregister(xr)
    comm.deregister(yr)
    allres = [None] * world
    dist.all_gather_object(allres, res)
    return {k: all(r.get(k) is True for r in allres) if all(isinstance(r.get(k), bool) for r in allres)
            else next(r[k] for r in allres if r.get(k) is not True) for k in res}


def multi_sweep(comm, dev, rank, world, send, recv, nvls, nvls_kind, nccl, big=GiB, sym_mode=-1):
    """N>1: latency / busbw over sizes -- libcf (CUDA graph and eager) next to
    NCCL 2.28 (comparison baseline only, never part of the product path) in a
    CUDA graph on default buffers AND on symmetric windows (ncclMemAlloc +
    ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)); the better NCCL mode is
    the bar.  L2 flushed between timed iterations below 64 MiB (both arms).
    Per-rank times; the caller takes the max over ranks."""
    import torch
    from paper_2504_09014_b200 import _lib
    rows = []
    # 1 KiB .. 1 GiB (x4); buffers of the largest size from the symmetric heap
    # (or registered once when there is none)
    if sym_mode >= 0:
        bs = comm.alloc_symmetric(big // 2, torch.bfloat16)
        br = comm.alloc_symmetric(big // 2, torch.bfloat16)
        bs.copy_(torch.randn(big // 2, device=dev).to(torch.bfloat16))
    else:
        bs = torch.randn(big // 2, device=dev).to(torch.bfloat16)
        br = torch.empty_like(bs)
        comm.register(bs)
        comm.register(br)
    flush = torch.empty(256 * MiB, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)
    sym = None
    if nccl is not None:
        try:   # symmetric windows, same size on every rank (collective calls)
            sp, rp = nccl.mem_alloc(big), nccl.mem_alloc(big)
            nccl.register_symmetric(sp, big)
            nccl.register_symmetric(rp, big)
            sym = (sp, rp)
        except Exception as e:
            rows.append({"bytes": 0, "kind": "nccl_symmetric", "error": f"{type(e).__name__}: {e}"[:200]})
        nz_s, nz_r = bs.clone(), torch.empty_like(br)   # NCCL's default (plain) buffers

    def eager(fn, iters):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            fn()
        e1.record(st)
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3 / iters

    def cur():
        return torch.cuda.current_stream(dev).cuda_stream

    def nccl_times(kind, nbytes_in, nbytes_out, iters, fl):
        """NCCL graph time on plain and on symmetric buffers (elements: 2 B)."""
        out = {}
        fn = {"allreduce": lambda s, r: nccl.all_reduce(s, r, nbytes_in // 2, "bf16", cur()),
              "allgather": lambda s, r: nccl.all_gather(s, r, nbytes_in // 2, "bf16", cur()),
              "reducescatter": lambda s, r: nccl.reduce_scatter(s, r, nbytes_out // 2, "bf16", cur())}[kind]
        out["nccl_graph_s"] = time_graph(dev, lambda: fn(nz_s.data_ptr(), nz_r.data_ptr()), iters, 3, fl)
        if sym is not None:
            out["nccl_sym_graph_s"] = time_graph(dev, lambda: fn(sym[0], sym[1]), iters, 3, fl)
        return out

    for nb in [KiB << (2 * i) for i in range(11)]:
        if nb > big:
            break
        cnt = nb // 2
        x, y = bs[:cnt], br[:cnt]
        iters = 50 if nb <= MiB else 10
        fl = flush if nb < 64 * MiB else None
        row = {"bytes": nb, "kind": "allreduce",
               "cf_graph_s": time_graph(dev, lambda: comm.all_reduce(x, y, algo="auto"), iters, 3, fl),
               "cf_eager_s": eager(lambda: comm.all_reduce(x, y, algo="auto"), iters)}
        # every algorithm on its own (the NVLink crossover table of the selector)
        for name, var, cap in (("1pa", "", 2 * MiB), ("2pa", "ll", 2 * MiB), ("2pa", "", None),
                               ("switch_2pa", "", None)):
            if (cap is not None and nb > cap) or (name == "switch_2pa" and not nvls):
                continue
            key = f"cf_{name}{'_' + var if var else ''}_graph_s"
            row[key] = time_graph(dev, lambda: comm.all_reduce(x, y, algo=name, variant=var), iters, 3, fl)
        if nccl is not None:
            row.update(nccl_times("allreduce", nb, nb, iters, fl))
        rows.append(row)
    # C2 / RS: AllGather (S = output bytes) and ReduceScatter (S = input bytes)
    for nb in [KiB << (2 * i) for i in range(11)]:
        if nb > big or nb // 2 < world:
            continue
        cnt = nb // 2 // world * world
        shard = cnt // world
        iters = 50 if nb <= MiB else 10
        fl = flush if nb < 64 * MiB else None
        for kind in ("allgather", "reducescatter"):
            if kind == "allgather":
                x, y = bs[:shard], br[:cnt]
                fn = lambda: comm.all_gather(x, y, algo="auto")  # noqa: E731
            else:
                x, y = bs[:cnt], br[:shard]
                fn = lambda: comm.reduce_scatter(x, y, algo="auto")  # noqa: E731
            row = {"bytes": cnt * 2, "kind": kind, "cf_graph_s": time_graph(dev, fn, iters, 3, fl)}
            if nccl is not None:
                row.update(nccl_times(kind, (shard if kind == "allgather" else cnt) * 2,
                                      (cnt if kind == "allgather" else shard) * 2, iters, fl))
            rows.append(row)
    # CTA budget sweep of the two-shot kernel at large sizes (default budget
    # one rank per GPU: 64 CTAs; the driver's 8-GPU run measures the choice)
    for nb in (64 * MiB, 256 * MiB):
        if nb > big:
            continue
        x, y = bs[:nb // 2], br[:nb // 2]
        row = {"bytes": nb, "kind": "allreduce", "budget_sweep": True}
        for ctas in (16, 32, 64, 128):
            comm.set_cta_budget(ctas, "2pa")
            row[f"cf_2pa_ctas{ctas}_graph_s"] = time_graph(dev, lambda: comm.all_reduce(x, y, algo="2pa"), 10, 3)
        comm.set_cta_budget(0, "2pa")
        rows.append(row)
    if nvls:
        for nb in [MiB << (2 * i) for i in range(6)]:
            if nb > big:
                break
            cnt = nb // 2
            x, y = bs[:cnt], br[:cnt]
            rows.append({"bytes": nb, "kind": nvls_kind, "cf_graph_s": time_graph(
                dev, lambda: comm.all_reduce(x, y, algo="switch_2pa"), 10, 3, flush if nb < 64 * MiB else None)})
    if sym_mode >= 0:
        comm.free_symmetric(bs)
        comm.free_symmetric(br)
    else:
        comm.deregister(bs)
        comm.deregister(br)
    del bs, br
    # C5: Llama-70B TP decode AllReduce [b, 8192] bf16 through DSL plans (K10)
    from paper_2504_09014_b200.algorithms import build_algo
    from paper_2504_09014_b200.lowering import LoweringParams, lower
    for name, var in (("2pa", "memory"), ("1pa", "")):
        for b in (1, 16, 256):
            elems = 8192 * b
            params = LoweringParams(world, elems, "bf16", "LL" if name == "1pa" else "HB")
            rt = comm.load_plan(lower(build_algo(name, params, variant=var), params), dtype="bf16")
            px, py = send[:rt.in_elems], recv[:rt.out_elems]
            t = time_graph(dev, lambda: rt.run(px, py), 20, 3, flush)
            rt.check_device_error()
            row = {"bytes": elems * 2, "kind": "allreduce", "plan": f"{name}{'_' + var if var else ''}",
                   "batch": b, "cf_plan_graph_s": t,
                   "cf_graph_s": time_graph(dev, lambda: comm.all_reduce(px[:elems], py[:elems], algo="auto"),
                                            20, 3, flush)}
            if nccl is not None and name == "2pa":
                row.update(nccl_times("allreduce", elems * 2, elems * 2, 20, flush))
            rows.append(row)
            rt.close()
    comm.check_device_error()
    return rows


def gather_max_over_ranks(t_local, e2e_local, rows_local, world, group=None):
    """All ranks: gather every rank's step time, e2e time and sweep rows
    (torch.distributed object all-gather over the bootstrap group) and reduce
    each time to its max over ranks; busbw per row uses the collective's bus
    factor (AllReduce 2(n-1)/n, AllGather / ReduceScatter (n-1)/n) and is
    also given as a percentage of 900 GB/s per direction (NVLink 5)."""
    import torch.distributed as dist
    times = [None] * world
    dist.all_gather_object(times, (t_local, e2e_local, rows_local), group=group)
    t = max(x[0] for x in times)
    te = max(x[1] for x in times)
    one_gpu = bool(os.environ.get("CF_BENCH_ONE_GPU"))
    sweep = []
    for i, row in enumerate(rows_local):
        nb = row["bytes"]
        kind = row.get("kind", "allreduce")
        out = {"bytes": nb}
        for k2 in ("plan", "batch", "kind", "error", "budget_sweep"):
            if k2 in row:
                out[k2] = row[k2]
        for key in [k for k in row if k.endswith("_s")]:
            tk = max(x[2][i][key] for x in times)   # max over ranks
            bw = busbw(nb, tk, world) if kind in ("allreduce", "nvls", "nvls_emulated") else \
                (nb / tk / 1e9 * (world - 1) / world if tk > 0 else 0.0)
            out[key[:-2]] = {"us": round(tk * 1e6, 2), "busbw": round(bw, 2)}
            if not one_gpu:
                out[key[:-2]]["pct_of_900"] = round(100 * bw / 900, 2)
        nc = [out[k]["us"] for k in ("nccl_graph", "nccl_sym_graph") if k in out]
        if nc and "cf_graph" in out:
            out["nccl_best_us"] = min(nc)
            out["cf_vs_nccl_best"] = round(min(nc) / out["cf_graph"]["us"], 3) if out["cf_graph"]["us"] else None
        sweep.append(out)
    return t, te, sweep


def run_multi_gpu(args):
    """N GPUs, one rank per process (torchrun, or self-launched by main()):
    the AllReduce over NVLink.  CF_BENCH_ONE_GPU=1 runs the same code with
    every rank on cuda:0 (a path check on a 1-GPU lease: time-sliced
    contexts, labelled as such, no NVLink figure)."""
    import torch
    import torch.distributed as dist
    from paper_2504_09014_b200.comm import Communicator
    from paper_2504_09014_b200.dtypes import torch_dtype
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    one_gpu = bool(os.environ.get("CF_BENCH_ONE_GPU"))
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", init_method="env://")
    comm = Communicator(device=local)
    dev = torch.device("cuda", local)
    nccl, nccl_err = nccl_setup(dev, rank, world)
    # symmetric heap (cfMemAlloc): every bench buffer lives there, so no
    # registration; with a multicast object (mode 1) switch_2pa runs in place
    # (multimem); on a 1-GPU path check the switch is emulated (mode 2)
    big = GiB if not one_gpu else 64 * MiB
    nvls_err = None
    try:
        sym_mode = comm.setup_symmetric(2 * big + 2 * HEAD_BYTES + 192 * MiB, mode="emulate" if one_gpu else "auto")
    except Exception as e:
        sym_mode, nvls_err = -1, f"{type(e).__name__}: {e}"[:200]
    nvls = sym_mode in (1, 2)
    nvls_kind = "nvls" if sym_mode == 1 else "nvls_emulated"
    parity = multi_parity(comm, dev, rank, world, nvls, sym_mode)
    if nvls and parity.get("allreduce_switch_2pa_symmetric") is not True:
        nvls = False    # a failed first multimem execution drops the NVLS rows, never the line
        if sym_mode == 1:
            comm.disable_switch()   # and AUTO stops picking it on every rank
    count = HEAD_BYTES // 2
    gen = torch.Generator(device=dev)
    gen.manual_seed(20250409 + 4000 + rank)
    alloc = (lambda numel: comm.alloc_symmetric(numel, torch_dtype(HEAD_DTYPE))) if sym_mode >= 0 else \
        (lambda numel: torch.empty(numel, device=dev, dtype=torch_dtype(HEAD_DTYPE)))
    send, recv = alloc(count), alloc(count)
    send.copy_(torch.randn(count, device=dev, generator=gen).to(torch_dtype(HEAD_DTYPE)))
    if sym_mode < 0:
        comm.register(send)
        comm.register(recv)
    stream = torch.cuda.current_stream(dev)
    # the selector's pick for the headline (AUTO: in-place NVLS on a multicast
    # heap, else the two-shot HB kernel)
    head_algo = "switch_2pa" if (nvls and sym_mode == 1) else "2pa"
    # measured selection over NVLink (Communicator.tune, max over ranks, one
    # table on every rank; NVLS start size on a multicast heap): the sweep's
    # 'auto' rows follow it
    tuned = None
    if not args.no_sweep:
        try:
            # (the bench runs no compute beside the collectives: budgets up to 128 CTAs)
            tr = comm.tune(kind="allreduce", dtype="bf16", iters=10, nvls=nvls and sym_mode == 1,
                           budgets=(32, 64, 96, 128))
            tuned = {"table": [[int(b), a] for b, a in tr["table"]], "nvls_min_bytes": tr["nvls_min_bytes"],
                     "cta_budget_2pa": tr["cta_budget_2pa"], "cta_budget_times_us": tr["cta_budget_times_us"],
                     "times_us": {a: [None if v is None else round(v * 1e6, 2) for v in ts]
                                  for a, ts in tr["times"].items()},
                     "sizes": tr["sizes"]}
        except Exception as e:   # the line still prints with the built-in table
            tuned = {"error": f"{type(e).__name__}: {e}"[:200]}
            comm.clear_device_error()
    head_pick = None
    if nvls:   # (emulated switch on a 1-GPU path check: exercises the same selection)
        # the headline size is above the tuning ladder: NVLS in place vs the
        # two-shot kernel measured here (max over ranks), the faster one is timed
        cand = {}
        for name in ("switch_2pa", "2pa"):
            for _ in range(2):
                comm.all_reduce(send, recv, algo=name)
            torch.cuda.synchronize(dev)
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(3):
                comm.all_reduce(send, recv, algo=name)
            b.record(stream)
            b.synchronize()
            cand[name] = a.elapsed_time(b) / 3
        allc = [None] * world
        dist.all_gather_object(allc, cand)
        worst = {k: max(c[k] for c in allc) for k in cand}
        head_algo = min(worst, key=worst.get)
        head_pick = {k: round(v * 1e3, 1) for k, v in worst.items()}   # us per call, max over ranks
    for _ in range(args.warmup):
        comm.all_reduce(send, recv, algo=head_algo)
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            comm.all_reduce(send, recv, algo=head_algo)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    dist.barrier()
    comm.check_device_error()
    t_local = e0.elapsed_time(e1) / 1e3 / args.steps
    # e2e: pinned host input -> device -> all_reduce -> pinned host output, per step
    host_in = send.cpu().pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    e2e_local = []
    for it in range(4):
        torch.cuda.synchronize(dev)
        dist.barrier()
        t0 = time.perf_counter()
        comm.all_reduce_host(host_in, host_out, algo="2pa")   # pipelined H2D / K3 / D2H
        torch.cuda.synchronize(dev)
        if it:
            e2e_local.append(time.perf_counter() - t0)
    rows_local = [] if args.no_sweep else multi_sweep(comm, dev, rank, world, send, recv, nvls, nvls_kind, nccl,
                                                       big, sym_mode)
    t, te, sweep = gather_max_over_ranks(t_local, float(np.mean(e2e_local)), rows_local, world)
    ok = all(v is True for v in parity.values())
    if rank == 0:
        # `value` is the whole-job aggregate (the contract): the bus bandwidth
        # of every GPU summed, N x the per-GPU busbw (nccl-tests definition,
        # reported beside it; the roofline and % of 900 GB/s are per GPU)
        per_gpu = busbw(HEAD_BYTES, t, world)
        value = world * per_gpu
        e2e_gpu = busbw(HEAD_BYTES, te, world)
        where = (f"{world} ranks sharing cuda:0 (time-sliced path check; not an NVLink measurement)"
                 if one_gpu else f"{world} ranks, one per GPU, peer loads/stores over NVLink 5 / NVSwitch")
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "busbw_per_gpu": round(per_gpu, 2),
            "value_definition": "aggregate over GPUs: n_gpus x per-GPU busbw (max-over-ranks time)",
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": HEAD_DTYPE,
            "data": "synthetic",
            "config": {"workload": f"AllReduce {HEAD_DTYPE}, {where}, {HEAD_BYTES // MiB} MiB per rank "
                                   "(C4 shape)", "ranks": world,
                       "algo": head_algo + (" (in place, symmetric buffers)" if head_algo == "switch_2pa" else ""),
                       "headline_pick_us": head_pick,
                       "buffers": "symmetric heap (cfMemAlloc)" if sym_mode >= 0 else "registered torch tensors",
                       "parallelism": f"{world} GPUs" if not one_gpu else f"{world} processes / 1 GPU",
                       "l2": "inputs larger than L2 (headline); sweep rows < 64 MiB flush L2 between "
                             "timed iterations (both arms)"},
            "parity": parity,
            "e2e": {"value": round(world * e2e_gpu, 3), "unit": "GB/s", "busbw_per_gpu": round(e2e_gpu, 3),
                    "h2d_bytes_per_step": world * HEAD_BYTES, "d2h_bytes_per_step": world * HEAD_BYTES,
                    "bytes_note": "all ranks (HEAD_BYTES per rank each way)",
                    "ms_per_step": round(te * 1e3, 3),
                    "api": "Communicator.all_reduce_host (cfAllReduceHostStaged), pinned host tensors"},
            "gpu_launches": args.steps, "clocks": clk.summary(), "tuned_selection": tuned,
            "sweep": {"config": "bf16 AllReduce (+ C5 DSL plans, AllGather, ReduceScatter, NVLS when the "
                                "box builds a multicast object): libcf (selector's pick) in a CUDA graph and "
                                "eager vs NCCL 2.28 in a CUDA graph on default buffers (nccl_graph) and on "
                                "symmetric windows (nccl_sym_graph); latency = max over ranks",
                      "nccl_version": Nccl_version(nccl), "nccl_error": nccl_err, "nvls": nvls_kind if nvls
                      else None, "nvls_error": nvls_err, "symmetric_heap_mode": sym_mode, "rows": sweep}}
        if one_gpu:
            line["roofline"] = None
        else:
            # north_star: every busbw also as a fraction of 900 GB/s per direction per GPU
            for row in sweep:
                for v in row.values():
                    if isinstance(v, dict) and v.get("busbw") is not None:
                        v["pct_of_900"] = round(100 * v["busbw"] / 900, 2)
            line["pct_of_900"] = round(100 * per_gpu / 900, 2)
            line["roofline"] = {"bound": "nvlink", "achieved": round(per_gpu, 1), "peak": 900.0,
                                "unit": "GB/s", "frac": round(per_gpu / 900, 4), "traffic": None,
                                "note": "busbw per GPU per direction vs nominal NVLink 5 (no measured "
                                        "NVLink peak in MEASURED_PEAKS.json)"}
        print(json.dumps(line))
    if nccl is not None:
        nccl.close()
    comm.close()
    dist.destroy_process_group()
    return 0 if ok else 1


def Nccl_version(nccl):
    if nccl is None:
        return None
    try:
        return nccl.version()
    except Exception:
        return None


def self_launch(args):
    """`bench.py --gpus N` without torchrun: spawn N ranks of this script on
    127.0.0.1 (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* as torchrun sets
    them); rank 0 prints the line.  Returns the worst exit code."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cf", choices=["cf", "reference"])
    ap.add_argument("--no-sweep", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "RANK" not in os.environ:
        return self_launch(args)
    if os.environ.get("CF_BENCH_MULTI") and "RANK" not in os.environ:
        os.environ.update(RANK="0", LOCAL_RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(29500 + os.getpid() % 1000))
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
