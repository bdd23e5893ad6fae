"""Golden vectors for the native DSL lowering: random user programs recorded
through the REFERENCE builder API (cf/lowering.py:133-293) and lowered by the
reference's own ``lower()`` (cf/lowering.py:629-648).  Each case stores the
recording as a list of builder calls plus the reference's canonical lowered
plan bytes (or the error code it raised), so tests/test_lowering.py can
replay the calls through paper_2504_09014_b200's ProgramGraph and compare.

Run in this container (needs /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_lower_fuzz.py
"""

from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"


def gen_calls(rng: random.Random):
    """One random program as builder calls (valid enough to usually lower)."""
    n = rng.choice([2, 2, 3, 4])
    proto = rng.choice(["HB", "HB", "LL", "LL"])
    inst = rng.choice([1, 1, 1, 2])
    unit = 2 if inst == 2 else 1
    calls = [["params", n, 16, "i32", proto, inst]]
    bufs = [("in", "input", 16), ("out", "output", 16)]
    for k in range(rng.randint(1, 3)):
        bufs.append((f"s{k}", "scratch", rng.choice([16, 32])))
    for b, kind, e in bufs:
        calls.append(["buffer", b, kind, "all", e])
    sizes = {b: e for b, _, e in bufs}
    chans = []
    for _ in range(rng.randint(1, 5)):
        src = rng.randrange(n)
        dst = rng.choice([r for r in range(n) if r != src])
        ctype = "port" if proto == "HB" and rng.random() < 0.4 else "memory"
        calls.append(["chan", ctype, src, dst])
        chans.append((ctype, src, dst))
    switch = None
    if rng.random() < 0.2:
        calls.append(["switch", list(range(n))])
        switch = list(range(n))

    def ref(buf=None, packet=False):
        b = buf or rng.choice(list(sizes))
        lim = sizes[b] // 2 if packet else sizes[b]
        size = rng.choice([u for u in (2, 4, 8) if u <= lim]) if rng.random() < 0.9 else unit
        size = max(unit, size - size % unit)
        off = rng.randrange(0, lim - size + 1)
        off -= off % unit
        return [b, off, size]

    scratch = [b for b, kind, _ in bufs if kind == "scratch"]
    nops = rng.randint(3, 18)
    for _ in range(nops):
        tb = rng.choice([0, 0, 0, 1])
        kind = rng.random()
        if kind < 0.22 and chans:
            ci = rng.randrange(len(chans))
            ctype, src, dst = chans[ci]
            if proto == "LL" and ctype == "memory":
                calls.append(["put_packets", ci, ref(packet=True), ref(), tb, None])
            elif rng.random() < 0.15:
                # group put over two thread blocks of the source rank
                r = ref()
                calls.append(["put", ci, r, [r[0], r[1], r[2]], 0, [0, 1]])
            else:
                calls.append(["put", ci, ref(), ref(), tb, None])
                if rng.random() < 0.6:
                    calls.append(["signal", ci, tb])
        elif kind < 0.32 and chans:
            ci = rng.randrange(len(chans))
            ctype, src, dst = chans[ci]
            if proto == "LL" and ctype == "memory":
                prior = [c[2] for c in calls if c[0] == "put_packets" and c[1] == ci]
                src = list(rng.choice(prior)) if prior and rng.random() < 0.8 else ref(packet=True)
                calls.append(["read_packets", ci, ref(), src, tb, None])
            else:
                calls.append(["wait", ci, tb, ref() if rng.random() < 0.7 else None])
        elif kind < 0.38 and chans:
            ci = rng.randrange(len(chans))
            if chans[ci][0] == "port":
                calls.append(["flush", ci, tb])
            elif proto == "HB":
                calls.append(["creduce", ci, ref(), ref(), tb])
        elif kind < 0.55:
            calls.append(["reduce", rng.randrange(n), ref(), ref(), tb])
        elif kind < 0.68:
            calls.append(["copy", rng.randrange(n), ref(), ref(), tb])
        elif kind < 0.76 and scratch and chans:
            # reduce into scratch then put it: the reduce_put fusion pattern
            mem = [i for i, c in enumerate(chans) if c[0] == "memory"]
            if mem and proto == "HB":
                ci = rng.choice(mem)
                r = chans[ci][1]
                s = ref(rng.choice(scratch))
                calls.append(["reduce", r, s, ref(), tb])
                if rng.random() < 0.3:
                    calls.append(["tb_sync", r, tb])
                calls.append(["put", ci, ref(), list(s), tb, None])
                if rng.random() < 0.5:
                    calls.append(["signal", ci, tb])
        elif kind < 0.84:
            calls.append(["tb_sync", rng.randrange(n), tb])
        elif kind < 0.88:
            calls.append(["device_barrier", rng.randrange(n), [0, 1]])
        elif switch is not None:
            caller = rng.randrange(n)
            if rng.random() < 0.5:
                calls.append(["sw_reduce", caller, ref(), ref(), tb])
            else:
                calls.append(["sw_bcast", caller, ref(), ref(), tb])
    passes = rng.choice([["sync", "fuse"], ["sync", "fuse"], ["sync"], ["fuse"], []])
    calls.append(["lower", passes])
    return calls


def replay(calls, api):
    """Replay builder calls through a module exposing the reference builder
    API (ProgramGraph, LoweringParams, lower); returns canonical bytes."""
    _, n, elems, dtype, proto, inst = calls[0]
    params = api.LoweringParams(n, elems, dtype, proto, instances=inst)
    g = api.ProgramGraph("fuzz", "custom", params)
    chans, sw = [], None
    for c in calls[1:]:
        op = c[0]
        if op == "buffer":
            g.buffer(c[1], c[2], c[3], c[4])
        elif op == "chan":
            chans.append(g.port_channel(c[2], c[3]) if c[1] == "port" else g.memory_channel(c[2], c[3]))
        elif op == "switch":
            sw = g.switch_channel(c[1])
        elif op == "put":
            chans[c[1]].put(dst=tuple(c[2]), src=tuple(c[3]), tb=c[4],
                            tb_group=tuple(c[5]) if c[5] else None)
        elif op == "put_packets":
            chans[c[1]].put_packets(dst=tuple(c[2]), src=tuple(c[3]), tb=c[4], flag=c[5])
        elif op == "read_packets":
            chans[c[1]].read_packets(dst=tuple(c[2]), src=tuple(c[3]), tb=c[4], flag=c[5])
        elif op == "signal":
            chans[c[1]].signal(tb=c[2])
        elif op == "wait":
            chans[c[1]].wait(tb=c[2], arrives=tuple(c[3]) if c[3] else None)
        elif op == "flush":
            chans[c[1]].flush(tb=c[2])
        elif op == "creduce":
            chans[c[1]].reduce(dst=tuple(c[2]), src=tuple(c[3]), tb=c[4])
        elif op == "reduce":
            g.reduce(c[1], dst=tuple(c[2]), src=tuple(c[3]), tb=c[4])
        elif op == "copy":
            g.copy(c[1], dst=tuple(c[2]), src=tuple(c[3]), tb=c[4])
        elif op == "tb_sync":
            g.tb_sync(c[1], tb=c[2])
        elif op == "device_barrier":
            g.device_barrier(c[1], c[2])
        elif op == "sw_reduce":
            sw.reduce(c[1], dst=tuple(c[2]), src=tuple(c[3]), tb=c[4])
        elif op == "sw_bcast":
            sw.broadcast(c[1], dst=tuple(c[2]), src=tuple(c[3]), tb=c[4])
        elif op == "lower":
            return api.lower(g, params, passes=tuple(c[1]))
    raise AssertionError("no lower call")


def main(count=500, seed=2504):
    sys.path.insert(0, REF)
    import commforge.lowering as L
    from commforge.errors import CommforgeError
    from commforge.plan import serialize_plan
    rng = random.Random(seed)
    cases, kinds = [], {}
    while len(cases) < count:
        calls = gen_calls(rng)
        try:
            plan = replay(calls, L)
            out = {"calls": calls, "plan": serialize_plan(plan).decode()}
            kinds["ok"] = kinds.get("ok", 0) + 1
        except CommforgeError as e:
            out = {"calls": calls, "error": e.code}
            kinds[e.code] = kinds.get(e.code, 0) + 1
        cases.append(out)
    with open(os.path.join(HERE, "lower_fuzz.json"), "w") as f:
        json.dump(cases, f, separators=(",", ":"))
        f.write("\n")
    print("lower_fuzz.json:", len(cases), kinds)


if __name__ == "__main__":
    main()
