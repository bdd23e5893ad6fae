"""Deterministic input generators shared by the golden script, the tests and
the bench (numpy PCG64 streams are stable across numpy versions).

Distributions
  int      i32 in [-1e6, 1e6)          (reference tests: test_acceptance.py:73-74)
  uniform  f32 U[-50, 50)              (reference tests: test_acceptance.py:105)
  wide     f32 N(0,1)*exp(U(-8,8))     (order-sensitive; exposes any reorder)
  bits     random 32-bit patterns as i32 (AllGather: bit-exact data movement)
  normal   N(0,1) * scale, for f16/bf16 (returned as f16 / bf16 bit patterns)
"""

from __future__ import annotations

import numpy as np


def gen_inputs(n: int, elems: int, dtype: str, dist: str, seed: int, scale: float = 1.0):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        if dist == "int":
            a = rng.integers(-10**6, 10**6, elems).astype(np.int32)
        elif dist == "uniform":
            a = (rng.random(elems) * 100 - 50).astype(np.float32)
        elif dist == "wide":
            a = (rng.standard_normal(elems) * np.exp(rng.uniform(-8, 8, elems))).astype(np.float32)
        elif dist == "bits":
            a = rng.integers(0, 2**32, elems, dtype=np.uint64).astype(np.uint32).view(np.int32)
        elif dist == "normal":
            a = (rng.standard_normal(elems) * scale).astype(np.float32)
        else:
            raise KeyError(dist)
        if dtype == "f16":
            a = a.astype(np.float32).astype(np.float16)
        elif dtype == "bf16":
            u = a.astype(np.float32).view(np.uint32).astype(np.uint64)
            a = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
        elif dtype == "f32":
            a = a.astype(np.float32)
        elif dtype == "i32":
            a = a.astype(np.int32)
        out.append(a)
    return out


def ag_bf16_shards(n: int, cnt: int, seed: int):
    """bf16 AllGather inputs of ag_bf16.json: random 16-bit patterns (NaNs
    included) as uint16, one array per rank."""
    rng = np.random.default_rng(seed)
    return [rng.integers(0, 1 << 16, cnt, dtype=np.uint32).astype(np.uint16) for _ in range(n)]
