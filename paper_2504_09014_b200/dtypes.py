"""Element types (reference: cf/dtypes.py:7-8 has i32/f32 only; f16/bf16 are
the B200 extension).  bf16 host arrays travel as np.uint16 bit patterns."""

from __future__ import annotations

import numpy as np

DTYPES = ("i32", "f32", "f16", "bf16")
CODES = {"i32": 0, "f32": 1, "f16": 2, "bf16": 3}
ELEM_SIZE = {"i32": 4, "f32": 4, "f16": 2, "bf16": 2}
NP_DTYPES = {"i32": np.dtype("<i4"), "f32": np.dtype("<f4"), "f16": np.dtype("<f2"),
             "bf16": np.dtype("<u2")}


def torch_dtype(name: str):
    import torch
    return {"i32": torch.int32, "f32": torch.float32, "f16": torch.float16,
            "bf16": torch.bfloat16}[name]


def from_torch(dt) -> str:
    import torch
    table = {torch.int32: "i32", torch.float32: "f32", torch.float16: "f16",
             torch.bfloat16: "bf16"}
    if dt not in table:
        raise KeyError(f"unsupported torch dtype {dt}")
    return table[dt]


def as_elems(raw: np.ndarray, dtype: str) -> np.ndarray:
    """View a uint8 byte array as elements of the given dtype (cf/dtypes.py:11-13)."""
    return raw.view(NP_DTYPES[dtype])


def to_bytes(values, dtype: str) -> np.ndarray:
    return np.asarray(values, NP_DTYPES[dtype]).view(np.uint8)
