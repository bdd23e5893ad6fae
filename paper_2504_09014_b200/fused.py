"""Compute-fused collectives: the C5 consumer's epilogue --
residual add + RMSNorm -- fused into the AllReduce (K13, ``cfAllReduceAddRMSNorm``).

The reference has no fused op; a reference user composes it from
``collective("allreduce", ...)`` (``cf/collectives.py:532-573``) and host
arithmetic.  Semantics per rank r, on ``[rows, hidden]`` tensors::

    h         = x_0 + x_1 + ... + x_{n-1}     f32 accumulate, rounded to dtype once
                                              (the same bits on every rank)
    resid_out = dtype(h + resid_in[r])
    norm_out  = dtype(resid_out * rsqrt(mean(resid_out ** 2, -1) + eps) * weight[r])

``algo``: ``"1pa_hb"`` (one-shot: each rank reduces every row -- latency
regime), ``"2pa"`` (two-shot: rank r owns a contiguous block of rows and
stores both results into every rank), or ``None`` (libcf picks).
"""

from __future__ import annotations

from . import _lib
from .dtypes import CODES, from_torch
from .errors import NoAlgoError, ShapeError

_ALGOS = {None: _lib.ALGOS["auto"], "auto": _lib.ALGOS["auto"], "1pa_hb": _lib.ALGOS["1pa_hb"],
          "2pa": _lib.ALGOS["2pa"]}


def allreduce_add_rmsnorm(world, inputs, residuals, weights, eps: float = 1e-6, algo: str | None = None,
                          resid_out=None, norm_out=None):
    """Fused AllReduce + residual + RMSNorm over a World (one entry per rank,
    CUDA tensors on the ranks' devices, all ``[rows, hidden]``; ``weights``
    ``[hidden]``, one per rank or a single shared tensor).  ``resid_out``
    defaults to updating ``residuals`` in place; ``norm_out`` defaults to fresh
    tensors.  Returns ``(norm_out, resid_out)``."""
    import torch
    n = world.num_ranks
    if len(inputs) != n or len(residuals) != n:
        raise ShapeError(f"expected {n} inputs and residuals, got {len(inputs)} and {len(residuals)}")
    if isinstance(weights, torch.Tensor):
        weights = [weights] * n
    if algo not in _ALGOS:
        raise NoAlgoError(f"fused allreduce+rmsnorm runs as 1pa_hb or 2pa, not {algo!r}")
    shape = tuple(inputs[0].shape)
    if len(shape) != 2:
        raise ShapeError(f"inputs must be [rows, hidden], got {shape}")
    rows, hidden = shape
    dtype = from_torch(inputs[0].dtype)
    for name, ts in (("input", inputs), ("residual", residuals)):
        for t in ts:
            if tuple(t.shape) != shape or t.dtype != inputs[0].dtype or not t.is_cuda or not t.is_contiguous():
                raise ShapeError(f"every {name} must be a contiguous CUDA tensor of shape {shape} "
                                 f"and dtype {inputs[0].dtype}")
    for w in weights:
        if tuple(w.shape) != (hidden,) or w.dtype != inputs[0].dtype or not w.is_contiguous():
            raise ShapeError(f"weight must be a contiguous [{hidden}] tensor of dtype {inputs[0].dtype}")
    if resid_out is None:
        resid_out = list(residuals)
    if norm_out is None:
        norm_out = [torch.empty_like(x) for x in inputs]
    _lib.check(_lib.lib().cfAllReduceAddRMSNorm(
        world.comm, _lib.ptr_array([t.data_ptr() for t in inputs]),
        _lib.ptr_array([t.data_ptr() for t in residuals]), _lib.ptr_array([t.data_ptr() for t in resid_out]),
        _lib.ptr_array([t.data_ptr() for t in norm_out]), _lib.ptr_array([t.data_ptr() for t in weights]),
        rows, hidden, float(eps), CODES[dtype], _ALGOS[algo], _lib.ptr_array(world.streams())))
    return norm_out, resid_out
