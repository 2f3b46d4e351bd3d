"""Thin wrappers over the ring kernels (``fss_ring_op``) for uint64 device tensors."""

from __future__ import annotations

import torch

from . import _dev, _lib

_OPS = {"add": 0, "sub": 1, "mul": 2, "neg": 3, "mask": 4}


def _run(op, a: torch.Tensor, b, n_bits: int) -> torch.Tensor:
    a = a.contiguous()
    if isinstance(b, torch.Tensor):
        if b.shape != a.shape:
            try:
                a, b = torch.broadcast_tensors(_dev.as_i64(a), _dev.as_i64(b))
            except RuntimeError:
                raise ValueError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}") from None
            a, b = _dev.as_u64(a.contiguous()), _dev.as_u64(b.contiguous())
        b = b.contiguous()
        bp, bs = _dev.ptr(b), 0
    else:
        bp, bs = None, (int(b) if b is not None else 0) & _dev.FULL64
    out = torch.empty_like(a)
    dev = a.device
    with _dev.on(dev):
        _lib.call("fss_ring_op", _OPS[op], n_bits, a.numel(), _dev.ptr(a), bp, bs, _dev.ptr(out),
                  _dev.stream_handle(dev))
    return out


def binary(op: str, a, b, n_bits: int) -> torch.Tensor:
    return _run(op, a, b, n_bits)


def neg(a, n_bits: int) -> torch.Tensor:
    return _run("neg", a, None, n_bits)


def mask(a, n_bits: int) -> torch.Tensor:
    if n_bits >= 64:
        return a.contiguous()
    return _run("mask", a, None, n_bits)


def sum(a, n_bits: int, axis=None) -> torch.Tensor:  # noqa: A001 (mirrors RingTensor.sum)
    v = _dev.as_i64(a)
    s = v.sum() if axis is None else v.sum(dim=axis)   # int64 wraps mod 2^64
    return mask(_dev.as_u64(s.reshape(s.shape)), n_bits)


def cumsum(a, n_bits: int, axis=-1) -> torch.Tensor:
    return mask(_dev.as_u64(_dev.as_i64(a).cumsum(dim=axis)), n_bits)
