"""Device plumbing shared by the drop-in modules: tensor conversion, raw
pointers and the current CUDA stream handed to the C ABI."""

from __future__ import annotations

import contextlib

import numpy as np
import torch

U64 = torch.uint64
I64 = torch.int64
U8 = torch.uint8

FULL64 = (1 << 64) - 1


def default_device(device=None) -> torch.device:
    if device is not None:
        dev = torch.device(device)
        if dev.type != "cuda":
            raise ValueError("the FSS path runs on CUDA devices only (no CPU fallback)")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        return dev
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 FSS path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_SIDE_STREAMS = {}


def side_streams(device: torch.device, k: int = 2) -> list:
    """k CUDA side streams of ``device`` for the calling thread, created once
    and reused (stream creation per call costs time, and the caching allocator
    pools free blocks per stream)."""
    import threading
    key = (str(device), threading.get_ident())
    got = _SIDE_STREAMS.get(key, [])
    while len(got) < k:
        got.append(torch.cuda.Stream(device))
    _SIDE_STREAMS[key] = got
    return got[:k]


try:
    _raw_stream = torch._C._cuda_getCurrentRawStream   # the cudaStream_t, without a Stream object
except AttributeError:  # pragma: no cover - older torch
    _raw_stream = None


def stream_handle(device: torch.device) -> int:
    """cudaStream_t of the calling thread's current stream on ``device``."""
    if _raw_stream is not None and device.index is not None:
        return _raw_stream(device.index)
    return torch.cuda.current_stream(device).cuda_stream


_NULL_CTX = contextlib.nullcontext()


def on(device):
    """``torch.cuda.device(device)``, skipped (a shared no-op context) when
    that device is already the calling thread's current one."""
    idx = device if isinstance(device, int) else getattr(device, "index", None)
    if idx is not None and torch._C._cuda_getDevice() == idx:
        return _NULL_CTX
    return torch.cuda.device(device)


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr() if t.numel() else None


def mask_int(w: int) -> int:
    return FULL64 if w >= 64 else (1 << w) - 1


def as_i64(t: torch.Tensor) -> torch.Tensor:
    """int64 view of a uint64 tensor (two's-complement arithmetic is identical mod 2^64)."""
    return t.view(I64) if t.dtype == U64 else t


def as_u64(t: torch.Tensor) -> torch.Tensor:
    return t.view(U64) if t.dtype == I64 else t


def to_device_u64(x, device: torch.device) -> torch.Tensor:
    """numpy / python ints / torch -> contiguous uint64 tensor on `device`."""
    if isinstance(x, torch.Tensor):
        if x.dtype == U64:
            t = x
        elif x.dtype in (torch.int64, torch.int32, torch.int16, torch.int8, torch.uint8, torch.bool,
                         torch.uint16, torch.uint32):
            t = x.to(torch.int64).view(U64)
        else:
            raise TypeError(f"ring values must be integer tensors, got {x.dtype}")
        return t.to(device, non_blocking=True).contiguous()
    arr = np.asarray(x)
    if arr.dtype != np.uint64:
        if arr.dtype.kind == "O":
            arr = np.array([int(v) & FULL64 for v in arr.reshape(-1)], dtype=np.uint64).reshape(arr.shape)
        else:
            arr = arr.astype(np.int64).astype(np.uint64)
    # np.ascontiguousarray would turn a 0-d array into shape (1,): keep the shape
    arr = np.require(arr, requirements="C")
    return torch.from_numpy(arr).to(device)


def to_device_u8(x, device: torch.device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=U8).contiguous()
    return torch.from_numpy(np.require(np.asarray(x, dtype=np.uint8), requirements="C")).to(device)


def to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def index_select(t: torch.Tensor, dim: int, idx: torch.Tensor) -> torch.Tensor:
    """Gather that also works for uint64 storage (via its int64 view)."""
    if t.dtype == U64:
        return t.view(I64).index_select(dim, idx).view(U64)
    return t.index_select(dim, idx)
