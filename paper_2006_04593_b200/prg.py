"""Drop-in for the reference's ``ariann.prg`` (pkg/src/ariann/prg.py).

G(x) = AES_k1(x) ^ x || AES_k2(x) ^ x || AES_k3(x) ^ x with the fixed public
keys 00..0f, 10..1f, 20..2f (prg.py:24-28). ``expand`` runs the sm_100a
T-table AES kernel (csrc/aes_ttable.cuh) through ``fss_aes_mmo_expand``.

Type convention of the drop-in: numpy in -> numpy out (host buffers are copied
to the device and back), torch CUDA tensor in -> torch CUDA tensor out.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _lib
from .ring import ring_mask

SEED_BITS = 127  # lambda
BLOCK_BYTES = 16
MAX_BLOCKS = 3

CIPHER_KEYS = (
    bytes(range(0x00, 0x10)),
    bytes(range(0x10, 0x20)),
    bytes(range(0x20, 0x30)),
)


def random_seeds(rng: np.random.Generator, count: int) -> np.ndarray:
    """(count, 16) uint8 seed blocks with the top bit cleared (prg.py:36-40).

    Host-side numpy draw, same call as the reference so the caller's rng
    advances identically. Bulk key generation draws its seeds on the device
    instead (fss._sample_tape -> fss_pcg64_tape)."""
    seeds = rng.integers(0, 256, size=(count, BLOCK_BYTES), dtype=np.uint8)
    seeds[:, 15] &= np.uint8(0x7F)
    return seeds


def _seeds_in(seeds):
    host = not isinstance(seeds, torch.Tensor)
    if host:
        arr = np.array(seeds, dtype=np.uint8, copy=True, order="C")
        if arr.ndim != 2 or arr.shape[1] != BLOCK_BYTES:
            raise ValueError("seeds must have shape (N, 16)")
        dev = _dev.default_device()
        t = torch.from_numpy(arr).to(dev)
    else:
        if seeds.ndim != 2 or seeds.shape[1] != BLOCK_BYTES:
            raise ValueError("seeds must have shape (N, 16)")
        t = seeds.to(dtype=torch.uint8).contiguous()
        dev = _dev.default_device(t.device)
    return t, dev, host


def expand(seeds, out_blocks: int):
    """Expand (N, 16) seed blocks to (N, 16*out_blocks) bytes (prg.py:43-60)."""
    if not 2 <= out_blocks <= MAX_BLOCKS:
        raise ValueError(f"out_blocks must be 2 or 3, got {out_blocks}")
    t, dev, host = _seeds_in(seeds)
    n = t.shape[0]
    out = torch.empty((n, out_blocks * BLOCK_BYTES), dtype=torch.uint8, device=dev)
    with _dev.on(dev):
        _lib.call("fss_aes_mmo_expand", _dev.ptr(t), n, out_blocks, _dev.ptr(out),
                  _dev.stream_handle(dev))
    return _dev.to_numpy(out) if host else out


def expand_one(seed: bytes, out_blocks: int) -> bytes:
    """Single-seed convenience wrapper (prg.py:63-68)."""
    if len(seed) != BLOCK_BYTES:
        raise ValueError("seed must be 16 bytes")
    arr = np.frombuffer(seed, dtype=np.uint8).reshape(1, BLOCK_BYTES).copy()
    return expand(arr, out_blocks).tobytes()


# ---------------------------------------------------------------------------
# Slice helpers (layout contract LAYOUT.md:23-46). The CUDA tree walks slice in
# registers; these are the API-level views, computed with device tensor ops.
# ---------------------------------------------------------------------------

def _bytes_in(raw, width, what):
    host = not isinstance(raw, torch.Tensor)
    t = (torch.from_numpy(np.ascontiguousarray(raw, dtype=np.uint8)).to(_dev.default_device())
         if host else raw.to(torch.uint8))
    if t.ndim != 2 or t.shape[1] < width:
        raise ValueError(what)
    return t, host


def _out(host, *ts):
    return tuple(_dev.to_numpy(x) for x in ts) if host else ts


def slice_eq(raw):
    """(N, 32) expansion bytes -> (sL, tL, sR, tR) (prg.py:71-86)."""
    t, host = _bytes_in(raw, 2 * BLOCK_BYTES, "equality slice needs (N, 32) bytes")
    if t.shape[1] != 2 * BLOCK_BYTES:
        raise ValueError("equality slice needs (N, 32) bytes")
    s_l = t[:, :16].clone()
    s_r = t[:, 16:32].clone()
    t_l = (s_l[:, 15] >> 7) & 1
    t_r = (s_r[:, 15] >> 7) & 1
    s_l[:, 15] &= 0x7F
    s_r[:, 15] &= 0x7F
    return _out(host, s_l, t_l, s_r, t_r)


def reassemble_eq(s_l, t_l, s_r, t_r):
    """Inverse of slice_eq (prg.py:89-96)."""
    host = not isinstance(s_l, torch.Tensor)
    dev = _dev.default_device() if host else s_l.device
    cv = (lambda a: _dev.to_device_u8(a, dev))
    s_l, t_l, s_r, t_r = cv(s_l), cv(t_l), cv(s_r), cv(t_r)
    out = torch.empty((s_l.shape[0], 2 * BLOCK_BYTES), dtype=torch.uint8, device=dev)
    out[:, :16] = s_l
    out[:, 16:] = s_r
    out[:, 15] |= t_l << 7
    out[:, 31] |= t_r << 7
    return _dev.to_numpy(out) if host else out


def slice_cmp(raw, n: int):
    """(N, 48) -> (sL, tL, sR, tR, sigmaL, tauL, sigmaR, tauR) (prg.py:99-119)."""
    t, host = _bytes_in(raw, 3 * BLOCK_BYTES, "comparison slice needs (N, 48) bytes")
    if n > 63:
        raise ValueError("comparison slice supports n <= 63")
    s_l, t_l, s_r, t_r = slice_eq(t[:, :32])
    lanes = t[:, 32:48].contiguous().view(torch.int64)
    mask = int(ring_mask(n))
    sigma_l = (lanes[:, 0] & mask).view(torch.uint64)
    sigma_r = (lanes[:, 1] & mask).view(torch.uint64)
    tau_l = (t[:, 39] >> 7).to(torch.uint8)
    tau_r = (t[:, 47] >> 7).to(torch.uint8)
    return _out(host, s_l, t_l, s_r, t_r, sigma_l, tau_l, sigma_r, tau_r)


def seed_to_ring(seeds, n: int):
    """LE u64 of bytes 0..7 reduced mod 2^n (prg.py:122-125)."""
    t, host = _bytes_in(seeds, BLOCK_BYTES, "seeds must have shape (N, 16)")
    v = t[:, :8].contiguous().view(torch.int64).reshape(-1)
    mask = int(ring_mask(n))
    if mask != _dev.FULL64:
        v = v & mask
    v = v.view(torch.uint64)
    return _dev.to_numpy(v) if host else v


def mask_stream(seed: bytes, round_idx: int, count: int, n_bits: int, device=None):
    """Deterministic ring-element stream for aggregation masks (prg.py:128-147):
    block i = seed ^ (round_idx LE bytes 0..7 || i LE bytes 8..15), top bit
    re-cleared, expanded to 2 MMO blocks = 4 u64 lanes. One fused kernel
    (fss_mask_stream); returns numpy like the reference unless ``device``
    is given, in which case the device tensor is returned."""
    if len(seed) != BLOCK_BYTES:
        raise ValueError("seed must be 16 bytes")
    ring_mask(n_bits)
    dev = _dev.default_device(device)
    lo = int.from_bytes(bytes(seed[:8]), "little")
    hi = int.from_bytes(bytes(seed[8:]), "little")
    out = torch.empty(int(count), dtype=torch.uint64, device=dev)
    with _dev.on(dev):
        _lib.call("fss_mask_stream", lo, hi, int(round_idx) & _dev.FULL64, int(count), n_bits,
                  _dev.ptr(out), _dev.stream_handle(dev))
    return out if device is not None else _dev.to_numpy(out)
