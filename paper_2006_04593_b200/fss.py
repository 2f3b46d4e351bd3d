"""Drop-in for the reference's ``ariann.fss`` (pkg/src/ariann/fss.py) on B200.

Same entry points, key types (field names, shapes, dtypes) and error classes
as the reference; key material lives in HBM as ``torch`` tensors in the
reference's struct-of-arrays layout, and every compute step is a sm_100a
kernel behind the C ABI (include/ariann_fss.h):

  _sample_tape        -> fss_pcg64_tape   (numpy PCG64 draws reproduced on device)
  _keygen_eq_core     -> fss_dpf_keygen
  _keygen_cmp_core    -> fss_dcf_keygen
  eval_eq / eval_cmp  -> fss_dpf_eval / fss_dcf_eval
  _pack_* / _unpack_* -> fss_arnk_pack / fss_arnk_unpack

Type convention: inputs given as numpy arrays / Python ints are host buffers
(copied in, results copied back to numpy); torch CUDA tensors stay on device.
``consumed`` bookkeeping stays a host numpy bool array (it is metadata, not key
material). ``take`` of a contiguous index range returns zero-copy column views
(the kernels take a level stride), other index sets are gathered on device.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _dev, _lib, _pcg, prg, ring_ops
from ._lib import PcgState
from .ring import RingTensor, ring_mask
from .runtime import FRAME_MASKED
from .sharing import AdditiveShare, _flat_u64, _pack, _peer_wire

LAMBDA = prg.SEED_BITS

MAGIC = b"ARNK"
VERSION = 1
KIND_EQ = 0
KIND_CMP = 1
KIND_TRIPLE = 2

_HEADER_BYTES = 13  # magic 4 | version 1 | kind 1 | n 1 | lambda 2 | count 4


class KeyFormatError(ValueError):
    """Malformed serialized key material."""


class KeyExhaustedError(RuntimeError):
    """More single-use keys requested than remain unconsumed."""


# ---------------------------------------------------------------------------
# Key containers (fss.py:59-166)
# ---------------------------------------------------------------------------

@dataclass
class FssTape:
    """Dealer randomness disclosed for cut-and-choose auditing (fss.py:59-68)."""

    alpha: torch.Tensor  # (count,) u64
    s0: torch.Tensor     # (count, 16) u8
    s1: torch.Tensor     # (count, 16) u8

    def take(self, idx) -> "FssTape":
        sel, _ = _index(idx, self.alpha.shape[0], self.alpha.device)
        return FssTape(_take1(self.alpha, sel), _take1(self.s0, sel), _take1(self.s1, sel))


def _index(idx, count: int, device):
    """Normalise an index spec -> (slice | device LongTensor, host selector of
    the ``consumed`` mask: a slice for contiguous ranges, else int64 indices)."""
    if isinstance(idx, slice) and idx.step in (None, 1):
        lo, hi, _ = idx.indices(count)
        hi = max(hi, lo)
        return slice(lo, hi), slice(lo, hi)
    if isinstance(idx, slice):
        arr = np.arange(count)[idx]
    elif isinstance(idx, torch.Tensor):
        arr = idx.detach().cpu().numpy().astype(np.int64).reshape(-1)
    else:
        arr = np.asarray(list(idx) if isinstance(idx, range) else idx, dtype=np.int64).reshape(-1)
    if arr.size and (arr.min() < -count or arr.max() >= count):
        raise IndexError(f"key index out of range for a batch of {count}")
    arr = np.where(arr < 0, arr + count, arr)
    if arr.size == 0:
        return slice(0, 0), arr
    lo = int(arr[0])
    if arr.size == 1 or np.all(np.diff(arr) == 1):
        return slice(lo, lo + arr.size), slice(lo, lo + arr.size)
    return torch.from_numpy(arr).to(device), arr


def _take1(t: torch.Tensor, sel):
    """Select along the element axis 0."""
    if isinstance(sel, slice):
        return t[sel]
    return _dev.index_select(t, 0, sel)


def _take2(t: torch.Tensor, sel):
    """Select along the element axis 1 of a level-major array."""
    if isinstance(sel, slice):
        return t[:, sel]
    return _dev.index_select(t, 1, sel)


def _check_party_tensors(k, names):
    dev = k.alpha_share.device
    for name in names:
        t = getattr(k, name)
        if not isinstance(t, torch.Tensor):
            raise KeyFormatError(f"{name} must be a torch tensor (device-resident key)")
        if t.device != dev:
            raise KeyFormatError(f"{name} lives on {t.device}, expected {dev}")


# Lazy slices: take_unused's O(1) hand-out of keys [lo, lo + m) of a batch
# whose arrays passed the eval layout check records (parent arrays, lo, m,
# level stride) instead of building six tensor views (~3.5 us of host time
# each, on the critical path of every online protocol). A field is created as
# a view of the parent's array when it is first read (cached per batch, so the
# same tensor object is returned on every read); the evaluation entry points
# take the device pointers straight from the parent arrays while no field of
# the batch has been assigned.
_LAZY_ROWS = ("scw", "tcw", "sigma_cw", "leaf_cw")   # level-major: element axis 1


def _lazy_field(obj, name):
    d = obj.__dict__
    lz = d.get("_lazy")
    if lz is None or name not in lz[0]:
        raise AttributeError(f"{type(obj).__name__!r} object has no attribute {name!r}")
    cache = d.setdefault("_lazyv", {})
    v = cache.get(name)
    if v is None:
        t, lo, m = lz[0][name], lz[1], lz[2]
        v = t[:, lo:lo + m] if name in _LAZY_ROWS else t[lo:lo + m]
        cache[name] = v
    return v


def _lazy_ptrs(k, names):
    """(parent arrays, lo, count, ld) of a lazy slice none of whose `names`
    fields was assigned, else None."""
    d = k.__dict__
    lz = d.get("_lazy")
    if lz is None or any(n in d for n in names):
        return None
    return lz


class _ConsumedMask:
    """The ``consumed`` field of the key batches (reference fss.py:92-102): a
    host numpy bool mask, as in the reference -- with the single-use hand-out
    of ``take_unused`` kept O(1) on its common path. While a batch's mask is
    a pure prefix (keys [0, front) spent, the rest untouched -- true of every
    freshly generated batch spent front to back), a hand-out only records the
    range; the recorded ranges are written into the array the next time the
    field is read (reading also ends the fast path: the caller may edit the
    array in place). A 9.6 M-key hand-out (config 4's argmax) thus costs no
    0.5 ms mask scan and fill per party."""

    def __get__(self, obj, objtype=None):
        if obj is None:
            return self
        d = obj.__dict__
        pend = d.get("_pend")
        if pend:
            arr = d["_cons"]
            for lo, hi in pend:
                arr[lo:hi] = True
            pend.clear()
        d["_front"] = None
        return d.get("_cons")

    def __set__(self, obj, value):
        obj.__dict__.update(_cons=value, _pend=[], _front=None)

    @staticmethod
    def fresh(obj, count: int):
        """A new all-unspent mask: the pure-prefix state with front 0."""
        obj.__dict__.update(_cons=np.zeros(count, dtype=bool), _pend=[], _front=0)

    @staticmethod
    def take_prefix(obj, m: int):
        """Spend [front, front + m) if the mask is a pure prefix with room;
        returns the start of the range or None (caller takes the slow path)."""
        d = obj.__dict__
        front = d.get("_front")
        if front is None or front + m > d["_cons"].shape[0]:
            return None
        if m:
            pend = d["_pend"]
            if pend and pend[-1][1] == front:
                pend[-1] = (pend[-1][0], front + m)
            else:
                pend.append((front, front + m))
        d["_front"] = front + m
        return front


@dataclass
class EqKeyBatch:
    """One party's batch of equality keys (struct-of-arrays, fss.py:71-105)."""

    party: int
    n_bits: int
    alpha_share: torch.Tensor   # (count,) u64
    seed0: torch.Tensor         # (count, 16) u8
    scw: torch.Tensor           # (n, count, 16) u8 seed corrections
    tcw: torch.Tensor           # (n, count) u8: bit0 = left t, bit1 = right t
    cw_final: torch.Tensor      # (count,) u64
    consumed: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.consumed is None:
            _ConsumedMask.fresh(self, self.count)

    @property
    def count(self) -> int:
        lz = self.__dict__.get("_lazy")
        return lz[2] if lz is not None else int(self.alpha_share.shape[0])

    @property
    def device(self):
        lz = self.__dict__.get("_lazy")
        return (lz[0]["alpha_share"] if lz is not None else self.alpha_share).device

    def __getattr__(self, name):   # reached only for names missing from __dict__
        return _lazy_field(self, name)

    def validate(self):
        n, count = self.n_bits, self.count
        if tuple(self.scw.shape) != (n, count, 16) or tuple(self.tcw.shape) != (n, count):
            raise KeyFormatError("correction word arrays do not match n_bits/count")
        if tuple(self.seed0.shape) != (count, 16) or tuple(self.cw_final.shape) != (count,):
            raise KeyFormatError("seed/final arrays do not match count")
        _check_party_tensors(self, ("seed0", "scw", "tcw", "cw_final"))

    def take(self, idx, _consumed=None) -> "EqKeyBatch":
        sel, arr = _index(idx, self.count, self.device)
        return _inherit_ready(self, EqKeyBatch(
            self.party, self.n_bits, _take1(self.alpha_share, sel), _take1(self.seed0, sel),
            _take2(self.scw, sel), _take2(self.tcw, sel), _take1(self.cw_final, sel),
            self.consumed[arr].copy() if _consumed is None else _consumed), sel)

    def take_unused(self, m: int) -> "EqKeyBatch":
        return _take_unused(self, m)


@dataclass
class CmpKeyBatch:
    """One party's batch of comparison keys (fss.py:108-154)."""

    party: int
    n_bits: int
    alpha_share: torch.Tensor   # (count,) u64
    seed0: torch.Tensor         # (count, 16) u8
    scw: torch.Tensor           # (n, count, 16) u8
    tcw: torch.Tensor           # (n, count) u8: bits 0..3 = tL, tR, tauL, tauR
    sigma_cw: torch.Tensor      # (n, count) u64
    leaf_cw: torch.Tensor       # (n+1, count) u64
    consumed: np.ndarray = field(default=None)
    out_bits: int = None

    def __post_init__(self):
        if self.consumed is None:
            _ConsumedMask.fresh(self, self.count)
        if self.out_bits is None:
            self.out_bits = self.n_bits

    @property
    def count(self) -> int:
        lz = self.__dict__.get("_lazy")
        return lz[2] if lz is not None else int(self.alpha_share.shape[0])

    @property
    def device(self):
        lz = self.__dict__.get("_lazy")
        return (lz[0]["alpha_share"] if lz is not None else self.alpha_share).device

    def __getattr__(self, name):   # reached only for names missing from __dict__
        return _lazy_field(self, name)

    def validate(self):
        n, count = self.n_bits, self.count
        if tuple(self.scw.shape) != (n, count, 16) or tuple(self.tcw.shape) != (n, count):
            raise KeyFormatError("correction word arrays do not match n_bits/count")
        if tuple(self.sigma_cw.shape) != (n, count) or tuple(self.leaf_cw.shape) != (n + 1, count):
            raise KeyFormatError("sigma/leaf arrays do not match n_bits/count")
        if tuple(self.seed0.shape) != (count, 16):
            raise KeyFormatError("seed array does not match count")
        _check_party_tensors(self, ("seed0", "scw", "tcw", "sigma_cw", "leaf_cw"))

    def take(self, idx, _consumed=None) -> "CmpKeyBatch":
        sel, arr = _index(idx, self.count, self.device)
        return _inherit_ready(self, CmpKeyBatch(
            self.party, self.n_bits, _take1(self.alpha_share, sel), _take1(self.seed0, sel),
            _take2(self.scw, sel), _take2(self.tcw, sel), _take2(self.sigma_cw, sel),
            _take2(self.leaf_cw, sel), self.consumed[arr].copy() if _consumed is None else _consumed,
            self.out_bits), sel)

    def take_unused(self, m: int) -> "CmpKeyBatch":
        return _take_unused(self, m)


@dataclass
class PackedKeyBatch:
    """One party's keys kept as their ARNK payload rows (count, elem) u8 on the
    device -- the element-major container layout of ``_pack_eq`` /
    ``_pack_cmp`` (fss.py:540-583, LAYOUT.md:48-71) -- instead of the
    level-major arrays. ``eval_eq`` / ``eval_cmp`` / ``sign_protocol`` /
    ``eq_protocol`` accept it and evaluate straight from the rows
    (fss_*_eval_packed), so a party that loads a key file
    (``keyfile.load_keys(..., packed=True)``) skips the unpack pass. New (no
    reference counterpart); ``unpack()`` gives the reference's typed batch."""

    kind: int                  # KIND_EQ / KIND_CMP
    party: int
    n_bits: int
    payload: torch.Tensor      # (count, elem_bytes) u8, device
    consumed: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.consumed is None:
            _ConsumedMask.fresh(self, self.count)

    @property
    def count(self) -> int:
        return int(self.payload.shape[0])

    @property
    def device(self):
        return self.payload.device

    @property
    def out_bits(self) -> int:
        return self.n_bits              # a container carries one ring width

    @property
    def alpha_share(self) -> torch.Tensor:
        """The w-byte little-endian alpha share at the front of every row."""
        w = _ring_width_bytes(self.n_bits)
        b = self.payload[:, :w].to(torch.int64)
        v = torch.zeros(self.count, dtype=torch.int64, device=self.device)
        for i in range(w):
            v |= b[:, i] << (8 * i)
        return v.view(torch.uint64)

    def validate(self):
        elem = eq_elem_bytes(self.n_bits) if self.kind == KIND_EQ else cmp_elem_bytes(self.n_bits)
        if self.kind not in (KIND_EQ, KIND_CMP):
            raise KeyFormatError(f"unknown key kind {self.kind}")
        if not isinstance(self.payload, torch.Tensor) or not self.payload.is_cuda:
            raise KeyFormatError("payload must be a device tensor")
        if self.payload.dtype != torch.uint8 or self.payload.ndim != 2 or self.payload.shape[1] != elem:
            raise KeyFormatError(f"payload must be (count, {elem}) uint8")
        if not self.payload.is_contiguous():
            raise KeyFormatError("payload rows must be contiguous")

    def take(self, idx, _consumed=None) -> "PackedKeyBatch":
        sel, arr = _index(idx, self.count, self.device)
        return PackedKeyBatch(self.kind, self.party, self.n_bits, _take1(self.payload, sel),
                              self.consumed[arr].copy() if _consumed is None else _consumed)

    def take_unused(self, m: int) -> "PackedKeyBatch":
        return _take_unused(self, m)

    def unpack(self):
        """The reference's typed batch (EqKeyBatch / CmpKeyBatch)."""
        self.validate()
        k = _unpack(self.kind, self.party, self.n_bits, self.count, self.payload.reshape(-1), self.device)
        k.consumed = self.consumed.copy()
        return k


for _cls in (EqKeyBatch, CmpKeyBatch, PackedKeyBatch):
    _cls.consumed = _ConsumedMask()   # after @dataclass: __init__ keeps its consumed=None default


def _eval_packed(party: int, k: PackedKeyBatch, x, out, m_own=None, m_peer=None):
    """Evaluation straight from payload rows (fss_dcf/dpf_eval_packed)."""
    k.validate()
    fn = "fss_dcf_eval_packed" if k.kind == KIND_CMP else "fss_dpf_eval_packed"
    n, count, dev = k.n_bits, k.count, k.device
    if m_own is not None:          # the masked round's opening happens in the kernel
        res = torch.empty(count, dtype=torch.uint64, device=dev)
        with _dev.on(dev):
            _lib.call(fn, int(party), n, count, _dev.ptr(k.payload), None, _dev.ptr(m_own),
                      _dev.ptr(m_peer), _dev.ptr(res), _dev.stream_handle(dev))
        return res
    out = _check_out(out, count, dev)
    xt, host = _prep_x(x, count, n, dev)

    def launch(xd, od, stream):
        with _dev.on(dev):
            _lib.call(fn, int(party), n, count, _dev.ptr(k.payload), _dev.ptr(xd), None, None,
                      _dev.ptr(od), stream)
    return _run_eval(launch, xt, host, count, dev, None, out)


_SPENT = np.ones(0, dtype=bool)


def _lazy_slice(batch, lo: int, m: int):
    """The lazy form of batch.take(slice(lo, lo + m)) for a spent hand-out, or
    None when the batch is not a ready level-major batch with contiguous
    per-element arrays (the caller then takes the eager views)."""
    if m == 0 or type(batch) not in (EqKeyBatch, CmpKeyBatch):
        return None
    d = batch.__dict__
    c = d.get("_ready")
    if c is None or "_lazy" in d or not _same_key(c[0], _ready_key(batch)):
        return None
    names = _LAZY_NAMES[type(batch)]
    P = {n: d[n] for n in names}
    if not (P["alpha_share"].is_contiguous() and P["seed0"].is_contiguous()
            and ("cw_final" not in P or P["cw_final"].is_contiguous())):
        return None
    child = object.__new__(type(batch))
    cd = child.__dict__
    cd.update(party=batch.party, n_bits=batch.n_bits, _lazy=(P, lo, m, c[1]))
    if type(batch) is CmpKeyBatch:
        cd["out_bits"] = batch.out_bits
    cd.update(_cons=_spent(m), _pend=[], _front=None)   # the consumed field: all spent
    return child


def _spent(m: int) -> np.ndarray:
    """A read-only all-True mask of m keys: the ``consumed`` field of a batch
    handed out by take_unused (every key of it is spent). One shared buffer,
    so a hand-out of millions of keys costs no mask allocation or copy."""
    global _SPENT
    if _SPENT.shape[0] < m:
        buf = np.ones(max(m, 2 * _SPENT.shape[0]), dtype=bool)
        buf.setflags(write=False)
        _SPENT = buf
    return _SPENT[:m]


def _take_unused(batch, m: int):
    """Single-use key hand-out (fss.py:157-166): the first m unconsumed keys.

    Keys are normally spent front to back. ``_free_hint`` h keeps the invariant
    consumed[:h] all True (consuming more keys never breaks it), so when
    consumed[h : h+m] are all free they ARE the first m free keys and go out as
    one contiguous zero-copy slice in O(m); otherwise the full scan is used.
    The handed-out batch is spent: its mask is a read-only all-True view."""
    _prime_ready(batch)
    if isinstance(getattr(type(batch), "consumed", None), _ConsumedMask):
        lo = _ConsumedMask.take_prefix(batch, m)
        if lo is not None:                 # O(1): no mask scan, no mask write now
            batch._free_hint = lo + m
            lazy = _lazy_slice(batch, lo, m)
            if lazy is not None:
                return lazy
            return batch.take(slice(lo, lo + m), _consumed=_spent(m))
    consumed = batch.consumed
    count = consumed.shape[0]
    h = min(getattr(batch, "_free_hint", 0), count)
    if h and not consumed[h - 1]:   # mask was replaced / edited: drop the hint
        h = 0
    if m == 0 or (h + m <= count and not consumed[h:h + m].any()):
        out = batch.take(slice(h, h + m), _consumed=_spent(m))
        if m:
            consumed[h:h + m] = True
        batch._free_hint = h + m
        return out
    free = np.flatnonzero(~consumed)
    if free.size < m:
        raise KeyExhaustedError(
            f"requested {m} keys but only {free.size} unconsumed remain (single-use)")
    idx = free[:m]
    out = batch.take(idx, _consumed=_spent(m))   # the view itself is spent once handed out
    consumed[idx] = True
    # everything before the next free key is now consumed
    batch._free_hint = int(free[m]) if free.size > m else count
    return out


# ---------------------------------------------------------------------------
# Randomness tape: numpy's Generator(PCG64) stream reproduced on device
# ---------------------------------------------------------------------------

def _device_tape_ok(n: int, rng) -> bool:
    return 1 <= n <= 63 and _pcg.is_pcg64(rng)


def _sample_tape(n: int, rng, count: int, alpha, device, shard=None, defer=None):
    """fss._sample_tape (fss.py:292-303): draw order alpha (unless given),
    alpha0, s0, s1 -- bit-identical to the reference's numpy draws.

    ``shard=(lo, m)`` materialises only the element slice [lo, lo + m) of the
    ``count``-element tape (a given ``alpha`` is then the slice's, shape (m,));
    ``rng`` still advances past the whole tape (see shard.py).

    ``defer`` (a list): on the device-tape paths the advance of ``rng`` (a
    128-bit LCG jump in Python, ~15 us) is appended as a callable instead of
    run, so keygen can launch its kernel first and advance the generator while
    the GPU works; the caller runs it before returning."""
    if shard is not None:
        return _sample_tape_slice(n, rng, count, alpha, device, *shard, defer=defer)
    if alpha is not None:
        alpha_t = _dev.to_device_u64(alpha, device)
        if tuple(alpha_t.shape) != (count,):
            raise ValueError("alpha must have shape (count,)")
        from . import ring_ops
        alpha_t = ring_ops.mask(alpha_t, n)
    if n == 64 and _pcg.is_pcg64(rng):
        # fss._uniform_ring's n == 64 branch (fss.py:48-50) is RingTensor.random's
        # two-call draw: the ring kernel, then the seeds-only tape
        from .ring import RingTensor
        a = alpha_t if alpha is not None else RingTensor.random((count,), 64, rng, device).data
        a0 = RingTensor.random((count,), 64, rng, device).data
        s0 = torch.empty((count, 16), dtype=torch.uint8, device=device)
        s1 = torch.empty((count, 16), dtype=torch.uint8, device=device)
        cst, st = _pcg.snapshot(rng)
        out_st = PcgState()
        with _dev.on(device):
            _lib.call("fss_pcg64_seeds", cst, count, _dev.ptr(s0), _dev.ptr(s1), out_st,
                      _dev.stream_handle(device))
        _pcg.commit(rng, st, out_st, count > 0)
        return a, a0, s0, s1
    if not _device_tape_ok(n, rng):
        # a non-PCG64 bit generator (MT19937, Philox, ...): the randomness source
        # is the caller's own host generator, drawn with the reference's calls.
        return _sample_tape_host(n, rng, count, alpha_t if alpha is not None else None, device)
    cst, st = _pcg.snapshot(rng)
    out_st = PcgState()
    draw_alpha = alpha is None
    a = torch.empty(count, dtype=torch.uint64, device=device) if draw_alpha else alpha_t
    a0 = torch.empty(count, dtype=torch.uint64, device=device)
    s0 = torch.empty((count, 16), dtype=torch.uint8, device=device)
    s1 = torch.empty((count, 16), dtype=torch.uint8, device=device)
    with _dev.on(device):
        _lib.call("fss_pcg64_tape", cst, n, count, int(draw_alpha),
                  _dev.ptr(a) if draw_alpha else None, _dev.ptr(a0), _dev.ptr(s0), _dev.ptr(s1),
                  out_st, _dev.stream_handle(device))
    _commit(rng, st, out_st, count > 0, defer)   # advance the caller's rng exactly as numpy would
    return a, a0, s0, s1


def _commit(rng, st, out_st, drawn: bool, defer):
    if defer is None:
        _pcg.commit(rng, st, out_st, drawn)
    else:
        defer.append(lambda: _pcg.commit(rng, st, out_st, drawn))


def _sample_tape_slice(n: int, rng, count: int, alpha, device, lo: int, m: int, defer=None):
    if not (0 <= lo and 0 <= m and lo + m <= count):
        raise ValueError(f"tape slice [{lo}, {lo + m}) outside a tape of {count}")
    alpha_t = None
    if alpha is not None:
        alpha_t = _dev.to_device_u64(alpha, device)
        if tuple(alpha_t.shape) != (m,):
            raise ValueError("alpha must have shape (slice length,)")
        from . import ring_ops
        alpha_t = ring_ops.mask(alpha_t, n)
    if not _device_tape_ok(n, rng):
        # n = 64 (RingTensor.random two-call draw) or a non-PCG64 generator: draw
        # the whole tape (on device / from the caller's generator) and keep the
        # slice. Only the n <= 63 PCG64 path generates the slice alone.
        full_alpha = None if alpha is None else torch.zeros(count, dtype=torch.uint64, device=device)
        a, a0, s0, s1 = _sample_tape(n, rng, count, full_alpha, device)
        a = alpha_t if alpha is not None else a[lo:lo + m].clone()
        return a, a0[lo:lo + m].clone(), s0[lo:lo + m].clone(), s1[lo:lo + m].clone()
    cst, st = _pcg.snapshot(rng)
    out_st = PcgState()
    draw_alpha = alpha is None
    a = torch.empty(m, dtype=torch.uint64, device=device) if draw_alpha else alpha_t
    a0 = torch.empty(m, dtype=torch.uint64, device=device)
    s0 = torch.empty((m, 16), dtype=torch.uint8, device=device)
    s1 = torch.empty((m, 16), dtype=torch.uint8, device=device)
    with _dev.on(device):
        _lib.call("fss_pcg64_tape_slice", cst, n, count, lo, m, int(draw_alpha),
                  _dev.ptr(a) if draw_alpha else None, _dev.ptr(a0), _dev.ptr(s0), _dev.ptr(s1),
                  out_st, _dev.stream_handle(device))
    _commit(rng, st, out_st, count > 0, defer)   # the generator moves past the WHOLE tape
    return a, a0, s0, s1


def _uniform_ring_host(rng, count, n):
    # fss._uniform_ring (fss.py:47-51) -- the reference's own numpy calls
    if n == 64:
        hi = rng.integers(0, 1 << 63, size=count, dtype=np.uint64) << np.uint64(1)
        return hi | rng.integers(0, 2, size=count, dtype=np.uint64)
    return rng.integers(0, 1 << n, size=count, dtype=np.uint64)


def _sample_tape_host(n, rng, count, alpha_t, device):
    a = alpha_t if alpha_t is not None else _dev.to_device_u64(_uniform_ring_host(rng, count, n), device)
    a0 = _dev.to_device_u64(_uniform_ring_host(rng, count, n), device)
    s0 = _dev.to_device_u8(prg.random_seeds(rng, count), device)
    s1 = _dev.to_device_u8(prg.random_seeds(rng, count), device)
    return a, a0, s0, s1


# ---------------------------------------------------------------------------
# Key generation (fss.py:173-340)
# ---------------------------------------------------------------------------

def _keygen_eq_core(n: int, alpha, alpha0, s0_init, s1_init):
    """fss._keygen_eq_core (fss.py:173-216) on device (fss_dpf_keygen)."""
    dev = alpha.device
    count = int(alpha.shape[0])
    alpha, alpha0 = alpha.contiguous(), alpha0.contiguous()
    s0_init, s1_init = s0_init.contiguous(), s1_init.contiguous()
    scw = torch.empty((n, count, 16), dtype=torch.uint8, device=dev)
    tcw = torch.empty((n, count), dtype=torch.uint8, device=dev)
    cw_final = torch.empty(count, dtype=torch.uint64, device=dev)
    alpha1 = torch.empty(count, dtype=torch.uint64, device=dev)
    with _dev.on(dev):
        _lib.call("fss_dpf_keygen", n, count, _dev.ptr(alpha), _dev.ptr(alpha0), _dev.ptr(s0_init),
                  _dev.ptr(s1_init), _dev.ptr(scw), _dev.ptr(tcw), _dev.ptr(cw_final),
                  _dev.ptr(alpha1), _dev.stream_handle(dev))
    k0 = EqKeyBatch(0, n, alpha0, s0_init, scw, tcw, cw_final)
    k1 = EqKeyBatch(1, n, alpha1, s1_init, scw, tcw, cw_final)
    return _born_ready(k0, count), _born_ready(k1, count)


def _keygen_cmp_core(n: int, alpha, alpha0, s0_init, s1_init, out_bits: int = None):
    """fss._keygen_cmp_core (fss.py:219-289) on device (fss_dcf_keygen)."""
    out_bits = n if out_bits is None else out_bits
    dev = alpha.device
    count = int(alpha.shape[0])
    alpha, alpha0 = alpha.contiguous(), alpha0.contiguous()
    s0_init, s1_init = s0_init.contiguous(), s1_init.contiguous()
    scw = torch.empty((n, count, 16), dtype=torch.uint8, device=dev)
    tcw = torch.empty((n, count), dtype=torch.uint8, device=dev)
    sigma_cw = torch.empty((n, count), dtype=torch.uint64, device=dev)
    leaf_cw = torch.empty((n + 1, count), dtype=torch.uint64, device=dev)
    alpha1 = torch.empty(count, dtype=torch.uint64, device=dev)
    with _dev.on(dev):
        _lib.call("fss_dcf_keygen", n, out_bits, count, _dev.ptr(alpha), _dev.ptr(alpha0),
                  _dev.ptr(s0_init), _dev.ptr(s1_init), _dev.ptr(scw), _dev.ptr(tcw),
                  _dev.ptr(sigma_cw), _dev.ptr(leaf_cw), _dev.ptr(alpha1), _dev.stream_handle(dev))
    k0 = CmpKeyBatch(0, n, alpha0, s0_init, scw, tcw, sigma_cw, leaf_cw, out_bits=out_bits)
    k1 = CmpKeyBatch(1, n, alpha1, s1_init, scw, tcw, sigma_cw, leaf_cw, out_bits=out_bits)
    return _born_ready(k0, count), _born_ready(k1, count)


def keygen_eq(n: int, rng: np.random.Generator, count: int = 1,
              alpha=None, device=None, _shard=None):
    """Generate ``count`` equality key pairs; returns (alpha, k0, k1) (fss.py:306-313).
    ``_shard=(lo, m)``: only keys [lo, lo + m) of the batch (shard.keygen_eq_shard)."""
    if not 4 <= n <= 64:
        raise ValueError("equality keys support 4 <= n <= 64")
    dev = _dev.default_device(device)
    pending = []
    try:
        a, a0, s0, s1 = _sample_tape(n, rng, count, alpha, dev, _shard, pending)
        k0, k1 = _keygen_eq_core(n, a, a0, s0, s1)
    finally:
        for advance in pending:   # the generator moves while the keygen kernel runs
            advance()
    return a, k0, k1


def keygen_eq_with_tape(n: int, rng: np.random.Generator, count: int = 1, device=None):
    alpha, k0, k1 = keygen_eq(n, rng, count, device=device)
    return alpha, k0, k1, FssTape(alpha, k0.seed0.clone(), k1.seed0.clone())


def keygen_cmp(n: int, rng: np.random.Generator, count: int = 1,
               alpha=None, out_bits: int = None, device=None, _shard=None):
    """Generate ``count`` comparison key pairs; returns (alpha, k0, k1) (fss.py:321-335).
    ``_shard=(lo, m)``: only keys [lo, lo + m) of the batch (shard.keygen_cmp_shard)."""
    if not 4 <= n <= 63:
        raise ValueError("comparison keys support 4 <= n <= 63")
    if out_bits is not None and not n <= out_bits <= 63:
        raise ValueError("out_bits must lie in [n, 63]")
    dev = _dev.default_device(device)
    pending = []
    try:
        a, a0, s0, s1 = _sample_tape(n, rng, count, alpha, dev, _shard, pending)
        k0, k1 = _keygen_cmp_core(n, a, a0, s0, s1, out_bits)
    finally:
        for advance in pending:   # the generator moves while the keygen kernel runs
            advance()
    return a, k0, k1


def keygen_cmp_with_tape(n: int, rng: np.random.Generator, count: int = 1, device=None):
    alpha, k0, k1 = keygen_cmp(n, rng, count, device=device)
    return alpha, k0, k1, FssTape(alpha, k0.seed0.clone(), k1.seed0.clone())


# ---------------------------------------------------------------------------
# Evaluation (fss.py:347-426)
# ---------------------------------------------------------------------------

def _broadcast_x(x, count: int, n: int, device):
    """fss._broadcast_x (fss.py:347-354); reduction mod 2^n happens in-kernel."""
    host = not isinstance(x, torch.Tensor)
    if host:
        arr = np.asarray(x, dtype=np.uint64) & ring_mask(n)
        if arr.ndim == 0:
            arr = np.full(count, arr, dtype=np.uint64)
        arr = arr.reshape(-1)
        if arr.shape[0] != count:
            raise ValueError(f"need one public input per key: {arr.shape[0]} != {count}")
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(device)
    else:
        if not x.is_cuda:
            host = "torch"  # host torch tensor (pinned for async copies): result comes back to host
        t = _dev.to_device_u64(x, device).reshape(-1)
        if t.numel() == 1 and count != 1:
            t = t.expand(count).contiguous()
        if t.shape[0] != count:
            raise ValueError(f"need one public input per key: {t.shape[0]} != {count}")
    return t, host


def _result(t: torch.Tensor, host):
    if not host:
        return t
    if host == "torch":
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return out
    return _dev.to_numpy(t)


def _level_stride(k, names) -> Optional[int]:
    """Common element stride of the level-major arrays, or None if not uniform."""
    ld = k.scw.stride(0) // 16 if k.scw.ndim == 3 and k.scw.shape[0] else k.count
    if k.scw.ndim == 3 and k.scw.shape[0] and (k.scw.stride(1) != 16 or k.scw.stride(2) != 1):
        return None
    for name in names:
        t = getattr(k, name)
        if t.shape[0] > 1 and (t.stride(0) != ld or t.stride(1) != 1):
            return None
        if t.shape[0] <= 1 and t.numel() and t.stride(-1) != 1:
            return None
    return max(ld, 1)


def _eval_operands(k, names):
    ld = _level_stride(k, names)
    if ld is None:
        for name in ("scw",) + tuple(names):
            setattr(k, name, getattr(k, name).contiguous())
        ld = max(k.count, 1)
    return ld


_EQ_LEVEL = ("tcw",)
_CMP_LEVEL = ("tcw", "sigma_cw", "leaf_cw")
_LAZY_NAMES = {EqKeyBatch: ("alpha_share", "seed0", "scw", "tcw", "cw_final"),
               CmpKeyBatch: ("alpha_share", "seed0", "scw", "tcw", "sigma_cw", "leaf_cw")}


def _ready_key(k):
    """Identity of a batch's arrays: while the fields hold the same tensor
    objects, validate() and the level-stride probe need not run again
    (assigning a field -- the way a batch's arrays are replaced -- changes it;
    key tensors are never resized in place)."""
    if isinstance(k, EqKeyBatch):
        return (k.n_bits, k.alpha_share, k.seed0, k.scw, k.tcw, k.cw_final)
    return (k.n_bits, k.out_bits, k.alpha_share, k.seed0, k.scw, k.tcw, k.sigma_cw, k.leaf_cw)


def _ready(k, names) -> int:
    """validate() + the common level stride of the level-major arrays, cached
    on the batch while its arrays stay the same objects; a contiguous take()
    of a ready batch inherits it (column views keep the level stride), so the
    batches take_unused hands to the online protocols skip both."""
    names_all = _LAZY_NAMES.get(type(k))
    lz = _lazy_ptrs(k, names_all) if names_all else None
    if lz is not None:      # an unassigned take_unused slice: the parent's check holds
        return lz[3]
    c = k.__dict__.get("_ready")
    if c is not None and _same_key(c[0], _ready_key(k)):
        return c[1]
    k.validate()
    ld = _eval_operands(k, names)
    k.__dict__["_ready"] = (_ready_key(k), ld)
    return ld


def _same_key(a, b) -> bool:
    return len(a) == len(b) and all(x is y or (type(x) is not torch.Tensor and x == y) for x, y in zip(a, b))


def _prime_ready(k):
    """Validate a batch once before it hands out keys, so the contiguous
    views that ``take_unused`` returns inherit the cached check (without it
    every online call would re-validate its fresh view). Never re-lays out
    the parent: a batch without a uniform level stride stays unprimed."""
    if not isinstance(k, (EqKeyBatch, CmpKeyBatch)) or "_ready" in k.__dict__:
        return
    try:
        k.validate()
    except KeyFormatError:
        return          # reported where the keys are used, as before
    ld = _level_stride(k, _EQ_LEVEL if isinstance(k, EqKeyBatch) else _CMP_LEVEL)
    if ld is not None:
        k.__dict__["_ready"] = (_ready_key(k), ld)


def _born_ready(k, count: int):
    """Mark a batch that keygen just built from fresh contiguous arrays of the
    validated shapes as checked, level stride = count (what validate() and the
    stride probe would find): the first take_unused of the online phase then
    skips both."""
    if "_ready" not in k.__dict__:
        k.__dict__["_ready"] = (_ready_key(k), max(count, 1))
    return k


def _inherit_ready(parent, child, sel):
    c = parent.__dict__.get("_ready")
    if isinstance(sel, slice) and c is not None and _same_key(c[0], _ready_key(parent)):
        child.__dict__["_ready"] = (_ready_key(child), c[1])
    return child


# Host-tensor inputs at least this large are streamed through the GPU in
# chunks on two CUDA streams, so the H2D copy of x, the evaluation kernel and
# the D2H copy of the shares of consecutive chunks overlap.
PIPELINE_MIN = 1 << 21
PIPELINE_CHUNK = 1 << 20


def _check_out(out, count: int, dev):
    """A caller-provided destination of the shares: ``count`` u64 words of device
    memory on ``dev`` (a torch tensor, or e.g. a peer-mapped shard.PeerGather slot)."""
    if out is None:
        return None
    if not getattr(out, "is_cuda", False) or torch.device(out.device) != dev:
        raise ValueError(f"out must be device memory on {dev}")
    if out.dtype not in (torch.uint64, torch.int64) or out.numel() != count:
        raise ValueError(f"out must hold {count} 64-bit words")
    if isinstance(out, torch.Tensor) and not out.is_contiguous():
        raise ValueError("out must be contiguous")
    return out


def _run_eval(launch, xt, host, count: int, dev, host_launch=None, out=None):
    """Run the evaluation over [0, count).

    Device input: ``launch(x_dev, out_dev, stream)`` once on the current
    stream. Pinned host torch input: the same launch on the host pointers
    (zero-copy) into a pinned host result. numpy input (pageable) of at least
    PIPELINE_MIN elements: ``host_launch(x_ptr, out_ptr, x_scratch, out_scratch,
    chunk, stage_ptr, stream_a, stream_b)`` -- one native call
    (fss_*_eval_host) staging chunks through pinned slots and streaming them
    over two CUDA streams so the host memcpy, H2D copy, kernel and D2H copy of
    consecutive chunks overlap; returns a numpy array."""
    big = count >= PIPELINE_MIN and host_launch is not None
    if out is not None:
        if host:
            raise ValueError("out= needs a device input x (device in, device out)")
        launch(xt, out, _dev.stream_handle(dev))
        return out
    if host == "torch_pinned":
        # Zero-copy: the evaluation kernel reads x straight from the caller's
        # pinned host buffer and stores the shares into a pinned host buffer
        # (UVA pointers, PCIe transfers issued by the kernel's own loads and
        # stores -- 8 B in and 8 B out per element, ~1 % of what the kernel
        # could stream). No staging copies, no chunk pipeline to fill and drain:
        # 2^24 DCF keys 4.42e8 vs 4.28e8 comparisons/s through the pipeline,
        # 2^20 keys 4.24e8 vs 3.35e8 (scripts/zerocopy_probe.py).
        out_host = torch.empty(count, dtype=torch.uint64, pin_memory=True)
        launch(xt, out_host, _dev.stream_handle(dev))
        torch.cuda.current_stream(dev).synchronize()
        return out_host
    if not big or host != "numpy":
        if host == "numpy":
            xt = torch.from_numpy(xt).to(dev, non_blocking=True)
        out = torch.empty(count, dtype=torch.uint64, device=dev)
        launch(xt, out, _dev.stream_handle(dev))
        return _result(out, {"numpy": True}.get(host, host))
    chunk = PIPELINE_CHUNK
    cur = torch.cuda.current_stream(dev)
    # device scratch on the current stream; the side streams wait for it and the
    # current stream waits for them, so the allocator cannot recycle it early
    scratch = torch.empty((2, 3 * chunk), dtype=torch.uint64, device=dev)   # 3 staging slots
    streams = _dev.side_streams(dev, 2)
    for st in streams:
        st.wait_stream(cur)
    out_host = _host_result(count)
    stage = torch.empty(6 * chunk, dtype=torch.uint64, pin_memory=True)
    host_launch(xt.ctypes.data, out_host.ctypes.data, scratch[0], scratch[1], chunk,
                stage.data_ptr(), streams[0].cuda_stream, streams[1].cuda_stream)
    for st in streams:
        cur.wait_stream(st)
    cur.synchronize()
    return out_host


# numpy results of the staged path up to this many bytes live in pinned memory
# from torch's caching host allocator (a numpy view that keeps the block
# alive): the pages are resident, so the pipeline's copy-out does not
# first-touch a fresh 2^24-element array, and the block is reused by the next
# call once the caller drops the array. Larger results stay plain np.empty.
PINNED_RESULT_MAX = 1 << 30
_PINNED_RESULTS = True


def _host_result(count: int) -> np.ndarray:
    if _PINNED_RESULTS and count * 8 <= PINNED_RESULT_MAX:
        return torch.empty(count, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    return np.empty(count, dtype=np.uint64)


def _prep_x(x, count: int, n: int, dev):
    """_broadcast_x plus the host fast paths (no upload here; the kernels reduce
    x mod 2^n themselves)."""
    if isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.uint64 \
            and x.numel() == count and x.device == dev and x.is_contiguous():
        return x.view(-1), False           # the online protocols' case: nothing to convert
    if isinstance(x, torch.Tensor) and not x.is_cuda and x.is_pinned() and x.is_contiguous() \
            and x.numel() == count and x.dtype in (torch.uint64, torch.int64):
        # contiguous pinned memory only: the zero-copy kernel reads it in place
        # (a non-contiguous view would be copied into pageable memory first)
        return x.reshape(-1), "torch_pinned"
    if isinstance(x, np.ndarray) and x.size == count and count >= PIPELINE_MIN \
            and x.dtype in (np.uint64, np.int64):
        return np.ascontiguousarray(x.reshape(-1)).view(np.uint64), "numpy"
    return _broadcast_x(x, count, n, dev)


def eval_eq(party: int, k: EqKeyBatch, x, out=None):
    """Per-party share of 1[x == alpha] (fss.py:357-377) via fss_dpf_eval.
    ``out``: as for eval_cmp. ``k`` may be a PackedKeyBatch."""
    if isinstance(k, PackedKeyBatch):
        return _eval_packed(party, k, x, out)
    ld = _ready(k, _EQ_LEVEL)
    n, count, dev = k.n_bits, k.count, k.device
    out = _check_out(out, count, dev)
    xt, host = _prep_x(x, count, n, dev)
    seed0, cw_final = k.seed0.contiguous(), k.cw_final.contiguous()

    def launch(xd, od, stream):   # whole batch: no column views to build
        with _dev.on(dev):
            _lib.call("fss_dpf_eval", int(party), n, count, ld, _dev.ptr(seed0), _dev.ptr(k.scw),
                      _dev.ptr(k.tcw), _dev.ptr(cw_final), _dev.ptr(xd), _dev.ptr(od), stream)

    def host_launch(xh, oh, xs, os_, chunk, stage, sa, sb):
        with _dev.on(dev):
            _lib.call("fss_dpf_eval_host", int(party), n, count, ld, _dev.ptr(seed0),
                      _dev.ptr(k.scw), _dev.ptr(k.tcw), _dev.ptr(cw_final), xh, oh,
                      _dev.ptr(xs), _dev.ptr(os_), chunk, stage, sa, sb)
    return _run_eval(launch, xt, host, count, dev, host_launch, out)


def eval_cmp(party: int, k: CmpKeyBatch, x, return_levels: bool = False, out=None):
    """Per-party share of 1[x <= alpha] (fss.py:380-426) via fss_dcf_eval.

    With return_levels the per-level output terms are also returned,
    shape (n+1, count); at most one level reconstructs to 1. ``out`` (device
    input only, extension): write the shares into this device buffer of count
    u64 words -- e.g. a slot of another GPU's gather buffer (shard.PeerGather),
    so the kernel's stores are the output collective. ``k`` may be a
    PackedKeyBatch (evaluated straight from its ARNK rows)."""
    if isinstance(k, PackedKeyBatch):
        if return_levels:
            return eval_cmp(party, k.unpack(), x, return_levels=True)
        return _eval_packed(party, k, x, out)
    ld = _ready(k, _CMP_LEVEL)
    n, count, dev = k.n_bits, k.count, k.device
    out = _check_out(out, count, dev)
    if out is not None and return_levels:
        raise ValueError("out= and return_levels are exclusive")
    xt, host = _prep_x(x, count, n, dev)
    seed0 = k.seed0.contiguous()
    if return_levels:
        if host == "torch_pinned":
            xt, host = xt.to(dev), "torch"
        elif host == "numpy":
            xt, host = torch.from_numpy(xt).to(dev), True
        out = torch.empty(count, dtype=torch.uint64, device=dev)
        levels = torch.empty((n + 1, count), dtype=torch.uint64, device=dev)
        with _dev.on(dev):
            _lib.call("fss_dcf_eval", int(party), n, int(k.out_bits), count, ld, _dev.ptr(seed0),
                      _dev.ptr(k.scw), _dev.ptr(k.tcw), _dev.ptr(k.sigma_cw), _dev.ptr(k.leaf_cw),
                      _dev.ptr(xt), _dev.ptr(out), _dev.ptr(levels), _dev.stream_handle(dev))
        return _result(out, host), _result(levels, host)

    def launch(xd, od, stream):   # whole batch: no column views to build
        with _dev.on(dev):
            _lib.call("fss_dcf_eval", int(party), n, int(k.out_bits), count, ld, _dev.ptr(seed0),
                      _dev.ptr(k.scw), _dev.ptr(k.tcw), _dev.ptr(k.sigma_cw), _dev.ptr(k.leaf_cw),
                      _dev.ptr(xd), _dev.ptr(od), None, stream)

    def host_launch(xh, oh, xs, os_, chunk, stage, sa, sb):
        with _dev.on(dev):
            _lib.call("fss_dcf_eval_host", int(party), n, int(k.out_bits), count, ld,
                      _dev.ptr(seed0), _dev.ptr(k.scw), _dev.ptr(k.tcw), _dev.ptr(k.sigma_cw),
                      _dev.ptr(k.leaf_cw), xh, oh, _dev.ptr(xs), _dev.ptr(os_), chunk, stage,
                      sa, sb)
    return _run_eval(launch, xt, host, count, dev, host_launch, out)


# ---------------------------------------------------------------------------
# Masked-input protocols (fss.py:433-491)
# ---------------------------------------------------------------------------

_sign_probe = None


def set_sign_probe(probe):
    """Install a harness callback probe(party, y_ring, out_ring, n_bits, out_bits)
    fired on every sign invocation (fss.py:436-441). Pass None to uninstall."""
    global _sign_probe
    _sign_probe = probe


def _masked_round(session, y, alpha_share, n: int, op: str):
    """The one online round of mask_and_reveal (sharing.py:214-230) up to the
    opening: returns this party's wire-packed m_j = y_j + alpha_j and the
    peer's. The opening x = m_0 + m_1 happens inside the evaluation kernel."""
    masked = _pack(0, _flat_u64(y.values), _flat_u64(alpha_share), n)
    peer = session.exchange(op, FRAME_MASKED, masked, elements=masked.numel())
    return masked, _peer_wire(peer, n, masked.numel(), masked.device)


def _eval_cmp_masked(party: int, k: CmpKeyBatch, m_own, m_peer) -> torch.Tensor:
    if isinstance(k, PackedKeyBatch):
        return _eval_packed(party, k, None, None, m_own, m_peer)
    lz = _lazy_ptrs(k, ("seed0", "scw", "tcw", "sigma_cw", "leaf_cw"))
    if lz is not None:      # a take_unused slice: pointers into the parent's arrays
        P, lo, count, ld = lz
        dev = P["scw"].device
        ptrs = (P["seed0"].data_ptr() + 16 * lo, P["scw"].data_ptr() + 16 * lo, P["tcw"].data_ptr() + lo,
                P["sigma_cw"].data_ptr() + 8 * lo, P["leaf_cw"].data_ptr() + 8 * lo)
    else:
        ld = _ready(k, _CMP_LEVEL)
        dev, count = k.device, k.count
        ptrs = (_dev.ptr(k.seed0.contiguous()), _dev.ptr(k.scw), _dev.ptr(k.tcw), _dev.ptr(k.sigma_cw),
                _dev.ptr(k.leaf_cw))
    out = torch.empty(count, dtype=torch.uint64, device=dev)
    with _dev.on(dev):
        _lib.call("fss_dcf_eval_masked", int(party), k.n_bits, int(k.out_bits), count, ld, *ptrs,
                  _dev.ptr(m_own), _dev.ptr(m_peer), _dev.ptr(out), _dev.stream_handle(dev))
    return out


def _eval_eq_masked(party: int, k: EqKeyBatch, m_own, m_peer) -> torch.Tensor:
    if isinstance(k, PackedKeyBatch):
        return _eval_packed(party, k, None, None, m_own, m_peer)
    lz = _lazy_ptrs(k, ("seed0", "scw", "tcw", "cw_final"))
    if lz is not None:      # a take_unused slice: pointers into the parent's arrays
        P, lo, count, ld = lz
        dev = P["scw"].device
        ptrs = (P["seed0"].data_ptr() + 16 * lo, P["scw"].data_ptr() + 16 * lo, P["tcw"].data_ptr() + lo,
                P["cw_final"].data_ptr() + 8 * lo)
    else:
        ld = _ready(k, _EQ_LEVEL)
        dev, count = k.device, k.count
        ptrs = (_dev.ptr(k.seed0.contiguous()), _dev.ptr(k.scw), _dev.ptr(k.tcw),
                _dev.ptr(k.cw_final.contiguous()))
    out = torch.empty(count, dtype=torch.uint64, device=dev)
    with _dev.on(dev):
        _lib.call("fss_dpf_eval_masked", int(party), k.n_bits, count, ld, *ptrs, _dev.ptr(m_own),
                  _dev.ptr(m_peer), _dev.ptr(out), _dev.stream_handle(dev))
    return out


def sign_protocol(session, y, keys: CmpKeyBatch):
    """Shares of 1[y <= 0] for an additively shared y. One online round (fss.py:444-473).

    The masked message m_j = y_j + alpha_j is wire-packed on device, exchanged,
    and opened inside the DCF evaluation kernel (fss_dcf_eval_masked)."""
    m = y.values.size
    if keys.out_bits != y.values.n_bits:
        raise ValueError("key output ring does not match the shared input")
    if keys.party != y.party:
        raise ValueError("key batch belongs to the other party")
    ks = keys.take_unused(m)
    if keys.n_bits != y.values.n_bits:
        # Narrow-domain keys: mask and reveal only the low domain bits.
        y = AdditiveShare(y.party, RingTensor(ring_ops.mask(y.values.data, keys.n_bits),
                                              keys.n_bits, _trusted=True), 0)
    m_own, m_peer = _masked_round(session, y, ks.alpha_share, keys.n_bits, "comparison")
    out = _eval_cmp_masked(y.party, ks, m_own, m_peer)
    if _sign_probe is not None:
        _sign_probe(y.party, y.values.data.reshape(-1), out, ks.n_bits, ks.out_bits)
    values = RingTensor(out.reshape(y.values.shape), ks.out_bits, _trusted=True)
    return AdditiveShare(y.party, values, precision=0)


def eq_protocol(session, y, keys: EqKeyBatch):
    """Shares of 1[y == 0] for an additively shared y. One online round, exact (fss.py:476-491)."""
    m = y.values.size
    if keys.n_bits != y.values.n_bits:
        raise ValueError("key ring width does not match the shared input")
    if keys.party != y.party:
        raise ValueError("key batch belongs to the other party")
    ks = keys.take_unused(m)
    m_own, m_peer = _masked_round(session, y, ks.alpha_share, keys.n_bits, "equality")
    out = _eval_eq_masked(y.party, ks, m_own, m_peer)
    values = RingTensor(out.reshape(y.values.shape), y.values.n_bits, _trusted=True)
    return AdditiveShare(y.party, values, precision=0)


# ---------------------------------------------------------------------------
# Serialization (container format in LAYOUT.md; fss.py:498-658)
# ---------------------------------------------------------------------------

@dataclass
class KeyBatch:
    """Dealer-side transport container holding both parties' payloads."""

    kind: int
    n_bits: int
    count: int
    payload0: bytes
    payload1: bytes


def _ring_width_bytes(n: int) -> int:
    return (n + 7) // 8


def eq_elem_bytes(n: int) -> int:
    """Serialized bytes per equality key element (one party), fss.py:513-516."""
    w = _ring_width_bytes(n)
    return w + 16 + n * 17 + w


def cmp_elem_bytes(n: int) -> int:
    """Serialized bytes per comparison key element (one party), fss.py:519-522."""
    w = _ring_width_bytes(n)
    return w + 16 + n * (17 + w) + (n + 1) * w


def cmp_key_bits(n: int, lam: int = LAMBDA) -> int:
    """Theoretical compressed comparison key size in bits (fss.py:525-527)."""
    return n * (lam + 2 * n + 4) + lam + 2 * n


def _pack_device(k) -> torch.Tensor:
    """Element-major ARNK payload of one party as a (count, elem) device tensor."""
    k.validate()
    if isinstance(k, CmpKeyBatch):
        if k.out_bits != k.n_bits:
            raise KeyFormatError("widened-output comparison keys are in-memory only")
        kind, elem, names = KIND_CMP, cmp_elem_bytes(k.n_bits), ("tcw", "sigma_cw", "leaf_cw")
    else:
        kind, elem, names = KIND_EQ, eq_elem_bytes(k.n_bits), ("tcw",)
    dev = k.device
    ld = _eval_operands(k, names)
    alpha, seed0 = k.alpha_share.contiguous(), k.seed0.contiguous()
    buf = torch.empty((k.count, elem), dtype=torch.uint8, device=dev)
    with _dev.on(dev):
        _lib.call("fss_arnk_pack", kind, k.n_bits, k.count, ld, _dev.ptr(alpha), _dev.ptr(seed0),
                  _dev.ptr(k.scw), _dev.ptr(k.tcw),
                  _dev.ptr(k.cw_final.contiguous()) if kind == KIND_EQ else None,
                  _dev.ptr(k.sigma_cw) if kind == KIND_CMP else None,
                  _dev.ptr(k.leaf_cw) if kind == KIND_CMP else None,
                  _dev.ptr(buf), _dev.stream_handle(dev))
    return buf


def _pack_eq(k: EqKeyBatch) -> bytes:
    return _dev.to_numpy(_pack_device(k)).tobytes()


def _pack_cmp(k: CmpKeyBatch) -> bytes:
    if k.out_bits != k.n_bits:
        raise KeyFormatError("widened-output comparison keys are in-memory only")
    return _dev.to_numpy(_pack_device(k)).tobytes()


def _unpack(kind: int, party: int, n: int, count: int, payload, device=None):
    dev = _dev.default_device(device)
    elem = eq_elem_bytes(n) if kind == KIND_EQ else cmp_elem_bytes(n)
    if isinstance(payload, torch.Tensor):
        buf = payload.to(dev).reshape(-1)
    else:
        buf = torch.frombuffer(bytearray(payload), dtype=torch.uint8).to(dev) if len(payload) else \
            torch.empty(0, dtype=torch.uint8, device=dev)
    if buf.numel() != count * elem:
        raise KeyFormatError(f"payload size mismatch: {buf.numel()} != {count * elem}")
    alpha = torch.empty(count, dtype=torch.uint64, device=dev)
    seed0 = torch.empty((count, 16), dtype=torch.uint8, device=dev)
    scw = torch.empty((n, count, 16), dtype=torch.uint8, device=dev)
    tcw = torch.empty((n, count), dtype=torch.uint8, device=dev)
    cw_final = sigma = leaf = None
    if kind == KIND_EQ:
        cw_final = torch.empty(count, dtype=torch.uint64, device=dev)
    else:
        sigma = torch.empty((n, count), dtype=torch.uint64, device=dev)
        leaf = torch.empty((n + 1, count), dtype=torch.uint64, device=dev)
    with _dev.on(dev):
        _lib.call("fss_arnk_unpack", kind, n, count, count, _dev.ptr(buf), _dev.ptr(alpha),
                  _dev.ptr(seed0), _dev.ptr(scw), _dev.ptr(tcw), _dev.ptr(cw_final),
                  _dev.ptr(sigma), _dev.ptr(leaf), _dev.stream_handle(dev))
    if kind == KIND_EQ:
        return EqKeyBatch(party, n, alpha, seed0, scw, tcw, cw_final)
    return CmpKeyBatch(party, n, alpha, seed0, scw, tcw, sigma, leaf)


def _unpack_eq(party: int, n: int, count: int, payload, device=None) -> EqKeyBatch:
    return _unpack(KIND_EQ, party, n, count, payload, device)


def _unpack_cmp(party: int, n: int, count: int, payload, device=None) -> CmpKeyBatch:
    return _unpack(KIND_CMP, party, n, count, payload, device)


def pack_keys(k0, k1) -> KeyBatch:
    """Bundle a key pair into the transport container (fss.py:605-613)."""
    if type(k0) is not type(k1) or k0.n_bits != k1.n_bits or k0.count != k1.count:
        raise ValueError("key batches do not form a pair")
    if isinstance(k0, EqKeyBatch):
        return KeyBatch(KIND_EQ, k0.n_bits, k0.count, _pack_eq(k0), _pack_eq(k1))
    if isinstance(k0, CmpKeyBatch):
        return KeyBatch(KIND_CMP, k0.n_bits, k0.count, _pack_cmp(k0), _pack_cmp(k1))
    if isinstance(k0, PackedKeyBatch):            # already payload rows: no kernel
        if k0.kind != k1.kind:
            raise ValueError("key batches do not form a pair")
        k0.validate()
        k1.validate()
        return KeyBatch(k0.kind, k0.n_bits, k0.count, _dev.to_numpy(k0.payload).tobytes(),
                        _dev.to_numpy(k1.payload).tobytes())
    raise TypeError(f"cannot pack {type(k0)!r}")


def unpack_keys(batch: KeyBatch, device=None):
    """Rebuild the typed key pair from a container (fss.py:616-624)."""
    if batch.kind == KIND_EQ:
        return (_unpack_eq(0, batch.n_bits, batch.count, batch.payload0, device),
                _unpack_eq(1, batch.n_bits, batch.count, batch.payload1, device))
    if batch.kind == KIND_CMP:
        return (_unpack_cmp(0, batch.n_bits, batch.count, batch.payload0, device),
                _unpack_cmp(1, batch.n_bits, batch.count, batch.payload1, device))
    raise KeyFormatError(f"cannot unpack kind {batch.kind}")


def serialize_keys(batch: KeyBatch) -> bytes:
    """ARNK header + both payloads (fss.py:627-630)."""
    header = (MAGIC + bytes([VERSION, batch.kind, batch.n_bits])
              + LAMBDA.to_bytes(2, "little") + batch.count.to_bytes(4, "little"))
    return header + batch.payload0 + batch.payload1


def deserialize_keys(data: bytes) -> KeyBatch:
    """Parse and validate an ARNK container (fss.py:633-658)."""
    if len(data) < _HEADER_BYTES:
        raise KeyFormatError("truncated header")
    if data[:4] != MAGIC:
        raise KeyFormatError("bad magic")
    version, kind, n = data[4], data[5], data[6]
    if version != VERSION:
        raise KeyFormatError(f"unsupported version {version}")
    lam = int.from_bytes(data[7:9], "little")
    if lam != LAMBDA:
        raise KeyFormatError(f"unsupported lambda {lam}")
    count = int.from_bytes(data[9:13], "little")
    body = data[_HEADER_BYTES:]
    if kind == KIND_EQ:
        per = eq_elem_bytes(n) * count
    elif kind == KIND_CMP:
        per = cmp_elem_bytes(n) * count
    elif kind == KIND_TRIPLE:
        if len(body) < 4:
            raise KeyFormatError("truncated triple payload")
        per = int.from_bytes(body[:4], "little") + 4
    else:
        raise KeyFormatError(f"unknown kind {kind}")
    if len(body) != 2 * per:
        raise KeyFormatError(f"payload size mismatch: {len(body)} != {2 * per}")
    return KeyBatch(kind, n, count, body[:per], body[per:])


# ---------------------------------------------------------------------------
# Cut-and-choose audit (fss.py:665-699)
# ---------------------------------------------------------------------------

def audit_keys(k0, k1, tape: FssTape, indices) -> list:
    """Replay keygen from the disclosed tape on device and byte-compare the
    packed keys with the issued ones. Returns the indices that do not match.
    Sampled keys are marked consumed in both batches."""
    from . import ring_ops

    indices = np.asarray(list(indices) if isinstance(indices, range) else indices,
                         dtype=np.int64).reshape(-1)
    if isinstance(k0, PackedKeyBatch):      # audit the unpacked sample, spend it in the packed batches
        sub0, sub1 = k0.take(indices).unpack(), k1.take(indices).unpack()
        k0.consumed[indices] = True
        k1.consumed[indices] = True
        bad = audit_keys(sub0, sub1, tape.take(indices), range(indices.size))
        return [int(indices[j]) for j in bad]
    sub0, sub1 = k0.take(indices), k1.take(indices)
    k0.consumed[indices] = True
    k1.consumed[indices] = True
    t = tape.take(indices)
    if isinstance(k0, EqKeyBatch):
        r0, r1 = _keygen_eq_core(k0.n_bits, t.alpha.contiguous(), sub0.alpha_share.contiguous(),
                                 t.s0.contiguous(), t.s1.contiguous())
    elif isinstance(k0, CmpKeyBatch):
        if k0.out_bits != k0.n_bits:
            raise KeyFormatError("widened-output comparison keys cannot be audited byte-wise")
        r0, r1 = _keygen_cmp_core(k0.n_bits, t.alpha.contiguous(), sub0.alpha_share.contiguous(),
                                  t.s0.contiguous(), t.s1.contiguous())
    else:
        raise TypeError(f"cannot audit {type(k0)!r}")
    if indices.size == 0:
        return []
    ok = (torch.all(_pack_device(sub0) == _pack_device(r0), dim=1)
          & torch.all(_pack_device(sub1) == _pack_device(r1), dim=1))
    recon = ring_ops.binary("add", sub0.alpha_share.contiguous(), sub1.alpha_share.contiguous(),
                            k0.n_bits)
    ok &= _dev.as_i64(recon) == _dev.as_i64(t.alpha.contiguous())
    ok = _dev.to_numpy(ok)
    return [int(i) for i, good in zip(indices, ok) if not good]
