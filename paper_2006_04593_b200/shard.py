"""Element-sharded dealer and output gather across ranks.

Every FSS element is independent, so a batch of ``total`` keys splits into
contiguous slices, one per rank (one process per GPU); each rank holds BOTH
parties' keys for its slice and runs keygen and evaluation with no data-path
collective. This module supplies the two pieces around that:

* ``keygen_cmp_shard`` / ``keygen_eq_shard``: rank r's slice of the keys that
  ``fss.keygen_cmp(n, rng, total)`` would deal on one device -- bit-identical,
  because the randomness tape of the slice is drawn straight from the caller's
  numpy PCG64 stream at the slice's offsets (``fss_pcg64_tape_slice``, LCG
  jump-ahead; no rank generates the other ranks' draws). Every rank passes a
  generator in the same state and every rank's generator then advances past the
  whole ``total``-element tape, exactly as the single-process dealer's would
  (``Dealer._generate``, reference dealer.py:96-103), so successive sharded
  calls stay in lock-step.
* ``gather_shards`` / ``all_gather_shards`` / ``gather_ring``: the one output
  collective of §8e -- the evaluated shares of every slice to rank ``dst`` (or to
  all ranks) for reconstruction; ``gather_ring`` ships them at the ring's wire
  width (4 B per element for n <= 32, the reference's ``pack_ring``,
  sharing.py:191-207) over NCCL.
* ``PeerGather``: the same gather fused into the evaluation -- every rank's eval
  kernel stores its shares straight into rank dst's result buffer through CUDA
  IPC peer memory (``fss.eval_cmp(..., out=gather.out(party))``).

The masked-message exchange between the two parties is the other collective and
lives in ``runtime`` (``DistTransport`` over NCCL, ``PeerTransport`` over peer
memory). Collectives use ``torch.distributed`` (NCCL for CUDA tensors on one
process per GPU; gloo for host tensors in the CPU tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _dev, fss


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced slice [lo, hi) of ``total`` elements owned by ``rank``
    (sizes differ by at most one; ranks in order)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside a world of {world}")
    if total < 0:
        raise ValueError("total must be non-negative")
    return total * rank // world, total * (rank + 1) // world


def _rank_world(rank, world, group=None) -> tuple[int, int]:
    if rank is None or world is None:
        if not (dist.is_available() and dist.is_initialized()):
            raise ValueError("pass rank and world, or initialise torch.distributed")
        rank = dist.get_rank(group) if rank is None else rank
        world = dist.get_world_size(group) if world is None else world
    return int(rank), int(world)


def keygen_cmp_shard(n: int, rng: np.random.Generator, total: int, rank: int = None,
                     world: int = None, alpha=None, out_bits: int = None, device=None, group=None):
    """Rank ``rank``'s slice of ``fss.keygen_cmp(n, rng, total, ...)``: returns
    (alpha, k0, k1) for elements [lo, hi) = ``shard_bounds(total, rank, world)``.
    A given ``alpha`` is the slice's (shape (hi - lo,))."""
    rank, world = _rank_world(rank, world, group)
    lo, hi = shard_bounds(total, rank, world)
    return fss.keygen_cmp(n, rng, total, alpha=alpha, out_bits=out_bits, device=device,
                          _shard=(lo, hi - lo))


def keygen_eq_shard(n: int, rng: np.random.Generator, total: int, rank: int = None,
                    world: int = None, alpha=None, device=None, group=None):
    """Rank ``rank``'s slice of ``fss.keygen_eq(n, rng, total, ...)`` (see keygen_cmp_shard)."""
    rank, world = _rank_world(rank, world, group)
    lo, hi = shard_bounds(total, rank, world)
    return fss.keygen_eq(n, rng, total, alpha=alpha, device=device, _shard=(lo, hi - lo))


def _comm_device(t: torch.Tensor, group=None) -> torch.device:
    # NCCL moves CUDA tensors (NVLink / NVSwitch); gloo moves host tensors
    return t.device if dist.get_backend(group) == "nccl" else torch.device("cpu")


def _collect(t: torch.Tensor, total: int, rank: int, world: int, dst, group):
    lo, hi = shard_bounds(total, rank, world)
    m = hi - lo
    if t.shape[0] != m:
        raise ValueError(f"rank {rank} holds {t.shape[0]} rows, its shard has {m}")
    per = -(-total // world) if world else 0
    tail = tuple(t.shape[1:])
    row_elems = int(np.prod(tail)) if tail else 1
    row_bytes = row_elems * t.element_size()
    dev = _comm_device(t, group)
    buf = torch.zeros((per, row_bytes), dtype=torch.uint8, device=dev)
    if m:
        buf[:m].copy_(t.contiguous().reshape(m, row_elems).view(torch.uint8))
    if dst is None:
        out = torch.empty((world * per, row_bytes), dtype=torch.uint8, device=dev)
        dist.all_gather_into_tensor(out, buf, group=group)
        parts = list(out.split(per))
    else:
        parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
        dist.gather(buf, parts, dst=dst, group=group)
        if rank != dst:
            return None
    rows = [parts[r][: shard_bounds(total, r, world)[1] - shard_bounds(total, r, world)[0]]
            for r in range(world)]
    flat = torch.cat(rows).to(t.device)
    return flat.view(t.dtype).reshape((total,) + tail)


def gather_shards(t: torch.Tensor, total: int, dst: int = 0, group=None):
    """Concatenate every rank's slice (shape (hi - lo, ...), any dtype) on rank
    ``dst``: returns the (total, ...) tensor there and None elsewhere."""
    rank, world = _rank_world(None, None, group)
    return _collect(t, total, rank, world, dst, group)


def all_gather_shards(t: torch.Tensor, total: int, group=None):
    """Every rank receives the concatenation of all slices, shape (total, ...)."""
    rank, world = _rank_world(None, None, group)
    return _collect(t, total, rank, world, None, group)


def gather_ring(values: torch.Tensor, n_bits: int, total: int, dst=0, group=None):
    """``gather_shards`` of ring values (u64, one per element) shipped at the
    ring's wire width (sharing.pack_ring: 4 B per element for n <= 32); the
    result is u64 again. ``dst=None`` gathers to every rank."""
    from . import sharing
    rank, world = _rank_world(None, None, group)
    v = values.reshape(-1)
    wire = sharing.pack_ring(v, n_bits) if v.is_cuda else v
    got = _collect(wire, total, rank, world, dst, group)
    if got is None:
        return None
    return sharing.unpack_ring(got, n_bits) if got.is_cuda else got


class _RawCuda:
    """__cuda_array_interface__ view of raw device memory (zero-copy torch view)."""

    def __init__(self, ptr: int, shape, typestr: str = "<i8"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class PeerGather:
    """The output gather fused with the evaluation over peer memory.

    Rank ``dst`` allocates a (slots, total) u64 result buffer -- one row per
    output, e.g. slot 0 / 1 for the two parties' shares -- and exports it with
    CUDA IPC; every rank maps it. ``out(slot)`` is this rank's [lo, hi) window
    of row ``slot``: passed as ``out=`` to ``fss.eval_cmp`` / ``fss.eval_eq``,
    it makes the evaluation kernel's own stores land in rank dst's HBM (NVLink /
    NVSwitch peer stores; the same HBM when the ranks share a GPU), so there is
    no separate gather collective and no staging copy. ``finish()`` orders the
    writes (stream sync on every rank, then a barrier) and returns the
    (slots, total) u64 tensor on rank dst -- a view valid until ``close()`` --
    and None elsewhere."""

    def __init__(self, total: int, slots: int = 2, dst: int = 0, group=None, device=None):
        import ctypes

        from . import _lib
        self._lib, self.group = _lib, group
        self.rank, self.world = _rank_world(None, None, group)
        self.total, self.slots, self.dst = int(total), int(slots), int(dst)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.lo, self.hi = shard_bounds(self.total, self.rank, self.world)
        hb = _lib.load().fss_ipc_handle_bytes()
        handle = torch.zeros(hb, dtype=torch.uint8)
        self._owned = None
        err, opened = None, False
        with _dev.on(self.device):
            if self.rank == self.dst:
                ptr = ctypes.c_void_p()
                try:
                    _lib.call("fss_ipc_alloc", max(8 * self.slots * self.total, 16), ctypes.byref(ptr))
                    self._owned = self.base = ptr.value
                    buf = (ctypes.c_uint8 * hb)()
                    _lib.call("fss_ipc_get_handle", ptr, buf)
                    handle = torch.tensor(list(buf), dtype=torch.uint8)
                except RuntimeError as e:      # still broadcast (zeros), then agree below
                    err = e
            nccl = dist.get_backend(group) == "nccl"
            comm = handle.to(self.device) if nccl else handle
            dist.broadcast(comm, src=self.dst, group=group)
            if self.rank != self.dst:
                if bool(comm.eq(0).all()):
                    err = "the destination rank exported no buffer"
                else:
                    raw = (ctypes.c_uint8 * hb)(*comm.cpu().tolist())
                    ptr = ctypes.c_void_p()
                    try:
                        _lib.call("fss_ipc_open_handle", raw, ctypes.byref(ptr))
                        self.base, opened = ptr.value, True
                    except RuntimeError as e:
                        err = e
            # every rank learns whether every mapping exists before any store:
            # a rank failing alone would leave the others in finish()'s barrier
            ok = torch.tensor([0 if err else 1], dtype=torch.int64,
                              device=self.device if nccl else "cpu")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            if int(ok.item()) != 1:
                if self._owned is not None:
                    _lib.call("fss_ipc_free", ctypes.c_void_p(self._owned))
                elif opened:
                    _lib.call("fss_ipc_close_handle", ctypes.c_void_p(self.base))
                self._closed = True
                from .runtime import PeerAccessError
                raise PeerAccessError("PeerGather: peer memory mapping failed on "
                                      + (f"this rank: {err}" if err else "another rank"))
        self._closed = False

    def out(self, slot: int):
        """This rank's window of row ``slot`` as a device buffer for ``out=``."""
        from .runtime import PeerBuffer
        if not 0 <= slot < self.slots:
            raise ValueError(f"slot {slot} outside [0, {self.slots})")
        ptr = self.base + 8 * (slot * self.total + self.lo)
        return PeerBuffer(ptr, self.hi - self.lo, torch.uint64, self.device)

    def _barrier(self):
        dist.barrier(group=self.group) if self.group is not None else dist.barrier()

    def finish(self):
        """Every rank's stores are complete and visible: the (slots, total) u64
        result on rank dst, None elsewhere."""
        torch.cuda.current_stream(self.device).synchronize()
        self._barrier()
        if self.rank != self.dst:
            return None
        return torch.as_tensor(_RawCuda(self.base, (self.slots, self.total)),
                               device=self.device).view(torch.uint64)

    def close(self):
        import ctypes
        if self._closed:
            return
        self._closed = True
        torch.cuda.current_stream(self.device).synchronize()
        self._barrier()                      # nobody writes or reads any more
        with _dev.on(self.device):
            if self.rank == self.dst:
                self._lib.call("fss_ipc_free", ctypes.c_void_p(self._owned))
            else:
                self._lib.call("fss_ipc_close_handle", ctypes.c_void_p(self.base))
