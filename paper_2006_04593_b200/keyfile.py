"""Streaming ARNK key files: dealer -> party key shipping on B200.

The reference ships preprocessing as one ARNK container per batch: the dealer
writes ``serialize_keys(pack_keys(k0, k1))`` to ``{kind}_{n}_{count}.arnk``
(``cli._cmd_keygen``, reference cli.py:195-214) and each party reads the whole
file back, unpacks both payloads and keeps its own (``cli._bench_split_role``,
cli.py:150-160). Both ends go through Python ``bytes`` of the full container.

``save_keys`` / ``load_keys`` produce and consume the identical file, but
stream it in chunks of keys through two pinned host buffers:

* save: device pack of chunk i+1 (``fss_arnk_pack`` on a column view) and its
  D2H copy overlap the file write of chunk i;
* load: the file read of chunk i+1 into pinned memory overlaps the H2D copy
  and the device unpack of chunk i, written straight into its column range of
  the full key arrays (``fss_arnk_unpack`` with the batch's level stride). A
  party reads only its own payload (half the file).

Each chunk is written / read at its file offset by IO_THREADS threads in
parallel (os.pwrite / os.preadv release the GIL).

Nothing of the container is ever materialised whole on the host.
"""

from __future__ import annotations

import os

import torch

from . import _dev, _lib, fss
from .fss import KIND_CMP, KIND_EQ, KeyFormatError

CHUNK = 1 << 18   # keys per chunk (cmp n = 32: 206 MiB per pinned buffer)
IO_THREADS = 4    # positional reads / writes of one chunk run in parallel
_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(IO_THREADS, thread_name_prefix="arnk-io")
    return _POOL


def _split(nbytes: int):
    """Byte ranges of one chunk for the I/O threads (>= 4 MiB each)."""
    parts = max(1, min(IO_THREADS, nbytes >> 22))
    step = -(-nbytes // parts)
    return [(a, min(nbytes, a + step)) for a in range(0, nbytes, step)]


def _pwrite_all(fd: int, mv: memoryview, offset: int):
    """Write mv at file offset with the I/O threads (os.pwrite releases the GIL;
    one core moves only a few GB/s into the page cache)."""
    def one(a, b):
        while a < b:
            a += os.pwrite(fd, mv[a:b], offset + a)
    for f in [_pool().submit(one, a, b) for a, b in _split(len(mv))]:
        f.result()


def _pread_all(fd: int, mv: memoryview, offset: int) -> int:
    def one(a, b):
        got = 0
        while a < b:
            k = os.preadv(fd, [mv[a:b]], offset + a)
            if k == 0:
                break
            a += k
            got += k
        return got
    return sum(f.result() for f in [_pool().submit(one, a, b) for a, b in _split(len(mv))])


def _header(kind: int, n: int, count: int) -> bytes:
    return (fss.MAGIC + bytes([fss.VERSION, kind, n]) + fss.LAMBDA.to_bytes(2, "little")
            + count.to_bytes(4, "little"))


def _elem(kind: int, n: int) -> int:
    return fss.eq_elem_bytes(n) if kind == KIND_EQ else fss.cmp_elem_bytes(n)


def read_header(fh, size: int):
    """Validate an ARNK header against the file size (fss.deserialize_keys,
    reference fss.py:633-658); returns (kind, n, count, per-party bytes)."""
    head = fh.read(fss._HEADER_BYTES)
    if len(head) < fss._HEADER_BYTES:
        raise KeyFormatError("truncated header")
    if head[:4] != fss.MAGIC:
        raise KeyFormatError("bad magic")
    version, kind, n = head[4], head[5], head[6]
    if version != fss.VERSION:
        raise KeyFormatError(f"unsupported version {version}")
    lam = int.from_bytes(head[7:9], "little")
    if lam != fss.LAMBDA:
        raise KeyFormatError(f"unsupported lambda {lam}")
    count = int.from_bytes(head[9:13], "little")
    if kind not in (KIND_EQ, KIND_CMP):
        raise KeyFormatError(f"key file of kind {kind}: only equality / comparison keys stream")
    per = _elem(kind, n) * count
    body = size - fss._HEADER_BYTES
    if body != 2 * per:
        raise KeyFormatError(f"payload size mismatch: {body} != {2 * per}")
    return kind, n, count, per


def save_keys(path, k0, k1, chunk: int = CHUNK) -> int:
    """Write the ARNK container of the key pair (byte-identical to
    ``serialize_keys(pack_keys(k0, k1))``); returns the bytes written."""
    if not isinstance(k0, (fss.EqKeyBatch, fss.CmpKeyBatch, fss.PackedKeyBatch)):
        raise TypeError(f"cannot save {type(k0).__name__} as an ARNK key file")
    if type(k0) is not type(k1) or k0.n_bits != k1.n_bits or k0.count != k1.count:
        raise ValueError("key batches do not form a pair")
    packed = isinstance(k0, fss.PackedKeyBatch)
    if packed:
        # payload rows already hold the container bytes: streamed as they are
        if k0.kind != k1.kind:
            raise ValueError("key batches do not form a pair")
        k0.validate()
        k1.validate()
        kind = k0.kind
    else:
        kind = KIND_EQ if isinstance(k0, fss.EqKeyBatch) else KIND_CMP
    if kind == KIND_CMP and k0.out_bits != k0.n_bits:
        raise KeyFormatError("widened-output comparison keys are in-memory only")
    n, count, dev = k0.n_bits, k0.count, k0.device
    elem = _elem(kind, n)
    chunk = max(1, min(chunk, max(count, 1)))
    pinned = [torch.empty(chunk * elem, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [None, None]
    side = _dev.side_streams(dev, 1)[0]
    written = 0
    per = elem * count
    fd = os.open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
    try:
        os.pwrite(fd, _header(kind, n, count), 0)
        written += fss._HEADER_BYTES
        jobs = [(p, k, lo, min(count, lo + chunk)) for p, k in ((0, k0), (1, k1))
                for lo in range(0, count, chunk)]

        def issue(i):
            _, k, lo, hi = jobs[i]
            b = i & 1
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                if packed:
                    buf = k.payload[lo:hi]                           # the rows themselves
                else:
                    buf = fss._pack_device(k.take(slice(lo, hi)))  # column view: no gather
                pinned[b][: buf.numel()].copy_(buf.reshape(-1), non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
                buf.record_stream(side)
            done[b] = (ev, buf.numel())

        if jobs:
            issue(0)
        for i in range(len(jobs)):
            b = i & 1
            ev, nbytes = done[b]
            if i + 1 < len(jobs):
                issue(i + 1)          # packs into the other pinned buffer meanwhile
            ev.synchronize()
            p, _, lo, _ = jobs[i]
            _pwrite_all(fd, memoryview(pinned[b].numpy())[:nbytes], fss._HEADER_BYTES + p * per + lo * elem)
            written += nbytes
    finally:
        os.close(fd)
    return written


def _alloc(kind: int, party: int, n: int, count: int, dev):
    alpha = torch.empty(count, dtype=torch.uint64, device=dev)
    seed0 = torch.empty((count, 16), dtype=torch.uint8, device=dev)
    scw = torch.empty((n, count, 16), dtype=torch.uint8, device=dev)
    tcw = torch.empty((n, count), dtype=torch.uint8, device=dev)
    if kind == KIND_EQ:
        cw_final = torch.empty(count, dtype=torch.uint64, device=dev)
        return fss.EqKeyBatch(party, n, alpha, seed0, scw, tcw, cw_final)
    sigma = torch.empty((n, count), dtype=torch.uint64, device=dev)
    leaf = torch.empty((n + 1, count), dtype=torch.uint64, device=dev)
    return fss.CmpKeyBatch(party, n, alpha, seed0, scw, tcw, sigma, leaf)


def load_keys(path, party: int = None, device=None, chunk: int = CHUNK, packed: bool = False):
    """Read an ARNK key file into HBM. ``party`` None -> (k0, k1) as
    ``unpack_keys(deserialize_keys(data))``; 0 or 1 -> that party's batch only
    (only its payload is read). ``packed=True``: keep the payload rows as they
    are (fss.PackedKeyBatch, evaluated straight from the rows) -- no unpack
    pass, and 824 instead of 1,088 bytes of HBM per DCF key at n = 32."""
    if party not in (None, 0, 1):
        raise ValueError("party must be 0, 1 or None")
    size = os.path.getsize(path)
    with open(path, "rb", buffering=0) as fh:
        kind, n, count, per = read_header(fh, size)
        dev = _dev.default_device(device)
        elem = _elem(kind, n)
        parties = (0, 1) if party is None else (party,)
        if packed:
            keys = {p: fss.PackedKeyBatch(kind, p, n, torch.empty((count, elem), dtype=torch.uint8,
                                                                  device=dev)) for p in parties}
        else:
            keys = {p: _alloc(kind, p, n, count, dev) for p in parties}
        chunk = max(1, min(chunk, max(count, 1)))
        pinned = [torch.empty(chunk * elem, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        staged = [] if packed else [torch.empty(chunk * elem, dtype=torch.uint8, device=dev) for _ in range(2)]
        used = [None, None]
        stream = torch.cuda.current_stream(dev)
        for p in parties:
            k = keys[p]
            for i, lo in enumerate(range(0, count, chunk)):
                hi = min(count, lo + chunk)
                b = i & 1
                if used[b] is not None:
                    used[b].synchronize()      # the copy that last read this pinned buffer is done
                view = memoryview(pinned[b].numpy())[: (hi - lo) * elem]
                got = _pread_all(fh.fileno(), view, fss._HEADER_BYTES + p * per + lo * elem)
                if got != (hi - lo) * elem:
                    raise KeyFormatError("truncated payload")
                if packed:                     # rows land in place: no unpack
                    k.payload[lo:hi].view(-1).copy_(pinned[b][: (hi - lo) * elem], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(stream)
                    used[b] = ev
                    continue
                dst = staged[b][: (hi - lo) * elem]
                dst.copy_(pinned[b][: (hi - lo) * elem], non_blocking=True)
                with _dev.on(dev):
                    _lib.call("fss_arnk_unpack", kind, n, hi - lo, count, _dev.ptr(dst),
                              _col(k.alpha_share, lo), _col(k.seed0, lo, 16), _col(k.scw, lo, 16),
                              _col(k.tcw, lo), _col(getattr(k, "cw_final", None), lo),
                              _col(getattr(k, "sigma_cw", None), lo), _col(getattr(k, "leaf_cw", None), lo),
                              stream.cuda_stream)
                ev = torch.cuda.Event()
                ev.record(stream)
                used[b] = ev
        torch.cuda.current_stream(dev).synchronize()
    if party is None:
        return keys[0], keys[1]
    return keys[party]


def _col(t, lo: int, width: int = 1):
    """Device pointer of column ``lo`` of a level-major (or element-major) array."""
    if t is None:
        return None
    return t.data_ptr() + lo * width * t.element_size()
