"""Drop-in for the reference's ``ariann.runtime`` (pkg/src/ariann/runtime.py):
sessions, framed exchanges and round accounting -- with device-resident
payloads.

The reference moves ``bytes`` frames over queues or TCP (runtime.py:50-210).
Here a payload is a device tensor (the wire-packed ring values produced by the
share layer's kernels) and the transports move it without leaving HBM:

* ``LocalTransport`` -- both parties in one process (one thread each, as
  ``run_local_pair`` in runtime.py:285-311). A send hands the tensor itself to
  the peer together with a CUDA event recorded on the sender's stream; the
  receiver's stream waits on that event, so the exchange is a stream-ordered
  device-to-device hand-off (zero copies, no host round trip).
* ``DistTransport`` -- one party per process (rank), over ``torch.distributed``
  point-to-point (NCCL over NVLink / NVSwitch on GPUs, gloo on CPU for tests).
  A 3-word header (tag, dtype code, numel) precedes each payload so frame
  desync and size errors are detected like the reference's frame checks
  (runtime.py:246-255).

Round semantics are the reference's: one ``exchange`` = one matched send and
receive = one round recorded in the ``RoundLedger`` with the payload bytes.
"""

from __future__ import annotations

import os
import queue
import threading
from dataclasses import dataclass, field

import torch

FRAME_REVEAL = 0x01
FRAME_MASKED = 0x02
FRAME_TRIPLE_DELTA = 0x03
FRAME_CONTROL = 0x04
FRAME_ABORT = 0x05

_FRAME_TAGS = {FRAME_REVEAL, FRAME_MASKED, FRAME_TRIPLE_DELTA, FRAME_CONTROL, FRAME_ABORT}

DEFAULT_TIMEOUT_MS = 30_000


def timeout_seconds() -> float:
    """ARIANN_TIMEOUT_MS, as in runtime.py:36-37."""
    return int(os.environ.get("ARIANN_TIMEOUT_MS", DEFAULT_TIMEOUT_MS)) / 1000.0


class SessionAbort(RuntimeError):
    """Protocol aborted: peer failure, timeout, or frame desync (runtime.py:40-41)."""


@dataclass
class Frame:
    """One message: a tag and a device (or host) tensor payload."""

    tag: int
    payload: torch.Tensor
    event: object = None  # torch.cuda.Event ordering the payload on the sender's stream


@dataclass
class RoundLedger:
    """Per-operation counters of online rounds, bytes, and elements (runtime.py:66-96)."""

    rounds: dict = field(default_factory=dict)
    bytes_sent: dict = field(default_factory=dict)
    bytes_received: dict = field(default_factory=dict)
    elements: dict = field(default_factory=dict)

    def record(self, op: str, sent: int, received: int, elements: int):
        self.rounds[op] = self.rounds.get(op, 0) + 1
        self.bytes_sent[op] = self.bytes_sent.get(op, 0) + sent
        self.bytes_received[op] = self.bytes_received.get(op, 0) + received
        self.elements[op] = self.elements.get(op, 0) + elements

    def total_rounds(self) -> int:
        return sum(self.rounds.values())

    def total_bytes_sent(self) -> int:
        return sum(self.bytes_sent.values())

    def as_dict(self) -> dict:
        return {"rounds": dict(self.rounds), "bytes_sent": dict(self.bytes_sent),
                "bytes_received": dict(self.bytes_received), "elements": dict(self.elements)}

    def snapshot(self) -> dict:
        return {op: n for op, n in self.rounds.items()}


def _nbytes(t: torch.Tensor) -> int:
    return t.numel() * t.element_size()


# ---------------------------------------------------------------------------
# Transports
# ---------------------------------------------------------------------------

class LocalTransport:
    """In-process duplex channel: FIFO queues of device-tensor frames (runtime.py:103-133)."""

    def __init__(self, inbox: queue.Queue, outbox: queue.Queue):
        self._inbox = inbox
        self._outbox = outbox
        self._closed = False

    def send(self, frame: Frame):
        if self._closed:
            raise SessionAbort("transport closed")
        p = frame.payload
        if frame.event is None and isinstance(p, torch.Tensor) and p.is_cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(p.device))
            frame = Frame(frame.tag, p, ev)
        self._outbox.put(frame)

    def recv(self) -> Frame:
        try:
            frame = self._inbox.get(timeout=timeout_seconds())
        except queue.Empty:
            raise SessionAbort("timed out waiting for peer") from None
        if frame is None:
            raise SessionAbort("peer closed the channel")
        if frame.event is not None:
            cur = torch.cuda.current_stream(frame.payload.device)
            cur.wait_event(frame.event)
            # the sender's allocator must not recycle the buffer before we read it
            frame.payload.record_stream(cur)
        return frame

    def close(self):
        if not self._closed:
            self._closed = True
            self._outbox.put(None)


def local_pair() -> tuple[LocalTransport, LocalTransport]:
    a, b = queue.Queue(), queue.Queue()
    return LocalTransport(a, b), LocalTransport(b, a)


_DTYPES = [torch.uint8, torch.int16, torch.int32, torch.int64, torch.uint16, torch.uint32,
           torch.uint64]
_DTYPE_CODE = {d: i for i, d in enumerate(_DTYPES)}
# NCCL / gloo move bytes; unsigned payloads travel as their signed views
_SIGNED = {torch.uint16: torch.int16, torch.uint32: torch.int32, torch.uint64: torch.int64}


class DistTransport:
    """One party per process over torch.distributed point-to-point.

    ``peer`` is the other party's global rank; ``group`` optionally restricts
    the communicator (e.g. a 2-rank pair inside an 8-GPU job). NCCL carries
    device tensors over NVLink / NVSwitch; gloo (CPU tensors) is used by the
    multi-process CPU tests.
    """

    def __init__(self, peer: int, group=None, device=None):
        import torch.distributed as dist
        self._dist = dist
        self.peer = peer
        self.group = group
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device())
            if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        self._closed = False

    def _wire(self, t: torch.Tensor) -> torch.Tensor:
        t = t.contiguous()
        return t.view(_SIGNED[t.dtype]) if t.dtype in _SIGNED else t

    def exchange_frames(self, frame: Frame) -> Frame:
        """Send our frame and receive the peer's (both directions in one batch)."""
        if self._closed:
            raise SessionAbort("transport closed")
        dist = self._dist
        p = frame.payload.to(self.device)
        tag, code, numel = self._swap_header(frame.tag, _DTYPE_CODE[p.dtype], p.numel())
        if frame.tag == FRAME_ABORT:
            # one-way, like the reference's abort frame: the peer raises on our
            # header and never enters the payload phase, so neither do we
            return Frame(tag, torch.empty(0, dtype=torch.uint8))
        if tag == FRAME_ABORT:
            raise SessionAbort("peer aborted")
        if code < 0 or code >= len(_DTYPES):
            raise SessionAbort("corrupt frame header")
        out = torch.empty(numel, dtype=_DTYPES[code], device=self.device)
        ops = []
        if p.numel():
            ops.append(dist.P2POp(dist.isend, self._wire(p).reshape(-1), self.peer, self.group))
        if numel:
            ops.append(dist.P2POp(dist.irecv, self._wire(out), self.peer, self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return Frame(tag, out)

    def _swap_header(self, tag: int, code: int, numel: int, timeout=None) -> tuple:
        dist = self._dist
        hdr = torch.tensor([tag, code, numel], dtype=torch.int64, device=self.device)
        peer_hdr = torch.empty(3, dtype=torch.int64, device=self.device)
        ops = [dist.P2POp(dist.isend, hdr, self.peer, self.group),
               dist.P2POp(dist.irecv, peer_hdr, self.peer, self.group)]
        for w in dist.batch_isend_irecv(ops):
            if timeout is None:
                w.wait()
            elif not w.wait(timeout):
                raise SessionAbort("peer did not take the abort frame")
        return tuple(int(v) for v in peer_hdr.tolist())

    def send_abort(self):
        # best effort, header only: the peer sees FRAME_ABORT in its next header
        # and raises before any payload is posted on either side
        import datetime
        try:
            if not self._closed:
                self._swap_header(FRAME_ABORT, 0, 0,
                                  timeout=datetime.timedelta(seconds=timeout_seconds()))
        except Exception:  # noqa: BLE001
            pass

    def close(self):
        self._closed = True


class PeerBuffer:
    """A peer process's device buffer mapped into this process (CUDA IPC).

    Duck-types the few tensor methods the share layer uses on an exchanged
    payload (dtype, numel, data_ptr, flat slicing), so the evaluation kernels
    read the peer's masked message in place: over NVLink / NVSwitch when the
    peer is another GPU, from the same HBM when both processes share one."""

    is_cuda = True

    def __init__(self, ptr: int, numel: int, dtype: torch.dtype, device: torch.device):
        self._ptr, self._numel, self.dtype, self.device = ptr, numel, dtype, device

    @property
    def shape(self):
        return (self._numel,)

    def numel(self) -> int:
        return self._numel

    def element_size(self) -> int:
        return torch.empty(0, dtype=self.dtype).element_size()

    def data_ptr(self) -> int:
        return self._ptr

    def to(self, device=None, *args, **kwargs):
        if device is not None and torch.device(device) != self.device:
            raise ValueError("a mapped peer buffer is only addressable from its own device")
        return self

    def reshape(self, *shape):
        if shape not in ((-1,), (self._numel,), ((-1,),), ((self._numel,),)):
            raise ValueError("mapped peer buffers are flat")
        return self

    def contiguous(self):
        return self

    def __getitem__(self, idx):
        if not isinstance(idx, slice) or idx.step not in (None, 1):
            raise TypeError("mapped peer buffers support contiguous slices only")
        lo, hi, _ = idx.indices(self._numel)
        hi = max(hi, lo)
        return PeerBuffer(self._ptr + lo * self.element_size(), hi - lo, self.dtype, self.device)

    def __repr__(self):
        return f"PeerBuffer(ptr=0x{self._ptr:x}, numel={self._numel}, dtype={self.dtype})"


class PeerTransport:
    """Same-node transport over CUDA IPC peer memory (one party per process).

    Each process owns two message slots in its HBM and maps the peer's two
    slots. ``exchange`` writes our wire-packed payload into our slot, makes it
    visible (stream sync), meets the peer at a barrier and returns the peer's
    slot as a :class:`PeerBuffer`: no copy of the peer's message is made -- the
    consuming kernel (e.g. fss_dcf_eval_masked) loads it directly over NVLink.
    Slots alternate per round, and every round starts with a stream sync +
    barrier, so a slot is only rewritten after the peer finished reading it.
    The small frame header (tag, dtype, size) goes through torch.distributed
    exactly as in :class:`DistTransport` and sizes grow both sides' slots in
    lock-step."""

    def __init__(self, peer: int, group=None, device=None, capacity: int = 1 << 20):
        import torch.distributed as dist
        from . import _lib
        self._dist, self._lib = dist, _lib
        self.peer, self.group = peer, group
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._hdr_device = (self.device if dist.get_backend(group) == "nccl"
                            else torch.device("cpu"))
        self._slots, self._peer_ptrs, self._cap, self._round = [], [], 0, 0
        self._closed = False
        self._aborted = False
        self._grow(capacity)

    def _swap(self, t: torch.Tensor) -> torch.Tensor:
        dist = self._dist
        t = t.to(self._hdr_device)
        out = torch.empty_like(t)
        ops = [dist.P2POp(dist.isend, t, self.peer, self.group),
               dist.P2POp(dist.irecv, out, self.peer, self.group)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        return out.cpu()

    def _grow(self, nbytes: int):
        import ctypes
        lib = self._lib
        torch.cuda.current_stream(self.device).synchronize()
        self._release()
        cap = max(int(nbytes), 1 << 12)
        hb = lib.load().fss_ipc_handle_bytes()
        mine = torch.zeros((2, hb), dtype=torch.uint8)
        with torch.cuda.device(self.device):
            for i in range(2):
                ptr = ctypes.c_void_p()
                lib.call("fss_ipc_alloc", cap, ctypes.byref(ptr))
                self._slots.append(ptr.value)
                buf = (ctypes.c_uint8 * hb)()
                lib.call("fss_ipc_get_handle", ptr, buf)
                mine[i] = torch.tensor(list(buf), dtype=torch.uint8)
        theirs = self._swap(mine)
        with torch.cuda.device(self.device):
            for i in range(2):
                raw = (ctypes.c_uint8 * hb)(*theirs[i].tolist())
                ptr = ctypes.c_void_p()
                lib.call("fss_ipc_open_handle", raw, ctypes.byref(ptr))
                self._peer_ptrs.append(ptr.value)
        self._cap = cap

    def _release(self):
        """Unmap the peer's slots and free ours (callers synchronise first)."""
        import ctypes
        with torch.cuda.device(self.device):
            for p in self._peer_ptrs:
                try:
                    self._lib.call("fss_ipc_close_handle", ctypes.c_void_p(p))
                except RuntimeError:
                    pass
            for p in self._slots:
                try:
                    self._lib.call("fss_ipc_free", ctypes.c_void_p(p))
                except RuntimeError:
                    pass
        self._peer_ptrs, self._slots = [], []

    def exchange_frames(self, frame: Frame) -> Frame:
        if self._closed:
            raise SessionAbort("transport closed")
        p = frame.payload.contiguous()
        nbytes = p.numel() * p.element_size()
        hdr = torch.tensor([frame.tag, _DTYPE_CODE[p.dtype], p.numel(), nbytes], dtype=torch.int64)
        tag, code, numel, peer_bytes = (int(v) for v in self._swap(hdr).tolist())
        if tag == FRAME_ABORT:
            # the aborting peer skips the closing barrier: so must we
            self._aborted = True
            raise SessionAbort("peer aborted")
        if code < 0 or code >= len(_DTYPES):
            raise SessionAbort("corrupt frame header")
        need = max(nbytes, peer_bytes)
        if need > self._cap:                    # both sides see both sizes: lock-step growth
            self._dist.barrier(group=self.group) if self.group is not None \
                else self._dist.barrier()       # the peer stopped reading the old slots
            self._grow(2 * need)
        slot = self._round & 1
        self._round += 1
        import ctypes
        with torch.cuda.device(self.device):
            self._lib.call("fss_memcpy_d2d", ctypes.c_void_p(self._slots[slot]),
                           ctypes.c_void_p(p.data_ptr() if nbytes else 0), nbytes,
                           ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
        # our message is in HBM and every earlier read of the peer's slots is done
        torch.cuda.current_stream(self.device).synchronize()
        self._dist.barrier(group=self.group) if self.group is not None else self._dist.barrier()
        return Frame(tag, PeerBuffer(self._peer_ptrs[slot], numel, _DTYPES[code], self.device))

    def send_abort(self):
        self._aborted = True
        try:
            self._swap(torch.tensor([FRAME_ABORT, 0, 0, 0], dtype=torch.int64))
        except Exception:  # noqa: BLE001
            pass

    def close(self):
        if not self._closed:
            import ctypes
            self._closed = True
            torch.cuda.current_stream(self.device).synchronize()
            if not self._aborted:
                # the peer may still be reading our slots: leave together
                self._dist.barrier(group=self.group) if self.group is not None \
                    else self._dist.barrier()
            self._release()


# ---------------------------------------------------------------------------
# Session
# ---------------------------------------------------------------------------

class Session:
    """One party's end of an online 2-party computation (runtime.py:217-282)."""

    def __init__(self, party: int, transport):
        if party not in (0, 1):
            raise ValueError("party must be 0 or 1")
        self.party = party
        self.transport = transport
        self.ledger = RoundLedger()
        self.open = True

    def exchange(self, op: str, tag: int, payload: torch.Tensor, elements: int) -> torch.Tensor:
        """Send one frame and receive the peer's matching frame (one round).

        ``payload`` is a tensor (normally the device wire buffer); the peer's
        payload comes back as a tensor on the same device, stream-ordered."""
        if not self.open:
            raise SessionAbort("session is closed")
        if tag not in _FRAME_TAGS:
            raise ValueError(f"unknown frame tag {tag}")
        frame = Frame(tag, payload)
        try:
            if isinstance(self.transport, (DistTransport, PeerTransport)):
                peer = self.transport.exchange_frames(frame)
            else:
                self.transport.send(frame)
                peer = self.transport.recv()
        except SessionAbort:
            self.open = False
            raise
        if peer.tag == FRAME_ABORT:
            self.open = False
            raise SessionAbort("peer aborted")
        if peer.tag != tag:
            self.open = False
            raise SessionAbort(f"frame desync: expected tag {tag}, got {peer.tag}")
        self.ledger.record(op, _nbytes(payload), _nbytes(peer.payload), elements)
        return peer.payload

    def abort(self, reason: str = ""):
        if self.open:
            try:
                if isinstance(self.transport, (DistTransport, PeerTransport)):
                    self.transport.send_abort()
                else:
                    self.transport.send(Frame(FRAME_ABORT, torch.empty(0, dtype=torch.uint8)))
            except Exception:  # noqa: BLE001
                pass
            self.open = False

    def close(self):
        self.open = False
        self.transport.close()


def run_session(party: int, transport, program):
    """Run ``program(session)``; returns (result, ledger) (runtime.py:272-282)."""
    session = Session(party, transport)
    try:
        result = program(session)
    except Exception:
        session.abort("program failed")
        raise
    finally:
        session.close()
    return result, session.ledger


_PARTY_STREAMS = {}


def _party_streams(dev) -> list:
    """The two party threads' CUDA streams on ``dev``, created once per device:
    the caching allocator keeps its free blocks per stream, so fresh streams on
    every call would make each online run cudaMalloc its buffers anew (measured:
    4 cudaMalloc per ReLU run, 8-430 ms online instead of ~3.5 ms)."""
    key = str(dev)
    if key not in _PARTY_STREAMS:
        _PARTY_STREAMS[key] = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    return _PARTY_STREAMS[key]


class _PartyWorkers:
    """Two long-lived party threads (one per party), reused by every
    run_local_pair call: starting two fresh threads per online run costs more
    host time than a small protocol's kernels (config 1: 2^16 comparisons).
    A job is a callable; the worker runs it and reports (result, error)."""

    def __init__(self):
        self._jobs = [queue.SimpleQueue(), queue.SimpleQueue()]
        self._done = [queue.SimpleQueue(), queue.SimpleQueue()]
        self.lock = threading.Lock()
        self.pid = os.getpid()
        self.threads = [threading.Thread(target=self._loop, args=(p,), daemon=True,
                                         name=f"ariann-party{p}") for p in (0, 1)]
        for t in self.threads:
            t.start()

    def _loop(self, party):
        while True:
            job = self._jobs[party].get()
            try:
                self._done[party].put((job(), None))
            except BaseException as exc:  # noqa: BLE001 -- handed to the caller
                self._done[party].put((None, exc))

    def run(self, job0, job1):
        self._jobs[0].put(job0)
        self._jobs[1].put(job1)
        return self._done[0].get(), self._done[1].get()


_WORKERS = None
_WORKERS_INIT = threading.Lock()


def _party_workers():
    global _WORKERS
    with _WORKERS_INIT:
        # a forked child inherits the object but not the threads: start anew
        if _WORKERS is None or _WORKERS.pid != os.getpid():
            _WORKERS = _PartyWorkers()
        return _WORKERS


def run_local_pair(program0, program1=None, device=None):
    """Two programs over the in-process transport, one thread per party
    (runtime.py:285-311). Each party thread runs on its own CUDA stream of
    ``device`` so the two parties' kernels can overlap; the exchange orders
    them. Returns ((result0, ledger0), (result1, ledger1)).

    The party threads are two persistent workers shared by all calls; a call
    made while they are busy (another thread's run, or a nested call from
    inside a party program) runs on two fresh threads instead."""
    if program1 is None:
        program1 = program0
    t0, t1 = local_pair()
    dev = None
    if torch.cuda.is_available():
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        parent = torch.cuda.current_stream(dev)
        streams = _party_streams(dev)
        for s in streams:
            s.wait_stream(parent)

    def job(party, transport, program):
        def run():
            try:
                if dev is not None:
                    with torch.cuda.device(dev), torch.cuda.stream(streams[party]):
                        return run_session(party, transport, program)
                return run_session(party, transport, program)
            except BaseException:
                transport.close()       # unblock the peer
                raise
        return run

    jobs = (job(0, t0, program0), job(1, t1, program1))
    workers = _party_workers()
    if workers.lock.acquire(blocking=False):
        try:
            outcome = workers.run(*jobs)
        finally:
            workers.lock.release()
    else:
        outcome = [[None, None], [None, None]]

        def fresh(p):
            try:
                outcome[p][0] = jobs[p]()
            except BaseException as exc:  # noqa: BLE001
                outcome[p][1] = exc
        ths = [threading.Thread(target=fresh, args=(p,)) for p in (0, 1)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
    if dev is not None:
        for s in streams:
            parent.wait_stream(s)
    for _, err in outcome:
        if err is not None:
            raise err
    return outcome[0][0], outcome[1][0]


def run_dist_party(party: int, peer: int, program, group=None, device=None):
    """This process plays ``party`` against the process of global rank ``peer``."""
    return run_session(party, DistTransport(peer, group, device), program)


def run_peer_party(party: int, peer: int, program, group=None, device=None, capacity=1 << 20):
    """As run_dist_party, but the masked messages are read in place from the
    peer's HBM through CUDA IPC (:class:`PeerTransport`)."""
    return run_session(party, PeerTransport(peer, group, device, capacity), program)
