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

import ctypes
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


class PeerAccessError(SessionAbort):
    """CUDA IPC mapping of the peer's buffers failed (no peer access between the
    two GPUs, or IPC unavailable). Raised on BOTH ranks: the mapping outcome is
    agreed before any peer load or store."""


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

class _Sched:
    """Scheduling words shared by the threads of an in-process party pair
    (csrc/host_sync.cu): frames posted to each party's inbox, the party whose
    turn it is to run Python, jobs posted to each party worker, jobs done.

    A waiting thread spins in the library with the GIL released instead of
    sleeping on a lock, and the running party hands the turn over when it
    blocks or finishes: the two parties' Python never contends for the GIL and
    no hand-over pays a kernel wake-up (measured: run_local_pair of an empty
    program 103 us, of one sign test 466 us, with blocking queues)."""

    INBOX0, INBOX1, TURN, JOB0, JOB1, DONE = range(6)
    GRACE_S = 0.002   # a waiter runs this long after its condition held, turn or not

    def __init__(self):
        from . import _lib
        self._lib = _lib.load()
        self._words = (ctypes.c_int64 * 8)()
        self._base = ctypes.addressof(self._words)

    def ptr(self, i: int) -> int:
        return self._base + 8 * i

    def event_rings(self, device) -> tuple:
        """Two timing-free CUDA events per party on ``device``, created once.
        A party records them alternately on its sends; exchanges are send
        then receive, so the peer has waited on an event before the party
        can send twice more and re-record it."""
        rings = self.__dict__.setdefault("_rings", {})
        key = device.index
        if key not in rings:
            import ctypes as ct
            from . import _dev
            evs = []
            with _dev.on(device):
                for _ in range(4):
                    h = ct.c_void_p()
                    self._lib_call("fss_event_create", ct.byref(h))
                    evs.append(h.value)
            rings[key] = ([evs[0], evs[1]], [evs[2], evs[3]])
        return rings[key]

    @staticmethod
    def _lib_call(name, *args):
        from . import _lib
        _lib.call(name, *args)

    def load(self, i: int) -> int:
        return self._lib.fss_host_load(self._base + 8 * i)

    def store(self, i: int, v: int):
        self._lib.fss_host_store(self._base + 8 * i, v)

    def add(self, i: int, d: int = 1) -> int:
        return self._lib.fss_host_add(self._base + 8 * i, d)

    def wait(self, i: int, target: int, me, timeout: float, pass_to: int = -1,
             bump: int = None, spin: float = 0.1) -> bool:
        """Until word i >= target (and, within GRACE_S, it is ``me``'s turn;
        ``me`` None: no turn). Before waiting, in the same native call: add 1
        to word ``bump`` and give the turn to ``pass_to`` (if >= 0). Spins for
        ``spin`` s before backing off to naps. False on timeout."""
        b = self._base
        turn = None if me is None and pass_to < 0 else b + 8 * self.TURN
        return self._lib.fss_host_wait(b + 8 * i, target, turn, -1 if me is None else me, pass_to,
                                       None if bump is None else b + 8 * bump, spin, self.GRACE_S,
                                       timeout) == 0


class LocalTransport:
    """In-process duplex channel: FIFO queues of device-tensor frames (runtime.py:103-133).

    With a scheduler (``local_pair``), a receive that finds its inbox empty
    passes the turn to the peer and spins until the peer's frame is posted."""

    def __init__(self, inbox, outbox, sched: _Sched = None, party: int = 0, events=None,
                 stream=None):
        self._inbox = inbox
        self._outbox = outbox
        self._closed = False
        self._sched = sched
        self._party = party
        self._seen = sched.load(_Sched.INBOX0 + party) if sched is not None else 0
        self._events = events     # [ev, ev] raw events of the scheduler's device, or None
        self._ev_dev = None
        self._ev_i = 0
        self._stream = stream     # this party's torch stream, or None
        if events is not None:
            from . import _dev, _lib
            self._dev, self._lib = _dev, _lib

    def _post(self, item):
        self._outbox.put(item)
        if self._sched is not None:
            self._sched.add(_Sched.INBOX0 + 1 - self._party)

    def send(self, frame: Frame):
        if self._closed:
            raise SessionAbort("transport closed")
        p = frame.payload
        if frame.event is None and isinstance(p, torch.Tensor) and p.is_cuda:
            if self._events is not None and self._stream is not None \
                    and p.device == self._stream.device:
                ev = self._events[self._ev_i]
                self._ev_i ^= 1
                self._lib.call("fss_event_record", ev, self._dev.stream_handle(p.device))
            else:
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream(p.device))
            frame = Frame(frame.tag, p, ev)
        self._post(frame)

    def recv(self) -> Frame:
        s = self._sched
        if s is not None:
            me = self._party
            self._seen += 1
            if s.load(_Sched.INBOX0 + me) < self._seen:
                # nothing posted yet: the peer runs while we wait
                if not s.wait(_Sched.INBOX0 + me, self._seen, me, timeout_seconds(), pass_to=1 - me):
                    raise SessionAbort("timed out waiting for peer")
            frame = self._inbox.get_nowait()
        else:
            try:
                frame = self._inbox.get(timeout=timeout_seconds())
            except queue.Empty:
                raise SessionAbort("timed out waiting for peer") from None
        if frame is None:
            raise SessionAbort("peer closed the channel")
        ev = frame.event
        if ev is not None:
            dev = frame.payload.device
            if isinstance(ev, int):          # a raw event of the scheduler's ring
                h = self._dev.stream_handle(dev)
                self._lib.call("fss_stream_wait_event", h, ev)
                st = self._stream
                cur = st if st is not None and st.cuda_stream == h else torch.cuda.current_stream(dev)
            else:
                cur = torch.cuda.current_stream(dev)
                cur.wait_event(ev)
            # the sender's allocator must not recycle the buffer before we read it
            frame.payload.record_stream(cur)
        return frame

    def close(self):
        if not self._closed:
            self._closed = True
            self._post(None)


def spin_enabled() -> bool:
    """ARIANN_LOCAL_SPIN=0 turns the spinning hand-over of the in-process pair
    off (blocking queues instead): for hosts with fewer free cores than the
    three threads of a run_local_pair call."""
    return os.environ.get("ARIANN_LOCAL_SPIN", "1") != "0"


def local_pair(sched: _Sched = None, device=None, streams=None) -> tuple[LocalTransport, LocalTransport]:
    """A connected transport pair. With a scheduler and ``device`` (the
    persistent party workers' run), frames of payloads on ``device`` are
    ordered by the scheduler's timing-free events, and ``streams`` are the
    parties' streams (the receivers' record_stream targets)."""
    a, b = queue.SimpleQueue(), queue.SimpleQueue()
    if sched is None and spin_enabled():
        sched = _Sched()
    rings = (sched.event_rings(device) if sched is not None and device is not None
             else (None, None))
    st = streams if streams is not None else (None, None)
    return (LocalTransport(a, b, sched, 0, rings[0], st[0]),
            LocalTransport(b, a, sched, 1, rings[1], st[1]))


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
        err = None
        with torch.cuda.device(self.device):
            try:
                for i in range(2):
                    ptr = ctypes.c_void_p()
                    lib.call("fss_ipc_alloc", cap, ctypes.byref(ptr))
                    self._slots.append(ptr.value)
                    buf = (ctypes.c_uint8 * hb)()
                    lib.call("fss_ipc_get_handle", ptr, buf)
                    mine[i] = torch.tensor(list(buf), dtype=torch.uint8)
            except RuntimeError as e:           # still swap (zeros), then agree below
                err = e
        theirs = self._swap(mine)
        with torch.cuda.device(self.device):
            try:
                for i in range(2):
                    if err is not None or bool(theirs[i].eq(0).all()):
                        err = err or "the peer exported no buffer"
                        break
                    raw = (ctypes.c_uint8 * hb)(*theirs[i].tolist())
                    ptr = ctypes.c_void_p()
                    lib.call("fss_ipc_open_handle", raw, ctypes.byref(ptr))
                    self._peer_ptrs.append(ptr.value)
            except RuntimeError as e:
                err = e
        # both sides learn whether both mappings exist before either uses one, so
        # a failed mapping fails the two parties alike (no side left blocked in
        # a later exchange waiting for a peer that raised)
        ok = self._swap(torch.tensor([0 if err else 1], dtype=torch.int64))
        if err is not None or int(ok[0]) != 1:
            self._release()
            self._closed = True
            raise PeerAccessError("peer memory mapping failed on "
                                  + (f"this rank: {err}" if err else "the peer"))
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
    A job is a callable; the worker runs it and reports (result, error).
    Idle workers spin on their job word (``_Sched``) for IDLE_SPIN_S after a
    job (back-to-back protocol runs find them awake), then block on their
    queue."""

    IDLE_SPIN_S = 0.1

    def __init__(self):
        self.sched = _Sched() if spin_enabled() else None
        self._jobs = [queue.SimpleQueue(), queue.SimpleQueue()]
        self._done = queue.SimpleQueue()
        self._out = [None, None]
        self.lock = threading.Lock()
        self.pid = os.getpid()
        self.threads = [threading.Thread(target=self._loop, args=(p,), daemon=True,
                                         name=f"ariann-party{p}") for p in (0, 1)]
        for t in self.threads:
            t.start()

    def _loop(self, party):
        s = self.sched
        if s is None:
            while True:
                job = self._jobs[party].get()
                try:
                    self._out[party] = (job(), None)
                except BaseException as exc:  # noqa: BLE001 -- handed to the caller
                    self._out[party] = (None, exc)
                self._done.put(party)
        seen, done = 0, False
        while True:
            seen += 1
            # report the previous job (DONE += 1, the peer's turn) and wait for the next
            if s.wait(_Sched.JOB0 + party, seen, party, self.IDLE_SPIN_S,
                      pass_to=1 - party if done else -1, bump=_Sched.DONE if done else None,
                      spin=self.IDLE_SPIN_S):
                job = self._jobs[party].get_nowait()
            else:
                job = self._jobs[party].get()
            try:
                self._out[party] = (job(), None)
            except BaseException as exc:  # noqa: BLE001 -- handed to the caller
                self._out[party] = (None, exc)
            done = True

    def run(self, job0, job1):
        s = self.sched
        if s is None:
            self._jobs[0].put(job0)
            self._jobs[1].put(job1)
            self._done.get()
            self._done.get()
            return self._out[0], self._out[1]
        target = s.load(_Sched.DONE) + 2
        s.store(_Sched.TURN, 2)               # neither party until both jobs are posted
        self._jobs[0].put(job0)
        self._jobs[1].put(job1)
        s.add(_Sched.JOB0 + 1)
        # post party 0's job and give it the turn as this thread starts waiting
        ok = s.wait(_Sched.DONE, target, None, 1.0, pass_to=0, bump=_Sched.JOB0, spin=1.0)
        while not ok:
            ok = s.wait(_Sched.DONE, target, None, 1.0, spin=0.0)
        return self._out[0], self._out[1]


_WORKERS = None
_WORKERS_INIT = threading.Lock()


def _party_workers():
    global _WORKERS
    with _WORKERS_INIT:
        # a forked child inherits the object but not the threads: start anew
        if (_WORKERS is None or _WORKERS.pid != os.getpid()
                or (_WORKERS.sched is not None) != spin_enabled()):
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
    dev = None
    if torch.cuda.is_available():
        from . import _dev, _lib
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        streams = _party_streams(dev)
        handles = [st.cuda_stream for st in streams]
        with _dev.on(dev):
            parent = _dev.stream_handle(dev)
            _lib.call("fss_streams_link", handles[0], handles[1], 2, parent, None, 1)   # fork
    workers = _party_workers()
    mine = workers.lock.acquire(blocking=False)
    try:
        sched = workers.sched if mine else None
        t0, t1 = local_pair(sched, dev if sched is not None else None,
                            streams if dev is not None else None)
    except BaseException:
        if mine:
            workers.lock.release()
        raise

    def job(party, transport, program):
        def run():
            try:
                if dev is not None:
                    # the party thread's device and stream (left set: the
                    # thread runs nothing but party programs)
                    if torch._C._cuda_getDevice() != dev.index:
                        torch.cuda.set_device(dev)
                    torch.cuda.set_stream(streams[party])
                return run_session(party, transport, program)
            except BaseException:
                transport.close()       # unblock the peer
                raise
        return run

    jobs = (job(0, t0, program0), job(1, t1, program1))
    if mine:
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
        with _dev.on(dev):
            _lib.call("fss_streams_link", parent, None, 1, handles[0], handles[1], 2)   # join
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
