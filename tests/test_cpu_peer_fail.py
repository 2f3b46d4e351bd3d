"""CPU tests (gloo) of the failure agreement in the two CUDA-IPC peer-memory
setups: shard.PeerGather (all ranks map rank dst's result buffer) and
runtime.PeerTransport (the two parties map each other's message slots).

When one rank cannot map (or export) its peer's buffer, EVERY rank must raise
runtime.PeerAccessError from the constructor and free what it allocated --
a rank failing alone would leave the others blocked in the next collective
(finish()'s barrier, the next frame exchange) until the process-group timeout.
The CUDA calls are replaced by a fake library so the agreement logic runs
without a GPU."""

import contextlib
import ctypes
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _FakeLib:
    """fss_ipc_* stand-ins: allocations are integers, handles 64 bytes of 1s."""

    def __init__(self, fail: str | None):
        self.fail, self.log, self._next = fail, [], 0x1000

    def load(self):
        return self

    def fss_ipc_handle_bytes(self):
        return 64

    def call(self, name, *args):
        self.log.append(name)
        if name == self.fail:
            raise RuntimeError(f"{name}: injected failure")
        if name in ("fss_ipc_alloc", "fss_ipc_open_handle"):
            args[-1]._obj.value = self._next
            self._next += 0x1000
        elif name == "fss_ipc_get_handle":
            ctypes.memset(args[1], 1, 64)
        return 0


def _patch(fake):
    from paper_2006_04593_b200 import _dev, _lib
    _lib.load, _lib.call = fake.load, fake.call
    _dev.on = lambda device: contextlib.nullcontext()
    torch.cuda.device = lambda device: contextlib.nullcontext()

    class _S:
        def synchronize(self):
            pass
    torch.cuda.current_stream = lambda device=None: _S()


def _gather_worker(rank, world, port, fail_rank, fail_call, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fake = _FakeLib(fail_call if rank == fail_rank else None)
        _patch(fake)
        from paper_2006_04593_b200 import shard
        from paper_2006_04593_b200.runtime import PeerAccessError
        try:
            shard.PeerGather(100, slots=2, dst=0, device="cpu")
            outcome = "ok"
        except PeerAccessError:
            outcome = "PeerAccessError"
        dist.barrier()            # every rank got here: nobody was left blocked
        q.put((rank, outcome, fake.log))
    finally:
        dist.destroy_process_group()


def _transport_worker(rank, port, fail_rank, fail_call, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        fake = _FakeLib(fail_call if rank == fail_rank else None)
        _patch(fake)
        from paper_2006_04593_b200.runtime import PeerAccessError, PeerTransport
        try:
            PeerTransport(1 - rank, device="cpu", capacity=4096)
            outcome = "ok"
        except PeerAccessError:
            outcome = "PeerAccessError"
        dist.barrier()
        q.put((rank, outcome, fake.log))
    finally:
        dist.destroy_process_group()


def _run(target, world, args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=target, args=(r, *((world,) if target is _gather_worker else ()),
                                              port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (o, log) for r, o, log in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    return res


@pytest.mark.parametrize("fail_rank,fail_call", [(2, "fss_ipc_open_handle"), (1, "fss_ipc_open_handle"),
                                                 (0, "fss_ipc_alloc"), (0, "fss_ipc_get_handle")])
def test_peer_gather_failure_is_agreed(fail_rank, fail_call):
    res = _run(_gather_worker, 3, (fail_rank, fail_call))
    assert all(o == "PeerAccessError" for o, _ in res.values()), res
    # the destination freed its buffer when it had one; the ranks that mapped it unmapped it
    if fail_call != "fss_ipc_alloc":
        assert "fss_ipc_free" in res[0][1]
    for r in (1, 2):
        opened = "fss_ipc_open_handle" in res[r][1] and not (r == fail_rank and fail_call ==
                                                               "fss_ipc_open_handle")
        assert ("fss_ipc_close_handle" in res[r][1]) == opened, (r, res[r])


def test_peer_gather_success_path():
    res = _run(_gather_worker, 3, (-1, None))
    assert all(o == "ok" for o, _ in res.values()), res


@pytest.mark.parametrize("fail_rank,fail_call", [(0, "fss_ipc_open_handle"), (1, "fss_ipc_open_handle"),
                                                 (1, "fss_ipc_alloc")])
def test_peer_transport_failure_is_agreed(fail_rank, fail_call):
    res = _run(_transport_worker, 2, (fail_rank, fail_call))
    assert all(o == "PeerAccessError" for o, _ in res.values()), res
    for r in (0, 1):
        log = res[r][1]
        # whatever a rank allocated or mapped, it released
        assert log.count("fss_ipc_free") == log.count("fss_ipc_alloc") - (
            1 if (r == fail_rank and fail_call == "fss_ipc_alloc") else 0)


def test_peer_transport_success_path():
    res = _run(_transport_worker, 2, (-1, None))
    assert all(o == "ok" for o, _ in res.values()), res
