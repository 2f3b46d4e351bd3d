"""CPU tests of the device-payload runtime (runtime.py): in-process pair over
LocalTransport and a real 2-process pair over torch.distributed (gloo,
world_size 2) -- the same DistTransport code that carries the masked message
over NCCL / NVLink on GPUs."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2006_04593_b200 import runtime


def test_local_pair_exchange_and_ledger():
    def prog(session):
        mine = torch.full((5,), 10 + session.party, dtype=torch.uint32)
        peer = session.exchange("comparison", runtime.FRAME_MASKED, mine, elements=5)
        peer2 = session.exchange("mul", runtime.FRAME_TRIPLE_DELTA,
                                 torch.arange(4, dtype=torch.uint8) + session.party, elements=4)
        return int(peer[0]), peer2.tolist()
    (r0, l0), (r1, l1) = runtime.run_local_pair(prog)
    assert r0 == (11, [1, 2, 3, 4]) and r1 == (10, [0, 1, 2, 3])
    assert l0.total_rounds() == 2 and l0.snapshot() == {"comparison": 1, "mul": 1}
    assert l0.total_bytes_sent() == 5 * 4 + 4
    assert l1.as_dict()["bytes_received"] == {"comparison": 20, "mul": 4}


def test_local_pair_desync_and_failure():
    def prog(session):
        tag = runtime.FRAME_MASKED if session.party == 0 else runtime.FRAME_REVEAL
        return session.exchange("x", tag, torch.zeros(1, dtype=torch.uint32), 1)
    with pytest.raises(runtime.SessionAbort):
        runtime.run_local_pair(prog)

    def bad(session):
        if session.party == 1:
            raise ValueError("boom")
        return session.exchange("x", runtime.FRAME_MASKED, torch.zeros(1), 1)
    with pytest.raises((ValueError, runtime.SessionAbort)):
        runtime.run_local_pair(bad)


def test_timeout(monkeypatch):
    monkeypatch.setenv("ARIANN_TIMEOUT_MS", "200")
    t0, _t1 = runtime.local_pair()
    s = runtime.Session(0, t0)
    with pytest.raises(runtime.SessionAbort):
        s.exchange("x", runtime.FRAME_MASKED, torch.zeros(1), 1)
    with pytest.raises(runtime.SessionAbort):
        s.exchange("x", runtime.FRAME_MASKED, torch.zeros(1), 1)  # session closed
    with pytest.raises(ValueError):
        runtime.Session(2, t0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dist_worker(rank, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        def prog(session):
            out = []
            for dt, vals in ((torch.uint32, [7, 8, 9]), (torch.uint64, [1 << 40, 3]),
                             (torch.uint8, [])):
                mine = torch.tensor([v + rank for v in vals], dtype=torch.int64).to(dt)
                peer = session.exchange("op", runtime.FRAME_MASKED, mine, elements=len(vals))
                assert peer.dtype == dt
                out.append([int(v) for v in peer.to(torch.int64)])
            return out
        res, ledger = runtime.run_dist_party(rank, 1 - rank, prog)
        q.put((rank, res, ledger.total_rounds(), ledger.total_bytes_sent()))
        # frame desync is detected on both sides
        tag = runtime.FRAME_MASKED if rank == 0 else runtime.FRAME_TRIPLE_DELTA
        try:
            runtime.run_dist_party(rank, 1 - rank,
                                   lambda s: s.exchange("x", tag, torch.zeros(2, dtype=torch.int32), 2))
            q.put((rank, "no-error"))
        except runtime.SessionAbort:
            q.put((rank, "abort"))
    finally:
        dist.destroy_process_group()


def test_dist_transport_gloo_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(4)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res = {g[0]: g[1:] for g in got if len(g) == 4}
    assert res[0][0] == [[8, 9, 10], [(1 << 40) + 1, 4], []]
    assert res[1][0] == [[7, 8, 9], [1 << 40, 3], []]
    assert res[0][1] == 3 and res[0][2] == 3 * 4 + 2 * 8
    assert sorted(g[1] for g in got if len(g) == 2) == ["abort", "abort"]


def test_peer_death_mid_round_aborts_not_hangs(monkeypatch):     # reference test_runtime.py:76-86
    monkeypatch.setenv("ARIANN_TIMEOUT_MS", "500")

    def party0(session):
        return session.exchange("a", runtime.FRAME_MASKED, torch.zeros(1, dtype=torch.uint8), 1)

    def party1(session):
        return None          # exits immediately, closing its transport

    with pytest.raises(runtime.SessionAbort):
        runtime.run_local_pair(party0, party1)


def test_large_payload_both_directions_no_deadlock():              # reference test_runtime.py:102-110
    blob = torch.zeros(2_000_000, dtype=torch.uint8)

    def program(session):
        return session.exchange("bulk", runtime.FRAME_MASKED, blob, blob.numel()).numel()

    (r0, _), (r1, _) = runtime.run_local_pair(program)
    assert r0 == blob.numel() and r1 == blob.numel()


def _abort_worker(rank, port, q):
    import datetime
    import time

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # a process-group timeout far above the test's bound: a hang would show
    dist.init_process_group("gloo", rank=rank, world_size=2, timeout=datetime.timedelta(seconds=90))
    try:
        def prog(session):
            session.exchange("a", runtime.FRAME_MASKED, torch.zeros(4, dtype=torch.int32), 4)
            if session.party == 1:
                raise ValueError("party 1 fails mid-program")
            # party 0 announces a large payload; the aborting side must not post
            # a receive for it (it would block until the group timeout)
            return session.exchange("b", runtime.FRAME_MASKED, torch.zeros(1 << 16, dtype=torch.int64),
                                    1 << 16)
        t0 = time.time()
        try:
            runtime.run_dist_party(rank, 1 - rank, prog)
            outcome = "no-error"
        except runtime.SessionAbort:
            outcome = "abort"
        except ValueError:
            outcome = "raised"
        dt = time.time() - t0
        # the pair is still in step: a fresh session exchanges normally
        res, _ = runtime.run_dist_party(
            rank, 1 - rank,
            lambda s: int(s.exchange("c", runtime.FRAME_MASKED, torch.full((3,), 5 + rank,
                                                                            dtype=torch.int32), 3)[0]))
        q.put((rank, outcome, dt, res))
    finally:
        dist.destroy_process_group()


def test_dist_abort_mid_program_fails_fast():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_abort_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0][1] == "abort" and got[1][1] == "raised"
    assert got[0][2] < 30 and got[1][2] < 30          # not the 90 s group timeout
    assert got[0][3] == 6 and got[1][3] == 5


def test_local_pair_reuses_workers_and_handles_nesting_and_errors():
    import threading as th
    names = []

    def prog(session):
        names.append(th.current_thread().name)
        return int(session.exchange("x", runtime.FRAME_MASKED,
                                    torch.full((2,), session.party, dtype=torch.int32), 2)[0])
    for _ in range(3):
        (r0, _), (r1, _) = runtime.run_local_pair(prog)
        assert (r0, r1) == (1, 0)
    assert set(names) == {"ariann-party0", "ariann-party1"}      # the persistent workers

    def nested(session):                 # a party program that runs its own pair
        inner = runtime.run_local_pair(prog)
        return inner[0][0]
    (a, _), (b, _) = runtime.run_local_pair(nested)
    assert a == 1 and b == 1

    def boom(session):
        if session.party == 0:
            raise KeyError("party 0 fails")
        return session.exchange("x", runtime.FRAME_MASKED, torch.zeros(1), 1)
    with pytest.raises((KeyError, runtime.SessionAbort)):
        runtime.run_local_pair(boom)
    (r0, _), (r1, _) = runtime.run_local_pair(prog)          # workers still healthy
    assert (r0, r1) == (1, 0)

    # concurrent callers: one gets the workers, the other fresh threads
    out = []
    ts = [th.Thread(target=lambda: out.append(runtime.run_local_pair(prog)[0][0])) for _ in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert out == [1, 1, 1, 1]


def _forked_child(q):
    def prog(session):
        return int(session.exchange("x", runtime.FRAME_MASKED,
                                    torch.full((1,), 7 + session.party, dtype=torch.int32), 1)[0])
    (a, _), (b, _) = runtime.run_local_pair(prog)
    q.put((a, b))


def test_local_pair_after_fork():
    # the parent's persistent workers do not exist in a forked child
    def prog(session):
        return session.party
    runtime.run_local_pair(prog)                      # parent starts its workers
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    p = ctx.Process(target=_forked_child, args=(q,))
    p.start()
    assert q.get(timeout=60) == (8, 7)
    p.join(timeout=30)
    assert p.exitcode == 0
