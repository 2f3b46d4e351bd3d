"""CPU tests of the in-process pair's hand-over (csrc/host_sync.cu through
runtime._Sched): the wait primitive's conditions, and LocalTransport / the
persistent party workers with the spinning scheduler on and off."""

import threading
import time

import pytest
import torch

from paper_2006_04593_b200 import runtime

S = runtime._Sched


def test_wait_ready_timeout_and_grace():
    s = S()
    assert s.wait(S.INBOX0, 0, None, 1.0)                 # already satisfied
    t0 = time.perf_counter()
    assert not s.wait(S.INBOX0, 1, None, 0.02, spin=0.005)  # never posted: times out
    assert time.perf_counter() - t0 >= 0.02
    s.add(S.INBOX0)
    s.store(S.TURN, 1)
    t0 = time.perf_counter()
    assert s.wait(S.INBOX0, 1, 0, 5.0)                    # posted, not our turn: grace
    assert S.GRACE_S <= time.perf_counter() - t0 < 1.0
    s.store(S.TURN, 0)
    t0 = time.perf_counter()
    assert s.wait(S.INBOX0, 1, 0, 5.0)                    # posted and our turn: at once
    assert time.perf_counter() - t0 < S.GRACE_S


def test_wait_bumps_and_passes_before_waiting():
    s = S()
    s.store(S.TURN, 0)
    assert s.wait(S.INBOX0, 0, 1, 1.0, pass_to=1, bump=S.DONE)
    assert s.load(S.DONE) == 1 and s.load(S.TURN) == 1
    assert s.add(S.DONE, 5) == 6


def test_turn_hand_over_between_threads():
    """A waiter whose word is posted still runs only once the poster passes
    the turn (well before the grace period)."""
    s = S()
    s.GRACE_S = 2.0            # only the hand-over may release the waiter here
    s.store(S.TURN, 0)
    order = []

    def waiter():
        assert s.wait(S.INBOX1, 1, 1, 5.0)
        order.append("waiter")

    t = threading.Thread(target=waiter)
    t.start()
    s.add(S.INBOX1)            # post: the waiter's condition holds, the turn is ours
    time.sleep(0.0005)
    order.append("poster")
    assert s.wait(S.INBOX0, 0, None, 1.0, pass_to=1)   # hand the turn over
    t.join()
    assert order == ["poster", "waiter"]


@pytest.mark.parametrize("spin", ["1", "0"])
def test_many_rounds_in_order(monkeypatch, spin):
    monkeypatch.setenv("ARIANN_LOCAL_SPIN", spin)

    def prog(session):
        got = []
        for r in range(50):
            mine = torch.full((3,), 100 * session.party + r, dtype=torch.int32)
            peer = session.exchange("op", runtime.FRAME_MASKED, mine, elements=3)
            got.append(int(peer[0]))
        return got
    for _ in range(3):
        (r0, l0), (r1, _) = runtime.run_local_pair(prog)
        assert r0 == [100 + r for r in range(50)] and r1 == list(range(50))
        assert l0.total_rounds() == 50
    assert (runtime._party_workers().sched is not None) == (spin == "1")


def test_failure_and_timeout_with_spinning_scheduler(monkeypatch):
    monkeypatch.setenv("ARIANN_LOCAL_SPIN", "1")

    def bad(session):
        if session.party == 1:
            raise ValueError("boom")
        return session.exchange("x", runtime.FRAME_MASKED, torch.zeros(1), 1)
    with pytest.raises((ValueError, runtime.SessionAbort)):
        runtime.run_local_pair(bad)

    monkeypatch.setenv("ARIANN_TIMEOUT_MS", "50")
    t0, _t1 = runtime.local_pair()
    start = time.perf_counter()
    with pytest.raises(runtime.SessionAbort, match="timed out"):
        t0.recv()
    assert time.perf_counter() - start >= 0.05


def test_nested_run_uses_fresh_threads():
    def inner(session):
        return session.exchange("in", runtime.FRAME_MASKED,
                                torch.tensor([session.party], dtype=torch.int32), 1)

    def outer(session):
        (a, _), (b, _) = runtime.run_local_pair(inner) if session.party == 0 else ((None, None), (None, None))
        peer = session.exchange("out", runtime.FRAME_MASKED,
                                torch.tensor([7 + session.party], dtype=torch.int32), 1)
        return (None if a is None else (int(a[0]), int(b[0]))), int(peer[0])
    (r0, _), (r1, _) = runtime.run_local_pair(outer)
    assert r0 == ((1, 0), 8) and r1 == (None, 7)
