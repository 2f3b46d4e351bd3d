"""run_local_pair orders the party streams after the caller's stream (fork)
and the caller's stream after the party streams (join), for the legacy
default stream (handle 0) and a side stream; the frames of the persistent
workers' event rings order the receiver after the sender."""

import pytest
import torch

from paper_2006_04593_b200 import runtime

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("caller", ["default", "side"])
def test_fork_and_join_follow_the_caller_stream(caller):
    dev = torch.device("cuda", 0)
    side = torch.cuda.Stream(dev)
    ctx = torch.cuda.stream(side) if caller == "side" else torch.cuda.stream(torch.cuda.default_stream(dev))
    with ctx:
        for rep in range(3):
            t = torch.zeros(1 << 20, dtype=torch.int64, device=dev)
            torch.cuda._sleep(100_000_000)          # the caller's stream is busy ...
            t.fill_(7 + rep)                        # ... before it writes the input
            out = torch.zeros(2, dtype=torch.int64, device=dev)

            def prog(s):
                torch.cuda._sleep(50_000_000)       # the party stream writes late
                out[s.party] = t.sum()
            runtime.run_local_pair(prog)
            # read on the caller's stream: it must have waited for both parties
            assert out.tolist() == [(7 + rep) << 20] * 2


def test_frames_order_receiver_after_sender():
    dev = torch.device("cuda", 0)

    def prog(s):
        msg = torch.zeros(1 << 16, dtype=torch.int64, device=dev)
        if s.party == 0:
            torch.cuda._sleep(100_000_000)          # party 0's payload is written late
        msg.fill_(11 + s.party)
        peer = s.exchange("op", runtime.FRAME_MASKED, msg, elements=msg.numel())
        return int(peer.sum())
    for _ in range(4):
        (r0, _), (r1, _) = runtime.run_local_pair(prog)
        assert r0 == 12 << 16 and r1 == 11 << 16
