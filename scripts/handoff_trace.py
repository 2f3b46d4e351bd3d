"""Where the host time of one in-process pair run goes: perf_counter marks at
the hand-over points of run_local_pair (dispatch, job start, session start,
program start/end, send, receive wait/return), medians over runs, for an empty
program and a one-round exchange of a small device tensor."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import runtime  # noqa: E402

M = []


def mark(tag):
    M.append((threading.current_thread().name[-1:], tag, time.perf_counter()))


def patch(obj, name, tag):
    fn = getattr(obj, name)

    def w(*a, **k):
        mark(tag + ">")
        try:
            return fn(*a, **k)
        finally:
            mark(tag + "<")
    setattr(obj, name, w)


patch(runtime, "run_session", "session")
patch(runtime.LocalTransport, "send", "send")
patch(runtime.LocalTransport, "recv", "recv")
patch(runtime._Sched, "wait", "wait")
x = torch.zeros(1024, dtype=torch.uint32, device="cuda")


def empty(s):
    mark("prog")


def one_round(s):
    mark("prog")
    s.exchange("op", runtime.FRAME_MASKED, x, elements=1024)
    mark("prog_end")


for name, prog in (("empty", empty), ("one round", one_round)):
    runs = []
    for i in range(60):
        M.clear()
        t0 = time.perf_counter()
        runtime.run_local_pair(prog)
        t1 = time.perf_counter()
        if i >= 10:
            runs.append([(th, tag, 1e6 * (t - t0)) for th, tag, t in M] + [("m", "end", 1e6 * (t1 - t0))])
    print(f"--- {name}: median us from the call")
    n = min(len(r) for r in runs)
    for j in range(n):
        vals = sorted(r[j][2] for r in runs)
        print(f"  {runs[0][j][0]:2s} {runs[0][j][1]:12s} {vals[len(vals) // 2]:8.1f}")
