"""Host (Python) cost of the online protocols, separated from GPU time.

1. One party's program against a loopback transport (exchange hands back the
   party's own frame): host microseconds per call of sign / eq / relu on tiny
   shapes, so nothing waits on the GPU; optional cProfile of each.
2. run_local_pair on the same tiny shapes: host wall per call (both parties,
   two threads, GIL-serialised glue).

  python scripts/host_cost.py [--profile]
"""
import cProfile
import dataclasses
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import dealer, fss, nn_ops, runtime  # noqa: E402
from paper_2006_04593_b200.sharing import encode_fixed, share  # noqa: E402

M = 2048


class Loopback:
    def __init__(self):
        self.q = None

    def send(self, frame):
        self.q = frame

    def recv(self):
        return self.q

    def close(self):
        pass


def fresh(k):
    """The same key arrays with an unspent mask (so loops can reuse them)."""
    return dataclasses.replace(k, consumed=None)


def per_party(name, prog, reps=400):
    s = runtime.Session(0, Loopback())
    for _ in range(20):
        prog(s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        prog(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:16s} one party, loopback: {1e6 * (t1 - t0) / reps:8.1f} us host per call", flush=True)
    if "--profile" in sys.argv:
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(reps):
            prog(s)
        pr.disable()
        torch.cuda.synchronize()
        pstats.Stats(pr).sort_stats(os.environ.get("SORT", "tottime")).print_stats(int(os.environ.get("TOP", "22")))


def pair(name, prog, reps=200):
    for _ in range(10):
        runtime.run_local_pair(prog)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        runtime.run_local_pair(prog)
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    ts.sort()
    print(f"{name:16s} run_local_pair host wall: median {1e6 * ts[len(ts) // 2]:8.1f} us", flush=True)


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(1)
    xs = share(encode_fixed(rng.uniform(-100, 100, M), 3, 32), rng, precision=3)
    d = dealer.make_dealer(32, seed=2)
    relu = [d.for_party(p).relu(M) for p in (0, 1)]
    eqk = [d.for_party(p).eq_keys(M) for p in (0, 1)]

    sign = lambda s: fss.sign_protocol(s, xs[s.party], fresh(relu[s.party].cmp))  # noqa: E731
    eq = lambda s: fss.eq_protocol(s, xs[s.party], fresh(eqk[s.party]))  # noqa: E731
    rl = lambda s: nn_ops.relu(s, xs[s.party], nn_ops.ReluPrep(  # noqa: E731
        fresh(relu[s.party].cmp), dataclasses.replace(relu[s.party].triple, consumed=False)))
    for name, prog in (("sign_protocol", sign), ("eq_protocol", eq), ("relu", rl)):
        per_party(name, prog)
    pair("empty program", lambda s: None)
    for name, prog in (("sign_protocol", sign), ("eq_protocol", eq), ("relu", rl)):
        pair(name, prog)


if __name__ == "__main__":
    main()
