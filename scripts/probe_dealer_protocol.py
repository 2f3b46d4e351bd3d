"""Wall time of config 1's protocol_with_dealer (dealer keygen inside the
in-process pair + one sign test, 2^16) over repeated runs, with the dealer's
cross-stream hand-over as shipped and with record_stream disabled."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import dealer, fss, runtime  # noqa: E402
from paper_2006_04593_b200.sharing import AdditiveShare, encode_fixed, share  # noqa: E402

N = 1 << 16
prng = np.random.default_rng(2)
xs = share(encode_fixed(prng.uniform(-100, 100, N), 3, 32), prng, precision=3)


def run(seed):
    d = dealer.make_dealer(32, seed=seed)

    def prog(session):
        keys = d.for_party(session.party).cmp_keys(N)
        return fss.sign_protocol(session, AdditiveShare(session.party, xs[session.party].values, 0), keys)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    runtime.run_local_pair(prog)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


for label in ("shipped", "no_record_stream", "shipped_again"):
    if label == "no_record_stream":
        orig = dealer._hand_over
        dealer._hand_over = lambda item, ready: torch.cuda.current_stream(ready.device).wait_event(ready.event)
    ts = [run(i) for i in range(12)]
    print(label, " ".join("%.3f" % t for t in ts), flush=True)
    if label == "no_record_stream":
        dealer._hand_over = orig
