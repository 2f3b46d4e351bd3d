"""Chrome trace (torch.profiler, CPU + CUDA) of one in-process two-party run of
a small online protocol, to find host gaps between the kernels:

  python scripts/trace_protocol.py [config1|config2|relu|argmax] [out.json]

config1 = dealer (keygen_cmp 2^16) + sign_protocol on 2^16 (the
protocol_with_dealer number of scripts/bench_configs.py); prints the wall time
of 20 runs (median) before tracing one more.
"""
import os
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import dealer, fss, nn_ops, runtime  # noqa: E402
from paper_2006_04593_b200.ring import RingTensor  # noqa: E402
from paper_2006_04593_b200.sharing import AdditiveShare, encode_fixed, share  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "config1"
out = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/trace_{what}.json"
N = 1 << 16 if what == "config1" else 1 << 20
prng = np.random.default_rng(2)
if what == "config1":
    xs = share(encode_fixed(prng.uniform(-100, 100, N), 3, 32), prng, precision=3)
elif what == "config2":
    xs = share(RingTensor.from_ints(prng.integers(-3, 4, N), 32), prng, precision=0)
elif what == "relu":
    shape = (1, 64, 112, 112)
    xs = share(encode_fixed(prng.uniform(-100, 100, shape), 3, 32), prng, precision=3)
else:
    shape = (16, 64, 56, 56)
    xs = share(encode_fixed(prng.uniform(-10, 10, shape), 3, 32), prng, precision=3)
    xs = [x.reshape(1024, 56, 56) for x in xs]


def run():
    d = dealer.make_dealer(32, seed=3)
    if what in ("relu", "argmax"):
        preps = []
        for p in (0, 1):
            v = d.for_party(p)
            preps.append(v.relu_shaped(shape) if what == "relu" else v.maxpool(56, 2, 2, planes=1024))

    def prog(session):
        view = d.for_party(session.party)
        if what == "config1":
            return fss.sign_protocol(session, AdditiveShare(session.party, xs[session.party].values, 0),
                                     view.cmp_keys(N))
        if what == "config2":
            return fss.eq_protocol(session, xs[session.party], view.eq_keys(N))
        if what == "relu":
            return nn_ops.relu(session, xs[session.party], preps[session.party])
        return nn_ops.maxpool(session, xs[session.party], 2, preps[session.party], 2)
    torch.cuda.synchronize()   # relu / argmax: material dealt before, online timed alone
    t0 = time.perf_counter()
    runtime.run_local_pair(prog)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for _ in range(3):
    run()
ts = sorted(run() for _ in range(20))
print(what, "wall ms median %.3f min %.3f" % (ts[10] * 1e3, ts[0] * 1e3), flush=True)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    run()
prof.export_chrome_trace(out)
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=20))
