"""torch.profiler view of one online protocol run (default: config 4 argmax
route MaxPool on 16x64x56x56, both parties in-process): where the time goes
between our kernels, torch glue and host work.

  python scripts/profile_protocol.py [k2|argmax|relu]
"""

import os
import sys
import time

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import dealer, nn_ops, runtime  # noqa: E402
from paper_2006_04593_b200.sharing import encode_fixed, share  # noqa: E402

route = sys.argv[1] if len(sys.argv) > 1 else "argmax"
rng = np.random.default_rng(4)
if route == "relu":
    shape = (1, 64, 112, 112)
    xs = share(encode_fixed(rng.uniform(-100, 100, shape), 3, 32), rng, precision=3)
else:
    shape = (16, 64, 56, 56)
    xs = share(encode_fixed(rng.uniform(-10, 10, shape), 3, 32), rng, precision=3)
    xs = [x.reshape(1024, 56, 56) for x in xs]


def once():
    d = dealer.make_dealer(32, seed=2)
    preps = []
    for p in (0, 1):
        v = d.for_party(p)
        if route == "relu":
            preps.append(v.relu_shaped(shape))
        elif route == "k2":
            preps.append(v.maxpool_k2(56, planes=1024))
        else:
            preps.append(v.maxpool(56, 2, 2, planes=1024))
    torch.cuda.synchronize()

    def prog(s):
        if route == "relu":
            return nn_ops.relu(s, xs[s.party], preps[s.party])
        if route == "k2":
            return nn_ops.maxpool_k2(s, xs[s.party], preps[s.party])
        return nn_ops.maxpool(s, xs[s.party], 2, preps[s.party], 2)
    t0 = time.perf_counter()
    runtime.run_local_pair(prog)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


once()
print("online wall ms:", once() * 1e3)
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    once()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
