"""Per-kernel GPU time of one online protocol run (torch.profiler / CUPTI, not
a bench number): which kernels besides the FSS evaluations cost time.

  python scripts/kernel_profile.py [relu|argmax|k2]
"""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import dealer, nn_ops, runtime  # noqa: E402
from paper_2006_04593_b200.sharing import encode_fixed, share  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "argmax"
rng = np.random.default_rng(4)
if what == "relu":
    shape = (1, 64, 112, 112)
    xs = share(encode_fixed(rng.uniform(-100, 100, shape), 3, 32), rng, precision=3)
else:
    xs = share(encode_fixed(rng.uniform(-10, 10, (16, 64, 56, 56)), 3, 32), rng, precision=3)
    xs = [x.reshape(1024, 56, 56) for x in xs]


def prep():
    d = dealer.make_dealer(32, seed=2)
    out = []
    for p in (0, 1):
        v = d.for_party(p)
        out.append(v.relu_shaped(shape) if what == "relu" else
                   v.maxpool(56, 2, 2, planes=1024) if what == "argmax" else v.maxpool_k2(56, planes=1024))
    torch.cuda.synchronize()
    return out


def prog_for(preps):
    def prog(s):
        if what == "relu":
            return nn_ops.relu(s, xs[s.party], preps[s.party])
        if what == "argmax":
            return nn_ops.maxpool(s, xs[s.party], 2, preps[s.party], 2)
        return nn_ops.maxpool_k2(s, xs[s.party], preps[s.party])
    return prog


for _ in range(3):
    runtime.run_local_pair(prog_for(prep()))
preps = prep()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    runtime.run_local_pair(prog_for(preps))
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
