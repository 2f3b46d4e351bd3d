"""Online latency of private ReLU (config 3, 1x64x112x112) through the
in-process two-party runtime: all runs listed (fresh dealer material each), plus
the allocator's cudaMalloc / retry counters, to separate kernel time from host
and allocator effects.

  python scripts/relu_latency.py [reps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import dealer, fss, nn_ops, runtime  # noqa: E402
from paper_2006_04593_b200.sharing import encode_fixed, share  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
shape = (1, 64, 112, 112)
rng = np.random.default_rng(4)
xs = share(encode_fixed(rng.uniform(-100, 100, shape), 3, 32), rng, precision=3)
stamps = {}


def prog_for(prep):
    def prog(s):
        t = stamps.setdefault(s.party, [])
        t.append(("start", time.perf_counter()))
        out = nn_ops.relu(s, xs[s.party], prep[s.party])
        t.append(("end", time.perf_counter()))
        return out
    return prog


for i in range(reps):
    d = dealer.make_dealer(32, seed=2)
    prep = [d.for_party(p).relu_shaped(shape) for p in (0, 1)]
    torch.cuda.synchronize()
    st0 = torch.cuda.memory_stats()
    stamps.clear()
    t0 = time.perf_counter()
    runtime.run_local_pair(prog_for(prep))
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st1 = torch.cuda.memory_stats()
    rel = {p: [(k, round((v - t0) * 1e3, 3)) for k, v in stamps[p]] for p in stamps}
    print(f"run {i}: wall {1e3 * (t2 - t0):.2f} ms (pair returned {1e3 * (t1 - t0):.2f}), "
          f"cudaMalloc +{st1.get('num_device_alloc', 0) - st0.get('num_device_alloc', 0)}, "
          f"retries +{st1.get('num_alloc_retries', 0) - st0.get('num_alloc_retries', 0)}, stamps {rel}",
          flush=True)
_, k0, _ = fss.keygen_cmp(32, np.random.default_rng(1), 802816)
x = torch.zeros(802816, dtype=torch.int64, device="cuda").view(torch.uint64)
fss.eval_cmp(0, k0, x)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    fss.eval_cmp(0, k0, x)
b.record()
b.synchronize()
print("eval_cmp 802816 ms", a.elapsed_time(b) / 10)
