"""Tune the pinned-host eval pipeline (fss._run_eval): host link bandwidth and
eval_cmp from pinned host x for several chunk sizes (2^24 DCF keys, n=32)."""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import fss  # noqa: E402

dev = torch.device("cuda", 0)
N = 1 << 24
out = {}
h = torch.empty(N, dtype=torch.int64, pin_memory=True)
d = torch.empty(N, dtype=torch.int64, device=dev)
for name, fn in (("h2d_GBps", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h_GBps", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    out[name] = 10 * N * 8 / (time.perf_counter() - t0) / 1e9
rng = np.random.default_rng(1)
alpha, k0, k1 = fss.keygen_cmp(32, rng, N, device=dev)
xh = alpha.view(torch.int64).cpu().pin_memory().view(torch.uint64)
xd = alpha
fss.eval_cmp(0, k0, xd)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    fss.eval_cmp(0, k0, xd)
    fss.eval_cmp(1, k1, xd)
torch.cuda.synchronize()
out["device_only_cmp_per_s"] = 5 * N / (time.perf_counter() - t0)
for chunk in (1 << 20, 1 << 21, 1 << 22, 1 << 20, 1 << 21, 1 << 22, 1 << 19, 1 << 20):
    fss.PIPELINE_CHUNK = chunk
    fss.eval_cmp(0, k0, xh)
    t0 = time.perf_counter()
    for _ in range(5):
        r0 = fss.eval_cmp(0, k0, xh)
        r1 = fss.eval_cmp(1, k1, xh)
    dt = time.perf_counter() - t0
    assert bool(((r0.view(torch.int64) + r1.view(torch.int64)) & 0xFFFFFFFF == 1).all())
    out.setdefault(f"pinned_chunk_2^{chunk.bit_length() - 1}_cmp_per_s", []).append(5 * N / dt)
print(json.dumps(out, indent=1))
