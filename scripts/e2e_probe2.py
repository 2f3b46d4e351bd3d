"""Variance study of the pinned-host eval pipeline: per-call wall times for
several chunk sizes, interleaved, 2^24 DCF keys."""
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
rng = np.random.default_rng(1)
alpha, k0, k1 = fss.keygen_cmp(32, rng, N, device=dev)
xh = alpha.view(torch.int64).cpu().pin_memory().view(torch.uint64)
res = {}
for rep in range(4):
    for chunk in (1 << 20, 1 << 21, 1 << 22):
        fss.PIPELINE_CHUNK = chunk
        ts = []
        for _ in range(6):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r0 = fss.eval_cmp(0, k0, xh)
            r1 = fss.eval_cmp(1, k1, xh)
            ts.append(time.perf_counter() - t0)
        res.setdefault(str(chunk), []).append([round(N / t / 1e6, 1) for t in ts])
print(json.dumps(res, indent=1))
