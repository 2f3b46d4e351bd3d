"""Small, single-kernel-dominated workloads for ncu captures (2^22 elements, n=32).

  python scripts/profile_target.py dcf_eval|dcf_eval_zerocopy|dpf_eval|dcf_keygen|dpf_keygen|arnk_pack|arnk_unpack
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import fss  # noqa: E402

what = sys.argv[1]
N = 1 << 22
dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)
if what.startswith("arnk"):
    alpha, k0, k1 = fss.keygen_cmp(32, rng, N, device=dev)
    buf = fss._pack_device(k0)
    if what == "arnk_unpack":
        fss._unpack(fss.KIND_CMP, 0, 32, N, buf.reshape(-1), dev)
elif what.startswith("dcf"):
    alpha, k0, k1 = fss.keygen_cmp(32, rng, N, device=dev)
    if what == "dcf_eval":
        fss.eval_cmp(0, k0, alpha)
    elif what == "dcf_eval_zerocopy":       # x in / shares out in pinned host memory
        fss.eval_cmp(0, k0, alpha.cpu().pin_memory())
else:
    alpha, k0, k1 = fss.keygen_eq(32, rng, N, device=dev)
    if what == "dpf_eval":
        fss.eval_eq(0, k0, alpha)
torch.cuda.synchronize()
