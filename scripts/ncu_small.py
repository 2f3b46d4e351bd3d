"""One eval launch of a given size through a given library, for ncu:

  python scripts/ncu_small.py [lib.so|tree] LOG2N dcf|dpf
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_04593_b200 import _dev, _lib, fss  # noqa: E402

path, log2n, kind = sys.argv[1], int(sys.argv[2]), sys.argv[3]
lib = _lib.load() if path == "tree" else ctypes.CDLL(path)
for fn in ("fss_dcf_eval", "fss_dpf_eval"):
    getattr(lib, fn).argtypes = _lib.SIGNATURES[fn]
N = 1 << log2n
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev).cuda_stream
x = torch.from_numpy(np.random.default_rng(2).integers(0, 1 << 32, N, dtype=np.uint64)
                     .view(np.int64)).to(dev).view(torch.uint64)
res = torch.empty(N, dtype=torch.uint64, device=dev)
if kind == "dcf":
    _, k, _ = fss.keygen_cmp(32, np.random.default_rng(1), N, device=dev)
    rc = lib.fss_dcf_eval(0, 32, 32, N, N, _dev.ptr(k.seed0), _dev.ptr(k.scw), _dev.ptr(k.tcw),
                          _dev.ptr(k.sigma_cw), _dev.ptr(k.leaf_cw), _dev.ptr(x), _dev.ptr(res), None, st)
else:
    _, k, _ = fss.keygen_eq(32, np.random.default_rng(1), N, device=dev)
    rc = lib.fss_dpf_eval(0, 32, N, N, _dev.ptr(k.seed0), _dev.ptr(k.scw), _dev.ptr(k.tcw),
                          _dev.ptr(k.cw_final), _dev.ptr(x), _dev.ptr(res), st)
assert rc == 0
torch.cuda.synchronize()
