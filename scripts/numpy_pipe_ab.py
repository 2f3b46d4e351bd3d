"""A/B of the staged (numpy) evaluation pipeline: both parties' fss.eval_cmp on
numpy x of 2^24 elements, keys resident, the in-tree library against a variant
library (FSS_VARIANT_LIB); alternating rounds, median wall time per step.

  FSS_VARIANT_LIB=path python scripts/numpy_pipe_ab.py
"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_04593_b200 import _lib, fss  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
tree = _lib.load()
libs = {"tree": tree}
vpath = os.environ.get("FSS_VARIANT_LIB")
if vpath:
    v = ctypes.CDLL(vpath)
    for name, argtypes in _lib.SIGNATURES.items():
        fn = getattr(v, name)
        fn.argtypes = argtypes
        fn.restype = _lib._RESTYPE.get(name, ctypes.c_int)
    libs["variant"] = v
N = 1 << 24
alpha, k0, k1 = fss.keygen_cmp(32, np.random.default_rng(3), N, device=dev)
x = np.random.default_rng(4).integers(0, 1 << 32, N, dtype=np.uint64)
times = {k: [] for k in libs}
ref = None
for rnd in range(7):
    for name, lib in libs.items():
        _lib._lib = lib
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        y0 = fss.eval_cmp(0, k0, x)
        y1 = fss.eval_cmp(1, k1, x)
        t = time.perf_counter() - t0
        if rnd:
            times[name].append(t)
        if ref is None:
            ref = (y0.copy(), y1.copy())
        else:
            assert np.array_equal(y0, ref[0]) and np.array_equal(y1, ref[1]), name
_lib._lib = tree
out = {k: {"ms_per_step": sorted(v)[len(v) // 2] * 1e3, "comparisons_per_s": N / (sorted(v)[len(v) // 2])}
       for k, v in times.items()}
print(json.dumps(out))
