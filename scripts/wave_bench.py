"""Launch-shape experiment of the eval kernels, DCF/DPF eval at the sizes of
the BASELINE protocol configs (802,816 = config 3 ReLU) and a few others; CUDA
events, median of 9. Compares the library under test ("balanced") with a
variant library at build/variants/lib_wave_off.so ("1024"). The recorded run
(profiles/r01_wave_bench.json) compared, with per-CTA contiguous element runs
(cta_span), a thread count trimmed so the last pass is full ("balanced")
against a constant 1024 threads ("1024", FSSB_BALANCE_WAVES=0 at the time):
1024 won at every size, and the trimming was removed.

  python scripts/wave_bench.py
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_04593_b200 import _dev, _lib, fss  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
libs = {"balanced": _lib.load()}
v = ctypes.CDLL(os.path.join(ROOT, "build", "variants", "lib_wave_off.so"))
v.fss_dcf_eval.argtypes = _lib.SIGNATURES["fss_dcf_eval"]
v.fss_dpf_eval.argtypes = _lib.SIGNATURES["fss_dpf_eval"]
libs["1024"] = v
out = {}
for N in (200_000, 802_816, 1 << 20, 2_408_448, 3_000_000, 1 << 22):
    _, k0, _ = fss.keygen_cmp(32, np.random.default_rng(1), N, device=dev)
    _, e0, _ = fss.keygen_eq(32, np.random.default_rng(1), N, device=dev)
    x = torch.zeros(N, dtype=torch.int64, device=dev).view(torch.uint64)
    res = torch.empty(N, dtype=torch.uint64, device=dev)
    row = {}
    for name, lib in libs.items():
        def dcf():
            lib.fss_dcf_eval(0, 32, 32, N, N, _dev.ptr(k0.seed0), _dev.ptr(k0.scw), _dev.ptr(k0.tcw),
                             _dev.ptr(k0.sigma_cw), _dev.ptr(k0.leaf_cw), _dev.ptr(x), _dev.ptr(res), None,
                             stream.cuda_stream)

        def dpf():
            lib.fss_dpf_eval(0, 32, N, N, _dev.ptr(e0.seed0), _dev.ptr(e0.scw), _dev.ptr(e0.tcw),
                             _dev.ptr(e0.cw_final), _dev.ptr(x), _dev.ptr(res), stream.cuda_stream)
        for kname, fn in (("dcf", dcf), ("dpf", dpf)):
            fn()
            ts = []
            for _ in range(9):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            row[f"{kname}_{name}_ms"] = sorted(ts)[4]
    out[N] = row
    print(N, json.dumps(row), flush=True)
with open(os.path.join(ROOT, "gpurun_out", "wave_bench.json"), "w") as fh:
    json.dump(out, fh, indent=1)
