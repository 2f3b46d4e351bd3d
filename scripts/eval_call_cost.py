"""Host cost of one public evaluation call (fss.eval_cmp / fss.eval_eq with a
device x) against the kernel it launches, at small batches where the host
part is visible in a single call's latency.

  * host_us: host time per call while the GPU runs behind (100 calls on a
    1-element batch whose kernel outlasts the host work; perf_counter)
  * call_us: CUDA events around one call on an idle stream (what
    scripts/bench_configs.py's sweep records), median of 15
  * kernel_us: CUDA events around the bare C-ABI launch with prepared
    pointers, median of 15

  python scripts/eval_call_cost.py [--out gpurun_out/eval_call_cost.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2006_04593_b200 import _dev, _lib, fss  # noqa: E402

DEV = torch.device("cuda", 0)


def med_events(fn, reps=15, warm=3):
    s = torch.cuda.current_stream(DEV)
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[len(ts) // 2]


def host_per_call(fn, calls=100):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(calls):
        fn()
    t = (time.perf_counter() - t0) / calls * 1e6
    torch.cuda.synchronize()
    return t


def bare(kind, k, x, out):
    s = _dev.stream_handle(DEV)
    ld = k.scw.stride(0) // 16
    if kind == "cmp":
        args = ("fss_dcf_eval", 0, k.n_bits, int(k.out_bits), k.count, ld, _dev.ptr(k.seed0),
                _dev.ptr(k.scw), _dev.ptr(k.tcw), _dev.ptr(k.sigma_cw), _dev.ptr(k.leaf_cw),
                _dev.ptr(x), _dev.ptr(out), None, s)
    else:
        args = ("fss_dpf_eval", 0, k.n_bits, k.count, ld, _dev.ptr(k.seed0), _dev.ptr(k.scw),
                _dev.ptr(k.tcw), _dev.ptr(k.cw_final), _dev.ptr(x), _dev.ptr(out), s)
    return lambda: _lib.call(*args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.set_device(DEV)
    _lib.load()
    res = {}
    for kind in ("cmp", "eq"):
        keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
        ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
        row = {}
        for log2n in (0, 16, 18):
            N = 1 << log2n
            alpha, k0, _ = keygen(32, np.random.default_rng(log2n), N, device=DEV)
            x = alpha.clone()
            out = torch.empty(N, dtype=torch.uint64, device=DEV)
            r = {"call_us": med_events(lambda: ev(0, k0, x)),
                 "kernel_us": med_events(bare(kind, k0, x, out))}
            if log2n == 0:
                r["host_us"] = host_per_call(lambda: ev(0, k0, x))
            r["call_over_kernel"] = r["call_us"] / r["kernel_us"]
            row[f"2^{log2n}"] = r
        res[kind] = row
    text = json.dumps(res, indent=1)
    print(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
