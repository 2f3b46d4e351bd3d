"""Where the time of one small keygen call goes (config 1: keygen_cmp(32, rng,
2^16) from a numpy Generator): CUDA events around the call on an idle stream,
host time per call, and the kernels it launches with their device times
(torch.profiler / CUPTI).

  python scripts/keygen_call_cost.py [--out gpurun_out/keygen_call_cost.json]
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

from paper_2006_04593_b200 import _lib, fss  # noqa: E402

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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.set_device(DEV)
    _lib.load()
    res = {}
    for kind, fn in (("dcf", fss.keygen_cmp), ("dpf", fss.keygen_eq)):
        for log2n in (10, 16, 20):
            N = 1 << log2n
            rng = np.random.default_rng(1)
            call = lambda: fn(32, rng, N, device=DEV)   # noqa: E731
            r = {"call_us": med_events(call)}
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(20):
                call()
            r["host_us_per_call_async"] = (time.perf_counter() - t0) / 20 * 1e6
            torch.cuda.synchronize()
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
                for _ in range(5):
                    call()
                torch.cuda.synchronize()
            kernels = {}
            for ev in prof.events():
                if ev.device_type.name == "CUDA":
                    k = kernels.setdefault(ev.name[:90], [0, 0.0])
                    k[0] += 1
                    k[1] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
            r["device_work_per_call_us"] = {k: round(v[1] / 5, 2) for k, v in kernels.items()}
            r["device_sum_us"] = round(sum(v[1] for v in kernels.values()) / 5, 2)
            res[f"{kind}_2^{log2n}"] = r
            print(kind, log2n, json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
