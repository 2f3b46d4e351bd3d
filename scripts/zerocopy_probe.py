"""Host-buffer evaluation two ways, 2^24 DCF keys (n = 32), party 0 + party 1
per step, pinned host x in / pinned host shares out:
  pipeline  -- fss.eval_cmp on the pinned tensor (since the zero-copy change
               this IS the zero-copy path; before it, the chunked 2-stream
               H2D / kernel / D2H pipeline);
  zerocopy  -- the C ABI called on the host pointers directly;
  numpy     -- fss.eval_cmp on a pageable numpy array (staged pipeline).
Wall time per step (median of 5) and bit-equality of the two.

  python scripts/zerocopy_probe.py [log2n]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import _dev, _lib, fss  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
N = 1 << log2n
dev = torch.device("cuda", 0)
_, k0, k1 = fss.keygen_cmp(32, np.random.default_rng(1), N, device=dev)
x = torch.empty(N, dtype=torch.int64, pin_memory=True)
x.copy_(torch.from_numpy(np.random.default_rng(2).integers(0, 1 << 32, N, dtype=np.uint64).view(np.int64)))
xu = x.view(torch.uint64)
outs = [torch.empty(N, dtype=torch.int64, pin_memory=True) for _ in range(2)]
stream = torch.cuda.current_stream(dev)


def pipeline():
    return fss.eval_cmp(0, k0, xu), fss.eval_cmp(1, k1, xu)


def zerocopy():
    for p, k in ((0, k0), (1, k1)):
        _lib.call("fss_dcf_eval", p, 32, 32, N, N, _dev.ptr(k.seed0), _dev.ptr(k.scw), _dev.ptr(k.tcw),
                  _dev.ptr(k.sigma_cw), _dev.ptr(k.leaf_cw), x.data_ptr(), outs[p].data_ptr(), None,
                  stream.cuda_stream)
    stream.synchronize()
    return outs


def timed(fn):
    fn()
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[2]


xn = x.numpy().view(np.uint64).copy()      # pageable numpy input (the reference's calling style)


def numpy_path():
    return fss.eval_cmp(0, k0, xn), fss.eval_cmp(1, k1, xn)


tp, tz, tn = timed(pipeline), timed(zerocopy), timed(numpy_path)
r0, r1 = pipeline()
z = zerocopy()
assert torch.equal(r0.view(torch.int64), z[0]) and torch.equal(r1.view(torch.int64), z[1])
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
xd = xu.to(dev)
a.record()
fss.eval_cmp(0, k0, xd)
fss.eval_cmp(1, k1, xd)
b.record()
b.synchronize()
print(f"N=2^{log2n}: device-resident {a.elapsed_time(b):.2f} ms, pipeline {tp * 1e3:.2f} ms, "
      f"zerocopy {tz * 1e3:.2f} ms, numpy {tn * 1e3:.2f} ms per step; comparisons/s pinned host "
      f"{N / tp:.4g} (fss.eval_cmp), zerocopy C-ABI {N / tz:.4g}, numpy (staged pipeline) {N / tn:.4g}")
