"""Host-side timeline of one in-process two-party online run (no profiler):
wraps the protocol's host entry points with perf_counter spans per party
thread and prints them relative to the run start, plus the wall time.

  python scripts/host_timeline.py [relu|config1|argmax|k2]
"""
import functools
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import beaver, dealer, fss, nn_ops, runtime, sharing  # noqa: E402
from paper_2006_04593_b200.sharing import AdditiveShare, encode_fixed, share  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "relu"
LOG = []


GPU = []   # (thread, label, event before the call, event after it) on the calling stream
GPU_LABELS = ("_eval_cmp_masked", "_eval_eq_masked", "beaver_protocol")


def wrap(mod, name, label=None):
    fn = getattr(mod, name)

    @functools.wraps(fn)
    def w(*a, **k):
        t0 = time.perf_counter()
        gpu = name in GPU_LABELS
        if gpu:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        try:
            return fn(*a, **k)
        finally:
            LOG.append((threading.current_thread().name, label or name, t0, time.perf_counter()))
            if gpu:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record()
                GPU.append((threading.current_thread().name, label or name, e0, e1))
    setattr(mod, name, w)


for mod, names in ((fss, ["sign_protocol", "eq_protocol", "_masked_round", "_eval_cmp_masked",
                          "_eval_eq_masked"]),
                   (beaver, ["beaver_protocol"]), (nn_ops, ["relu", "argmax", "maxpool"])):
    for n in names:
        wrap(mod, n, f"{mod.__name__.split('.')[-1]}.{n}")
if os.environ.get("FINE"):   # finer host spans of the prologue up to the first evaluation launch
    for mod, names in ((nn_ops, ["_plus_public", "mul_protocol"]), (fss, ["_pack", "_peer_wire"]),
                       (runtime, ["run_session"])):
        for n in names:
            if hasattr(mod, n):
                wrap(mod, n, f"{mod.__name__.split('.')[-1]}.{n}")
    wrap(fss.CmpKeyBatch, "take_unused", "CmpKeyBatch.take_unused")
_orig_ex = runtime.Session.exchange


def _ex(self, *a, **k):
    t0 = time.perf_counter()
    try:
        return _orig_ex(self, *a, **k)
    finally:
        LOG.append((threading.current_thread().name, "exchange", t0, time.perf_counter()))


runtime.Session.exchange = _ex
rng = np.random.default_rng(4)
if what == "relu":
    shape = (1, 64, 112, 112)
    xs = share(encode_fixed(rng.uniform(-100, 100, shape), 3, 32), rng, precision=3)
elif what == "config1":
    xs = share(encode_fixed(rng.uniform(-100, 100, 1 << 16), 3, 32), rng, precision=3)
else:
    xs = share(encode_fixed(rng.uniform(-10, 10, (16, 64, 56, 56)), 3, 32), rng, precision=3)
    xs = [x.reshape(1024, 56, 56) for x in xs]


def once():
    d = dealer.make_dealer(32, seed=2)
    preps = []
    for p in (0, 1):
        v = d.for_party(p)
        if what == "relu":
            preps.append(v.relu_shaped(shape))
        elif what == "config1":
            preps.append(v.cmp_keys(1 << 16))
        elif what == "k2":
            preps.append(v.maxpool_k2(56, planes=1024))
        else:
            preps.append(v.maxpool(56, 2, 2, planes=1024))
    torch.cuda.synchronize()

    def prog(s):
        if what == "relu":
            return nn_ops.relu(s, xs[s.party], preps[s.party])
        if what == "config1":
            return fss.sign_protocol(s, AdditiveShare(s.party, xs[s.party].values, 0), preps[s.party])
        if what == "k2":
            return nn_ops.maxpool_k2(s, xs[s.party], preps[s.party])
        return nn_ops.maxpool(s, xs[s.party], 2, preps[s.party], 2)
    LOG.clear()
    GPU.clear()
    start = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    start.record()
    runtime.run_local_pair(prog)
    t1 = time.perf_counter()
    end = torch.cuda.Event(enable_timing=True)
    end.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    gpu = [(th, name, start.elapsed_time(a), start.elapsed_time(b)) for th, name, a, b in GPU]
    return t0, t1, t2, gpu, start.elapsed_time(end)


for _ in range(5):
    once()
walls, spans, gspans, gends = [], {}, {}, []
for _ in range(11):
    t0, t1, t2, gpu, gend = once()
    walls.append(t2 - t0)
    gends.append(gend)
    seen = {}
    for th, name, a, b in sorted(LOG, key=lambda r: r[2]):
        key = (th[-12:], name, seen.setdefault((th, name), 0))
        seen[(th, name)] += 1
        spans.setdefault(key, []).append(((a - t0) * 1e3, (b - t0) * 1e3))
    seen = {}
    for th, name, a, b in gpu:
        key = (th[-12:], name, seen.setdefault((th, name), 0))
        seen[(th, name)] += 1
        gspans.setdefault(key, []).append((a, b))


def med(v):
    return sorted(v)[len(v) // 2]


print(what, "online wall ms: median %.3f over %d runs; GPU start->end event median %.3f ms"
      % (med(walls) * 1e3, len(walls), med(gends)))
print("host spans (median start -> median end, ms from the run start):")
for key, v in sorted(spans.items(), key=lambda kv: med([a for a, _ in kv[1]])):
    print("  %-12s %-28s %8.3f -> %8.3f" % (key[0], key[1], med([a for a, _ in v]), med([b for _, b in v])))
print("GPU spans of the same calls (CUDA events on the party stream before / after the call):")
for key, v in sorted(gspans.items(), key=lambda kv: med([a for a, _ in kv[1]])):
    print("  %-12s %-28s %8.3f -> %8.3f" % (key[0], key[1], med([a for a, _ in v]), med([b for _, b in v])))
