"""Host microseconds of the torch calls on the online path's glue (device and
stream contexts, events, record_stream, small allocations, ctypes launches)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import _dev, _lib  # noqa: E402


def t(name, fn, reps=20000):
    for _ in range(200):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    print(f"{name:44s} {1e6 * dt / reps:7.2f} us", flush=True)


dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
s = torch.cuda.Stream(dev)
x = torch.zeros(1024, dtype=torch.uint64, device=dev)
ev = torch.cuda.Event()
lib = _lib.load()


def ctx_device():
    with torch.cuda.device(dev):
        pass


def ctx_stream():
    with torch.cuda.stream(s):
        pass


def event_new_record():
    e = torch.cuda.Event()
    e.record(torch.cuda.current_stream(dev))


def ring_op():
    out = torch.empty(1024, dtype=torch.uint64, device=dev)
    _lib.call("fss_ring_op", 0, 32, 1024, _dev.ptr(x), _dev.ptr(x), 0, _dev.ptr(out),
              _dev.stream_handle(dev))


t("with torch.cuda.device(dev)", ctx_device)
t("with torch.cuda.stream(s)", ctx_stream)
t("torch.cuda.current_stream(dev)", lambda: torch.cuda.current_stream(dev))
t("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
t("_dev.stream_handle(dev)", lambda: _dev.stream_handle(dev))
t("torch.cuda.current_device()", torch.cuda.current_device)
t("Event() + record(current_stream)", event_new_record)
t("ev.record()", lambda: ev.record())
t("current_stream().wait_event(ev)", lambda: torch.cuda.current_stream().wait_event(ev))
t("x.record_stream(s)", lambda: x.record_stream(s))
t("s.wait_stream(current)", lambda: s.wait_stream(torch.cuda.current_stream()))
t("torch.empty(1024, u64, cuda)", lambda: torch.empty(1024, dtype=torch.uint64, device=dev))
t("x.data_ptr()", x.data_ptr)
t("_dev.ptr(x)", lambda: _dev.ptr(x))
t("x.reshape(-1)", lambda: x.reshape(-1))
t("x[:512]", lambda: x[:512])
t("x.view(torch.int64)", lambda: x.view(torch.int64))
t("lib.fss_host_load (ctypes, 1 arg)", lambda: lib.fss_host_load(None))
w = (__import__("ctypes").c_int64 * 2)()
wa = __import__("ctypes").addressof(w)
t("lib.fss_host_wait (ctypes, 8 args, ready)", lambda: lib.fss_host_wait(wa, 0, None, -1, -1, None, 0.0, 1.0))
t("getattr(_lib.load(), name) + check", lambda: _lib.check(getattr(_lib.load(), "fss_host_load")(None), "x"))
t("ring op: empty + _lib.call (8 args) + launch", ring_op)
