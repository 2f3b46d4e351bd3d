"""Per-element cost of DCF / DPF eval (n = 32, plain device x) across batch
sizes, for the in-tree library and optional variant libraries
(FSS_VARIANT_LIBS=name=path,name=path): CUDA events around single launches,
median of 15 after 3 warm-ups. Reports ms per launch, ns per element and the
rate relative to the 2^22 launch of the same library.

  python scripts/small_batch_probe.py [out.json]
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
libs = {"tree": _lib.load()}
for item in filter(None, os.environ.get("FSS_VARIANT_LIBS", "").split(",")):
    name, path = item.split("=", 1)
    v = ctypes.CDLL(path)
    for fn in ("fss_dcf_eval", "fss_dpf_eval", "fss_dcf_keygen", "fss_dpf_keygen"):
        getattr(v, fn).argtypes = _lib.SIGNATURES[fn]
        getattr(v, fn).restype = ctypes.c_int
    libs[name] = v

SIZES = [1, 32, 148 * 32, 1 << 14, 1 << 15, 1 << 16, 1 << 17, 200_000, 802_816, 1 << 20, 1 << 22]
NMAX = max(SIZES)
_, k0, _ = fss.keygen_cmp(32, np.random.default_rng(1), NMAX, device=dev)
_, e0, _ = fss.keygen_eq(32, np.random.default_rng(1), NMAX, device=dev)
_tape_rng = np.random.default_rng(5)
TAPE = [torch.from_numpy(_tape_rng.integers(0, 1 << 32, NMAX, dtype=np.uint64).view(np.int64)).to(dev)
        .view(torch.uint64) for _ in range(2)]
TAPE += [torch.from_numpy(_tape_rng.integers(0, 256, (NMAX, 16), dtype=np.uint8)).to(dev) for _ in range(2)]
x = torch.from_numpy(np.random.default_rng(2).integers(0, 1 << 32, NMAX, dtype=np.uint64)
                     .view(np.int64)).to(dev).view(torch.uint64)
res = torch.empty(NMAX, dtype=torch.uint64, device=dev)
ref = {}
out = {}
for name, lib in libs.items():
    rows = {}
    for N in SIZES:
        def dcf():
            rc = lib.fss_dcf_eval(0, 32, 32, N, NMAX, _dev.ptr(k0.seed0), _dev.ptr(k0.scw), _dev.ptr(k0.tcw),
                                  _dev.ptr(k0.sigma_cw), _dev.ptr(k0.leaf_cw), _dev.ptr(x), _dev.ptr(res),
                                  None, stream.cuda_stream)
            assert rc == 0

        def dpf():
            rc = lib.fss_dpf_eval(0, 32, N, NMAX, _dev.ptr(e0.seed0), _dev.ptr(e0.scw), _dev.ptr(e0.tcw),
                                  _dev.ptr(e0.cw_final), _dev.ptr(x), _dev.ptr(res), stream.cuda_stream)
            assert rc == 0
        kg = {}

        def dcf_kg():
            kg["c"] = [torch.empty((32, N, 16), dtype=torch.uint8, device=dev),
                       torch.empty((32, N), dtype=torch.uint8, device=dev),
                       torch.empty((32, N), dtype=torch.uint64, device=dev),
                       torch.empty((33, N), dtype=torch.uint64, device=dev),
                       torch.empty(N, dtype=torch.uint64, device=dev)]
            c = kg["c"]
            rc = lib.fss_dcf_keygen(32, 32, N, _dev.ptr(tape[0]), _dev.ptr(tape[1]), _dev.ptr(tape[2]),
                                    _dev.ptr(tape[3]), _dev.ptr(c[0]), _dev.ptr(c[1]), _dev.ptr(c[2]),
                                    _dev.ptr(c[3]), _dev.ptr(c[4]), stream.cuda_stream)
            assert rc == 0

        def dpf_kg():
            kg["e"] = [torch.empty((32, N, 16), dtype=torch.uint8, device=dev),
                       torch.empty((32, N), dtype=torch.uint8, device=dev),
                       torch.empty(N, dtype=torch.uint64, device=dev),
                       torch.empty(N, dtype=torch.uint64, device=dev)]
            c = kg["e"]
            rc = lib.fss_dpf_keygen(32, N, _dev.ptr(tape[0]), _dev.ptr(tape[1]), _dev.ptr(tape[2]),
                                    _dev.ptr(tape[3]), _dev.ptr(c[0]), _dev.ptr(c[1]), _dev.ptr(c[2]),
                                    _dev.ptr(c[3]), stream.cuda_stream)
            assert rc == 0
        tape = [t[:N].contiguous() for t in TAPE]
        row = {}
        for kname, fn in (("dcf_keygen", dcf_kg), ("dpf_keygen", dpf_kg)):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(15):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            got = kg["c" if kname == "dcf_keygen" else "e"]
            if name == "tree":
                ref[(kname, N)] = [g.clone() for g in got]
            else:
                for g, w in zip(got, ref[(kname, N)]):
                    assert torch.equal(g.view(torch.uint8), w.view(torch.uint8)), (name, kname, N)
            ms = sorted(ts)[7]
            row[kname] = {"ms": ms, "ns_per_elem": ms * 1e6 / N}
        for kname, fn in (("dcf", dcf), ("dpf", dpf)):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(15):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            ms = sorted(ts)[7]
            # parity of the variant against the in-tree library on this size
            got = res[:N].clone()
            if name == "tree":
                ref[(kname, N)] = got
            else:
                assert torch.equal(got.view(torch.int64), ref[(kname, N)].view(torch.int64)), (name, kname, N)
            row[kname] = {"ms": ms, "ns_per_elem": ms * 1e6 / N}
        rows[N] = row
        print(name, N, json.dumps(row), flush=True)
    for N, row in rows.items():
        for kname in ("dcf", "dpf", "dcf_keygen", "dpf_keygen"):
            row[kname]["rel_to_2p22"] = rows[1 << 22][kname]["ns_per_elem"] / row[kname]["ns_per_elem"]
    out[name] = rows
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "small_batch_probe.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
