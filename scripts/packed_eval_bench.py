"""Evaluation straight from ARNK payload rows (fss.PackedKeyBatch,
fss_*_eval_packed) vs the level-major keys, 2^log2n keys (n = 32), device x,
CUDA events, median of 5; and the receiving party's flow "payload in HBM ->
shares": unpack + eval vs packed eval.

  python scripts/packed_eval_bench.py [log2n]
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_04593_b200 import fss  # noqa: E402


def timed(fn, stream):
    fn()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[2]


def main(log2n: int = 24):
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    N = 1 << log2n
    out = {"N": N}
    for kind in ("cmp", "eq"):
        keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
        ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
        code = fss.KIND_CMP if kind == "cmp" else fss.KIND_EQ
        alpha, k0, _ = keygen(32, np.random.default_rng(1), N, device=dev)
        x = alpha.clone()
        pk = fss.PackedKeyBatch(code, 0, 32, fss._pack_device(k0))
        assert torch.equal(ev(0, pk, x).view(torch.int64), ev(0, k0, x).view(torch.int64))
        t_unpacked = timed(lambda: ev(0, k0, x), stream)
        t_packed = timed(lambda: ev(0, pk, x), stream)
        t_unpack = timed(lambda: pk.unpack(), stream)
        row = {"eval_levelmajor_ms": t_unpacked, "eval_packed_ms": t_packed,
               "unpack_ms": t_unpack, "unpack_plus_eval_ms": t_unpack + t_unpacked,
               "packed_vs_unpack_plus_eval": (t_unpack + t_unpacked) / t_packed,
               "party_evals_per_s_packed": N / t_packed * 1e3}
        out[kind] = row
        print(kind, json.dumps(row), flush=True)
        del alpha, k0, x, pk
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "packed_eval.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 24)
