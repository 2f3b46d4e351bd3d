"""The BASELINE north-star batch, run for real on one B200: DCF and DPF keygen +
eval at n = 32 on a 2^28-element batch, every element checked.

The 2^28 keys of both parties do not fit one GPU in the reference layout
(≈ 300 GB for DCF), so the batch is dealt as 4 shards of 2^26 with the sharded
dealer (shard.keygen_*_shard: shard r is bit-identical to elements
[r * 2^26, (r+1) * 2^26) of ONE keygen of the whole 2^28 batch -- exactly what
rank r of a 4-GPU job would hold). Each shard is generated, evaluated by both
parties on x (half the elements x = alpha, the rest uniform) and every share
pair is reconstructed on device and compared with the predicate; then the
shard is freed. Times are CUDA-event times summed over the shards (nothing
extrapolated; one untimed warm-up shard first so that the allocator's one-time
cudaMalloc of the shard-sized buffers is not counted as keygen). Output:
gpurun_out/full_2p28.json.

  python scripts/full_2p28.py [log2_total] [log2_shards]
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2006_04593_b200 import fss, shard  # noqa: E402


def main(log2_total: int = 28, log2_shards: int = 2):
    dev = torch.device("cuda", 0)
    total, world = 1 << log2_total, 1 << log2_shards
    stream = torch.cuda.current_stream(dev)
    out = {"total": total, "shards": world, "n": 32}
    t_wall = time.perf_counter()
    for kind in ("cmp", "eq"):
        # untimed warm-up shard: the caching allocator takes the shard-sized
        # device memory once (cudaMalloc of ~75 GB is not part of keygen)
        warm = (shard.keygen_cmp_shard if kind == "cmp" else shard.keygen_eq_shard)(
            32, np.random.default_rng(1), total, 0, world, device=dev)
        del warm
        kg_ms = ev_ms = 0.0
        checked = 0
        for r in range(world):
            rng = np.random.default_rng(2028)           # every shard starts from the same dealer state
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if kind == "cmp":
                alpha, k0, k1 = shard.keygen_cmp_shard(32, rng, total, r, world, device=dev)
            else:
                alpha, k0, k1 = shard.keygen_eq_shard(32, rng, total, r, world, device=dev)
            b.record(stream)
            b.synchronize()
            kg_ms += a.elapsed_time(b)
            m = alpha.shape[0]
            g = torch.Generator(device=dev).manual_seed(31 + r)
            x = torch.randint(0, 1 << 32, (m,), device=dev, dtype=torch.int64, generator=g)
            hit = torch.rand(m, device=dev, generator=g) < 0.5
            x = torch.where(hit, alpha.view(torch.int64), x).view(torch.uint64)
            ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
            a.record(stream)
            y0 = ev(0, k0, x)
            y1 = ev(1, k1, x)
            b.record(stream)
            b.synchronize()
            ev_ms += a.elapsed_time(b)
            rec = (y0.view(torch.int64) + y1.view(torch.int64)) & 0xFFFFFFFF
            xs, al = x.view(torch.int64), alpha.view(torch.int64)
            want = (xs <= al) if kind == "cmp" else (xs == al)
            assert torch.equal(rec, want.to(torch.int64)), f"{kind} shard {r}: reconstruction mismatch"
            checked += m
            del alpha, k0, k1, x, y0, y1, rec, want, hit   # the next shard reuses the memory
        name = "dcf" if kind == "cmp" else "dpf"
        out[name] = {"elements_checked": checked, "keygen_ms": kg_ms, "keygen_pairs_per_s": total / kg_ms * 1e3,
                     "eval_ms_both_parties": ev_ms, "party_evals_per_s": 2 * total / ev_ms * 1e3,
                     "comparisons_per_s" if kind == "cmp" else "equality_tests_per_s": total / ev_ms * 1e3}
        print(name, json.dumps(out[name]), flush=True)
    out["wall_s"] = time.perf_counter() - t_wall
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "full_2p28.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main(*(int(v) for v in sys.argv[1:3]))
