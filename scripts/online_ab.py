"""A/B of the in-process pair's hand-over (ARIANN_LOCAL_SPIN=1 spinning
scheduler vs 0 blocking queues) on the online protocols: config 1 (2^16 sign
tests with dealer), config 3 (ReLU on 1x64x112x112, online), wall ms, median.

  python scripts/online_ab.py [reps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_04593_b200 import dealer, fss, nn_ops, runtime  # noqa: E402
from paper_2006_04593_b200.sharing import AdditiveShare, encode_fixed, share  # noqa: E402


def wall(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
    print(f"cpus: os.cpu_count={os.cpu_count()} affinity={len(os.sched_getaffinity(0))}", flush=True)
    rng = np.random.default_rng(4)
    x1 = share(encode_fixed(rng.uniform(-100, 100, 1 << 16), 3, 32), rng, precision=3)
    shape = (1, 64, 112, 112)
    x3 = share(encode_fixed(rng.uniform(-100, 100, shape), 3, 32), rng, precision=3)
    res = {}
    for mode in ("0", "1", "0", "1"):
        os.environ["ARIANN_LOCAL_SPIN"] = mode
        c1, c3 = [], []
        for rep in range(reps + 3):
            d = dealer.make_dealer(32, seed=3)

            def prog1(s):
                keys = d.for_party(s.party).cmp_keys(1 << 16)
                return fss.sign_protocol(s, AdditiveShare(s.party, x1[s.party].values, 0), keys)
            _, t1 = wall(lambda: runtime.run_local_pair(prog1))
            preps = [d.for_party(p).relu_shaped(shape) for p in (0, 1)]
            _, t3 = wall(lambda: runtime.run_local_pair(lambda s: nn_ops.relu(s, x3[s.party], preps[s.party])))
            if rep >= 3:
                c1.append(t1 * 1e3)
                c3.append(t3 * 1e3)
        res.setdefault(mode, []).append((float(np.median(c1)), float(np.median(c3))))
        print(f"spin={mode}: config1 sign+dealer {np.median(c1):.3f} ms  relu online {np.median(c3):.3f} ms",
              flush=True)


if __name__ == "__main__":
    main()
