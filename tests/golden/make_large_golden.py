"""Digest fixtures of the UNMODIFIED Python reference at the BASELINE sizes.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_large_golden.py

Key material at 2^16 / 2^20 elements is far too large to commit, so this
records, for each case, the numpy seeds and the sha256 of the reference's own
outputs: the ARNK container ``serialize_keys(pack_keys(k0, k1))`` (every key
byte of both parties), ``alpha``, both parties' eval shares on a seeded input
(30 % of x equal to alpha), and a fingerprint of the generator state after
keygen. Cases: DCF n=32 at N = 1, 7, 2^16 (BASELINE config 1); DPF n=32 at
N = 1, 7, 2^20 (config 2). tests/test_gpu_large_golden.py recomputes the same
digests from the B200 path. Output: tests/golden/large_digests.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u8").tobytes()).hexdigest()


def xs_for(seed: int, alpha: np.ndarray, n: int) -> np.ndarray:
    """Public inputs: uniform in Z_2^n, 30 % replaced by alpha (hits)."""
    r = np.random.default_rng(seed)
    x = r.integers(0, 1 << n, size=alpha.shape[0], dtype=np.uint64)
    hit = r.random(alpha.shape[0]) < 0.3
    x[hit] = alpha[hit]
    return x


def main():
    sys.path.insert(0, REF)
    from ariann import fss  # noqa: E402  (the reference)

    cases = [("cmp", 32, 1), ("cmp", 32, 7), ("cmp", 32, 1 << 16),
             ("eq", 32, 1), ("eq", 32, 7), ("eq", 32, 1 << 20)]
    out = {"generator": "tests/golden/make_large_golden.py (reference ariann, numpy "
                        + np.__version__ + ")", "cases": {}}
    for kind, n, N in cases:
        seed, xseed = 77_000 + N, 88_000 + N
        t0 = time.time()
        rng = np.random.default_rng(seed)
        keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
        alpha, k0, k1 = keygen(n, rng, N)
        nxt = rng.integers(0, 1 << 32, size=4, dtype=np.uint64)
        x = xs_for(xseed, alpha, n)
        ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
        y0, y1 = ev(0, k0, x), ev(1, k1, x)
        blob = fss.serialize_keys(fss.pack_keys(k0, k1))
        mask = np.uint64((1 << n) - 1)
        rec = (y0 + y1) & mask
        want = (x <= alpha) if kind == "cmp" else (x == alpha)
        assert np.array_equal(rec, want.astype(np.uint64))
        name = f"{kind}_n{n}_N{N}"
        out["cases"][name] = {"kind": kind, "n": n, "N": N, "seed": seed, "x_seed": xseed,
                              "arnk_sha256": sha(blob), "arnk_bytes": len(blob),
                              "alpha_sha256": sha(alpha), "y0_sha256": sha(y0), "y1_sha256": sha(y1),
                              "next_draws": [int(v) for v in nxt],
                              "reference_seconds": round(time.time() - t0, 2)}
        print(name, out["cases"][name], flush=True)
    with open(os.path.join(HERE, "large_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
