"""Golden vectors for prg.mask_stream (pkg/src/ariann/prg.py:128-147), produced
by the UNMODIFIED reference in the build container:

    python tests/golden/make_prg_extra.py
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from ariann import prg  # noqa: E402
    cases = [(bytes(range(16)), 0, 100, 32), (bytes(range(16)), 1, 100, 32),
             (bytes([0xFF] * 16), 7, 1, 16), (bytes(range(100, 116)), 123456789, 1027, 64),
             (bytes(range(16)), (1 << 63) + 5, 4096, 40), (bytes(16), 0, 0, 32)]
    out = {}
    for i, (seed, rnd, count, n) in enumerate(cases):
        out[f"seed{i}"] = np.frombuffer(seed, dtype=np.uint8)
        out[f"meta{i}"] = np.array([rnd, count, n], dtype=np.uint64)
        out[f"out{i}"] = prg.mask_stream(seed, rnd, count, n)
    np.savez_compressed(os.path.join(HERE, "mask_stream.npz"), cases=np.int64(len(cases)), **out)
    print("wrote", len(cases), "mask_stream cases")


if __name__ == "__main__":
    main()
