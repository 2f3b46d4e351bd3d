"""Dealer -> party key shipping through ARNK files: the streaming path
(keyfile.save_keys / load_keys: pinned double buffers, device pack/unpack)
vs the reference's bytes path (serialize_keys(pack_keys(...)) + write;
read + deserialize_keys + unpack_keys, cli.py:195-214 / 150-160), on
2^log2n DCF keys (n = 32). Files go to /dev/shm when present so the number
is the pipeline's, not the disk's. Wall-clock, best of 3.

  python scripts/keyfile_bench.py [--log2n 21]
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(log2n: int):
    import numpy as np
    import torch

    from paper_2006_04593_b200 import fss, keyfile

    dev = torch.device("cuda", 0)
    N = 1 << log2n
    _, k0, k1 = fss.keygen_cmp(32, np.random.default_rng(5), N, device=dev)
    d = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
    path = os.path.join(d, "fss_keyfile_bench.arnk")
    size = fss._HEADER_BYTES + 2 * N * fss.cmp_elem_bytes(32)

    def best(fn):
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    def save_bytes():
        with open(path, "wb") as fh:
            fh.write(fss.serialize_keys(fss.pack_keys(k0, k1)))

    def load_bytes(party=None):
        with open(path, "rb") as fh:
            pair = fss.unpack_keys(fss.deserialize_keys(fh.read()), device=dev)
        return pair if party is None else pair[party]

    out = {"keys": N, "file_bytes": size, "dir": d}
    try:
        out["stream_save_s"] = best(lambda: keyfile.save_keys(path, k0, k1))
        out["stream_load_both_s"] = best(lambda: keyfile.load_keys(path, device=dev))
        out["stream_load_party_s"] = best(lambda: keyfile.load_keys(path, party=1, device=dev))
        r1 = keyfile.load_keys(path, party=1, device=dev)
        assert torch.equal(r1.scw, k1.scw)
        out["bytes_save_s"] = best(save_bytes)
        out["bytes_load_both_s"] = best(load_bytes)
        out["bytes_load_party_s"] = best(lambda: load_bytes(1))
    finally:
        if os.path.exists(path):
            os.remove(path)
    for key in [k for k in out if k.endswith("_s")]:
        out[key[:-2] + "_gb_per_s"] = (size if "both" in key or "save" in key else size / 2) / out[key] / 1e9
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "keyfile_bench.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[sys.argv.index("--log2n") + 1]) if "--log2n" in sys.argv else 21)
