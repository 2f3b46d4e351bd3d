"""ARNK pack / unpack against the HBM bandwidth of THEIR read:write mix.

MEASURED_PEAKS.json's hbm_gbs is a 1:1 copy; the transposes move 1,088 B read :
824 B written per DCF key (pack) and the reverse (unpack). This script builds
and runs scripts/hbm_mix_probe.cu (streaming kernel, same byte mix, no reuse)
and times the shipped kernels (fss._pack_device / fss._unpack, 2^22 keys, CUDA
events, best of 5 after a warm-up), then reports each kernel as a fraction of
the 1:1 copy roof and of its own mix roof.

  python scripts/arnk_mix_roof.py [--out gpurun_out/arnk_mix_roof.json]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def probe() -> list:
    exe = "/tmp/hbm_mix_probe"
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                           os.path.join(ROOT, "scripts", "hbm_mix_probe.cu")])
    out = subprocess.check_output([exe], text=True)
    return [json.loads(line) for line in out.splitlines() if line.startswith("{")]


def kernels(log2n: int) -> dict:
    import numpy as np
    import torch

    from paper_2006_04593_b200 import _lib, fss
    _lib.load()
    dev = torch.device("cuda", 0)
    N = 1 << log2n
    stream = torch.cuda.current_stream(dev)

    def timed(fn):
        fn()
        best = None
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            t = a.elapsed_time(b) / 1e3
            best = t if best is None else min(best, t)
        return best

    rng = np.random.default_rng(5)
    res = {}
    for kind, keygen, kcode in (("dcf", fss.keygen_cmp, fss.KIND_CMP), ("dpf", fss.keygen_eq, fss.KIND_EQ)):
        _, k0, _ = keygen(32, rng, N, device=dev)
        payload = fss._pack_device(k0).reshape(-1)
        pay_b = payload.numel() // N
        arr_b = sum(getattr(k0, f).numel() * getattr(k0, f).element_size() for f in
                    (("alpha_share", "seed0", "scw", "tcw", "sigma_cw", "leaf_cw") if kind == "dcf"
                     else ("alpha_share", "seed0", "scw", "tcw", "cw_final"))) // N
        tp = timed(lambda: fss._pack_device(k0))
        tu = timed(lambda: fss._unpack(kcode, 0, 32, N, payload, dev))
        res[kind] = {"payload_B_per_key": pay_b, "arrays_B_per_key": arr_b,
                     "pack_ms": tp * 1e3, "pack_GBps": N * (pay_b + arr_b) / tp / 1e9,
                     "unpack_ms": tu * 1e3, "unpack_GBps": N * (pay_b + arr_b) / tu / 1e9}
        del k0, payload
        torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=22)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    mixes = probe()
    best = {}
    for m in mixes:
        if "mix" in m:
            best[m["mix"]] = max(best.get(m["mix"], 0.0), m["GBps"])
    ks = kernels(args.log2n)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    copy_peak = peaks.get("hbm_gbs")
    roof_of = {("dcf", "pack"): "dcf_pack_1088to824", ("dcf", "unpack"): "dcf_unpack_824to1088",
               ("dpf", "pack"): "dpf_pack_576to568", ("dpf", "unpack"): "dpf_unpack_568to576"}
    for (kind, op), mix in roof_of.items():
        gbps = ks[kind][f"{op}_GBps"]
        ks[kind][f"{op}_mix_roof_GBps"] = best.get(mix)
        ks[kind][f"{op}_frac_mix_roof"] = gbps / best[mix] if best.get(mix) else None
        ks[kind][f"{op}_frac_copy_peak"] = gbps / copy_peak if copy_peak else None
    out = {"what": "ARNK kernels vs the streaming bandwidth of their own read:write byte mix "
                   "(scripts/hbm_mix_probe.cu, best over 2 / 4 CTAs per SM)",
           "copy_peak_measured_peaks_json": copy_peak, "mix_probe": mixes, "mix_best_GBps": best,
           "kernels_2p%d" % args.log2n: ks}
    text = json.dumps(out, indent=1)
    print(text)
    if args.out:
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        with open(args.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
