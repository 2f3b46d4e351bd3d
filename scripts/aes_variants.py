"""AES-kernel design experiments: build libariann_fss variants with different
compile-time choices (CPU side) and time their DCF/DPF eval on the GPU on the
same HBM-resident keys (made by the main library), checking bit-exactness.

  python scripts/aes_variants.py build            # here (nvcc, no GPU)
  python scripts/aes_variants.py run [--log2n 22] # on the box (gpurun)
"""

from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "build", "variants")

VARIANTS = {
    "default": [],
}
# round-1 sweep g (profiles/r01_aes_variants_g_unroll.json): unrolling the DCF
# level loop x2 = +0.1 % (noise), x4 = -3.3 % (register pressure): off.
# round-1 sweep b (profiles/r01_aes_variants_b.json): 512/640/768/1024 threads
# x prefetch; more resident warps win (1024: DCF 92.9 %, DPF 85.5 % of the
# lookup roof vs 88.2 % / 72.8 % at 512).
# round-1 result (profiles/r01_aes_variants.json): moving the byte-0/3 address
# arithmetic to IMAD (FSSB_IMAD_ADDR=1) was 10-12 % SLOWER than one PRMT.


def build():
    from paper_2006_04593_b200 import _build
    os.makedirs(VDIR, exist_ok=True)
    for name, defs in VARIANTS.items():
        print(name, _build.build(force=True, defines=defs, lib=os.path.join(VDIR, f"lib_{name}.so")))


def run(log2n: int):
    import numpy as np
    import torch

    from paper_2006_04593_b200 import _dev, _lib, fss

    dev = torch.device("cuda", 0)
    N = 1 << log2n
    rng = np.random.default_rng(5)
    alpha, k0, k1 = fss.keygen_cmp(32, rng, N, device=dev)
    x = torch.from_numpy(np.random.default_rng(6).integers(0, 1 << 32, N, dtype=np.uint64)).to(dev)
    ref0 = fss.eval_cmp(0, k0, x)
    ea, e0, e1 = fss.keygen_eq(32, rng, N, device=dev)
    xe = ea.clone()
    ref_e = fss.eval_eq(0, e0, xe)
    stream = torch.cuda.current_stream(dev)
    peaks = _lib.probe_peaks()
    out = {"N": N, "peaks": peaks}
    for name in VARIANTS:
        lib = ctypes.CDLL(os.path.join(VDIR, f"lib_{name}.so"))
        for fn, argt in (("fss_dcf_eval", _lib.SIGNATURES["fss_dcf_eval"]),
                         ("fss_dpf_eval", _lib.SIGNATURES["fss_dpf_eval"])):
            getattr(lib, fn).argtypes = argt
        res = torch.empty(N, dtype=torch.uint64, device=dev)

        def dcf():
            rc = lib.fss_dcf_eval(0, 32, 32, N, N, _dev.ptr(k0.seed0), _dev.ptr(k0.scw),
                                  _dev.ptr(k0.tcw), _dev.ptr(k0.sigma_cw), _dev.ptr(k0.leaf_cw),
                                  _dev.ptr(x), _dev.ptr(res), None, stream.cuda_stream)
            assert rc == 0

        def dpf():
            rc = lib.fss_dpf_eval(0, 32, N, N, _dev.ptr(e0.seed0), _dev.ptr(e0.scw), _dev.ptr(e0.tcw),
                                  _dev.ptr(e0.cw_final), _dev.ptr(xe), _dev.ptr(res),
                                  stream.cuda_stream)
            assert rc == 0

        row = {}
        # lookups per party-eval: DCF 32 x (160 + 149: sigma block at out_bits <= 32), DPF 32 x 160
        for kname, fn, ref, aes, lk in (("dcf_eval", dcf, ref0, 64, 9888),
                                        ("dpf_eval", dpf, ref_e, 32, 5120)):
            fn()
            torch.cuda.synchronize()
            assert torch.equal(res.view(torch.int64), ref.view(torch.int64)), (name, kname)
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b) / 1e3)
            t = sorted(ts)[len(ts) // 2]
            row[kname] = {"ms": t * 1e3, "party_evals_per_s": N / t, "aes_per_s": N * aes / t,
                          "frac_lds_roof": N * lk / t / (peaks["lds_wavefronts_per_s"] * 32)}
        out[name] = row
        print(name, json.dumps(row), flush=True)
    # T-table vs bitsliced AES on the PRG expand (2^24 seeds, 3 blocks each)
    M = 1 << 24
    seeds = torch.randint(0, 256, (M, 16), dtype=torch.uint8, device=dev)
    res = torch.empty((M, 48), dtype=torch.uint8, device=dev)
    ref = torch.empty_like(res)
    main = _lib.load()
    sys.path.insert(0, os.path.join(ROOT, "scripts", "research", "bitsliced"))
    import build as bs_build                      # research record, not in the product ABI
    bs = ctypes.CDLL(bs_build.build())
    bs.fss_aes_mmo_expand_bitsliced.argtypes = _lib.SIGNATURES["fss_aes_mmo_expand"]
    for name, fn in (("expand_ttable", main.fss_aes_mmo_expand),
                     ("expand_bitsliced", bs.fss_aes_mmo_expand_bitsliced)):
        def go(fn=fn, o=(ref if name == "expand_ttable" else res)):
            assert fn(_dev.ptr(seeds), M, 3, _dev.ptr(o), stream.cuda_stream) == 0
        go()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            go()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        t = sorted(ts)[2]
        out[name] = {"ms": t * 1e3, "aes_per_s": 3 * M / t}
        print(name, json.dumps(out[name]), flush=True)
    assert torch.equal(res, ref)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "aes_variants.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(peaks))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        n = int(sys.argv[sys.argv.index("--log2n") + 1]) if "--log2n" in sys.argv else 22
        run(n)
        if "--small" in sys.argv:
            run(16)
