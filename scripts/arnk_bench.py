"""ARNK (de)serialisation kernels on the GPU: the tiled shared-memory transpose
(csrc/arnk_kernels.cu, the shipped path) vs the round-1 naive kernel (built as
a variant with FSSB_ARNK_NAIVE=1), bit-exact against each other, timed with
CUDA events and reported against the HBM roof.

  python scripts/arnk_bench.py build          # here (nvcc, no GPU)
  python scripts/arnk_bench.py run [--log2n 22]

Algorithmic bytes per element and direction (n = 32, reference in-memory
layout): payload 824 (cmp) / 568 (eq) + key arrays alpha 8, seed 16, scw 512,
tcw 32, sigma 256 + leaf 264 (cmp) / cw_final 8 (eq) = 1,912 / 1,144 B.
"""

from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "build", "variants")
ROUNDS = int(os.environ.get("ARNK_ROUNDS", "6"))
# variant name -> compile-time defines (the shipped library is "main")
VARIANTS = {
    "naive": ["FSSB_ARNK_NAIVE=1"],
    # r02 pack study: the LDGSTS-staged kernel (shipped before the TMA tensor-map pack),
    # TMA staging depth / CTA size / L2 promotion of the tensor maps
    "ldgsts": ["FSSB_ARNK_TMA_PACK=0"],
    "cmp_s2": ["FSSB_ARNK_TMA_STAGES_CMP=2"],
    "eq_s3": ["FSSB_ARNK_TMA_STAGES_EQ=3"],
    "tma256": ["FSSB_ARNK_TMA_THREADS=256"],
    "promo0": ["FSSB_ARNK_TMA_L2PROMO=0"],
    # r02 unpack study: CTA size and tile size of the unpack tile kernel
    "un512": ["FSSB_ARNK_UNPACK_THREADS=512"],
    "un_t32": ["FSSB_ARNK_UNPACK_TILE_KB=60"],
    "un512_t32": ["FSSB_ARNK_UNPACK_THREADS=512", "FSSB_ARNK_UNPACK_TILE_KB=60"],
    "un128": ["FSSB_ARNK_UNPACK_THREADS=128"],
    "un_t128": ["FSSB_ARNK_UNPACK_TILE_KB=215"],
    "un_t128_512": ["FSSB_ARNK_UNPACK_TILE_KB=215", "FSSB_ARNK_UNPACK_THREADS=512"],
    "un_t128_1024": ["FSSB_ARNK_UNPACK_TILE_KB=215", "FSSB_ARNK_UNPACK_THREADS=1024"],
    # TMA pack with 32-key tiles (2 or 3 staging buffers)
    "tma32": ["FSSB_ARNK_TMA_LNB=1"],
    "tma32_s2": ["FSSB_ARNK_TMA_LNB=1", "FSSB_ARNK_TMA_STAGES_CMP=2"],
    "tma32_1024": ["FSSB_ARNK_TMA_LNB=1", "FSSB_ARNK_TMA_THREADS=1024"],
    "cmp32_s4": ["FSSB_ARNK_TMA_STAGES_CMP=4"],
    "cmp32_256": ["FSSB_ARNK_TMA_THREADS=256"],
    "eq32_s3": ["FSSB_ARNK_TMA_LNB_EQ=1", "FSSB_ARNK_TMA_STAGES_EQ=3"],
    "eq32_1024": ["FSSB_ARNK_TMA_LNB_EQ=1", "FSSB_ARNK_TMA_THREADS=1024"],
}
if os.environ.get("ARNK_VARIANTS"):
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in os.environ["ARNK_VARIANTS"].split(",")}


def vlib(name):
    return os.path.join(VDIR, f"lib_arnk_{name}.so")


def build():
    from paper_2006_04593_b200 import _build
    os.makedirs(VDIR, exist_ok=True)
    for name, defs in VARIANTS.items():
        print(_build.build(force=True, defines=defs, lib=vlib(name)))


def key_bytes(kind: int, n: int) -> int:
    base = 8 + 16 + 16 * n + n
    return base + (8 * n + 8 * (n + 1) if kind == 1 else 8)


def run(log2n: int):
    import numpy as np
    import torch

    from paper_2006_04593_b200 import _dev, _lib, fss

    dev = torch.device("cuda", 0)
    N = 1 << log2n
    stream = torch.cuda.current_stream(dev)
    libs = {"main": _lib.load()}
    for name in VARIANTS:
        lib = ctypes.CDLL(vlib(name))
        for fn in ("fss_arnk_pack", "fss_arnk_unpack"):
            getattr(lib, fn).argtypes = _lib.SIGNATURES[fn]
        libs[name] = lib
    main = libs["main"]
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except (OSError, ValueError):
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    out = {"N": N, "hbm_peak_gbs": hbm}
    for kind, name in ((1, "cmp"), (0, "eq")):
        rng = np.random.default_rng(3)
        _, k0, _ = (fss.keygen_cmp if kind else fss.keygen_eq)(32, rng, N, device=dev)
        elem = int(main.fss_arnk_elem_bytes(kind, 32))
        algo = elem + key_bytes(kind, 32)
        bufs = {lib: torch.empty(N * elem, dtype=torch.uint8, device=dev) for lib in libs}
        fields = ["alpha_share", "seed0", "scw", "tcw"] + (["sigma_cw", "leaf_cw"] if kind else ["cw_final"])
        outs = {lib: {f: torch.empty_like(getattr(k0, f)) for f in fields} for lib in libs}

        def ptrs(src):
            return [_dev.ptr(src["alpha_share"]), _dev.ptr(src["seed0"]), _dev.ptr(src["scw"]),
                    _dev.ptr(src["tcw"]), _dev.ptr(src.get("cw_final")), _dev.ptr(src.get("sigma_cw")),
                    _dev.ptr(src.get("leaf_cw"))]

        src = {f: getattr(k0, f) for f in fields}
        fns = {}
        for libname, lib in libs.items():
            def pack(lib=lib, libname=libname):
                assert lib.fss_arnk_pack(kind, 32, N, N, *ptrs(src), _dev.ptr(bufs[libname]),
                                         stream.cuda_stream) == 0

            def unpack(lib=lib, libname=libname):
                assert lib.fss_arnk_unpack(kind, 32, N, N, _dev.ptr(bufs[libname]), *ptrs(outs[libname]),
                                           stream.cuda_stream) == 0
            fns[libname] = {"pack": pack, "unpack": unpack}
            pack()
            unpack()
        # round-robin over the libraries (ROUNDS x 5 launches each) so clock /
        # thermal drift hits every variant alike; median over all launches
        times = {ln: {"pack": [], "unpack": []} for ln in libs}
        for _ in range(ROUNDS):
            for libname in libs:
                for op in ("pack", "unpack"):
                    for _ in range(5):
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(stream)
                        fns[libname][op]()
                        b.record(stream)
                        b.synchronize()
                        times[libname][op].append(a.elapsed_time(b) / 1e3)
        for libname in libs:
            row = {}
            for op in ("pack", "unpack"):
                ts = sorted(times[libname][op])
                t = ts[len(ts) // 2]
                row[op] = {"ms": t * 1e3, "keys_per_s": N / t, "gb_per_s": N * algo / t / 1e9,
                           "frac_hbm": N * algo / t / 1e9 / hbm, "launches": len(ts)}
            out[f"{name}_{libname}"] = row
            print(name, libname, "pack %.4f ms frac %.4f | unpack %.4f ms frac %.4f" % (
                row["pack"]["ms"], row["pack"]["frac_hbm"], row["unpack"]["ms"], row["unpack"]["frac_hbm"]),
                flush=True)
        for libname in libs:
            assert torch.equal(bufs["main"], bufs[libname]), ("pack payloads differ", libname)
            for f in fields:
                a, b = outs[libname][f], getattr(k0, f)
                assert torch.equal(a.view(torch.uint8), b.contiguous().view(torch.uint8)), (libname, f)
        out[f"{name}_algorithmic_bytes_per_key"] = algo
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "arnk_bench.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(int(sys.argv[sys.argv.index("--log2n") + 1]) if "--log2n" in sys.argv else 22)
