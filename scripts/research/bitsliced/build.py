"""Build the bitsliced-AES research library (not part of the product ABI):
scripts/_variants/libfss_bitsliced.so exporting fss_aes_mmo_expand_bitsliced.

  python scripts/research/bitsliced/build.py
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(HERE)))
CSRC = os.path.join(ROOT, "paper_2006_04593_b200", "csrc")     # aes_consts.h
OUT = os.path.join(ROOT, "scripts", "_variants", "libfss_bitsliced.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "bitsliced_kernels.cu")
    deps = [src, os.path.join(HERE, "aes_bitsliced.cuh"), os.path.join(CSRC, "aes_consts.h")]
    if not force and os.path.exists(OUT) and all(os.path.getmtime(d) <= os.path.getmtime(OUT) for d in deps):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
                    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-I", HERE, "-I", CSRC,
                    src, "-o", OUT], check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
