"""CPU check of the bitsliced AES circuit (scripts/research/bitsliced/aes_bitsliced.cuh, the measured
alternative to the T-table AES): the same header is compiled for the host with
g++ and must reproduce the reference's PRG vectors and the oracle's expand
bit-exactly."""

import json
import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

CSRC = os.path.join(ROOT, "paper_2006_04593_b200", "csrc")          # aes_consts.h
BSDIR = os.path.join(ROOT, "scripts", "research", "bitsliced")     # aes_bitsliced.cuh


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    out = str(tmp_path_factory.mktemp("bs") / "bitsliced_host")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", BSDIR, "-I", CSRC,
                    os.path.join(ROOT, "tests", "native", "bitsliced_host.cpp"), "-o", out],
                   check=True)
    return out


def _run(exe, seeds):
    r = subprocess.run([exe], input=seeds.tobytes(), capture_output=True, check=True)
    return np.frombuffer(r.stdout, dtype=np.uint8).reshape(-1, 48)


def test_bitsliced_prg_vectors(exe):
    with open(os.path.join(GOLDEN, "prg_vectors.json")) as fh:
        vecs = json.load(fh)["vectors"]
    seeds = np.zeros((32, 16), dtype=np.uint8)
    for i, (s, _) in enumerate(vecs):
        seeds[i] = np.frombuffer(bytes.fromhex(s), dtype=np.uint8)
    out = _run(exe, seeds)
    for i, (_, e) in enumerate(vecs):
        assert out[i].tobytes().hex() == e


def test_bitsliced_matches_oracle(exe, oracle):
    seeds = np.random.default_rng(3).integers(0, 256, (32 * 64, 16), dtype=np.uint8)
    assert np.array_equal(_run(exe, seeds), oracle.expand(seeds, 3))
