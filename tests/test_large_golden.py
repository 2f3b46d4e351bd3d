"""Parity at the BASELINE sizes against digests of the UNMODIFIED reference
(tests/golden/large_digests.json, made by tests/golden/make_large_golden.py):
DCF n=32 at N = 1, 7, 2^16 (config 1) and DPF n=32 at N = 1, 7, 2^20
(config 2). Every key byte of both parties (sha256 of the ARNK container),
alpha, both parties' eval shares and the generator state after keygen must
match. CPU: the C oracle; GPU: the B200 path through the drop-in API."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "large_digests.json")) as _fh:
    CASES = json.load(_fh)["cases"]


def sha(a) -> str:
    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).astype("<u8").tobytes()).hexdigest()


def xs_for(seed, alpha, n):
    r = np.random.default_rng(seed)
    x = r.integers(0, 1 << n, size=alpha.shape[0], dtype=np.uint64)
    hit = r.random(alpha.shape[0]) < 0.3
    x[hit] = alpha[hit]
    return x


def _header(kind, n, N):
    return b"ARNK" + bytes([1, 0 if kind == "eq" else 1, n]) + (127).to_bytes(2, "little") \
        + N.to_bytes(4, "little")


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_digests(oracle, name):
    c = CASES[name]
    kind, n, N = c["kind"], c["n"], c["N"]
    rng = np.random.default_rng(c["seed"])
    keygen = oracle.keygen_cmp if kind == "cmp" else oracle.keygen_eq
    alpha, k0, k1 = keygen(n, rng, N)
    assert rng.integers(0, 1 << 32, size=4, dtype=np.uint64).tolist() == c["next_draws"]
    assert sha(alpha) == c["alpha_sha256"]
    blob = _header(kind, n, N) + oracle.pack(k0) + oracle.pack(k1)
    assert len(blob) == c["arnk_bytes"] and sha(blob) == c["arnk_sha256"]
    x = xs_for(c["x_seed"], alpha, n)
    ev = oracle.eval_cmp if kind == "cmp" else oracle.eval_eq
    assert sha(ev(0, k0, x)) == c["y0_sha256"] and sha(ev(1, k1, x)) == c["y1_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_b200_matches_reference_digests(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2006_04593_b200 import fss
    c = CASES[name]
    kind, n, N = c["kind"], c["n"], c["N"]
    rng = np.random.default_rng(c["seed"])
    keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    alpha, k0, k1 = keygen(n, rng, N, device=torch.device("cuda", 0))
    assert rng.integers(0, 1 << 32, size=4, dtype=np.uint64).tolist() == c["next_draws"]
    a = alpha.cpu().numpy()
    assert sha(a) == c["alpha_sha256"]
    blob = fss.serialize_keys(fss.pack_keys(k0, k1))
    assert len(blob) == c["arnk_bytes"] and sha(blob) == c["arnk_sha256"]
    x = xs_for(c["x_seed"], a, n)
    ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
    assert sha(ev(0, k0, x)) == c["y0_sha256"] and sha(ev(1, k1, x)) == c["y1_sha256"]
