"""Pin the CPU oracle (oracle/) against the reference: its committed PRG vectors
and golden fixtures produced by running the Python reference (tests/golden/)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_golden


def _vectors():
    with open(os.path.join(GOLDEN, "prg_vectors.json")) as fh:
        return [(bytes.fromhex(s), bytes.fromhex(e)) for s, e in json.load(fh)["vectors"]]


@pytest.mark.parametrize("aesni", [False, True])
def test_prg_vectors(oracle, aesni):
    # pkg/tests/test_prg.py:26-34 -- the 15 pinned vectors, both AES paths.
    oracle.use_aesni(aesni)
    try:
        vecs = _vectors()
        assert len(vecs) == 15
        for seed, want in vecs:
            assert oracle.expand(np.frombuffer(seed, np.uint8), 3).tobytes() == want
        # first row: standard AES-128 KAT (key 00..0f, zero plaintext)
        assert oracle.aes128(0, bytes(16)).hex() == "c6a13b37878f5b826f4f8162a1c8d879"
    finally:
        oracle.use_aesni(True)


def test_prg_expand_golden(oracle):
    g = load_golden("prg")
    assert np.array_equal(oracle.expand(g["seeds"], 3), g["exp3"])
    assert np.array_equal(oracle.expand(g["seeds"], 2), g["exp2"])
    # expand does not clear the top bit of its input (prg.py:43-60)
    assert np.array_equal(oracle.expand(g["raw_seeds"], 3), g["raw_exp3"])


@pytest.mark.parametrize("tag", golden_cases())
def test_keygen_and_eval_golden(oracle, tag):
    g = load_golden(tag)
    n, N, ob = int(g["n"]), int(g["N"]), int(g["out_bits"])
    kind = "eq" if tag.startswith("fss_eq") else "cmp"
    # tape replay: same numpy draws as fss._sample_tape
    rng = np.random.default_rng(int(g["seed"]))
    alpha, a0, s0, s1 = oracle.sample_tape(n, rng, N)
    assert np.array_equal(alpha, g["alpha"]) and np.array_equal(a0, g["alpha0"])
    assert np.array_equal(s0, g["s0"]) and np.array_equal(s1, g["s1"])
    assert np.array_equal(rng.integers(0, 1 << 32, size=4, dtype=np.uint64), g["next_draws"])
    if kind == "eq":
        k0, k1 = oracle.keygen_eq_core(n, alpha, a0, s0, s1)
        assert np.array_equal(k0["cw_final"], g["cw_final"])
        y0, y1 = oracle.eval_eq(0, k0, g["x"]), oracle.eval_eq(1, k1, g["x"])
    else:
        k0, k1 = oracle.keygen_cmp_core(n, alpha, a0, s0, s1, ob)
        assert np.array_equal(k0["sigma_cw"], g["sigma_cw"])
        assert np.array_equal(k0["leaf_cw"], g["leaf_cw"])
        y0, lv0 = oracle.eval_cmp(0, k0, g["x"], return_levels=True)
        y1, lv1 = oracle.eval_cmp(1, k1, g["x"], return_levels=True)
        assert np.array_equal(lv0, g["lv0"]) and np.array_equal(lv1, g["lv1"])
    assert np.array_equal(k0["scw"], g["scw"]) and np.array_equal(k0["tcw"], g["tcw"])
    assert np.array_equal(k1["alpha_share"], g["alpha1"])
    assert np.array_equal(y0, g["y0"]) and np.array_equal(y1, g["y1"])
    mask = np.uint64(oracle.ring_mask(ob))
    want = (g["x"] == g["alpha"]) if kind == "eq" else (g["x"] <= g["alpha"])
    assert np.array_equal((y0 + y1) & mask, want.astype(np.uint64))
    if "arnk" in g:
        blob = g["arnk"].tobytes()
        body = blob[13:]
        half = len(body) // 2
        assert oracle.pack(k0) == body[:half] and oracle.pack(k1) == body[half:]
        r0 = oracle.unpack(kind, 0, n, N, body[:half])
        assert oracle.pack(r0) == body[:half]


@pytest.mark.parametrize("n", [4, 5])
def test_exhaustive_golden(oracle, n):
    g = load_golden(f"exhaustive_n{n}")
    size = 1 << n
    idx = np.repeat(np.arange(size), size)
    xs = np.tile(np.arange(size, dtype=np.uint64), size)
    for kind in ("eq", "cmp"):
        body = g[f"{kind}_arnk"].tobytes()[13:]
        half = len(body) // 2
        k0 = oracle.unpack(kind, 0, n, size, body[:half])
        k1 = oracle.unpack(kind, 1, n, size, body[half:])
        take = lambda k: {key: (v[:, idx] if key in ("scw", "tcw", "sigma_cw", "leaf_cw") else
                                (v[idx] if isinstance(v, np.ndarray) else v)) for key, v in k.items()}
        ev = oracle.eval_eq if kind == "eq" else oracle.eval_cmp
        y0, y1 = ev(0, take(k0), xs), ev(1, take(k1), xs)
        assert np.array_equal(y0, g[f"{kind}_y0"]) and np.array_equal(y1, g[f"{kind}_y1"])
