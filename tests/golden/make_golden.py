"""Generate golden fixtures by running the UNMODIFIED Python reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``ariann`` from /root/reference/pkg/src, runs its own keygen / eval /
serialization entry points on fixed numpy seeds and writes the inputs and
outputs to tests/golden/*.npz + prg_vectors.json. Nothing here is imported at
test time; the GPU box only sees the committed fixtures.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _next_draws(rng):
    # Fingerprint of the generator state after keygen: lets tests check that the
    # drop-in advances the caller's rng exactly like the reference does.
    return rng.integers(0, 1 << 32, size=4, dtype=np.uint64)


def _xs(rng_x, alpha, n, N):
    xs = rng_x.integers(0, 1 << min(n, 63), size=N, dtype=np.uint64)
    if n == 64:
        xs = (xs << np.uint64(1)) | rng_x.integers(0, 2, size=N, dtype=np.uint64)
    hit = rng_x.random(N) < 0.3
    xs[hit] = alpha[hit]
    near = (~hit) & (rng_x.random(N) < 0.3)
    mask = np.uint64((1 << n) - 1) if n < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    xs[near] = (alpha[near] + np.uint64(1)) & mask
    return xs


def main():
    sys.path.insert(0, REF)
    from ariann import fss, prg  # noqa: E402  (the reference)

    vec_path = "/root/reference/pkg/prg_vectors.txt"
    vectors = []
    with open(vec_path) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                s, e = line.split()
                vectors.append([s, e])
    rng = np.random.default_rng(2024)
    seeds = prg.random_seeds(rng, 64)
    raw_seeds = rng.integers(0, 256, size=(64, 16), dtype=np.uint8)  # top bit NOT cleared
    with open(os.path.join(HERE, "prg_vectors.json"), "w") as fh:
        json.dump({"source": "pkg/prg_vectors.txt (reference, 15 rows)", "vectors": vectors}, fh,
                  indent=1)
    np.savez_compressed(os.path.join(HERE, "prg.npz"), seeds=seeds, exp3=prg.expand(seeds, 3),
                        exp2=prg.expand(seeds, 2), raw_seeds=raw_seeds,
                        raw_exp3=prg.expand(raw_seeds, 3))

    cases = []
    for n in (4, 5, 6, 7, 8, 9, 10, 12, 16, 24, 32):
        cases.append(("eq", n, None, 64 if n < 32 else 256))
        cases.append(("cmp", n, None, 64 if n < 32 else 256))
    cases += [("eq", 33, None, 32), ("eq", 64, None, 32), ("cmp", 33, None, 32),
              ("cmp", 63, None, 32), ("cmp", 12, 40, 64), ("cmp", 16, 32, 64)]
    out = {}
    for ci, (kind, n, ob, N) in enumerate(cases):
        seed = 1000 + ci
        rng = np.random.default_rng(seed)
        if kind == "eq":
            alpha, k0, k1, tape = fss.keygen_eq_with_tape(n, rng, N)
        elif ob is None:
            alpha, k0, k1, tape = fss.keygen_cmp_with_tape(n, rng, N)
        else:
            alpha, k0, k1 = fss.keygen_cmp(n, rng, N, out_bits=ob)
        nxt = _next_draws(rng)
        xs = _xs(np.random.default_rng(seed + 7), alpha, n, N)
        tag = f"{kind}_n{n}" + (f"_ob{ob}" if ob else "")
        d = dict(seed=np.int64(seed), n=np.int64(n), N=np.int64(N),
                 out_bits=np.int64(ob if ob else n), alpha=alpha, alpha0=k0.alpha_share,
                 alpha1=k1.alpha_share, s0=k0.seed0, s1=k1.seed0, next_draws=nxt, x=xs,
                 scw=k0.scw, tcw=k0.tcw)
        if kind == "eq":
            d["cw_final"] = k0.cw_final
            d["y0"] = fss.eval_eq(0, k0, xs)
            d["y1"] = fss.eval_eq(1, k1, xs)
        else:
            d["sigma_cw"] = k0.sigma_cw
            d["leaf_cw"] = k0.leaf_cw
            d["y0"], d["lv0"] = fss.eval_cmp(0, k0, xs, return_levels=True)
            d["y1"], d["lv1"] = fss.eval_cmp(1, k1, xs, return_levels=True)
        if ob is None:
            blob = fss.serialize_keys(fss.pack_keys(k0, k1))
            d["arnk"] = np.frombuffer(blob, dtype=np.uint8)
        out[tag] = d
    for tag, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"fss_{tag}.npz"), **d)

    # Exhaustive n=4,5 with alpha = arange (test_fss.py:36-50 shape).
    for n in (4, 5):
        rng = np.random.default_rng(n)
        size = 1 << n
        alphas = np.arange(size, dtype=np.uint64)
        _, e0, e1 = fss.keygen_eq(n, rng, count=size, alpha=alphas)
        _, c0, c1 = fss.keygen_cmp(n, rng, count=size, alpha=alphas)
        idx = np.repeat(np.arange(size), size)
        xs = np.tile(np.arange(size, dtype=np.uint64), size)
        np.savez_compressed(
            os.path.join(HERE, f"exhaustive_n{n}.npz"),
            eq_arnk=np.frombuffer(fss.serialize_keys(fss.pack_keys(e0, e1)), dtype=np.uint8),
            cmp_arnk=np.frombuffer(fss.serialize_keys(fss.pack_keys(c0, c1)), dtype=np.uint8),
            eq_y0=fss.eval_eq(0, e0.take(idx), xs), eq_y1=fss.eval_eq(1, e1.take(idx), xs),
            cmp_y0=fss.eval_cmp(0, c0.take(idx), xs), cmp_y1=fss.eval_cmp(1, c1.take(idx), xs),
            next_draws=_next_draws(rng))
    print("wrote", len(out) + 3, "fixtures to", HERE)


if __name__ == "__main__":
    main()
