"""All five BASELINE.json configs on one B200, beyond bench.py's headline line.

  python scripts/bench_configs.py [--sweep-max 28] [--out gpurun_out/configs.json]

1. DCF keygen + eval, 2^16 int32, two parties in-process (+ the online sign protocol)
2. DPF keygen + eval, 2^20 (+ the online equality protocol)
3. Private ReLU on 1x64x112x112 shares: dealer (keys + triple) and online (2 rounds),
   output shares checked against the reference's digest (tests/golden/protocols.json)
4. Private 2x2 MaxPool on 16x64x56x56: k2 route (digest-checked) and the argmax
   route (9.6 M DCF + 3.2 M DPF), all 1,024 planes batched in one call
5. Sweep 2^16 .. 2^28 of DCF / DPF keygen and eval, timed separately; above
   2^26 keys are generated and evaluated in 2^26 chunks (both parties' keys for
   2^28 DCF elements take ~300 GB in the reference layout)

Device times are CUDA events on the launching stream (median of 5 after 2
warm-ups for the sweep); protocol times are host wall-clock around a
synchronised run (they include the party threads and the exchanges): median
of 10 (config 1), 9 (config 3) and 5 (config 4) runs after warm-up.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2006_04593_b200 import dealer, fss, nn_ops, runtime  # noqa: E402
from paper_2006_04593_b200.sharing import AdditiveShare, encode_fixed, share  # noqa: E402

DEV = torch.device("cuda", 0)


def digest(*ts):
    h = hashlib.sha256()
    for t in ts:
        h.update(np.ascontiguousarray(t.detach().cpu().numpy().astype("<u8")).tobytes())
    return h.hexdigest()


def wall(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def ev_time(fn, reps=5, warm=2):
    s = torch.cuda.current_stream(DEV)
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    return sorted(ts)[len(ts) // 2]


def golden(name):
    with open(os.path.join(ROOT, "tests", "golden", "protocols.json")) as fh:
        return json.load(fh)["cases"][name]


def config12(kind, N):
    rng = np.random.default_rng(1)
    keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
    t_kg = ev_time(lambda: keygen(32, rng, N, device=DEV))
    alpha, k0, k1 = keygen(32, rng, N, device=DEV)
    x = alpha.clone()
    t_ev = ev_time(lambda: (ev(0, k0, x), ev(1, k1, x)))
    # online protocol through the two-party runtime (keys from the dealer)
    prng = np.random.default_rng(2)
    if kind == "cmp":
        xs = share(encode_fixed(prng.uniform(-100, 100, N), 3, 32), prng, precision=3)
    else:
        from paper_2006_04593_b200.ring import RingTensor
        xs = share(RingTensor.from_ints(prng.integers(-3, 4, N), 32), prng, precision=0)
    d = dealer.make_dealer(32, seed=3)

    def prog(session):
        view = d.for_party(session.party)
        if kind == "cmp":
            keys = view.cmp_keys(N)
            return fss.sign_protocol(session, AdditiveShare(session.party, xs[session.party].values, 0),
                                     keys)
        return fss.eq_protocol(session, xs[session.party], view.eq_keys(N))
    # dealer + online, median of 10 after 3 warm-ups (the first runs also fill
    # the caching allocator and the party streams)
    runs = []
    for rep in range(13):
        d = dealer.make_dealer(32, seed=3)
        ((_, l0), _), t_run = wall(lambda: runtime.run_local_pair(prog))
        if rep >= 3:
            runs.append(t_run)
    t_total = sorted(runs)[len(runs) // 2]
    return {"N": N, "keygen_pairs_per_s": N / t_kg, "keygen_ms": t_kg * 1e3,
            "eval_both_parties_ms": t_ev * 1e3, "comparisons_per_s" if kind == "cmp" else
            "equality_tests_per_s": N / t_ev,
            "protocol_with_dealer_ms": t_total * 1e3, "rounds": l0.total_rounds()}


def config3():
    c = golden("config3_relu_1x64x112x112")
    shape = tuple(c["shape"])
    rng = np.random.default_rng(c["seed"])
    xs = share(encode_fixed(rng.uniform(c["lo"], c["hi"], shape), 3, 32), rng, precision=3)
    deal_ms, on_ms = [], []
    for rep in range(10):                   # rep 0 warms up; median of reps 1-9
        d = dealer.make_dealer(32, seed=c["dealer_seed"])
        preps = [None, None]

        def deal():
            # both parties' material, in the reference's request order
            preps[0] = d.for_party(0).relu_shaped(shape)
            preps[1] = d.for_party(1).relu_shaped(shape)
        _, t_deal = wall(deal)
        ((r0, l0), (r1, _)), t_on = wall(lambda: runtime.run_local_pair(
            lambda s: nn_ops.relu(s, xs[s.party], preps[s.party])))
        if rep:
            deal_ms.append(t_deal * 1e3)
            on_ms.append(t_on * 1e3)
    return {"dealer_ms": sorted(deal_ms)[len(deal_ms) // 2], "online_ms": sorted(on_ms)[len(on_ms) // 2],
            "online_ms_runs": on_ms,
            "rounds": l0.total_rounds(), "bytes_sent": l0.total_bytes_sent(),
            "bit_exact_vs_reference": digest(r0.values.data, r1.values.data) == c["out_digest"],
            "reference_cpu_total_s": 43.9,
            "reference_cpu_note": "tests/golden/make_protocol_golden.py run of the Python reference "
                                  "(dealer + online, 1 process) in the build container"}


def config4():
    out = {}
    c = golden("config4_maxpoolk2_16x64x56x56")
    shape = tuple(c["shape"])
    planes = shape[0] * shape[1]
    rng = np.random.default_rng(c["seed"])
    xs = share(encode_fixed(rng.uniform(c["lo"], c["hi"], shape), 3, 32), rng, precision=3)
    xp = [x.reshape(planes, 56, 56) for x in xs]
    for route in ("k2", "argmax"):
        deal_ms, on_ms = [], []
        for rep in range(6):                # rep 0 warms up; median of reps 1-5
            preps = None
            torch.cuda.synchronize()
            d = dealer.make_dealer(32, seed=c["dealer_seed"])
            preps = [None, None]

            def deal():
                for p in (0, 1):
                    v = d.for_party(p)
                    preps[p] = v.maxpool_k2(56, planes=planes) if route == "k2" else \
                        v.maxpool(56, 2, 2, planes=planes)
            _, t_deal = wall(deal)

            def prog(s):
                if route == "k2":
                    return nn_ops.maxpool_k2(s, xp[s.party], preps[s.party])
                return nn_ops.maxpool(s, xp[s.party], 2, preps[s.party], 2)
            ((r0, l0), (r1, _)), t_on = wall(lambda: runtime.run_local_pair(prog))
            if rep:
                deal_ms.append(t_deal * 1e3)
                on_ms.append(t_on * 1e3)
        o = {"dealer_ms": sorted(deal_ms)[len(deal_ms) // 2], "online_ms": sorted(on_ms)[len(on_ms) // 2],
             "online_ms_runs": on_ms,
             "rounds": l0.total_rounds(),
             "bytes_sent": l0.total_bytes_sent(),
             "dcf": planes * 784 * (3 if route == "k2" else 12),
             "dpf": 0 if route == "k2" else planes * 784 * 4}
        if route == "k2":
            o["bit_exact_vs_reference"] = digest(r0.values.data, r1.values.data) == c["out_digest"]
            o["reference_cpu_total_s"] = 126.2
        else:
            ca = golden("config4_maxpool_argmax_16x64x56x56")
            o["bit_exact_vs_reference"] = digest(r0.values.data, r1.values.data) == ca["out_digest"]
            o["reference_cpu_total_s"] = 472.0
            o["reference_cpu_note"] = ("tests/golden/make_protocol_golden.py --only "
                                       "config4_maxpool_argmax_16x64x56x56 (1 process, build container)")
        out[route] = o
        del preps
        torch.cuda.empty_cache()
    return out


def sweep(lo, hi):
    rows = []
    chunk_max = 1 << 26
    for log2n in range(lo, hi + 1, 2):
        N = 1 << log2n
        for kind in ("cmp", "eq"):
            keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
            ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
            chunk = min(N, chunk_max)
            rng = np.random.default_rng(log2n)
            t_kg = ev_time(lambda: keygen(32, rng, chunk, device=DEV))   # median of 5 after 2 warm-ups
            alpha, k0, k1 = keygen(32, rng, chunk, device=DEV)
            x = alpha.clone()
            t_e0 = ev_time(lambda: ev(0, k0, x))
            t_e1 = ev_time(lambda: ev(1, k1, x))
            rec = (ev(0, k0, x).view(torch.int64) + ev(1, k1, x).view(torch.int64)) & 0xFFFFFFFF
            assert bool((rec == 1).all())
            del alpha, k0, k1, x, rec
            torch.cuda.empty_cache()
            chunks = N // chunk
            rows.append({"kind": "DCF" if kind == "cmp" else "DPF", "log2n": log2n, "chunks": chunks,
                         "keygen_ms": t_kg * chunks * 1e3, "keygen_pairs_per_s": N / (t_kg * chunks),
                         "eval_ms_per_party": (t_e0 + t_e1) / 2 * chunks * 1e3,
                         "party_evals_per_s": 2 * N / ((t_e0 + t_e1) * chunks),
                         "note": "timed per 2^26 chunk x chunks" if chunks > 1 else ""})
            print(json.dumps(rows[-1]), flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep-max", type=int, default=28)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    ap.add_argument("--only", default="1,2,3,4,5")
    a = ap.parse_args()
    torch.cuda.set_device(DEV)
    only = set(a.only.split(","))
    out = {"gpu": torch.cuda.get_device_name(DEV)}
    if "1" in only:
        out["config1_dcf_2^16"] = config12("cmp", 1 << 16)
        print(json.dumps(out["config1_dcf_2^16"]), flush=True)
    if "2" in only:
        out["config2_dpf_2^20"] = config12("eq", 1 << 20)
        print(json.dumps(out["config2_dpf_2^20"]), flush=True)
    if "3" in only:
        out["config3_relu_1x64x112x112"] = config3()
        print(json.dumps(out["config3_relu_1x64x112x112"]), flush=True)
    if "4" in only:
        out["config4_maxpool_16x64x56x56"] = config4()
        print(json.dumps(out["config4_maxpool_16x64x56x56"]), flush=True)
    if "5" in only:
        out["config5_sweep"] = sweep(16, a.sweep_max)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
