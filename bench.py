#!/usr/bin/env python
"""Benchmark of the FSS hot path on B200 (contract: see DESIGN.md "Measurement").

Metric (BASELINE.json): FSS comparisons/sec, DCF eval, n = 32. One comparison =
the evaluation of one element's DCF key by BOTH parties (two party-evals).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Default workload (`config.workload`): 2^24 DCF keys per GPU (n = out_bits = 32),
keys resident in HBM in the reference's SoA layout (≈18 GB per GPU, far larger
than the 126 MB L2, so no L2 flush is needed between steps). A step = eval_cmp
for party 0 and party 1 over every element (two kernel launches).

`e2e` = the same metric through the public drop-in API with host buffers: per
step eval_cmp for both parties on a pinned host x (keys dealt beforehand and
resident in HBM, as in `value`), the shares returned in pinned host memory.
The host path is zero-copy: the eval kernel reads x from and stores the shares
to the pinned host buffers itself (UVA, over PCIe), so the 2 x 8 B per element
cross the bus inside the timed kernel.
`e2e.with_keygen` additionally runs keygen_cmp(32, rng, N) from the host numpy
Generator (tape drawn on device from its PCG64 state) inside every step.

`--impl reference` times the CPU restatement of the reference's algorithm
(oracle/, C + AES-NI + OpenMP on all host cores; the Python reference itself
cannot travel to the GPU box) on a bounded sample of the same workload.
Multi-GPU (torchrun): the N * 2^log2n keys are ONE global batch dealt by the
sharded dealer (shard.keygen_cmp_shard: rank r draws only slice r of the shared
PCG64 tape, bit-identical to a single-device keygen); every rank holds both
parties' keys for its slice (weak scaling, no data-path collective in the timed
step); time = max over ranks. Secondary (N >= 2): the output gather of both
parties' shares to rank 0 (shard.gather_ring over NCCL) and the two-GPU sign
protocol over NCCL and over peer memory.

`--global-log2n G` (north-star shape): ONE batch of 2^G keys (G = 28: the
target's 2^28-element batch) split over the N ranks -- strong scaling. A rank's
slice above 2^chunk-log2n keys (default 2^26, ~75 GB of keys) is streamed in
chunks: per chunk keygen (timed separately) then both parties' eval (timed);
`value` = 2^G x steps / (max over ranks of the summed eval time).

`--gpus N` must equal the launcher's WORLD_SIZE. Without a launcher and N > 1,
bench.py re-launches itself under torch.distributed.run with N ranks (one per
GPU); with fewer visible GPUs than N it exits non-zero. It never prints a line
for a different N than asked.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_BITS = 32
BYTES_PER_EVAL = 16 + 32 * 16 + 32 + 32 * 8 + 33 * 8 + 8 + 8   # 1096 B
AES_PER_EVAL = 64                                              # 32 levels x 2 blocks
LDS_PER_AES = 160                                              # T-table lookups per block
# Lookups the T-table DCF evaluation needs per party-eval at out_bits <= 32 (the
# bench's ring): per level one full block (160) + the sigma block's rounds 1-9
# (144) + its last-round bytes that the output reads (4 for sigma mod 2^32, 1
# for the tau bit) = 309.
LOOKUPS_PER_EVAL = 32 * (160 + 149)                            # 9,888
# one conflict-free LDS.32 wavefront serves 32 lanes' lookups
LOP3_PER_AES_BITSLICED = 356.25                                # SURVEY.md §8d bitsliced floor


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--log2n", type=int, default=24, help="DCF keys per GPU = 2^log2n (weak scaling)")
    p.add_argument("--global-log2n", type=int, default=None,
                   help="strong scaling: one batch of 2^G keys split over the ranks")
    p.add_argument("--chunk-log2n", type=int, default=26,
                   help="strong scaling: largest resident key chunk per rank (2^k keys)")
    p.add_argument("--cpu-log2n", type=int, default=None,
                   help="CPU sample (reference arm / cpu_baseline); default: the GPU arm's per-GPU "
                        "batch when host memory allows")
    p.add_argument("--cpu-single-log2n", type=int, default=16,
                   help="single-thread CPU sample (SURVEY 8d item (i))")
    p.add_argument("--no-numa", action="store_true", help="do not bind host buffers to the GPU's node")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-secondary", action="store_true")
    return p.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------- workload

METRIC = "FSS comparisons/sec (DCF eval, n=32)"
L2_NOTE = ("inputs larger than L2: every step reads each key's 1,064 B of correction words once "
           "(>= 2^16 keys = 70 MB per launch at the smallest sample, 18 GB at the default 2^24); "
           "no L2 flush between steps")


def workload_config(args, ws: int) -> dict:
    """The `config` of BOTH arms (identical dicts: the driver compares them)."""
    if args.global_log2n is not None:
        return {"workload": f"DCF eval n=32 out_bits=32, one batch of 2^{args.global_log2n} keys over "
                            f"{ws} GPU(s), both parties per step",
                "global_batch": 1 << args.global_log2n, "parallelism": f"dp{ws} (element shards)",
                "l2": L2_NOTE}
    return {"workload": f"DCF eval n=32 out_bits=32, 2^{args.log2n} keys per GPU, both parties per step",
            "global_batch": ws << args.log2n, "parallelism": f"dp{ws} (element shards)",
            "l2": L2_NOTE}


def cpu_sample_log2n(args) -> int:
    """CPU sample: the GPU arm's per-GPU batch when the host has room for the
    oracle's keys (1,112 B per key plus the tape and x), else the largest power
    of two that fits in a quarter of the available memory."""
    want = args.global_log2n if args.global_log2n is not None else args.log2n
    if args.cpu_log2n is not None:
        return args.cpu_log2n
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = 0
    per_key = 1112 + 48 + 3 * 8
    k = want
    while k > 16 and (per_key << k) > avail // 4:
        k -= 1
    return k


def _oracle_eval_rate(log2n: int, threads: int, min_s: float, max_reps: int, seed: int = 1):
    """(comparisons/s, reps, threads) of the oracle's eval_cmp for both parties
    on 2^log2n keys (keygen untimed), checked against the predicate."""
    import numpy as np

    import oracle
    oracle.build()
    oracle.set_threads(threads)
    N = 1 << log2n
    alpha, k0, k1 = oracle.keygen_cmp(N_BITS, np.random.default_rng(seed), N)
    x = (alpha + np.random.default_rng(seed + 1).integers(0, 2000, N, dtype=np.uint64)
         - np.uint64(1000)) & np.uint64(0xFFFFFFFF)
    reps, t_total, y0, y1 = 0, 0.0, None, None
    while reps < 1 or (t_total < min_s and reps < max_reps):
        t0 = time.perf_counter()
        y0 = oracle.eval_cmp(0, k0, x)
        y1 = oracle.eval_cmp(1, k1, x)
        t_total += time.perf_counter() - t0
        reps += 1
    assert np.array_equal((y0 + y1) & np.uint64(0xFFFFFFFF), (x <= alpha).astype(np.uint64))
    return N * reps / t_total, reps, oracle.threads()


def single_thread_baseline(args) -> dict:
    """the CPU port on ONE host thread."""
    import oracle
    v, reps, _ = _oracle_eval_rate(args.cpu_single_log2n, 1, 3.0, 50)
    return {"value": v, "unit": "comparisons/s", "cores": 1, "kind": "port",
            "sample": f"{reps} x 2^{args.cpu_single_log2n} DCF keys (n=32), eval_cmp party 0 + party 1, "
                      f"oracle/fss_oracle.c on 1 thread (AES-NI={oracle.aesni()})"}


def run_reference(args, ws, rank):
    """CPU arm: the oracle restatement of the reference algorithm on host cores,
    on the GPU arm's per-GPU workload (each step = both parties' eval of every
    key of the sample)."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    oracle.build()
    # all the host threads this process may use: torchrun exports
    # OMP_NUM_THREADS=1 to every rank, but only rank 0 runs this arm
    oracle.set_threads(len(os.sched_getaffinity(0)))
    log2n = cpu_sample_log2n(args)
    N = 1 << log2n
    rng = np.random.default_rng(1)
    alpha, k0, k1 = oracle.keygen_cmp(N_BITS, rng, N)
    x = (alpha + np.random.default_rng(2).integers(0, 2000, N, dtype=np.uint64)
         - np.uint64(1000)) & np.uint64(0xFFFFFFFF)
    for _ in range(args.warmup):
        oracle.eval_cmp(0, k0, x)
        oracle.eval_cmp(1, k1, x)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        y0 = oracle.eval_cmp(0, k0, x)
        y1 = oracle.eval_cmp(1, k1, x)
        times.append(time.perf_counter() - t0)
    rec = (y0 + y1) & np.uint64(0xFFFFFFFF)
    assert np.array_equal(rec, (x <= alpha).astype(np.uint64))
    del alpha, k0, k1, x, y0, y1, rec
    t = sum(times) / len(times)
    v = N / t
    cores = oracle.threads()
    cfg = workload_config(args, ws)
    per_gpu = cfg["global_batch"] // ws
    same = (N == per_gpu and ws == 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": v,
        "unit": "comparisons/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.global_log2n is not None else "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": cfg,
        "sample_matches_config": same,
        "cpu_baseline": {"value": v, "unit": "comparisons/s", "cores": cores, "kind": "port",
                         "sample": f"2^{log2n} DCF keys (n=32) per step, eval_cmp party 0 + party 1, "
                                   f"oracle/fss_oracle.c (AES-NI={oracle.aesni()}, OpenMP)"
                                   + ("" if same else f"; the config's batch is {cfg['global_batch']} keys "
                                      "-- per-key cost is size-independent beyond L3")},
        "single_thread": single_thread_baseline(args),
        "e2e": {"value": v, "unit": "comparisons/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- ours

def cpu_baseline_line(args):
    import oracle
    log2n = min(cpu_sample_log2n(args), 22)      # bounded: ~10-30 s of CPU work
    v, reps, cores = _oracle_eval_rate(log2n, len(os.sched_getaffinity(0)), 10.0, 100)
    return {"value": v, "unit": "comparisons/s", "cores": cores, "kind": "port",
            "sample": f"{reps} x 2^{log2n} DCF keys (n=32), eval_cmp party 0 + party 1, oracle C "
                      f"restatement with AES-NI={oracle.aesni()}, OpenMP",
            "single_thread": single_thread_baseline(args)}


def load_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_dcf_eval.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_unit", d.get("dram_bytes_per_party_eval"))
    except (OSError, ValueError):
        return None


def measure_secondary(dev, args):
    """Keygen and DPF numbers beside the headline (keygen and eval timed
    separately): CUDA events on the launching stream, 2^22
    elements, best of 3 after one warm-up."""
    import numpy as np
    import torch

    from paper_2006_04593_b200 import fss

    N = 1 << min(22, args.log2n)
    stream = torch.cuda.current_stream(dev)

    def timed(fn):
        fn()
        best = None
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            t = a.elapsed_time(b) / 1e3
            best = t if best is None else min(best, t)
        return best

    out = {"elements": N}
    rng = np.random.default_rng(77)
    t = timed(lambda: fss.keygen_cmp(N_BITS, rng, N, device=dev))
    out["dcf_keygen_pairs_per_s"] = N / t
    out["dcf_keygen_aes_per_s"] = N * 192 / t
    t = timed(lambda: fss.keygen_eq(N_BITS, rng, N, device=dev))
    out["dpf_keygen_pairs_per_s"] = N / t
    alpha, e0, e1 = fss.keygen_eq(N_BITS, rng, N, device=dev)
    x = alpha.clone()
    t = timed(lambda: fss.eval_eq(0, e0, x))
    out["dpf_eval_party_evals_per_s"] = N / t
    out["dpf_eval_aes_per_s"] = N * 32 / t
    rec = (fss.eval_eq(0, e0, x).view(torch.int64) + fss.eval_eq(1, e1, x).view(torch.int64)) & 0xFFFFFFFF
    assert bool((rec == 1).all()), "DPF reconstruction mismatch"
    del alpha, e0, e1, x, rec
    # ARNK key (de)serialisation of one party's DCF keys (fss_arnk_pack /
    # fss_arnk_unpack): HBM-bound byte transposes; algorithmic bytes per key =
    # the 824-B payload + the 1,088 B of key arrays, each moved once
    _, c0, _ = fss.keygen_cmp(N_BITS, rng, N, device=dev)
    payload = fss._pack_device(c0).reshape(-1)
    per_key = fss.cmp_elem_bytes(N_BITS) + 8 + 16 + 16 * N_BITS + N_BITS + 8 * N_BITS + 8 * (N_BITS + 1)
    t = timed(lambda: fss._pack_device(c0))
    out["arnk_pack_keys_per_s"] = N / t
    out["arnk_pack_gb_per_s"] = N * per_key / t / 1e9
    t = timed(lambda: fss._unpack(fss.KIND_CMP, 0, N_BITS, N, payload, dev))
    out["arnk_unpack_keys_per_s"] = N / t
    out["arnk_unpack_gb_per_s"] = N * per_key / t / 1e9
    out["arnk_algorithmic_bytes_per_key"] = per_key
    out["arnk_note"] = ("arnk_*_frac_hbm is against MEASURED_PEAKS' 1:1 copy. Pack reads 1,088 B and writes "
                        "824 B per key, a read-heavy mix that streams faster than a copy (read-only 7.36, "
                        "write-only 6.36 TB/s on this part, scripts/hbm_mix_probe.cu), so pack can exceed 1; "
                        "the time-additive roof of its mix is 6.89 TB/s, of unpack's (824 : 1,088) 6.76 TB/s "
                        "(profiles/r02_arnk_tma_pack_tiles.json)")
    back = fss._unpack(fss.KIND_CMP, 0, N_BITS, N, payload, dev)
    assert torch.equal(back.scw, c0.scw) and torch.equal(back.leaf_cw.view(torch.int64),
                                                         c0.leaf_cw.view(torch.int64)), "ARNK round trip"
    del c0, payload, back
    torch.cuda.empty_cache()
    return out


def measure_exchange(dev, xdev, rank, ws, N, barrier, max_over_ranks):
    """The one online message of a comparison when the two parties sit on
    different GPUs: rank r (party r % 2) swaps its wire-packed masked inputs
    (N x u32 at n = 32) with rank r ^ 1 through runtime.DistTransport (NCCL
    point-to-point over NVLink / NVSwitch). Max over ranks, 5 exchanges."""
    import torch

    from paper_2006_04593_b200 import runtime

    sess = runtime.Session(rank % 2, runtime.DistTransport(rank ^ 1, device=xdev))
    msg = torch.full((N,), rank, dtype=torch.int32, device=dev)   # u32 wire words
    peer = sess.exchange("comparison", runtime.FRAME_MASKED, msg, N)
    assert int(peer[0]) == (rank ^ 1)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        sess.exchange("comparison", runtime.FRAME_MASKED, msg, N)
    torch.cuda.synchronize()
    t = max_over_ranks((time.perf_counter() - t0) / 5)
    return {"bytes_each_way_per_rank": 4 * N, "ms": t * 1e3, "GBps_each_way": 4 * N / t / 1e9,
            "pairs": ws // 2, "note": "wall clock incl. the 24-byte frame header round trip"}


def measure_pair_protocol(dev, xdev, rank, barrier, max_over_ranks, M=1 << 22, reps=5):
    """The online sign test with the two parties on two GPUs: rank r plays party
    r % 2 against rank r ^ 1 (mask -> exchange -> DCF eval, one round), once
    with the message over NCCL (DistTransport) and once read in place from the
    peer's HBM by the eval kernel (PeerTransport, CUDA IPC over NVLink).
    Max over ranks of the wall time per call."""
    import numpy as np
    import torch

    from paper_2006_04593_b200 import dealer, fss, runtime
    from paper_2006_04593_b200.sharing import AdditiveShare, encode_fixed, share

    party, peer, pair = rank % 2, rank ^ 1, rank // 2
    rng = np.random.default_rng(88 + pair)
    xs = share(encode_fixed(rng.uniform(-100, 100, M), 3, 32, device=dev), rng, precision=3)
    y = AdditiveShare(party, xs[party].values, 0)
    out = {"elements_per_pair": M}
    for name, make in (("nccl", lambda: runtime.DistTransport(peer, device=xdev)),
                       ("peer_memory", lambda: runtime.PeerTransport(peer, device=dev,
                                                                     capacity=8 * M))):
        try:
            transport = make()
        except runtime.PeerAccessError as e:     # raised on both ranks of the pair alike
            out[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
            continue
        keys = dealer.make_dealer(32, seed=77 + pair).for_party(party).cmp_keys(M * (reps + 1))
        sess = runtime.Session(party, transport)
        fss.sign_protocol(sess, y, keys)          # warm-up
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            r = fss.sign_protocol(sess, y, keys)
        torch.cuda.synchronize()
        t = max_over_ranks((time.perf_counter() - t0) / reps)
        sess.close()
        out[name] = {"ms_per_call": t * 1e3, "comparisons_per_s_per_pair": M / t}
        del keys, r
    return out


def measure_gather(k0, k1, x, total, rank, barrier, max_over_ranks, reps=5):
    """The output collective of SURVEY §8e, three ways, per step of BOTH parties'
    evaluation of this rank's slice (max over ranks of the wall time):
    * eval_only   -- the two eval launches, shares stay local (the `value` step);
    * nccl_gather -- + both parties' shares to rank 0 at wire width
                     (shard.gather_ring: 4 B per element per party, NCCL);
    * peer_fused  -- the eval kernels store their shares straight into rank 0's
                     result buffer through CUDA IPC peer memory
                     (shard.PeerGather, fss.eval_cmp(out=...)), then finish().
    Rank 0 checks that both gathers reconstruct to bits."""
    import torch

    from paper_2006_04593_b200 import fss, shard

    def eval_only():
        return fss.eval_cmp(0, k0, x), fss.eval_cmp(1, k1, x)

    def nccl():
        y0, y1 = eval_only()
        return shard.gather_ring(y0, N_BITS, total, dst=0), shard.gather_ring(y1, N_BITS, total, dst=0)

    from paper_2006_04593_b200.runtime import PeerAccessError
    try:
        g = shard.PeerGather(total, slots=2, dst=0)
    except PeerAccessError as e:                 # agreed over all ranks: all skip it
        g, peer_error = None, f"{type(e).__name__}: {e}"[:300]

    def fused():
        fss.eval_cmp(0, k0, x, out=g.out(0))
        fss.eval_cmp(1, k1, x, out=g.out(1))
        return g.finish()

    def check(r0, r1):
        if rank == 0:
            rec = (r0.view(torch.int64) + r1.view(torch.int64)) & 0xFFFFFFFF
            assert bool(((rec == 0) | (rec == 1)).all()), "gathered shares do not reconstruct to bits"

    check(*nccl())
    if g is not None:
        res = fused()
        if rank == 0:
            check(res[0], res[1])
    out = {"elements": total, "bytes_to_rank0_wire": 2 * total * 4, "bytes_to_rank0_fused": 2 * total * 8}
    variants = [("eval_only", eval_only), ("nccl_gather", nccl)]
    if g is not None:
        variants.append(("peer_fused", fused))
    else:
        out["peer_fused_error"] = peer_error
    for name, fn in variants:
        fn()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        out[f"{name}_ms_per_step"] = max_over_ranks((time.perf_counter() - t0) / reps) * 1e3
    if g is not None:
        g.close()
    return out


def numa_bind(dev) -> dict:
    """Bind this process's host threads to the NUMA node of its GPU (read from
    sysfs by PCI address) so the pinned e2e buffers are first-touched there.
    Returns what was done; the caller restores the previous affinity."""
    import torch
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    info = {"gpu_pci": bus, "node": None, "cpus": None}
    try:
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as fh:
            node = int(fh.read().strip())
        info["node"] = node
        if node >= 0:
            with open(f"/sys/devices/system/node/node{node}/cpulist") as fh:
                cpulist = fh.read().strip()
            cpus = set()
            for part in cpulist.split(","):
                lo, _, hi = part.partition("-")
                cpus.update(range(int(lo), int(hi or lo) + 1))
            cpus &= os.sched_getaffinity(0) or cpus
            if cpus:
                os.sched_setaffinity(0, cpus)
                info["cpus"] = cpulist
    except (OSError, ValueError) as exc:
        info["error"] = str(exc)
    return info


def roofline_blocks(N: int, avg_launch_s: float, peaks_live: dict, hbm_peak: float, hbm_src: str,
                    traffic, label: str) -> dict:
    """The roofline objects of the dominant kernel (dcf_eval_kernel), for
    launches of N party-evals averaging avg_launch_s."""
    aes_rate = N * AES_PER_EVAL / avg_launch_s
    lookup_rate = N * LOOKUPS_PER_EVAL / avg_launch_s
    lds_peak_lookups = peaks_live["lds_wavefronts_per_s"] * 32
    alu_peak_aes = peaks_live["lop3_lane_ops_per_s"] / LOP3_PER_AES_BITSLICED
    achieved_gbs = N * BYTES_PER_EVAL / avg_launch_s / 1e9
    return {
        "roofline": {"bound": "smem-lookup", "achieved": lookup_rate, "peak": lds_peak_lookups,
                     "unit": "T-table lookups/s", "frac": lookup_rate / lds_peak_lookups,
                     "traffic": (traffic * N if traffic else None),
                     "kernel": "dcf_eval_kernel",
                     "binding": ("shared-memory LDS wavefronts: the AES rounds are T-table lookups, one "
                                 "conflict-free LDS.32 wavefront per 32 lanes; ncu shows the shared pipe "
                                 "at ~95 % and DRAM at ~15 % (profiles/ncu_dcf_eval.json). alu_roofline "
                                 "frac > 1 is expected: that roof prices a bitsliced AES at 356.25 LOP3 "
                                 "per block, work the T-table kernel does not execute, so it does not "
                                 "bound this kernel (DESIGN.md section 3)"),
                     "aes_blocks_per_s": aes_rate,
                     "note": (f"{LOOKUPS_PER_EVAL} algorithmic lookups per party-eval (32 levels x "
                              "[160 for the child block + 149 for the sigma block: rounds 1-9 and the 5 "
                              "last-round bytes that sigma mod 2^32 and tau read]) x "
                              f"{label} party-evals per launch / CUDA-event launch time; "
                              "peak = 32 x the measured conflict-free LDS wavefront rate on this GPU "
                              f"({peaks_live['lds_wavefronts_per_s']:.4g}/s, fss_probe_peaks); "
                              "traffic = ncu DRAM bytes per launch (profiles/ncu_dcf_eval.json x N)")},
        "alu_roofline": {"bound": "alu", "achieved": aes_rate, "peak": alu_peak_aes,
                         "unit": "AES-blocks/s", "frac": aes_rate / alu_peak_aes,
                         "note": (f"bitsliced-AES ALU roof of SURVEY.md 8d: measured LOP3 rate "
                                  f"{peaks_live['lop3_lane_ops_per_s']:.4g} lane-ops/s / "
                                  f"{LOP3_PER_AES_BITSLICED} LOP3 per block (not binding, see "
                                  "roofline.binding)")},
        "hbm_roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved_gbs / hbm_peak,
                         "note": f"{BYTES_PER_EVAL} algorithmic B per party-eval; peak = {hbm_src}"},
    }


def _hbm_peak():
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except (OSError, ValueError):
        pass
    if "hbm_gbs" in peaks:
        return float(peaks["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    return 6650.0, "fallback 6.65 TB/s of B200_PROFILING.md (MEASURED_PEAKS.json absent on this box)"


class _Ctx:
    """Per-run distributed plumbing shared by the weak and strong modes."""

    def __init__(self, args, ws, rank, local):
        import torch
        import torch.distributed as dist
        self.args, self.ws, self.rank = args, ws, rank
        # Test-only: FSS_BENCH_SAME_GPU=1 puts every rank on cuda:0 over gloo so the
        # N>1 code path can be exercised on a single-GPU box (numbers meaningless).
        self.same_gpu = os.environ.get("FSS_BENCH_SAME_GPU") == "1"
        self.local = 0 if self.same_gpu else local
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if ws > 1:
            import datetime
            timeout = datetime.timedelta(minutes=10)
            if self.same_gpu:
                dist.init_process_group("gloo", timeout=timeout)
            else:
                dist.init_process_group("nccl", device_id=self.dev, timeout=timeout)
        self.xdev = torch.device("cpu") if self.same_gpu else self.dev   # device for collectives
        self.stream = torch.cuda.current_stream(self.dev)

    def barrier(self):
        import torch.distributed as dist
        if self.ws > 1:
            dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        import torch
        import torch.distributed as dist
        if self.ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=self.xdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def finish(self):
        import torch.distributed as dist
        if self.ws > 1:
            dist.destroy_process_group()


def strong_plan(global_log2n: int, chunk_log2n: int, rank: int, ws: int):
    """Rank's slice [lo, hi) of the 2^G batch (shard.shard_bounds) and its chunks
    of at most 2^chunk_log2n keys, in order."""
    from paper_2006_04593_b200 import shard
    lo, hi = shard.shard_bounds(1 << global_log2n, rank, ws)
    cmax = 1 << chunk_log2n
    return lo, hi, [(c, min(hi, c + cmax)) for c in range(lo, hi, cmax)]


def run_strong(args, ctx):
    """One global batch of 2^G keys, rank r evaluates slice r (shard_bounds),
    streamed in chunks of <= 2^chunk_log2n keys. Per chunk: keygen of the
    chunk's keys from the shared tape (fss.keygen_cmp with the chunk's offsets,
    bit-identical to a single-device keygen of 2^G; timed separately), then
    both parties' eval (timed). Resident when the slice is one chunk."""
    import numpy as np
    import torch

    from paper_2006_04593_b200 import _lib, fss, shard

    ws, rank, dev, stream = ctx.ws, ctx.rank, ctx.dev, ctx.stream
    total = 1 << args.global_log2n
    lo, hi, chunks = strong_plan(args.global_log2n, args.chunk_log2n, rank, ws)
    cmax = 1 << args.chunk_log2n
    resident = len(chunks) == 1

    def deal(c_lo, c_hi):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        alpha, k0, k1 = fss.keygen_cmp(N_BITS, np.random.default_rng(1000), total, device=dev,
                                       _shard=(c_lo, c_hi - c_lo))
        y = torch.randint(-(1 << 20), 1 << 20, (c_hi - c_lo,), device=dev, dtype=torch.int64)
        x = ((alpha.view(torch.int64) + y) & 0xFFFFFFFF).view(torch.uint64)
        ev1.record(stream)
        return alpha, k0, k1, x, (ev0, ev1)

    def check(alpha, k0, k1, x):
        rec = (fss.eval_cmp(0, k0, x).view(torch.int64) + fss.eval_cmp(1, k1, x).view(torch.int64)) \
            & 0xFFFFFFFF
        assert torch.equal(rec, (x.view(torch.int64) <= alpha.view(torch.int64)).to(torch.int64)), \
            "DCF reconstruction mismatch"

    keys = deal(*chunks[0])
    check(*keys[:4])
    # e2e through the public API with host buffers: each chunk's x in pinned
    # host memory, the shares back in pinned host memory (zero-copy kernel)
    x_host = None if args.no_e2e else torch.empty(max(b - a for a, b in chunks), dtype=torch.int64,
                                                  pin_memory=True)
    for _ in range(args.warmup):
        fss.eval_cmp(0, keys[1], keys[3])
        fss.eval_cmp(1, keys[2], keys[3])
    torch.cuda.synchronize()
    sampler = ClockSampler(ctx.local)
    sampler.start()
    eval_evs, kg_evs, launch_n, host_evs = [], [], [], []
    ctx.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    for _ in range(args.steps):
        for ci, (c_lo, c_hi) in enumerate(chunks):
            if not resident:
                keys = None                      # the previous chunk's memory is reused
                keys = deal(c_lo, c_hi)
                kg_evs.append(keys[4])
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(stream)
            fss.eval_cmp(0, keys[1], keys[3])
            b.record(stream)
            fss.eval_cmp(1, keys[2], keys[3])
            c.record(stream)
            eval_evs.append((a, b, c))
            launch_n += [c_hi - c_lo] * 2
            if x_host is not None:
                xh = x_host[:c_hi - c_lo]
                xh.copy_(keys[3].view(torch.int64), non_blocking=True)
                h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                h0.record(stream)
                fss.eval_cmp(0, keys[1], xh.view(torch.uint64))
                fss.eval_cmp(1, keys[2], xh.view(torch.uint64))
                h1.record(stream)
                host_evs.append((h0, h1))
    torch.cuda.synchronize()
    ctx.barrier()
    wall = time.perf_counter() - t_wall
    clocks = sampler.stop()
    if not resident:
        check(*keys[:4])
    launch_ms = []
    for a, b, c in eval_evs:
        launch_ms += [a.elapsed_time(b), b.elapsed_time(c)]
    t_eval = ctx.max_over_ranks(sum(launch_ms) / 1e3)
    t_kg = ctx.max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in kg_evs) / 1e3) if kg_evs else None
    t_host = ctx.max_over_ranks(sum(e0.elapsed_time(e1) for e0, e1 in host_evs) / 1e3) if host_evs else None
    wall = ctx.max_over_ranks(wall)
    value = total * args.steps / t_eval
    avg_launch_s = sum(launch_ms) / len(launch_ms) / 1e3
    n_avg = sum(launch_n) / len(launch_n)
    del keys
    torch.cuda.empty_cache()
    if rank != 0:
        return
    hbm_peak, hbm_src = _hbm_peak()
    peaks_live = _lib.probe_peaks()
    line = {
        "metric": METRIC, "value": value, "unit": "comparisons/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_eval / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(args, ws),
        "chunking": {"keys_per_rank": hi - lo, "chunks_per_rank": len(chunks), "chunk_keys": cmax,
                     "resident": resident,
                     "note": ("eval time summed over the chunks (CUDA events around each chunk's two "
                              "launches); keygen of each chunk from the shared 2^%d tape runs between "
                              "them and is timed separately" % args.global_log2n) if not resident
                     else "slice resident in HBM, dealt once before the timed steps"},
        "keygen": ({"pairs_per_s": total * args.steps / t_kg, "ms_per_step": t_kg / args.steps * 1e3}
                   if t_kg else None),
        "wall_ms_per_step_incl_keygen": wall / args.steps * 1e3,
        "wall_note": ("host wall clock per step: every chunk's keygen, its device-x eval of both "
                      "parties (the timed value) and, unless --no-e2e, the same eval again from "
                      "pinned host x (e2e)"),
        **roofline_blocks(int(n_avg), avg_launch_s, peaks_live, hbm_peak, hbm_src,
                          load_traffic(), f"2^{int(np.log2(n_avg))}"),
        "peaks_probe": peaks_live,
        "kernel_ms_per_launch": avg_launch_s * 1e3,
        "clocks": clocks,
        "gpu_launches": len(launch_ms),
        "e2e": ({"value": total * args.steps / t_host, "unit": "comparisons/s",
                 "h2d_bytes_per_step": 2 * total * 8, "d2h_bytes_per_step": 2 * total * 8,
                 "step": "fss.eval_cmp(party 0 and 1) per chunk with the chunk's x in pinned host memory "
                         "and the shares returned in pinned host memory (zero-copy kernel); summed over "
                         "the chunks, max over ranks"} if t_host else None),
        "cpu_baseline": None,
    }
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import numpy as np
    import torch

    from paper_2006_04593_b200 import _lib, fss, shard

    _lib.load()  # fail loudly without the CUDA library
    ctx = _Ctx(args, ws, rank, local)
    try:
        if args.global_log2n is not None:
            run_strong(args, ctx)
        else:
            run_weak(args, ctx, np, torch, _lib, fss, shard)
    finally:
        ctx.finish()


def run_weak(args, ctx, np, torch, _lib, fss, shard):
    ws, rank, dev, xdev, stream = ctx.ws, ctx.rank, ctx.dev, ctx.xdev, ctx.stream
    barrier, max_over_ranks = ctx.barrier, ctx.max_over_ranks
    N = 1 << args.log2n

    # ---- value: keys resident in HBM, device inputs ------------------------
    # rank r holds slice r of ONE global batch of N * ws keys (shard.py: the
    # slice's tape is drawn at its offsets in the shared PCG64 stream, so the
    # union over ranks is bit-identical to a single-device keygen of N * ws)
    alpha, k0, k1 = shard.keygen_cmp_shard(N_BITS, np.random.default_rng(1000), N * ws, rank, ws,
                                           device=dev)
    y = torch.randint(-(1 << 20), 1 << 20, (N,), device=dev, dtype=torch.int64)
    x = ((alpha.view(torch.int64) + y) & 0xFFFFFFFF).view(torch.uint64)
    out0 = out1 = None
    for _ in range(args.warmup):
        out0 = fss.eval_cmp(0, k0, x)
        out1 = fss.eval_cmp(1, k1, x)
    torch.cuda.synchronize()
    rec = (out0.view(torch.int64) + out1.view(torch.int64)) & 0xFFFFFFFF
    assert torch.equal(rec, (x.view(torch.int64) <= alpha.view(torch.int64)).to(torch.int64)), \
        "DCF reconstruction mismatch"

    sampler = ClockSampler(ctx.local)
    sampler.start()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
    barrier()
    torch.cuda.synchronize()
    evs[0].record(stream)
    for s in range(args.steps):
        fss.eval_cmp(0, k0, x)
        evs[2 * s + 1].record(stream)
        fss.eval_cmp(1, k1, x)
        evs[2 * s + 2].record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    launch_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(2 * args.steps)]
    t_local = evs[0].elapsed_time(evs[-1]) / 1e3
    t = max_over_ranks(t_local)
    value = ws * N * args.steps / t
    avg_launch_s = sum(launch_ms) / len(launch_ms) / 1e3

    hbm_peak, hbm_src = _hbm_peak()
    peaks_live = _lib.probe_peaks()   # measured on this box, this run
    roof = roofline_blocks(N, avg_launch_s, peaks_live, hbm_peak, hbm_src, load_traffic(),
                           f"2^{args.log2n}")
    secondary = measure_secondary(dev, args) if not args.no_secondary else None
    if secondary:
        for op in ("pack", "unpack"):
            secondary[f"arnk_{op}_frac_hbm"] = secondary[f"arnk_{op}_gb_per_s"] / hbm_peak
    if ws >= 2 and ws % 2 == 0 and not args.no_secondary:
        secondary = dict(secondary or {})
        secondary["nccl_masked_exchange"] = measure_exchange(dev, xdev, rank, ws, N, barrier,
                                                             max_over_ranks)
        secondary["two_gpu_sign_protocol"] = measure_pair_protocol(dev, xdev, rank, barrier,
                                                                   max_over_ranks)
    if ws >= 2 and not args.no_secondary:
        secondary = dict(secondary or {})
        secondary["output_gather"] = measure_gather(k0, k1, x, N * ws, rank, barrier,
                                                    max_over_ranks)
    del out0, out1, rec

    # ---- e2e through the public API with host buffers ----------------------
    e2e = None
    numa = None
    if not args.no_e2e:
        prev_affinity = os.sched_getaffinity(0)
        numa = None if args.no_numa else numa_bind(dev)
        x_host = torch.empty(N, dtype=torch.int64, pin_memory=True)
        x_host.copy_(torch.from_numpy(np.random.default_rng(5 + rank).integers(
            0, 1 << 32, N, dtype=np.uint64).view(np.int64)))
        x_host = x_host.view(torch.uint64)

        def timed_host(step, steps):
            barrier()
            torch.cuda.synchronize()
            e_start = torch.cuda.Event(enable_timing=True)
            e_end = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e_start.record(stream)
            for _ in range(steps):
                step()
            e_end.record(stream)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            return max_over_ranks(max(e_start.elapsed_time(e_end) / 1e3, wall))

        # (1) online comparison through the public API: keys resident in HBM
        # (dealt before, like the reference arm's keys), pinned host x in,
        # pinned host shares out -- every step copies x up and both shares down.
        def e2e_step():
            r0 = fss.eval_cmp(0, k0, x_host)      # pinned host in -> pinned host out
            r1 = fss.eval_cmp(1, k1, x_host)
            return r0, r1

        # warm-up: the first host-pipeline calls also set up pinned staging
        # blocks and side streams (one-time costs a long-running caller never sees)
        for _ in range(max(args.warmup, 5)):
            r0, r1 = e2e_step()
        want = (x_host.view(torch.int64) <= alpha.view(torch.int64).cpu()).to(torch.int64)
        assert torch.equal((r0.view(torch.int64) + r1.view(torch.int64)) & 0xFFFFFFFF, want)
        t_e2e = timed_host(e2e_step, args.steps)
        e2e = {"value": ws * N * args.steps / t_e2e, "unit": "comparisons/s",
               "h2d_bytes_per_step": 2 * N * 8, "d2h_bytes_per_step": 2 * N * 8,
               "step": "fss.eval_cmp(party 0 and 1, HBM-resident keys, pinned host x of 2^%d u64) "
                       "-> pinned host shares; zero-copy: the kernel loads x from and stores the "
                       "shares to pinned host memory over PCIe" % args.log2n,
               "numa": numa}

        # (1b) the reference caller's convention (fss.py:347-354): numpy x in,
        # numpy shares out -- pageable memory, staged through pinned slots by the
        # library's 2-stream pipeline
        x_np = x_host.view(torch.int64).numpy().view(np.uint64).copy()

        def numpy_step():
            return fss.eval_cmp(0, k0, x_np), fss.eval_cmp(1, k1, x_np)

        for _ in range(3):
            n0, n1 = numpy_step()
        assert np.array_equal((n0 + n1) & np.uint64(0xFFFFFFFF), want.numpy().view(np.uint64))
        t_np = timed_host(numpy_step, max(3, args.steps // 2))
        e2e["numpy"] = {"value": ws * N * max(3, args.steps // 2) / t_np, "unit": "comparisons/s",
                        "h2d_bytes_per_step": 2 * N * 8, "d2h_bytes_per_step": 2 * N * 8,
                        "step": "fss.eval_cmp(party 0 and 1, numpy uint64 x of 2^%d) -> numpy shares "
                                "(pageable host memory, staged pipeline)" % args.log2n}
        del x_np, n0, n1, r0, r1
        del k0, k1, alpha, x, y
        torch.cuda.empty_cache()

        # (2) dealer + online: keygen_cmp from the host numpy Generator (tape
        # drawn on device from its PCG64 state) inside every step as well.
        rng2 = np.random.default_rng(2000 + rank)

        def e2e_keygen_step():
            _, q0, q1 = fss.keygen_cmp(N_BITS, rng2, N, device=dev)
            return fss.eval_cmp(0, q0, x_host), fss.eval_cmp(1, q1, x_host)

        for _ in range(3):   # fills the allocator's cache for two generations of keys
            e2e_keygen_step()
        ksteps = max(3, args.steps // 4)
        t_kg = timed_host(e2e_keygen_step, ksteps)
        e2e["with_keygen"] = {"value": ws * N * ksteps / t_kg, "unit": "comparisons/s",
                              "steps": ksteps,
                              "step": "keygen_cmp(32, numpy Generator, 2^%d) + the eval step above"
                                      % args.log2n}
        os.sched_setaffinity(0, prev_affinity)

    if rank != 0:
        return
    cpu = None if (args.no_cpu or ws > 1) else cpu_baseline_line(args)
    cfg = workload_config(args, ws)
    line = {
        "metric": METRIC,
        "value": value, "unit": "comparisons/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "dtype_note": "AES on 32-bit words / u8 key bytes, ring sums mod 2^32 (u64 storage, "
                      "reference layout)", "data": "synthetic",
        "config": cfg,
        "residency": "keys resident in HBM; inputs larger than L2 (%.1f GB of keys per GPU, L2 126 MB), "
                     "so no L2 flush between steps" % (N * (1064 + 2 * 24) / 1e9),
        **roof,
        "peaks_probe": peaks_live,
        "secondary": secondary,
        "kernel_ms_per_launch": avg_launch_s * 1e3,
        "clocks": clocks,
        "gpu_launches": 2 * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    args = _args()
    ws, rank, local = _dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # asked for N GPUs without a launcher: launch N ranks ourselves
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus and os.environ.get("FSS_BENCH_SAME_GPU") != "1":
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible\n")
            sys.exit(2)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if ws != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but the launcher started {ws} rank(s)\n")
        sys.exit(2)
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
