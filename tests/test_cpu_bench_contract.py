"""bench.py's reference arm runs without a GPU (the oracle C port on host
cores): check it prints one JSON line with the contract's keys."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "2", "--warmup", "1", "--cpu-log2n", "12"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e", "impl"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_under_torchrun_uses_all_host_threads():
    """The driver launches the reference arm with torchrun for N > 1: rank 0
    alone prints the line, and it must not inherit torchrun's
    OMP_NUM_THREADS=1."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "2",
                        "--warmup", "1", "--cpu-log2n", "12"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


def test_gpus_flag_never_misreported():
    """--gpus N with a different number of ranks (or of visible GPUs) exits
    non-zero instead of printing a line for another N."""
    for env_extra in ({}, {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}):
        env = dict(os.environ, **env_extra)
        env.pop("FSS_BENCH_SAME_GPU", None)
        if not env_extra:
            env.pop("WORLD_SIZE", None)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                            "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
        assert r.returncode != 0
        assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        assert "--gpus 2" in r.stderr


def test_strong_plan_covers_the_batch_once():
    sys.path.insert(0, ROOT)
    import bench
    for G, C, ws in ((28, 26, 1), (28, 26, 2), (28, 26, 8), (20, 17, 3), (10, 12, 4)):
        seen = []
        for r in range(ws):
            lo, hi, chunks = bench.strong_plan(G, C, r, ws)
            assert chunks[0][0] == lo and chunks[-1][1] == hi
            assert all(b - a <= 1 << C and b > a for a, b in chunks)
            assert all(chunks[i][1] == chunks[i + 1][0] for i in range(len(chunks) - 1))
            seen += chunks
        assert seen[0][0] == 0 and seen[-1][1] == 1 << G
        assert sum(b - a for a, b in seen) == 1 << G
    assert len(bench.strong_plan(28, 26, 0, 1)[2]) == 4 and len(bench.strong_plan(28, 26, 3, 4)[2]) == 1


def test_reference_arm_config_equals_product_config():
    """Both arms print the same `config` dict for the same flags (the driver
    compares the arms' configs)."""
    sys.path.insert(0, ROOT)
    import bench
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1", "--log2n", "12", "--cpu-single-log2n", "10"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    import argparse
    ns = argparse.Namespace(global_log2n=None, log2n=12)
    assert d["config"] == bench.workload_config(ns, 1)
    assert d["sample_matches_config"] is True and d["config"]["global_batch"] == 1 << 12
    st = d["single_thread"]
    assert st["cores"] == 1 and st["value"] > 0 and st["kind"] == "port"
