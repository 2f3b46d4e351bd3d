"""bench.py's N>1 code path (torchrun, one process per rank, max-over-ranks
timing, the sharded dealer, the NCCL masked-exchange and output-gather
secondaries) exercised on a single-GPU box:
FSS_BENCH_SAME_GPU=1 puts both ranks on cuda:0 over gloo. Only the contract
is checked -- numbers from two ranks sharing one GPU are meaningless."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)


def test_two_rank_bench_contract():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, FSS_BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--log2n", "18"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1                        # rank 0 prints one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["config"]["global_batch"] == 2 << 18
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] == 6
    ex = d["secondary"]["nccl_masked_exchange"]
    assert ex["bytes_each_way_per_rank"] == 4 << 18 and ex["pairs"] == 1
    pp = d["secondary"]["two_gpu_sign_protocol"]
    assert pp["nccl"]["comparisons_per_s_per_pair"] > 0
    assert pp["peer_memory"]["comparisons_per_s_per_pair"] > 0
    g = d["secondary"]["output_gather"]   # both parties' shares of 2 x 2^18 elements to rank 0
    assert g["elements"] == 2 << 18 and g["bytes_to_rank0_wire"] == 2 * (2 << 18) * 4
    assert g["eval_only_ms_per_step"] > 0 and g["nccl_gather_ms_per_step"] > 0
    assert g["peer_fused_ms_per_step"] > 0


def test_strong_scaling_mode_self_launched():
    """`python bench.py --gpus 2 --global-log2n G` without a launcher re-launches
    itself with 2 ranks (same-GPU gloo mode here) and reports ONE strong-scaling
    line over the 2^G batch, each rank streaming its slice in chunks."""
    env = dict(os.environ, FSS_BENCH_SAME_GPU="1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
                        "--warmup", "3", "--global-log2n", "18", "--chunk-log2n", "16"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["global_batch"] == 1 << 18
    c = d["chunking"]
    assert c["keys_per_rank"] == 1 << 17 and c["chunks_per_rank"] == 2 and not c["resident"]
    assert d["gpu_launches"] == 3 * 2 * 2 and d["value"] > 0 and d["keygen"]["pairs_per_s"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 2 * 8 << 18
