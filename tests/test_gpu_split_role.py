"""The reference's split-role flow (cli._cmd_keygen + cli._bench_split_role,
reference cli.py:140-214) on the B200 stack: a dealer writes one ARNK key
file; two party processes each read only their own payload (kept packed --
evaluated straight from the rows), derive consistent shares of the same
input from a shared seed, and run the one-round sign protocol against each
other (masked messages read in place from the peer's HBM, CUDA IPC); the
reconstructed result equals the in-process run on the unpacked keys. Both
processes share cuda:0 here; on a multi-GPU box each would own a GPU."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

N, NBITS, SEED = 5000, 32, 11


def _shares():
    from paper_2006_04593_b200.sharing import AdditiveShare, encode_fixed, share
    pub = np.random.default_rng(SEED)                 # both parties derive the same sharing
    values = pub.uniform(-100, 100, N)
    ys = share(encode_fixed(values, 3, NBITS), pub)
    return [AdditiveShare(p, ys[p].values, 0) for p in (0, 1)], values


def _party(rank, port, path, q):
    import torch.distributed as dist

    from paper_2006_04593_b200 import fss, keyfile, runtime
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        keys = keyfile.load_keys(path, party=rank, packed=True)   # only this party's payload
        ys, _ = _shares()
        res, ledger = runtime.run_peer_party(rank, 1 - rank,
                                             lambda s: fss.sign_protocol(s, ys[s.party], keys))
        q.put((rank, res.values.numpy().tobytes(), ledger.total_rounds(), bool(keys.consumed.all())))
    finally:
        dist.destroy_process_group()


def test_split_role_sign_protocol(tmp_path):
    from paper_2006_04593_b200 import fss, keyfile, runtime
    _, k0, k1 = fss.keygen_cmp(NBITS, np.random.default_rng(SEED + 1), N)   # the dealer
    path = str(tmp_path / f"cmp_{NBITS}_{N}.arnk")
    keyfile.save_keys(path, k0, k1)
    ys, values = _shares()
    (w0, _), (w1, _) = runtime.run_local_pair(
        lambda s: fss.sign_protocol(s, ys[s.party], {0: k0, 1: k1}[s.party]))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_party, args=(r, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in procs:
        rank, raw, rounds, consumed = q.get(timeout=300)
        got[rank] = np.frombuffer(raw, dtype=np.uint64)
        assert rounds == 1 and consumed
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got[0], w0.values.numpy()) and np.array_equal(got[1], w1.values.numpy())
    rec = (got[0] + got[1]) & np.uint64(0xFFFFFFFF)
    assert np.mean(rec == (np.floor(values * 1000) <= 0)) > 0.999
