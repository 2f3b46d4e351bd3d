"""Element-sharded dealer (shard.py, fss_pcg64_tape_slice) on the GPU.

Every rank's slice of a sharded keygen must be bit-identical to the same slice
of the single-device keygen of the whole batch -- which the other test files
pin to the reference -- for DCF and DPF keys, n on both sides of the 32-bit /
64-bit draw split, with and without numpy's buffered half-word at the start,
given or drawn alpha, uneven and empty slices; and every rank's generator must
end in the single-device generator's state. A two-process run (both ranks on
cuda:0, gloo) then evaluates its slice and gathers the shares to rank 0."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

from paper_2006_04593_b200 import fss, shard  # noqa: E402

DEV = torch.device("cuda", 0)


def _rng(seed, buffered):
    rng = np.random.default_rng(seed)
    if buffered:  # one 32-bit draw leaves numpy's buffered half-word behind
        rng.integers(0, 1 << 20, size=1, dtype=np.uint64)
        assert rng.bit_generator.state["has_uint32"] == 1
    return rng


def _fields(kind):
    common = ["alpha_share", "seed0"]
    if kind == "cmp":
        return common, ["scw", "tcw", "sigma_cw", "leaf_cw"]
    return common, ["scw", "tcw", "cw_final"]


def _cat(parts, axis):
    return torch.cat([p.view(torch.int64) if p.dtype == torch.uint64 else p for p in parts], dim=axis)


def _same_state(a, b):
    if isinstance(a, dict):
        return a.keys() == b.keys() and all(_same_state(a[k], b[k]) for k in a)
    if isinstance(a, np.ndarray):
        return np.array_equal(a, b)
    return a == b


def _check_sharded(kind, n, total, world, buffered, given_alpha, rng_factory=None, out_bits=None):
    make = rng_factory or (lambda: _rng(11, buffered))
    galpha = None
    if given_alpha:
        galpha = np.random.default_rng(3).integers(0, 1 << min(n, 63), total, dtype=np.uint64)
    r_full = make()
    if kind == "cmp":
        full = fss.keygen_cmp(n, r_full, total, alpha=galpha, out_bits=out_bits, device=DEV)
    else:
        full = fss.keygen_eq(n, r_full, total, alpha=galpha, device=DEV)
    parts, rngs = [], []
    for r in range(world):
        rr = make()
        lo, hi = shard.shard_bounds(total, r, world)
        a_sl = None if galpha is None else galpha[lo:hi]
        if kind == "cmp":
            parts.append(shard.keygen_cmp_shard(n, rr, total, r, world, alpha=a_sl, out_bits=out_bits,
                                                device=DEV))
        else:
            parts.append(shard.keygen_eq_shard(n, rr, total, r, world, alpha=a_sl, device=DEV))
        rngs.append(rr)
    alpha, k0, k1 = full
    assert torch.equal(_cat([p[0] for p in parts], 0), alpha.view(torch.int64))
    per_party, shared = _fields(kind)
    for j, kf in ((1, k0), (2, k1)):
        for f in per_party:
            assert torch.equal(_cat([getattr(p[j], f) for p in parts], 0),
                               getattr(kf, f).view(torch.int64) if getattr(kf, f).dtype == torch.uint64
                               else getattr(kf, f)), (f, j)
    for f in shared:
        ref = getattr(k0, f)
        axis = 0 if f == "cw_final" else 1
        got = _cat([getattr(p[1], f) for p in parts], axis)
        assert torch.equal(got, ref.view(torch.int64) if ref.dtype == torch.uint64 else ref), f
    want_state = r_full.bit_generator.state
    nxt = r_full.integers(0, 1 << 30, 5)
    for rr in rngs:
        assert _same_state(rr.bit_generator.state, want_state)
        assert np.array_equal(rr.integers(0, 1 << 30, 5), nxt)


@pytest.mark.parametrize("n", [8, 32, 40, 63])
@pytest.mark.parametrize("buffered", [False, True])
def test_sharded_cmp_keygen_equals_slices(n, buffered):
    for total, world in ((1, 1), (7, 3), (1000, 4), (4099, 5), (3, 5)):
        _check_sharded("cmp", n, total, world, buffered, given_alpha=False)


@pytest.mark.parametrize("n", [5, 32, 33, 64])
def test_sharded_eq_keygen_equals_slices(n):
    for buffered in (False, True):
        for total, world in ((1000, 3), (17, 2)):
            _check_sharded("eq", n, total, world, buffered, given_alpha=False)


@pytest.mark.parametrize("kind,n", [("cmp", 32), ("cmp", 48), ("eq", 16), ("eq", 64)])
def test_sharded_keygen_given_alpha(kind, n):
    _check_sharded(kind, n, 999, 4, buffered=True, given_alpha=True)


def test_sharded_keygen_widened_out_bits_and_mt19937():
    _check_sharded("cmp", 12, 513, 3, False, False, out_bits=40)
    mt = lambda: np.random.Generator(np.random.MT19937(5))  # noqa: E731 - host-drawn tape
    _check_sharded("cmp", 32, 300, 2, False, False, rng_factory=mt)
    _check_sharded("eq", 32, 300, 3, False, True, rng_factory=mt)


def test_sharded_keygen_large_slice():
    # a 2^22 batch over 8 ranks: only the last rank's slice is generated
    total, world = 1 << 22, 8
    _, k0, k1 = fss.keygen_cmp(32, np.random.default_rng(21), total, device=DEV)
    a, s0, s1 = shard.keygen_cmp_shard(32, np.random.default_rng(21), total, world - 1, world, device=DEV)
    lo, hi = shard.shard_bounds(total, world - 1, world)
    assert torch.equal(s0.scw, k0.scw[:, lo:hi]) and torch.equal(s1.seed0, k1.seed0[lo:hi])
    assert torch.equal(s0.leaf_cw.view(torch.int64), k0.leaf_cw[:, lo:hi].view(torch.int64))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, total, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        x = np.random.default_rng(8).integers(0, 1 << 32, total, dtype=np.uint64)
        alpha, k0, k1 = shard.keygen_cmp_shard(32, np.random.default_rng(4), total, device=DEV)
        lo, hi = shard.shard_bounds(total, rank, 2)
        xs = torch.from_numpy(x[lo:hi].view(np.int64)).to(DEV).view(torch.uint64)
        y0, y1 = fss.eval_cmp(0, k0, xs), fss.eval_cmp(1, k1, xs)
        g0 = shard.gather_ring(y0, 32, total, dst=0)
        g1 = shard.gather_ring(y1, 32, total, dst=0)
        ga = shard.gather_shards(alpha, total, dst=0)
        ok = True
        if rank == 0:
            fa, f0, f1 = fss.keygen_cmp(32, np.random.default_rng(4), total, device=DEV)
            xd = torch.from_numpy(x.view(np.int64)).to(DEV).view(torch.uint64)
            w0, w1 = fss.eval_cmp(0, f0, xd), fss.eval_cmp(1, f1, xd)
            ok = (torch.equal(g0.view(torch.int64), w0.view(torch.int64))
                  and torch.equal(g1.view(torch.int64), w1.view(torch.int64))
                  and torch.equal(ga.view(torch.int64), fa.view(torch.int64)))
            rec = (g0.view(torch.int64) + g1.view(torch.int64)) & 0xFFFFFFFF
            ok = ok and torch.equal(rec.cpu(), torch.from_numpy((x <= fa.cpu().numpy()).astype(np.int64)))
        else:
            ok = g0 is None and g1 is None and ga is None
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_two_process_sharded_keygen_eval_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    total = 20001
    procs = [ctx.Process(target=_worker, args=(r, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)


def _worker_peer(rank, port, total, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        x = np.random.default_rng(8).integers(0, 1 << 32, total, dtype=np.uint64)
        alpha, k0, k1 = shard.keygen_cmp_shard(32, np.random.default_rng(4), total, device=DEV)
        lo, hi = shard.shard_bounds(total, rank, 2)
        xs = torch.from_numpy(x[lo:hi].view(np.int64)).to(DEV).view(torch.uint64)
        g = shard.PeerGather(total, slots=2, dst=1)
        for rnd in range(2):                  # the buffer is reusable round after round
            fss.eval_cmp(0, k0, xs, out=g.out(0))
            fss.eval_cmp(1, k1, xs, out=g.out(1))
            res = g.finish()
        ok = True
        if rank == 1:
            fa, f0, f1 = fss.keygen_cmp(32, np.random.default_rng(4), total, device=DEV)
            xd = torch.from_numpy(x.view(np.int64)).to(DEV).view(torch.uint64)
            w0, w1 = fss.eval_cmp(0, f0, xd), fss.eval_cmp(1, f1, xd)
            ok = (tuple(res.shape) == (2, total)
                  and torch.equal(res[0].view(torch.int64), w0.view(torch.int64))
                  and torch.equal(res[1].view(torch.int64), w1.view(torch.int64)))
        else:
            ok = res is None
        g.close()
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_two_process_peer_gather_fused_with_eval():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker_peer, args=(r, port, 30001, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)


def test_eval_out_argument():
    _, k0, _ = fss.keygen_cmp(32, np.random.default_rng(2), 1000, device=DEV)
    _, e0, _ = fss.keygen_eq(32, np.random.default_rng(2), 1000, device=DEV)
    x = torch.arange(1000, device=DEV).view(torch.uint64)
    buf = torch.empty(1000, dtype=torch.uint64, device=DEV)
    assert fss.eval_cmp(0, k0, x, out=buf) is buf
    assert torch.equal(buf.view(torch.int64), fss.eval_cmp(0, k0, x).view(torch.int64))
    assert fss.eval_eq(0, e0, x, out=buf) is buf
    assert torch.equal(buf.view(torch.int64), fss.eval_eq(0, e0, x).view(torch.int64))
    with pytest.raises(ValueError):
        fss.eval_cmp(0, k0, x, out=buf[:999])
    with pytest.raises(ValueError):
        fss.eval_cmp(0, k0, np.zeros(1000, dtype=np.uint64), out=buf)   # host input
    with pytest.raises(ValueError):
        fss.eval_cmp(0, k0, x, out=torch.empty(1000, dtype=torch.uint64))  # host buffer
    with pytest.raises(ValueError):
        fss.eval_cmp(0, k0, x, return_levels=True, out=buf)
