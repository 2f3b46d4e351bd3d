"""GPU tests of the share layer (ring / sharing / beaver / nn_ops drop-ins)
against numpy restatements of the reference's formulas
(ring.py:99-162, sharing.py:65-264, beaver.py:257-300, nn_ops.py:83-190)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2006_04593_b200 import beaver, dealer, nn_ops, runtime, sharing  # noqa: E402
from paper_2006_04593_b200.ring import RingTensor, ring_mask  # noqa: E402


def _u(n):
    return np.uint64(ring_mask(n))


@pytest.mark.parametrize("n", [4, 8, 9, 16, 17, 31, 32, 33, 63, 64])
def test_ring_ops_vs_numpy(n):
    rng = np.random.default_rng(n)
    a = rng.integers(0, np.iinfo(np.uint64).max, 1000, dtype=np.uint64, endpoint=True) & _u(n)
    b = rng.integers(0, np.iinfo(np.uint64).max, 1000, dtype=np.uint64, endpoint=True) & _u(n)
    A, B = RingTensor(a, n), RingTensor(b, n)
    with np.errstate(over="ignore"):
        assert np.array_equal((A + B).numpy(), (a + b) & _u(n))
        assert np.array_equal((A - B).numpy(), (a - b) & _u(n))
        assert np.array_equal((A * B).numpy(), (a * b) & _u(n))
        assert np.array_equal((-A).numpy(), (np.uint64(0) - a) & _u(n))
        assert np.array_equal((A * 12345).numpy(), (a * np.uint64(12345)) & _u(n))
        assert int(A.sum().numpy()) == int(np.sum(a, dtype=np.uint64) & _u(n))
        assert np.array_equal(A.cumsum().numpy(), np.cumsum(a, dtype=np.uint64) & _u(n))
    half = np.uint64(1) << np.uint64(n - 1)
    want = a.astype(np.int64) - ((a >= half).astype(np.int64) << np.int64(n)) if n < 64 else \
        a.view(np.int64)
    assert np.array_equal(A.signed().cpu().numpy(), want)
    for i in (1, n // 2, n):
        assert np.array_equal(A.bit(i).cpu().numpy(),
                              ((a >> np.uint64(n - i)) & np.uint64(1)).astype(np.uint8))


@pytest.mark.parametrize("n,width", [(4, 1), (8, 1), (9, 2), (16, 2), (17, 4), (32, 4), (33, 8),
                                     (64, 8)])
def test_wire_packing_widths(n, width):
    rng = np.random.default_rng(n)
    a = rng.integers(0, np.iinfo(np.uint64).max, 777, dtype=np.uint64, endpoint=True) & _u(n)
    w = sharing.pack_ring(RingTensor(a, n), n)
    assert w.element_size() == width and w.numel() == 777
    # bytes on the wire == the reference's pack_ring (sharing.py:201-203)
    ref = a.astype({1: "<u1", 2: "<u2", 4: "<u4", 8: "<u8"}[width]).tobytes()
    assert w.cpu().view(torch.uint8).numpy().tobytes() == ref
    assert np.array_equal(sharing.unpack_ring(w, n).cpu().numpy(), a)


def test_share_reconstruct_encode_decode_and_guard():
    rng = np.random.default_rng(5)
    v = rng.uniform(-1000, 1000, (13, 7))
    enc = sharing.encode_fixed(v, 3, 32)
    s0, s1 = sharing.share(enc, rng, precision=3)
    assert np.allclose(sharing.decode_pair(s0, s1), np.floor(v * 1e3) / 1e3)
    with pytest.raises(sharing.FixedPointOverflow):
        sharing.encode_fixed([3e6], 3, 32)
    with sharing.forbid_reconstruction("audit"):
        with pytest.raises(sharing.ReconstructionForbidden):
            sharing.reconstruct(s0, s1)
        with sharing.allow_reconstruction():
            sharing.reconstruct(s0, s1)
    with pytest.raises(ValueError):
        sharing.reconstruct(s0, s0)


@pytest.mark.parametrize("n,digits", [(32, 3), (64, 3), (40, 1)])
def test_truncate_matches_reference_formula(n, digits):
    rng = np.random.default_rng(n + digits)
    vals = rng.integers(-10 ** 6, 10 ** 6, 5000)
    enc = RingTensor.from_ints(vals, n)
    s0, s1 = sharing.share(enc, rng, precision=digits)
    t0, t1 = sharing.truncate(s0, digits), sharing.truncate(s1, digits)
    div = np.uint64(10 ** digits)
    a0, a1 = s0.values.numpy(), s1.values.numpy()
    want0 = a0 // div
    neg = (np.uint64(0) - a1) & _u(n)
    want1 = (np.uint64(0) - (neg // div)) & _u(n)
    assert np.array_equal(t0.values.numpy(), want0) and np.array_equal(t1.values.numpy(), want1)
    got = sharing.reconstruct(t0, t1).signed().cpu().numpy()
    assert np.max(np.abs(got - np.floor_divide(vals, 10 ** digits))) <= 1


def test_reveal_and_beaver_product():
    rng = np.random.default_rng(8)
    x = RingTensor.from_ints(rng.integers(-5000, 5000, (20, 30)), 32)
    y = RingTensor.from_ints(rng.integers(-5000, 5000, (20, 30)), 32)
    xs, ys = sharing.share(x, rng), sharing.share(y, rng)
    t0, t1 = beaver.gen_triple(beaver.OP_MUL, beaver.ElemwiseGeometry((20, 30)), 32, rng)
    tri = [t0, t1]

    def prog(s):
        z = beaver.mul_protocol(s, xs[s.party], ys[s.party], tri[s.party])
        return sharing.reveal(s, z)
    (z0, l0), (z1, _) = runtime.run_local_pair(prog)
    assert z0 == z1 and z0 == x * y
    assert l0.snapshot() == {"mul": 1, "reveal": 1}
    with pytest.raises(beaver.TripleReuseError):
        runtime.run_local_pair(lambda s: beaver.mul_protocol(s, xs[s.party], ys[s.party],
                                                             tri[s.party]))
    with pytest.raises(NotImplementedError):
        beaver.gen_triple(beaver.OP_MATMUL, beaver.MatmulGeometry(2, 2, 2), 32, rng)
    blob = beaver.pack_triples(t0, t1)
    u0, u1 = beaver.unpack_triples(blob)
    assert u0.a == t0.a and u1.c == t1.c and u0.geometry == t0.geometry


@pytest.mark.parametrize("route", ["argmax", "k2"])
def test_batched_maxpool_is_the_plaintext_max(route):
    # planes (P, m, m) pooled in one 3- / 4-round call; values at p=3 are distinct
    # with overwhelming probability, so the result is the exact encoded maximum
    rng = np.random.default_rng(17)
    P, m = 6, 10
    v = rng.uniform(-10, 10, (P, m, m))
    xs = sharing.share(sharing.encode_fixed(v, 3, 32), rng, precision=3)
    d = dealer.make_dealer(32, seed=18)

    def prog(s):
        view = d.for_party(s.party)
        if route == "k2":
            return nn_ops.maxpool_k2(s, xs[s.party], view.maxpool_k2(m, planes=P))
        return nn_ops.maxpool(s, xs[s.party], 2, view.maxpool(m, 2, 2, planes=P), 2)
    (r0, l0), (r1, _) = runtime.run_local_pair(prog)
    got = sharing.decode_pair(r0, r1)
    want = (np.floor(v * 1e3) / 1e3).reshape(P, m // 2, 2, m // 2, 2).max(axis=(2, 4))
    assert got.shape == (P, m // 2, m // 2)
    assert np.mean(np.abs(got - want) < 1e-9) > 0.99
    assert l0.total_rounds() == (3 if route == "argmax" else 4)


def test_triple_container_bytes_match_reference():
    # kind-2 ARNK container of an elementwise triple (beaver.py:319-330), bytes
    # produced by the reference for the same rng seed (tests/golden/triple_arnk.npz)
    import os

    from conftest import GOLDEN
    from paper_2006_04593_b200 import fss
    with np.load(os.path.join(GOLDEN, "triple_arnk.npz")) as g:
        want, seed = g["arnk"].tobytes(), int(g["seed"])
    rng = np.random.default_rng(seed)
    t0, t1 = beaver.gen_triple(beaver.OP_MUL, beaver.ElemwiseGeometry((3, 4)), 32, rng)
    blob = fss.serialize_keys(beaver.pack_triples(t0, t1))
    assert blob == want
    u0, u1 = beaver.unpack_triples(fss.deserialize_keys(blob))
    assert u0.a == t0.a and u1.b == t1.b and u1.c == t1.c


@pytest.mark.parametrize("n", [6, 8, 12])
def test_protocols_at_narrow_rings(n):
    # masked messages at 1- and 2-byte wire widths, opened inside the eval kernels
    from paper_2006_04593_b200 import fss
    rng = np.random.default_rng(n)
    vals = rng.integers(-2, 3, 4000)
    ys = sharing.share(RingTensor.from_ints(vals, n), rng)
    d = dealer.make_dealer(n, seed=n + 1)

    def prog(s):
        view = d.for_party(s.party)
        e = fss.eq_protocol(s, ys[s.party], view.eq_keys(4000))
        c = fss.sign_protocol(s, ys[s.party], view.cmp_keys(4000))
        return e, c
    ((e0, c0), l0), ((e1, c1), _) = runtime.run_local_pair(prog)
    assert l0.bytes_sent == {"equality": 4000 * (1 if n <= 8 else 2),
                             "comparison": 4000 * (1 if n <= 8 else 2)}
    eq = sharing.reconstruct(e0, e1).numpy()
    assert np.array_equal(eq, (vals == 0).astype(np.uint64))
    cmp = sharing.reconstruct(c0, c1).numpy()
    # sign test fails with probability |y| / 2^n per element (fss.py:444-473)
    assert np.mean(cmp != (vals <= 0).astype(np.uint64)) < 8 * 2.0 / 2 ** n + 0.01


@pytest.mark.parametrize("n", [4, 13, 32, 63, 64])
def test_bit_decompose_recompose(n):
    from paper_2006_04593_b200.ring import bit_decompose, recompose
    rng = np.random.default_rng(n)
    a = rng.integers(0, np.iinfo(np.uint64).max, (5, 7), dtype=np.uint64, endpoint=True) & _u(n)
    A = RingTensor(a, n)
    bits = bit_decompose(A).cpu().numpy()
    want = np.stack([((a >> np.uint64(n - 1 - i)) & np.uint64(1)).astype(np.uint8)
                     for i in range(n)])
    assert np.array_equal(bits, want)
    assert recompose(bits, n) == A


@pytest.mark.parametrize("n,m,lead", [(32, 4, (3, 5)), (8, 2, (7,)), (64, 9, (2, 3)), (17, 5, (1,))])
def test_pairwise_and_group_sum_kernels_vs_numpy(n, m, lead):
    """fss_ring_pairwise / fss_ring_group_sum against the reference's numpy
    formulas (nn_ops.py:111-116): off-diagonal x_i - x_j grouped by j, and
    group sums plus party 0's public constant."""
    rng = np.random.default_rng(m * 100 + n)
    v = rng.integers(0, np.iinfo(np.uint64).max, lead + (m,), dtype=np.uint64, endpoint=True) & _u(n)
    with np.errstate(over="ignore"):
        want = (v[..., None, :] - v[..., :, None])[..., ~np.eye(m, dtype=bool)] & _u(n)
    got = nn_ops._pairwise_diffs(torch.from_numpy(v).cuda(), m, n)
    assert got.shape == want.shape and np.array_equal(got.cpu().numpy(), want)
    for party in (0, 1):
        share = sharing.AdditiveShare(party, RingTensor(want, n), 0)
        out = nn_ops._group_sum(share, m - 1, -(m - 1))
        with np.errstate(over="ignore"):
            ref = want.reshape(lead + (m, m - 1)).sum(axis=-1, dtype=np.uint64)
            if party == 0:
                ref = ref + np.uint64((-(m - 1)) & ((1 << 64) - 1))
        assert out.shape == lead + (m,) and np.array_equal(out.values.numpy(), ref & _u(n))
