"""The reference's unit tests of the layers around the FSS path -- pkg/tests/
test_ring.py, test_sharing.py, test_beaver.py (elementwise part),
test_nn_ops.py (ReLU / argmax / MaxPool) and test_dealer.py -- restated
one-to-one against the B200 drop-in (same names, seeds, inputs, assertions;
each cites the reference line). Out of scope and therefore not mirrored:
matmul / conv triples and protocols, break_ties, BatchNorm / Newton, the MLP
training plan. Device types: ring data are torch CUDA tensors,
read through RingTensor.numpy() / .cpu().
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

from hypothesis import given, settings, strategies as st  # noqa: E402
from scipy import stats  # noqa: E402

from paper_2006_04593_b200 import beaver, dealer, fss, nn_ops, sharing  # noqa: E402
from paper_2006_04593_b200.beaver import (ElemwiseGeometry, TripleReuseError, gen_triple,  # noqa: E402
                                          unroll)
from paper_2006_04593_b200.ring import (RingTensor, bit_decompose, recompose, ring_mask,  # noqa: E402
                                        signed_value)
from paper_2006_04593_b200.runtime import run_local_pair  # noqa: E402
from paper_2006_04593_b200.sharing import (FixedPointOverflow, ReconstructionForbidden,  # noqa: E402
                                           allow_reconstruction, decode_fixed, decode_pair,
                                           encode_fixed, forbid_reconstruction, mask_and_reveal,
                                           reconstruct, share, truncate)


def L(t):
    """Python list of a RingTensor / tensor / array."""
    if isinstance(t, RingTensor):
        return t.numpy().tolist()
    if isinstance(t, torch.Tensor):
        return t.cpu().tolist()
    return np.asarray(t).tolist()


# ------------------------------------------------------------ test_ring.py

def test_add_wraps_mod_2n():                                     # test_ring.py:8-11
    assert L(RingTensor.from_ints([250], 8) + RingTensor.from_ints([10], 8)) == [4]


def test_neg_is_two_complement():                                # test_ring.py:14-16
    assert L(-RingTensor.from_ints([1], 8)) == [255]


def test_mul_wraps():                                            # test_ring.py:19-21
    a = RingTensor.from_ints([16], 8)
    assert L(a * a) == [0]


def test_scalar_broadcast():                                     # test_ring.py:24-26
    assert L(RingTensor.from_ints([1, 2, 3], 8) + 254) == [255, 0, 1]


def test_ring_width_mismatch_rejected():                         # test_ring.py:29-33
    with pytest.raises(ValueError, match="width mismatch"):
        RingTensor.from_ints([1], 8) + RingTensor.from_ints([1], 16)


def test_shape_mismatch_rejected():                              # test_ring.py:36-40
    with pytest.raises(ValueError, match="shape mismatch"):
        RingTensor.from_ints([1, 2, 3], 8) + RingTensor.from_ints([1, 2], 8)


def test_bit_decompose_examples():                               # test_ring.py:43-46
    assert L(bit_decompose(RingTensor.from_ints([5], 4))[:, 0]) == [0, 1, 0, 1]
    assert L(bit_decompose(RingTensor.from_ints([0], 4))[:, 0]) == [0, 0, 0, 0]
    assert L(bit_decompose(RingTensor.from_ints([128], 8))[:, 0]) == [1, 0, 0, 0, 0, 0, 0, 0]


@pytest.mark.parametrize("n", [4, 6, 8, 10])
def test_bit_roundtrip_exhaustive(n):                            # test_ring.py:49-52
    a = RingTensor(np.arange(1 << n, dtype=np.uint64), n)
    assert recompose(bit_decompose(a), n) == a


@pytest.mark.parametrize("n", [16, 32, 64])
def test_bit_roundtrip_random(n):                                # test_ring.py:55-59
    a = RingTensor.random((1000,), n, np.random.default_rng(n))
    assert recompose(bit_decompose(a), n) == a


def test_signed_examples():                                      # test_ring.py:62-64
    assert L(signed_value(RingTensor.from_ints([255, 127, 128], 8))) == [-1, 127, -128]


def test_signed_roundtrip_exhaustive_n8():                       # test_ring.py:67-70
    vals = np.arange(-128, 128)
    assert np.array_equal(RingTensor.from_ints(vals, 8).signed().cpu().numpy(), vals)


@given(st.integers(min_value=4, max_value=64), st.data())
@settings(max_examples=50, deadline=None)
def test_additive_inverse_property(n, data):                     # test_ring.py:73-78
    vals = data.draw(st.lists(st.integers(0, (1 << n) - 1), min_size=1, max_size=8))
    a = RingTensor(np.array(vals, dtype=np.uint64), n)
    assert np.all((a + (-a)).numpy() == 0)


def test_mask_rejects_bad_widths():                              # test_ring.py:90-94
    with pytest.raises(ValueError):
        ring_mask(3)
    with pytest.raises(ValueError):
        ring_mask(65)


# ------------------------------------------------------------ test_sharing.py

def test_encode_examples():                                      # test_sharing.py:15-17
    assert L(encode_fixed(1.5, 3, 32)) == 1500
    assert L(encode_fixed(-2.0, 3, 32)) == 2**32 - 2000


def test_encode_overflow_rejected():                             # test_sharing.py:20-23
    with pytest.raises(FixedPointOverflow):
        encode_fixed(1e7, 3, 32)
    encode_fixed(1e7, 3, 32, allow_wrap=True)


@given(st.lists(st.floats(-100, 100), min_size=1, max_size=20))
@settings(max_examples=200, deadline=None)
def test_fixed_point_roundtrip(vals):                            # test_sharing.py:26-31
    back = decode_fixed(encode_fixed(vals, 3, 32), 3)
    assert np.all(np.abs(back - np.asarray(vals)) <= 1e-3)


def test_share_reconstruct_roundtrip():                          # test_sharing.py:34-38
    rng = np.random.default_rng(0)
    secret = RingTensor.random((4, 7), 32, rng)
    s0, s1 = share(secret, rng)
    assert reconstruct(s0, s1) == secret


def test_share_of_zero_is_negation_pair():                       # test_sharing.py:41-44
    s0, s1 = share(RingTensor.zeros((10,), 16), np.random.default_rng(1))
    assert np.array_equal(s0.values.numpy(), (-s1.values).numpy())


def test_share_uniformity_smoke():                               # test_sharing.py:47-53
    rng = np.random.default_rng(2)
    big0, _ = share(RingTensor(np.full(10_000, 42, dtype=np.uint64), 32), rng)
    raw = sharing.pack_ring(big0.values.data, 32).cpu().view(torch.uint8).numpy()
    assert stats.chisquare(np.bincount(raw, minlength=256)).pvalue > 1e-3


def test_reconstruction_linearity():                             # test_sharing.py:56-62
    rng = np.random.default_rng(3)
    a = RingTensor.random((50,), 32, rng)
    b = RingTensor.random((50,), 32, rng)
    a0, a1 = share(a, rng)
    b0, b1 = share(b, rng)
    assert reconstruct(a0 + b0, a1 + b1) == a + b


def test_reconstruct_rejects_metadata_mismatch():                # test_sharing.py:65-70
    s0, s1 = share(RingTensor.zeros((3,), 16), np.random.default_rng(4))
    s1.precision = 5
    with pytest.raises(ValueError):
        reconstruct(s0, s1)


def test_add_public_and_mul_public():                            # test_sharing.py:73-86
    rng = np.random.default_rng(5)
    s0, s1 = share(encode_fixed([1.0, -2.0], 3, 32), rng, precision=3)
    const = encode_fixed([0.5, 0.5], 3, 32)
    r = reconstruct(s0.add_public(const), s1.add_public(const))
    assert np.allclose(decode_fixed(r, 3), [1.5, -1.5])
    r2 = reconstruct(s0.mul_public_int(3), s1.mul_public_int(3))
    assert np.allclose(decode_fixed(r2, 3), [3.0, -6.0])
    f0, f1 = s0.mul_public_fixed(0.5), s1.mul_public_fixed(0.5)
    assert f0.precision == 6
    assert np.allclose(decode_fixed(reconstruct(truncate(f0, 3), truncate(f1, 3)), 3), [0.5, -1.0],
                       atol=2e-3)


def _reveal_with_alpha(y_vals, alpha_vals, n):                   # test_sharing.py:93-104
    rng = np.random.default_rng(6)
    ys = share(RingTensor.from_ints(y_vals, n), rng)
    a0, a1 = share(RingTensor.from_ints(alpha_vals, n), rng)
    alpha_shares = {0: a0.values.data, 1: a1.values.data}

    def program(session):
        return mask_and_reveal(session, ys[session.party], alpha_shares[session.party], op="comparison")

    (x0, l0), (x1, _) = run_local_pair(program)
    assert x0 == x1
    return x0, l0


def test_mask_and_reveal_examples():                             # test_sharing.py:107-112
    x, ledger = _reveal_with_alpha([5], [10], 8)
    assert L(x) == [15]
    assert ledger.rounds == {"comparison": 1}
    x, _ = _reveal_with_alpha([250], [10], 8)
    assert L(x) == [4]


def test_masked_value_uniform_over_fresh_masks():                # test_sharing.py:115-123
    rng = np.random.default_rng(7)
    trials = 20_000
    y = np.full(trials, 77, dtype=np.uint64)
    alpha = rng.integers(0, 256, trials, dtype=np.uint64)
    x = (y + alpha) & ring_mask(8)
    assert stats.chisquare(np.bincount(x.astype(np.int64), minlength=256)).pvalue > 1e-3


def test_truncate_example():                                     # test_sharing.py:130-134
    s0, s1 = share(RingTensor.from_ints([3_000_000], 32), np.random.default_rng(8), precision=6)
    r = reconstruct(truncate(s0, 3), truncate(s1, 3))
    assert abs(int(r.signed()[0]) - 3000) <= 1


def test_truncate_zero_digits_is_identity():                     # test_sharing.py:137-141
    s0, s1 = share(RingTensor.from_ints([1234], 32), np.random.default_rng(9), precision=3)
    t0 = truncate(s0, 0)
    assert t0.precision == 3 and np.array_equal(t0.values.numpy(), s0.values.numpy())


def test_truncate_monte_carlo_error_bound():                     # test_sharing.py:144-156
    rng = np.random.default_rng(10)
    trials = 100_000
    vals = rng.uniform(-1e4, 1e4, trials)
    s0, s1 = share(encode_fixed(vals, 6, 48), rng, precision=6)
    out = reconstruct(truncate(s0, 3), truncate(s1, 3))
    ok = np.abs(decode_fixed(out, 3) - vals) <= 2e-3
    assert np.mean(ok) >= 0.999 and np.mean(~ok) <= 0.001


def test_truncate_wrap_rate_tracks_magnitude_over_ring():        # test_sharing.py:159-169
    rng = np.random.default_rng(13)
    trials = 200_000
    vals = np.full(trials, 2000.0)
    s0, s1 = share(encode_fixed(vals, 6, 32), rng, precision=6)
    out = reconstruct(truncate(s0, 3), truncate(s1, 3))
    wraps = np.abs(decode_fixed(out, 3) - vals) > 1.0
    expected = 2000.0 * 1e6 / 2**32
    sigma = np.sqrt(trials * expected * (1 - expected))
    assert abs(wraps.sum() - trials * expected) <= 4 * sigma + 5


def test_truncate_rejects_over_truncation():                     # test_sharing.py:172-176
    s0, _ = share(RingTensor.from_ints([10], 32), np.random.default_rng(11), precision=2)
    with pytest.raises(ValueError):
        truncate(s0, 3)


def test_guard_blocks_and_allows():                              # test_sharing.py:183-191
    s0, s1 = share(RingTensor.zeros((2,), 16), np.random.default_rng(12))
    with forbid_reconstruction("unit test"):
        with pytest.raises(ReconstructionForbidden):
            reconstruct(s0, s1)
        with allow_reconstruction():
            reconstruct(s0, s1)
    reconstruct(s0, s1)


# ------------------------------------------------------------ test_beaver.py (elementwise)

def _run_protocol(xs, ys, triples, proto):                       # test_beaver.py:16-20
    def program(session):
        return proto(session, xs[session.party], ys[session.party], triples[session.party])
    return run_local_pair(program)


def test_triple_reconstructs_to_product():                       # test_beaver.py:23-29
    t0, t1 = gen_triple("mul", ElemwiseGeometry((4,)), 32, np.random.default_rng(0))
    assert (t0.c + t1.c) == (t0.a + t1.a) * (t0.b + t1.b)


def test_mul_protocol_examples():                                # test_beaver.py:50-59
    rng = np.random.default_rng(3)
    for x_val, y_val, want in [(5, 6, 30), (0, 9, 0)]:
        xs = share(RingTensor.from_ints([x_val], 32), rng)
        ys = share(RingTensor.from_ints([y_val], 32), rng)
        triples = gen_triple("mul", ElemwiseGeometry((1,)), 32, rng)
        (r0, l0), (r1, _) = _run_protocol(xs, ys, triples, beaver.mul_protocol)
        assert L(reconstruct(r0, r1))[0] == want
        assert l0.rounds == {"mul": 1}


def test_mul_protocol_fixed_point():                             # test_beaver.py:62-74
    rng = np.random.default_rng(4)
    xs = share(encode_fixed([1.5], 3, 32), rng, precision=3)
    ys = share(encode_fixed([2.0], 3, 32), rng, precision=3)
    triples = gen_triple("mul", ElemwiseGeometry((1,)), 32, rng)

    def program(session):
        return truncate(beaver.mul_protocol(session, xs[session.party], ys[session.party],
                                            triples[session.party]), 3)

    (r0, _), (r1, _) = run_local_pair(program)
    assert abs(decode_pair(r0, r1)[0] - 3.0) <= 2e-3


def test_unroll_example_and_edge():                              # test_beaver.py:184-195
    x = RingTensor.from_ints(np.arange(16, dtype=np.int64).reshape(4, 4), 32)
    u = unroll(x, 2, 2)
    assert u.shape == (4, 4)
    assert L(u)[0] == [0, 1, 4, 5] and L(u)[3] == [10, 11, 14, 15]
    whole = unroll(x, 4, 1)
    assert whole.shape == (1, 16) and L(whole)[0] == list(range(16))
    with pytest.raises(ValueError):
        unroll(x, 5, 1)


def test_triple_reuse_rejected():                                # test_beaver.py:213-226
    rng = np.random.default_rng(12)
    xs = share(RingTensor.from_ints([1], 32), rng)
    ys = share(RingTensor.from_ints([2], 32), rng)
    triples = gen_triple("mul", ElemwiseGeometry((1,)), 32, rng)

    def program(session):
        beaver.mul_protocol(session, xs[session.party], ys[session.party], triples[session.party])
        return beaver.mul_protocol(session, xs[session.party], ys[session.party], triples[session.party])

    with pytest.raises(TripleReuseError):
        run_local_pair(program)


def test_shape_mismatch_rejected():                              # test_beaver.py:229-240
    rng = np.random.default_rng(13)
    xs = share(RingTensor.from_ints([1, 2], 32), rng)
    ys = share(RingTensor.from_ints([2, 3], 32), rng)
    triples = gen_triple("mul", ElemwiseGeometry((3,)), 32, rng)
    with pytest.raises(ValueError, match="geometry"):
        _run_protocol(xs, ys, triples, beaver.mul_protocol)


def test_revealed_deltas_look_uniform():                         # test_beaver.py:243-250
    rng = np.random.default_rng(14)
    trials = 20_000
    x = RingTensor.from_ints(np.full(trials, 1234, dtype=np.int64), 32)
    t0, t1 = gen_triple("mul", ElemwiseGeometry((trials,)), 32, rng)
    delta = (x - (t0.a + t1.a)).numpy()
    raw = np.frombuffer(delta.astype("<u4").tobytes(), dtype=np.uint8)
    assert stats.chisquare(np.bincount(raw, minlength=256)).pvalue > 1e-3


def test_triple_container_roundtrip():                           # test_beaver.py:253-262 (elementwise geometry)
    t0, t1 = gen_triple("mul", ElemwiseGeometry((3, 5)), 32, np.random.default_rng(15))
    batch = fss.deserialize_keys(fss.serialize_keys(beaver.pack_triples(t0, t1)))
    assert batch.kind == fss.KIND_TRIPLE
    r0, r1 = beaver.unpack_triples(batch)
    assert r0.op_tag == "mul" and r0.geometry == ElemwiseGeometry((3, 5))
    assert (r0.a + r1.a) == (t0.a + t1.a) and (r0.c + r1.c) == (t0.c + t1.c)


# ------------------------------------------------------------ test_nn_ops.py (FSS layers)

N_BITS, P = 32, 3


def _run(program, n=N_BITS):                                     # test_nn_ops.py:13-19
    d = dealer.make_dealer(n, seed=101)
    return run_local_pair(lambda session: program(session, d.for_party(session.party)))


def _shared(values, rng, precision=P, n=N_BITS):                 # test_nn_ops.py:22-23
    return share(encode_fixed(values, precision, n), rng, precision=precision)


def test_relu_examples_and_rounds():                             # test_nn_ops.py:26-36
    xs = _shared([-2.0, 0.0, 3.0], np.random.default_rng(0))
    (r0, l0), (r1, _) = _run(lambda s, prep: nn_ops.relu(s, xs[s.party], prep.relu(3)))
    assert np.allclose(decode_pair(r0, r1), [0.0, 0.0, 3.0])
    assert l0.total_rounds() == 2 and l0.rounds == {"comparison": 1, "mul": 1}


def test_relu_all_negative_is_zero():                            # test_nn_ops.py:39-47
    xs = _shared([-5.0, -0.001, -99.9], np.random.default_rng(1))
    (r0, _), (r1, _) = _run(lambda s, prep: nn_ops.relu(s, xs[s.party], prep.relu(3)))
    assert np.allclose(decode_pair(r0, r1), 0.0)


def test_relu_matches_plaintext_in_bulk():                       # test_nn_ops.py:50-61
    rng = np.random.default_rng(2)
    vals = rng.uniform(-100, 100, 10_000)
    xs = _shared(vals, rng)
    (r0, _), (r1, _) = _run(lambda s, prep: nn_ops.relu(s, xs[s.party], prep.relu(vals.size)))
    assert np.allclose(decode_pair(r0, r1), np.maximum(np.floor(vals * 1000) / 1000, 0.0), atol=1e-9)


def test_relu_plus_negated_relu_is_abs():                        # test_nn_ops.py:64-78
    rng = np.random.default_rng(3)
    vals = rng.uniform(-50, 50, 200)
    vals[np.abs(vals) < 0.01] = 1.0
    xs = _shared(vals, rng)

    def program(session, prep):
        x = xs[session.party]
        return nn_ops.relu(session, x, prep.relu(vals.size)) + nn_ops.relu(session, -x, prep.relu(vals.size))

    (r0, _), (r1, _) = _run(program)
    assert np.allclose(decode_pair(r0, r1), np.abs(np.floor(vals * 1000) / 1000), atol=1e-9)


def test_argmax_basic_tie_and_rounds():                          # test_nn_ops.py:81-99
    rng = np.random.default_rng(4)
    xs = _shared([1.0, 3.0, 2.0], rng)
    (r0, l0), (r1, _) = _run(lambda s, prep: nn_ops.argmax(s, xs[s.party], prep.argmax(1, 3)))
    assert L(reconstruct(r0, r1)) == [0, 1, 0]
    assert l0.total_rounds() == 2 and l0.rounds == {"comparison": 1, "equality": 1}
    ties = _shared([5.0, 5.0, 1.0], rng)
    (r0, _), (r1, _) = _run(lambda s, prep: nn_ops.argmax(s, ties[s.party], prep.argmax(1, 3)))
    assert L(reconstruct(r0, r1)) == [1, 1, 0]


def test_argmax_output_sum_equals_max_multiplicity():            # test_nn_ops.py:102-114
    rows = np.array([[1.0, 4.0, 4.0, 0.0], [7.0, 7.0, 7.0, 7.0], [0.0, 1.0, 2.0, 3.0]])
    xs = _shared(rows, np.random.default_rng(5))
    (r0, _), (r1, _) = _run(lambda s, prep: nn_ops.argmax(s, xs[s.party], prep.argmax(3, 4)))
    assert reconstruct(r0, r1).numpy().astype(np.int64).sum(axis=-1).tolist() == [2, 4, 1]


def test_argmax_bulk_matches_numpy():                            # test_nn_ops.py:117-134
    rng = np.random.default_rng(6)
    rows = rng.uniform(-10, 10, (1000, 10))
    q = np.sort(np.floor(rows * 1000), axis=-1)
    rows = rows[(q[:, -1] - q[:, -2]) >= 1]
    m = rows.shape[0]
    xs = _shared(rows, rng, n=40)
    (r0, _), (r1, _) = _run(lambda s, prep: nn_ops.argmax(s, xs[s.party], prep.argmax(m, 10)), n=40)
    onehot = reconstruct(r0, r1).numpy().astype(np.int64)
    assert np.array_equal(np.argmax(onehot, axis=-1), np.argmax(rows, axis=-1))
    assert np.all(onehot.sum(axis=-1) == 1)


def test_maxpool_example_constant_and_rounds():                  # test_nn_ops.py:181-198
    rng = np.random.default_rng(11)
    xs = _shared([[1.0, 2.0], [3.0, 4.0]], rng)
    (r0, l0), (r1, _) = _run(lambda s, prep: nn_ops.maxpool(s, xs[s.party], 2, prep.maxpool(2, 2)))
    assert np.allclose(decode_pair(r0, r1), [[4.0]])
    assert l0.total_rounds() == 3
    const = _shared(np.full((4, 4), 2.5), rng)
    (r0, _), (r1, _) = _run(lambda s, prep: nn_ops.maxpool(s, const[s.party], 2, prep.maxpool(4, 2)))
    assert np.allclose(decode_pair(r0, r1), 2.5 - 1e-3, atol=2e-3)


def test_maxpool_random_matches_plaintext():                     # test_nn_ops.py:201-214
    rng = np.random.default_rng(12)
    for trial in range(20):
        vals = rng.uniform(-10, 10, (8, 8))
        xs = _shared(vals, rng)
        (r0, _), (r1, _) = _run(lambda s, prep: nn_ops.maxpool(s, xs[s.party], 2, prep.maxpool(8, 2)))
        want = np.floor(vals * 1000).reshape(4, 2, 4, 2).transpose(0, 2, 1, 3)
        want = want.reshape(4, 4, 4).max(axis=-1) / 1000
        assert np.allclose(decode_pair(r0, r1), want, atol=1e-9), trial


def test_maxpool_k2_matches_and_uses_four_rounds():              # test_nn_ops.py:217-234
    rng = np.random.default_rng(13)
    xs = _shared(rng.uniform(-10, 10, (6, 6)), rng)
    (t0, lt), (t1, _) = _run(lambda s, prep: nn_ops.maxpool_k2(s, xs[s.party], prep.maxpool_k2(6)))
    (a0, la), (a1, _) = _run(lambda s, prep: nn_ops.maxpool(s, xs[s.party], 2, prep.maxpool(6, 2)))
    assert np.allclose(decode_pair(t0, t1), decode_pair(a0, a1))
    assert lt.total_rounds() == 4 and la.total_rounds() == 3
    assert la.elements["comparison"] / lt.elements["comparison"] == 4.0


def test_prep_plans_match_published_formulas():                  # test_nn_ops.py:312-319 (FSS layers)
    assert nn_ops.relu_plan(100) == [("cmp", 100), ("triple", "mul", ElemwiseGeometry((100,)))]
    assert nn_ops.argmax_plan(1, 10)[0] == ("cmp", 90)
    assert nn_ops.argmax_plan(1, 10)[1] == ("eq", 10)
    plan = nn_ops.maxpool_plan(8, 2)
    assert plan[0] == ("cmp", 16 * 4 * 3) and plan[1] == ("eq", 16 * 4)


# ------------------------------------------------------------ test_dealer.py

def test_relu_plan_yields_published_counts():                   # test_dealer.py:8-14
    b0, b1, _ = dealer.preprocess(nn_ops.relu_plan(100), 32, np.random.default_rng(0))
    assert isinstance(b0.items[0], fss.CmpKeyBatch) and b0.items[0].count == 100
    assert isinstance(b0.items[1], beaver.BeaverTriple)
    assert b0.items[1].geometry == ElemwiseGeometry((100,))
    assert b1.items[0].count == 100


def test_same_plan_same_seed_identical_bundles():                # test_dealer.py:17-24
    plan = nn_ops.relu_plan(10) + nn_ops.argmax_plan(1, 4)
    a0, a1, _ = dealer.preprocess(plan, 16, np.random.default_rng(7))
    b0, b1, _ = dealer.preprocess(plan, 16, np.random.default_rng(7))
    assert fss.serialize_keys(fss.pack_keys(a0.items[0], a1.items[0])) == \
        fss.serialize_keys(fss.pack_keys(b0.items[0], b1.items[0]))
    assert np.array_equal(a0.items[1].a.numpy(), b0.items[1].a.numpy())


def test_preprocess_keeps_audit_tapes_on_request():              # test_dealer.py:46-52
    b0, b1, tapes = dealer.preprocess([("cmp", 5), ("eq", 3)], 16, np.random.default_rng(2),
                                      keep_tapes=True)
    assert len(tapes) == 2
    assert fss.audit_keys(b0.items[0], b1.items[0], tapes[0], range(5)) == []
    assert fss.audit_keys(b0.items[1], b1.items[1], tapes[1], range(3)) == []


def test_plan_is_data_independent():                             # test_dealer.py:55-61
    b0, b1, _ = dealer.preprocess(nn_ops.relu_plan(4), 32, np.random.default_rng(3))
    rec = (b0.items[0].alpha_share.view(torch.int64) + b1.items[0].alpha_share.view(torch.int64)) \
        & int(ring_mask(32))
    assert tuple(rec.shape) == (4,)


def test_streaming_dealer_detects_desync():                      # test_dealer.py:64-69
    d = dealer.make_dealer(16, seed=4)
    p0, p1 = d.for_party(0), d.for_party(1)
    p0.cmp_keys(3)
    with pytest.raises(RuntimeError, match="desync"):
        p1.eq_keys(3)


def test_streaming_dealer_frees_delivered_slots():               # test_dealer.py:72-78
    d = dealer.make_dealer(16, seed=5)
    p0, p1 = d.for_party(0), d.for_party(1)
    for _ in range(4):
        p0.cmp_keys(2)
        p1.cmp_keys(2)
    assert d._made == {}
