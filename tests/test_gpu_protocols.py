"""GPU parity of the online protocols (sign / eq / ReLU / argmax / MaxPool,
batched MaxPool and the two full-size BASELINE configs) against fixtures the
unmodified reference produced (tests/golden/make_protocol_golden.py).

Inputs are regenerated here from the recorded numpy seeds with the drop-in's
own encode_fixed / share / dealer, the protocol runs on cuda:0 through the
in-process two-party runtime, and the output shares of BOTH parties must be
bit-identical to the reference's (array compare for small cases, sha256 of the
full share arrays for the big ones), with the same round and byte ledger.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2006_04593_b200 import dealer, fss, nn_ops, runtime  # noqa: E402
from paper_2006_04593_b200.ring import RingTensor  # noqa: E402
from paper_2006_04593_b200.sharing import (AdditiveShare, encode_fixed, reconstruct,  # noqa: E402
                                           share)

with open(os.path.join(GOLDEN, "protocols.json")) as fh:
    CASES = json.load(fh)["cases"]


def digest(*tensors) -> str:
    h = hashlib.sha256()
    for t in tensors:
        h.update(np.ascontiguousarray(t.detach().cpu().numpy().astype("<u8")).tobytes())
    return h.hexdigest()


def _inputs(c):
    rng = np.random.default_rng(c["seed"])
    if c["kind"] == "eq":
        vals = rng.integers(c["lo"], c["hi"], c["shape"][0])
        enc = RingTensor.from_ints(vals, c["n"])
        return share(enc, rng, precision=0)
    x = rng.uniform(c["lo"], c["hi"], tuple(c["shape"]))
    return share(encode_fixed(x, c["p"], c["n"]), rng, precision=c["p"])


def _program(c, xs):
    d = dealer.make_dealer(c["n"], seed=c["dealer_seed"])
    kind = c["kind"]
    shape = tuple(c["shape"])

    if kind == "compare":
        def prog(session):
            keys = d.for_party(session.party, cmp_bits=c["cmp_bits"]).cmp_keys(shape[0])
            return fss.sign_protocol(session, AdditiveShare(session.party, xs[session.party].values, 0),
                                     keys)
    elif kind == "eq":
        def prog(session):
            return fss.eq_protocol(session, xs[session.party],
                                   d.for_party(session.party).eq_keys(shape[0]))
    elif kind == "relu":
        def prog(session):
            return nn_ops.relu(session, xs[session.party],
                               d.for_party(session.party).relu_shaped(shape))
    elif kind == "argmax":
        def prog(session):
            return nn_ops.argmax(session, xs[session.party],
                                 d.for_party(session.party).argmax(shape[0], shape[1]))
    elif kind in ("maxpool", "maxpool_batched"):
        k, stride = c["k"], c["stride"]
        planes = 1 if kind == "maxpool" else int(np.prod(shape[:-2]))
        side = shape[-1]

        def prog(session):
            view = d.for_party(session.party)
            x = xs[session.party]
            if kind == "maxpool_batched":
                x = x.reshape(planes, side, side)
            if c["route"] == "argmax":
                return nn_ops.maxpool(session, x, k, view.maxpool(side, k, stride, planes=planes),
                                      stride)
            return nn_ops.maxpool_k2(session, x, view.maxpool_k2(side, planes=planes))
    else:
        raise AssertionError(kind)
    return prog


@pytest.mark.parametrize("name", sorted(CASES))
def test_protocol_matches_reference(name):
    c = CASES[name]
    xs = _inputs(c)
    assert digest(xs[0].values.data, xs[1].values.data) == c["in_digest"]
    (r0, l0), (r1, l1) = runtime.run_local_pair(_program(c, xs))
    torch.cuda.synchronize()
    assert list(r0.values.shape) == c["out_shape"]
    assert r0.precision == c["out_precision"] and r0.values.n_bits == c["out_bits"]
    assert l0.total_rounds() == c["rounds"] and l1.total_rounds() == c["rounds"]
    assert l0.total_bytes_sent() == c["bytes_sent"]
    assert l0.snapshot() == c["rounds_by_op"]
    path = os.path.join(GOLDEN, f"proto_{name}.npz")
    if os.path.exists(path):
        with np.load(path) as g:
            assert np.array_equal(r0.values.numpy().reshape(g["out0"].shape), g["out0"])
            assert np.array_equal(r1.values.numpy().reshape(g["out1"].shape), g["out1"])
    assert digest(r0.values.data, r1.values.data) == c["out_digest"]


def test_relu_values_and_sign_failure_law():
    # plaintext check of ReLU on a larger batch: exact except the rare sign-wrap
    # failures (probability |y| / 2^32 per element, nn_ops.py:83-94)
    rng = np.random.default_rng(99)
    x = rng.uniform(-100, 100, (1 << 16,))
    xs = share(encode_fixed(x, 3, 32), rng, precision=3)
    d = dealer.make_dealer(32, seed=100)

    def prog(session):
        return nn_ops.relu(session, xs[session.party], d.for_party(session.party).relu(1 << 16))
    (r0, _), (r1, _) = runtime.run_local_pair(prog)
    got = reconstruct(r0, r1).signed().cpu().numpy() / 1e3
    want = np.maximum(np.floor(x * 1e3) / 1e3, 0)
    bad = np.abs(got - want) > 1e-6
    assert bad.sum() <= 2


def test_single_use_keys_and_desync():
    d = dealer.make_dealer(32, seed=5)
    rng = np.random.default_rng(6)
    xs = share(encode_fixed(rng.uniform(-1, 1, 8), 3, 32), rng, precision=3)

    def prog(session):
        keys = d.for_party(session.party).cmp_keys(8)
        me = AdditiveShare(session.party, xs[session.party].values, 0)
        fss.sign_protocol(session, me, keys)
        return fss.sign_protocol(session, me, keys)   # keys are spent
    with pytest.raises(fss.KeyExhaustedError):
        runtime.run_local_pair(prog)


def test_dealer_material_survives_cross_stream_release():
    """Material generated on party 0's stream and consumed on party 1's must not
    be recycled by party 0's allocator pool while party 1's kernels still read
    it: the dealer marks every tensor as used on the consumer stream."""
    M = 1 << 20
    d = dealer.make_dealer(32, seed=9)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s0):
        k0 = d.for_party(0).cmp_keys(M)
    x = torch.from_numpy(np.random.default_rng(1).integers(0, 1 << 32, M, dtype=np.uint64)
                         .view(np.int64)).cuda().view(torch.uint64)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        k1 = d.for_party(1).cmp_keys(M)
        want = fss.eval_cmp(1, k1, x).clone()
        s1.synchronize()
        outs = [fss.eval_cmp(1, k1, x) for _ in range(30)]    # ~tens of ms of reads queued
    del k0, k1
    with torch.cuda.stream(s0):                               # reuse party 0's pool at once
        junk = [torch.full((32, M, 16), 0xFF, dtype=torch.uint8, device="cuda") for _ in range(2)]
        junk += [torch.full((33, M), -1, dtype=torch.int64, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o.view(torch.int64), want.view(torch.int64))
    del junk
