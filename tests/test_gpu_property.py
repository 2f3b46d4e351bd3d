"""Randomised parity (hypothesis): for random ring widths, output widths,
batch sizes, parties, generator states (incl. numpy's buffered half-word) and
inputs, the B200 keygen and evaluation equal the C oracle's restatement of
the reference byte for byte -- keys, rng advance, shares, per-level terms."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402

from paper_2006_04593_b200 import fss  # noqa: E402

# FSS_HYPOTHESIS_EXAMPLES raises the example count for a long soak run
SETTINGS = dict(max_examples=int(os.environ.get("FSS_HYPOTHESIS_EXAMPLES", "60")), deadline=None,
                suppress_health_check=[HealthCheck.function_scoped_fixture])


def _rng(seed, pre):
    rng = np.random.default_rng(seed)
    if pre:
        rng.integers(0, 1 << 20, size=pre, dtype=np.uint64)   # odd pre-draws leave a buffered half-word
    return rng


@settings(**SETTINGS)
@given(n=st.integers(4, 63), extra=st.integers(0, 20), count=st.integers(1, 300),
       seed=st.integers(0, 2**32 - 1), pre=st.integers(0, 3), hits=st.floats(0, 1))
def test_dcf_random_parity(oracle, n, extra, count, seed, pre, hits):
    out_bits = min(63, n + extra)
    r_gpu, r_ref = _rng(seed, pre), _rng(seed, pre)
    alpha, k0, k1 = fss.keygen_cmp(n, r_gpu, count, out_bits=out_bits)
    a, a0, s0, s1 = oracle.sample_tape(n, r_ref, count)
    assert r_gpu.bit_generator.state == r_ref.bit_generator.state
    assert np.array_equal(alpha.cpu().numpy(), a)
    c0, c1 = oracle.keygen_cmp_core(n, a, a0, s0, s1, out_bits)
    assert np.array_equal(k0.scw.cpu().numpy(), c0["scw"]) and np.array_equal(k0.tcw.cpu().numpy(), c0["tcw"])
    assert np.array_equal(k0.sigma_cw.cpu().view(torch.int64).numpy().view(np.uint64), c0["sigma_cw"])
    assert np.array_equal(k0.leaf_cw.cpu().view(torch.int64).numpy().view(np.uint64), c0["leaf_cw"])
    xr = np.random.default_rng(seed ^ 0x5A5A)
    x = xr.integers(0, 1 << n, count, dtype=np.uint64)
    hit = xr.random(count) < hits
    x[hit] = a[hit]
    for party, (kg, kr) in enumerate(((k0, c0), (k1, c1))):
        y, lv = fss.eval_cmp(party, kg, x, return_levels=True)
        yr, lvr = oracle.eval_cmp(party, kr, x, return_levels=True)
        assert np.array_equal(y, yr) and np.array_equal(lv, lvr)
        # the hot instantiation (no per-level output) too
        assert np.array_equal(fss.eval_cmp(party, kg, x), yr)


# Batches large enough that the eval launch runs 1,024-thread CTAs with several
# strided passes per CTA (>= 148 x 1,024 elements) and ragged final passes.
@settings(**dict(SETTINGS, max_examples=int(os.environ.get("FSS_HYPOTHESIS_LARGE", "8"))))
@given(n=st.integers(4, 63), extra=st.integers(0, 12), count=st.integers(1 << 16, 1 << 18),
       seed=st.integers(0, 2**32 - 1), pre=st.integers(0, 3), hits=st.floats(0, 1),
       device_x=st.booleans())
def test_dcf_large_batch_random_parity(oracle, n, extra, count, seed, pre, hits, device_x):
    out_bits = min(63, n + extra)
    r_gpu, r_ref = _rng(seed, pre), _rng(seed, pre)
    alpha, k0, k1 = fss.keygen_cmp(n, r_gpu, count, out_bits=out_bits)
    a, a0, s0, s1 = oracle.sample_tape(n, r_ref, count)
    assert r_gpu.bit_generator.state == r_ref.bit_generator.state
    c0, c1 = oracle.keygen_cmp_core(n, a, a0, s0, s1, out_bits)
    assert np.array_equal(k0.scw.cpu().numpy(), c0["scw"])
    assert np.array_equal(k0.leaf_cw.cpu().view(torch.int64).numpy().view(np.uint64), c0["leaf_cw"])
    xr = np.random.default_rng(seed ^ 0x3C3C)
    x = xr.integers(0, 1 << n, count, dtype=np.uint64)
    hit = xr.random(count) < hits
    x[hit] = a[hit]
    xin = torch.from_numpy(x.view(np.int64)).cuda().view(torch.uint64) if device_x else x
    for party, (kg, kr) in enumerate(((k0, c0), (k1, c1))):
        y = fss.eval_cmp(party, kg, xin)
        y = y.view(torch.int64).cpu().numpy().view(np.uint64) if device_x else y
        assert np.array_equal(y, oracle.eval_cmp(party, kr, x))


@settings(**dict(SETTINGS, max_examples=int(os.environ.get("FSS_HYPOTHESIS_LARGE", "8"))))
@given(n=st.integers(4, 64), count=st.integers(1 << 16, 1 << 18), seed=st.integers(0, 2**32 - 1),
       hits=st.floats(0, 1))
def test_dpf_large_batch_random_parity(oracle, n, count, seed, hits):
    r_gpu, r_ref = _rng(seed, 0), _rng(seed, 0)
    alpha, k0, k1 = fss.keygen_eq(n, r_gpu, count)
    a, a0, s0, s1 = oracle.sample_tape(n, r_ref, count)
    c0, c1 = oracle.keygen_eq_core(n, a, a0, s0, s1)
    xr = np.random.default_rng(seed ^ 0xC3C3)
    x = xr.integers(0, 1 << min(n, 63), count, dtype=np.uint64)
    hit = xr.random(count) < hits
    x[hit] = a[hit]
    for party, (kg, kr) in enumerate(((k0, c0), (k1, c1))):
        assert np.array_equal(fss.eval_eq(party, kg, x), oracle.eval_eq(party, kr, x))


@settings(**SETTINGS)
@given(n=st.integers(4, 64), count=st.integers(1, 300), seed=st.integers(0, 2**32 - 1),
       pre=st.integers(0, 3), hits=st.floats(0, 1))
def test_dpf_random_parity(oracle, n, count, seed, pre, hits):
    r_gpu, r_ref = _rng(seed, pre), _rng(seed, pre)
    alpha, k0, k1 = fss.keygen_eq(n, r_gpu, count)
    a, a0, s0, s1 = oracle.sample_tape(n, r_ref, count)
    assert r_gpu.bit_generator.state == r_ref.bit_generator.state
    c0, c1 = oracle.keygen_eq_core(n, a, a0, s0, s1)
    assert np.array_equal(k0.scw.cpu().numpy(), c0["scw"])
    xr = np.random.default_rng(seed ^ 0xA5A5)
    x = xr.integers(0, 1 << min(n, 63), count, dtype=np.uint64)
    if n == 64:
        x = (x << np.uint64(1)) | xr.integers(0, 2, count, dtype=np.uint64)
    hit = xr.random(count) < hits
    x[hit] = a[hit]
    for party, (kg, kr) in enumerate(((k0, c0), (k1, c1))):
        assert np.array_equal(fss.eval_eq(party, kg, x), oracle.eval_eq(party, kr, x))
