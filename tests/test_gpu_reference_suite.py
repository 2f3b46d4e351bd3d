"""The reference's own FSS test cases (pkg/tests/test_fss.py, test_acceptance.py)
restated against the drop-in on the GPU: DCF examples, the at-most-one-level
property, determinism, widened outputs, the sign-failure law (c02), key sizes
(c03) and the single-key byte-uniformity view."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2006_04593_b200 import fss  # noqa: E402
from paper_2006_04593_b200.ring import ring_mask  # noqa: E402


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _rec(a, b, n):
    return (np.asarray(a) + np.asarray(b)) & ring_mask(n)


def test_cmp_examples_n8():                         # test_fss.py:53-59
    rng = np.random.default_rng(2)
    _, k0, k1 = fss.keygen_cmp(8, rng, alpha=np.array([7], dtype=np.uint64))
    for x, want in [(3, 1), (200, 0), (7, 1), (0, 1)]:
        assert _rec(fss.eval_cmp(0, k0, x), fss.eval_cmp(1, k1, x), 8)[0] == want


def test_eq_hit_and_miss():                         # test_fss.py:15-33
    rng = np.random.default_rng(1)
    alpha, k0, k1 = fss.keygen_eq(16, rng, count=100)
    a = _np(alpha)
    assert np.all(_rec(fss.eval_eq(0, k0, a), fss.eval_eq(1, k1, a), 16) == 1)
    miss = (a + np.uint64(1)) & ring_mask(16)
    assert np.all(_rec(fss.eval_eq(0, k0, miss), fss.eval_eq(1, k1, miss), 16) == 0)


def test_cmp_at_most_one_level_fires():             # test_fss.py:62-71
    for n, count in ((8, 64), (32, 4096)):
        rng = np.random.default_rng(3)
        _, k0, k1 = fss.keygen_cmp(n, rng, count=count)
        xs = np.random.default_rng(4).integers(0, 1 << n, count, dtype=np.uint64)
        _, lv0 = fss.eval_cmp(0, k0, xs, return_levels=True)
        _, lv1 = fss.eval_cmp(1, k1, xs, return_levels=True)
        per_level = (lv0 + lv1) & ring_mask(n)
        assert per_level.shape == (n + 1, count)
        assert np.all((per_level == 0) | (per_level == 1))
        assert np.all(per_level.sum(axis=0) <= 1)


def test_keygen_deterministic_given_rng_state():    # test_fss.py:86-90
    a = fss.keygen_cmp(16, np.random.default_rng(42), count=4)
    b = fss.keygen_cmp(16, np.random.default_rng(42), count=4)
    assert fss.serialize_keys(fss.pack_keys(a[1], a[2])) == \
        fss.serialize_keys(fss.pack_keys(b[1], b[2]))


def test_wide_output_narrow_domain_keys():          # test_fss.py:93-101
    rng = np.random.default_rng(5)
    alpha, k0, k1 = fss.keygen_cmp(12, rng, count=256, out_bits=32)
    xs = rng.integers(0, 1 << 12, 256, dtype=np.uint64)
    rec = _rec(fss.eval_cmp(0, k0, xs), fss.eval_cmp(1, k1, xs), 32)
    assert np.array_equal(rec, (xs <= _np(alpha)).astype(np.uint64))
    with pytest.raises(fss.KeyFormatError):
        fss.pack_keys(k0, k1)


@pytest.mark.parametrize("y", [16, -16, 256, -256, 1024, -1024])
def test_c02_sign_failure_rate(y):                  # test_acceptance.py:58-78
    n, trials = 16, 100_000
    rng = np.random.default_rng(2000 + y)
    alpha, k0, k1 = fss.keygen_cmp(n, rng, count=trials)
    x = (_np(alpha) + np.uint64(y & 0xFFFF)) & ring_mask(n)
    rec = _rec(fss.eval_cmp(0, k0, x), fss.eval_cmp(1, k1, x), n)
    fails = int(np.sum(rec != np.uint64(1 if y <= 0 else 0)))
    q = abs(y) / 2.0 ** n
    expected, sigma = trials * q, np.sqrt(trials * q * (1 - q))
    assert abs(fails - expected) <= 3 * sigma


def test_c03_key_sizes():                           # test_acceptance.py:85-101
    assert fss.cmp_elem_bytes(32) == 824 <= 885 and fss.eq_elem_bytes(32) == 568
    rng = np.random.default_rng(6)
    _, k0, k1 = fss.keygen_cmp(32, rng, count=10)
    blob = fss.serialize_keys(fss.pack_keys(k0, k1))
    assert len(blob) == 13 + 2 * 10 * 824
    assert fss.cmp_key_bits(32) == 6431


def test_single_key_view_byte_distribution():       # test_fss.py:255-271
    from scipy import stats
    rng = np.random.default_rng(18)
    count = 10_000
    _, k0, _ = fss.keygen_cmp(8, rng, count=count, alpha=np.full(count, 123, dtype=np.uint64))
    pools = [_np(k0.alpha_share).astype(np.uint8), _np(k0.seed0)[:, :15].reshape(-1),
             _np(k0.scw)[:, :, :15].reshape(-1), _np(k0.sigma_cw).astype(np.uint8).reshape(-1),
             _np(k0.leaf_cw).astype(np.uint8).reshape(-1)]
    counts = np.bincount(np.concatenate(pools), minlength=256)
    assert stats.chisquare(counts).pvalue > 1e-3
