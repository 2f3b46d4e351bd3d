"""Share-level parity at the sizes the bench numbers are quoted on.

* 2^24 DCF keys at n = 32 -- the bench's per-GPU workload, dealt exactly as
  ``bench.py`` deals it (``shard.keygen_cmp_shard`` of ``default_rng(1000)``,
  one rank) and evaluated by both parties with the hot launch shape (plain-x
  ``dcf_eval_kernel<W32, no levels>``, 1,024 threads per CTA, many strided
  passes per CTA). A random sample of 2^16 elements is checked against the C
  oracle (restatement of reference fss.py:219-289 / 380-426): every key field
  of both parties and both parties' shares.
* one 2^26 shard (rank 1 of 4) of the 2^28-key batch of the north-star target.
  The tape entries of the sampled elements are recomputed independently with
  numpy's own PCG64 jump-ahead (``PCG64.advance``) at their offsets in the
  2^28-element tape (draw order alpha, alpha0, s0, s1 of fss._sample_tape,
  fss.py:292-303); the recomputation is pinned against ``oracle.sample_tape`` on
  a small tape first.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2006_04593_b200 import fss, shard  # noqa: E402

M32 = 0xFFFFFFFF


def _np64(t):
    return t.detach().view(torch.int64).cpu().numpy().view(np.uint64)


def _np8(t):
    return t.detach().cpu().numpy()


def _check_keys(k0, k1, idx, c0, c1):
    """Device key batches at columns idx == oracle key dicts (already sliced)."""
    ii = torch.as_tensor(idx, device=k0.scw.device)
    assert np.array_equal(_np8(k0.scw.index_select(1, ii)), c0["scw"])
    assert np.array_equal(_np8(k0.tcw.index_select(1, ii)), c0["tcw"])
    assert np.array_equal(_np64(k0.sigma_cw.index_select(1, ii)), c0["sigma_cw"])
    assert np.array_equal(_np64(k0.leaf_cw.index_select(1, ii)), c0["leaf_cw"])
    for k, c in ((k0, c0), (k1, c1)):
        assert np.array_equal(_np8(k.seed0.index_select(0, ii)), c["seed0"])
        assert np.array_equal(_np64(k.alpha_share.index_select(0, ii)), c["alpha_share"])
    # the two parties share the correction-word arrays (reference fss.py:214-215)
    assert k0.scw is k1.scw and k0.leaf_cw is k1.leaf_cw


def _check_eval(oracle, k0, k1, x_dev, idx, c0, c1):
    x_s = _np64(x_dev)[idx]
    y0, y1 = _np64(fss.eval_cmp(0, k0, x_dev)), _np64(fss.eval_cmp(1, k1, x_dev))
    assert np.array_equal(y0[idx], oracle.eval_cmp(0, c0, x_s))
    assert np.array_equal(y1[idx], oracle.eval_cmp(1, c1, x_s))
    return y0, y1


def test_bench_shape_2p24_sampled_vs_oracle(oracle):
    N = 1 << 24
    alpha, k0, k1 = shard.keygen_cmp_shard(32, np.random.default_rng(1000), N, 0, 1, device="cuda")
    ref_rng = np.random.default_rng(1000)
    a, a0, s0, s1 = oracle.sample_tape(32, ref_rng, N)
    assert np.array_equal(_np64(alpha), a)
    idx = np.sort(np.random.default_rng(7).choice(N, 1 << 16, replace=False))
    idx[:3] = (0, 1, 2)
    idx[-3:] = (N - 3, N - 2, N - 1)                   # first and last CTA runs
    c0, c1 = oracle.keygen_cmp_core(32, a[idx], a0[idx], s0[idx], s1[idx])
    _check_keys(k0, k1, idx, c0, c1)
    del s0, s1
    # the bench's inputs: x = alpha + y, |y| < 2^20 ...
    y = torch.randint(-(1 << 20), 1 << 20, (N,), device="cuda", dtype=torch.int64,
                      generator=torch.Generator("cuda").manual_seed(3))
    x = ((alpha.view(torch.int64) + y) & M32).view(torch.uint64)
    y0, y1 = _check_eval(oracle, k0, k1, x, idx, c0, c1)
    xs = _np64(x)
    assert np.array_equal((y0 + y1) & np.uint64(M32), (xs <= a).astype(np.uint64))
    # ... and uniform x
    xu = torch.from_numpy(np.random.default_rng(9).integers(0, 1 << 32, N, dtype=np.uint64)
                          .view(np.int64)).cuda().view(torch.uint64)
    _check_eval(oracle, k0, k1, xu, idx, c0, c1)
    del k0, k1, alpha, x, xu, y
    torch.cuda.empty_cache()


class _TapeAt:
    """Tape entries of single elements of fss._sample_tape(32, rng, total) for a
    fresh ``default_rng(seed)``, reached by PCG64 jump-ahead: n = 32 draws are
    32-bit words, two per 64-bit output (low half first); the stream holds
    alpha (total words), alpha0 (total), s0 (4 words per seed), s1 (4 each)."""

    def __init__(self, seed: int, total: int):
        self.state = np.random.PCG64(seed).state
        self.total = total

    def _word(self, w: int) -> int:
        bg = np.random.PCG64()
        bg.state = self.state
        bg.advance(int(w) // 2)
        v = int(bg.random_raw())
        return v & M32 if w % 2 == 0 else v >> 32

    def __call__(self, idx):
        T = self.total
        a = np.array([self._word(k) for k in idx], dtype=np.uint64)
        a0 = np.array([self._word(T + k) for k in idx], dtype=np.uint64)
        seeds = []
        for base in (2 * T, 6 * T):
            s = np.array([[self._word(base + 4 * k + q) for q in range(4)] for k in idx],
                         dtype="<u4").view(np.uint8).reshape(len(idx), 16)
            s[:, 15] &= 0x7F
            seeds.append(s)
        return a, a0, seeds[0], seeds[1]


def test_tape_jump_ahead_restatement_is_pinned(oracle):
    T = 5000
    a, a0, s0, s1 = oracle.sample_tape(32, np.random.default_rng(31), T)
    idx = np.array([0, 1, 2, 1234, T - 2, T - 1])
    for got, want in zip(_TapeAt(31, T)(idx), (a, a0, s0, s1)):
        assert np.array_equal(got, want[idx])


def test_2p28_batch_shard_sampled_vs_oracle(oracle):
    total, world, rank = 1 << 28, 4, 1
    rng = np.random.default_rng(2028)
    alpha, k0, k1 = shard.keygen_cmp_shard(32, rng, total, rank, world, device="cuda")
    lo, hi = shard.shard_bounds(total, rank, world)
    assert k0.count == hi - lo == 1 << 26
    # every rank's generator advances past the whole 2^28 tape
    ref = np.random.default_rng(2028)
    ref.bit_generator.advance(10 * total // 2)
    got, want = rng.bit_generator.state, ref.bit_generator.state
    assert got["state"] == want["state"] and got["has_uint32"] == want["has_uint32"] == 0
    idx = np.sort(np.random.default_rng(8).choice(hi - lo, 4096, replace=False))
    idx[0], idx[-1] = 0, hi - lo - 1
    a, a0, s0, s1 = _TapeAt(2028, total)(idx + lo)
    assert np.array_equal(_np64(alpha)[idx], a)
    c0, c1 = oracle.keygen_cmp_core(32, a, a0, s0, s1)
    _check_keys(k0, k1, idx, c0, c1)
    xu = torch.from_numpy(np.random.default_rng(10).integers(0, 1 << 32, hi - lo, dtype=np.uint64)
                          .view(np.int64)).cuda()
    xu[::5] = alpha.view(torch.int64)[::5]
    xu = xu.view(torch.uint64)
    y0, y1 = _check_eval(oracle, k0, k1, xu, idx, c0, c1)
    rec = (y0 + y1) & np.uint64(M32)
    assert np.array_equal(rec, (_np64(xu) <= _np64(alpha)).astype(np.uint64))
    del k0, k1, alpha, xu
    torch.cuda.empty_cache()
