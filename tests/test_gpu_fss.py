"""GPU parity of the drop-in prg/fss against the reference's golden fixtures
and the CPU oracle (bit-exact: integer/byte work)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2006_04593_b200 import fss, prg  # noqa: E402


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def _mask(w):
    return np.uint64((1 << w) - 1) if w < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)


def test_prg_vectors():
    with open(os.path.join(GOLDEN, "prg_vectors.json")) as fh:
        vecs = json.load(fh)["vectors"]
    assert len(vecs) == 15
    for s, e in vecs:
        assert prg.expand_one(bytes.fromhex(s), 3).hex() == e
        assert prg.expand_one(bytes.fromhex(s), 2).hex() == e[:64]


def test_prg_expand_golden_and_device_io():
    g = load_golden("prg")
    assert np.array_equal(prg.expand(g["seeds"], 3), g["exp3"])
    assert np.array_equal(prg.expand(g["seeds"], 2), g["exp2"])
    assert np.array_equal(prg.expand(g["raw_seeds"], 3), g["raw_exp3"])
    dev = torch.from_numpy(g["seeds"]).cuda()
    out = prg.expand(dev, 3)
    assert out.is_cuda and np.array_equal(_np(out), g["exp3"])
    with pytest.raises(ValueError):
        prg.expand(g["seeds"], 4)


def test_prg_expand_large_vs_oracle(oracle):
    rng = np.random.default_rng(11)
    seeds = rng.integers(0, 256, size=(1 << 20, 16), dtype=np.uint8)
    assert np.array_equal(prg.expand(seeds, 3), oracle.expand(seeds, 3))


def test_slices_match_layout():
    g = load_golden("prg")
    raw = g["exp3"]
    sl, tl, sr, tr, gl, ul, gr, ur = prg.slice_cmp(raw, 32)
    assert np.array_equal(tl, raw[:, 15] >> 7) and np.array_equal(ur, raw[:, 47] >> 7)
    assert np.array_equal(gl, raw[:, 32:40].copy().view("<u8").reshape(-1) & np.uint64(0xFFFFFFFF))
    assert np.array_equal(prg.reassemble_eq(*prg.slice_eq(raw[:, :32])), raw[:, :32])
    assert np.array_equal(prg.seed_to_ring(raw[:, :16], 16),
                          raw[:, :8].copy().view("<u8").reshape(-1) & np.uint64(0xFFFF))


@pytest.mark.parametrize("tag", golden_cases())
def test_keygen_eval_golden(tag):
    g = load_golden(tag)
    n, N, ob = int(g["n"]), int(g["N"]), int(g["out_bits"])
    kind = "eq" if tag.startswith("fss_eq") else "cmp"
    rng = np.random.default_rng(int(g["seed"]))
    if kind == "eq":
        alpha, k0, k1 = fss.keygen_eq(n, rng, N)
    else:
        alpha, k0, k1 = fss.keygen_cmp(n, rng, N, out_bits=(ob if ob != n else None))
    # the caller's generator advanced exactly like the reference's
    assert np.array_equal(rng.integers(0, 1 << 32, size=4, dtype=np.uint64), g["next_draws"])
    assert np.array_equal(_np(alpha), g["alpha"])
    assert np.array_equal(_np(k0.alpha_share), g["alpha0"])
    assert np.array_equal(_np(k1.alpha_share), g["alpha1"])
    assert np.array_equal(_np(k0.seed0), g["s0"]) and np.array_equal(_np(k1.seed0), g["s1"])
    assert np.array_equal(_np(k0.scw), g["scw"]) and np.array_equal(_np(k0.tcw), g["tcw"])
    assert k0.scw is k1.scw  # CWs shared between the parties (fss.py:214-215)
    x = g["x"]
    if kind == "eq":
        assert np.array_equal(_np(k0.cw_final), g["cw_final"])
        y0, y1 = fss.eval_eq(0, k0, x), fss.eval_eq(1, k1, x)
    else:
        assert np.array_equal(_np(k0.sigma_cw), g["sigma_cw"])
        assert np.array_equal(_np(k0.leaf_cw), g["leaf_cw"])
        y0, lv0 = fss.eval_cmp(0, k0, x, return_levels=True)
        y1, lv1 = fss.eval_cmp(1, k1, x, return_levels=True)
        assert np.array_equal(lv0, g["lv0"]) and np.array_equal(lv1, g["lv1"])
    assert isinstance(y0, np.ndarray) and y0.dtype == np.uint64
    assert np.array_equal(y0, g["y0"]) and np.array_equal(y1, g["y1"])
    # device-resident inputs give device-resident outputs with the same values
    xd = torch.from_numpy(x).cuda()
    yd = fss.eval_eq(0, k0, xd) if kind == "eq" else fss.eval_cmp(0, k0, xd)
    assert yd.is_cuda and np.array_equal(_np(yd), g["y0"])
    if "arnk" in g:
        blob = fss.serialize_keys(fss.pack_keys(k0, k1))
        assert blob == g["arnk"].tobytes()
        r0, r1 = fss.unpack_keys(fss.deserialize_keys(blob))
        assert fss.serialize_keys(fss.pack_keys(r0, r1)) == blob
    else:
        with pytest.raises(fss.KeyFormatError):
            fss.pack_keys(k0, k1)


@pytest.mark.parametrize("n", [4, 5])
def test_exhaustive_golden(n):
    g = load_golden(f"exhaustive_n{n}")
    size = 1 << n
    rng = np.random.default_rng(n)
    alphas = np.arange(size, dtype=np.uint64)
    _, e0, e1 = fss.keygen_eq(n, rng, count=size, alpha=alphas)
    _, c0, c1 = fss.keygen_cmp(n, rng, count=size, alpha=alphas)
    assert np.array_equal(rng.integers(0, 1 << 32, size=4, dtype=np.uint64), g["next_draws"])
    assert fss.serialize_keys(fss.pack_keys(e0, e1)) == g["eq_arnk"].tobytes()
    assert fss.serialize_keys(fss.pack_keys(c0, c1)) == g["cmp_arnk"].tobytes()
    idx = np.repeat(np.arange(size), size)
    xs = np.tile(np.arange(size, dtype=np.uint64), size)
    assert np.array_equal(fss.eval_eq(0, e0.take(idx), xs), g["eq_y0"])
    assert np.array_equal(fss.eval_eq(1, e1.take(idx), xs), g["eq_y1"])
    assert np.array_equal(fss.eval_cmp(0, c0.take(idx), xs), g["cmp_y0"])
    assert np.array_equal(fss.eval_cmp(1, c1.take(idx), xs), g["cmp_y1"])


@pytest.mark.parametrize("n", range(4, 11))
def test_exhaustive_exactness(n):
    # test_acceptance.py::test_c01 -- every (alpha, x) pair for n = 4..10
    size = 1 << n
    rng = np.random.default_rng(n)
    alphas = np.arange(size, dtype=np.uint64)
    _, e0, e1 = fss.keygen_eq(n, rng, count=size, alpha=alphas)
    _, c0, c1 = fss.keygen_cmp(n, rng, count=size, alpha=alphas)
    idx = torch.arange(size, device="cuda").repeat_interleave(size)
    xs = torch.arange(size, device="cuda").repeat(size)
    m = (1 << n) - 1
    rec_c = (fss.eval_cmp(0, c0.take(idx), xs).view(torch.int64)
             + fss.eval_cmp(1, c1.take(idx), xs).view(torch.int64)) & m
    rec_e = (fss.eval_eq(0, e0.take(idx), xs).view(torch.int64)
             + fss.eval_eq(1, e1.take(idx), xs).view(torch.int64)) & m
    a = idx.to(torch.int64)
    assert torch.equal(rec_c, (xs <= a).to(torch.int64))
    assert torch.equal(rec_e, (xs == a).to(torch.int64))


@pytest.mark.parametrize("kind,n,N", [("cmp", 32, 1 << 16), ("eq", 32, 1 << 20), ("cmp", 16, 4099),
                                      ("eq", 63, 777), ("cmp", 63, 515), ("eq", 64, 300),
                                      ("cmp", 8, 1), ("eq", 4, 3)])
def test_large_vs_oracle(oracle, kind, n, N):
    seed = 77 + n + N
    rng = np.random.default_rng(seed)
    keygen = fss.keygen_eq if kind == "eq" else fss.keygen_cmp
    alpha, k0, k1 = keygen(n, rng, N)
    ref_rng = np.random.default_rng(seed)
    a, a0, s0, s1 = oracle.sample_tape(n, ref_rng, N)
    assert np.array_equal(_np(alpha), a) and np.array_equal(_np(k0.alpha_share), a0)
    assert np.array_equal(_np(k0.seed0), s0) and np.array_equal(_np(k1.seed0), s1)
    assert np.array_equal(rng.integers(0, 1 << 32, 3, dtype=np.uint64),
                          ref_rng.integers(0, 1 << 32, 3, dtype=np.uint64))
    core = oracle.keygen_eq_core if kind == "eq" else oracle.keygen_cmp_core
    r0, r1 = core(n, a, a0, s0, s1)
    for name in ("scw", "tcw") + (("cw_final",) if kind == "eq" else ("sigma_cw", "leaf_cw")):
        assert np.array_equal(_np(getattr(k0, name)), r0[name]), name
    xs = np.random.default_rng(seed + 1).integers(0, 1 << min(n, 63), N, dtype=np.uint64)
    xs[::3] = a[::3]
    ev, oev = (fss.eval_eq, oracle.eval_eq) if kind == "eq" else (fss.eval_cmp, oracle.eval_cmp)
    y0, y1 = ev(0, k0, xs), ev(1, k1, xs)
    assert np.array_equal(y0, oev(0, r0, xs)) and np.array_equal(y1, oev(1, r1, xs))
    want = (xs == a) if kind == "eq" else (xs <= a)
    assert np.array_equal((y0 + y1) & _mask(n), want.astype(np.uint64))


def test_buffered_half_word_state(oracle):
    # A Dealer stream can leave numpy's 32-bit half-word buffered (has_uint32=1).
    for pre in (1, 3):
        rng = np.random.default_rng(5)
        rng.integers(0, 2, size=pre, dtype=np.uint64)
        assert rng.bit_generator.state["has_uint32"] == 1
        ref = np.random.default_rng(5)
        ref.integers(0, 2, size=pre, dtype=np.uint64)
        for n in (16, 32, 40):
            alpha, k0, k1 = fss.keygen_cmp(n, rng, 33)
            a, a0, s0, s1 = oracle.sample_tape(n, ref, 33)
            assert np.array_equal(_np(alpha), a) and np.array_equal(_np(k0.alpha_share), a0)
            assert np.array_equal(_np(k1.seed0), s1)
            assert rng.bit_generator.state == ref.bit_generator.state


def test_take_views_gather_and_single_use():
    rng = np.random.default_rng(3)
    alpha, k0, k1 = fss.keygen_cmp(16, rng, 64)
    xs = np.random.default_rng(4).integers(0, 1 << 16, 64, dtype=np.uint64)
    full = fss.eval_cmp(0, k0, xs)
    v = k0.take(np.arange(10, 30))            # contiguous -> zero-copy views
    assert v.scw.data_ptr() == k0.scw[:, 10:].data_ptr()
    assert np.array_equal(fss.eval_cmp(0, v, xs[10:30]), full[10:30])
    idx = np.array([5, 1, 63, 7, 7])
    assert np.array_equal(fss.eval_cmp(0, k0.take(idx), xs[idx]), full[idx])
    s = k0.take_unused(60)
    assert s.count == 60 and k0.consumed[:60].all()
    with pytest.raises(fss.KeyExhaustedError):
        k0.take_unused(5)


def test_validate_and_errors():
    rng = np.random.default_rng(20)
    _, k0, _ = fss.keygen_cmp(16, rng, count=2)
    k0.scw = k0.scw[:-1]
    with pytest.raises(fss.KeyFormatError):
        fss.eval_cmp(0, k0, np.zeros(2, dtype=np.uint64))
    _, e0, _ = fss.keygen_eq(16, rng, count=2)
    e0.n_bits = 12
    with pytest.raises(fss.KeyFormatError):
        fss.eval_eq(0, e0, np.zeros(2, dtype=np.uint64))
    _, e0, _ = fss.keygen_eq(16, rng, count=2)
    with pytest.raises(ValueError):
        fss.eval_eq(0, e0, np.zeros(3, dtype=np.uint64))
    with pytest.raises(ValueError):
        fss.keygen_cmp(64, rng, 1)
    with pytest.raises(ValueError):
        fss.keygen_cmp(12, rng, 1, out_bits=8)
    with pytest.raises(ValueError):
        fss.keygen_eq(3, rng, 1)


def test_empty_batch_and_scalar_x():
    rng = np.random.default_rng(10)
    alpha, k0, k1 = fss.keygen_eq(8, rng, count=1)
    a = int(_np(alpha)[0])
    rec = (fss.eval_eq(0, k0, a) + fss.eval_eq(1, k1, a)) & np.uint64(255)
    assert rec[0] == 1
    empty0, empty1 = k0.take(np.array([], dtype=np.int64)), k1.take(np.array([], dtype=np.int64))
    blob = fss.serialize_keys(fss.pack_keys(empty0, empty1))
    assert len(blob) == 13 and fss.deserialize_keys(blob).count == 0
    assert fss.eval_eq(0, empty0, np.zeros(0, dtype=np.uint64)).shape == (0,)
    _, z0, z1 = fss.keygen_cmp(12, rng, count=0)
    assert z0.count == 0


def test_audit_on_device():
    rng = np.random.default_rng(14)
    _, k0, k1, tape = fss.keygen_cmp_with_tape(16, rng, count=20)
    sample = [0, 3, 7, 11, 19, 4, 9, 15, 2, 6]
    assert fss.audit_keys(k0, k1, tape, sample) == []
    assert k0.consumed[sample].all() and not k0.consumed[[1, 5, 8]].any()
    rng = np.random.default_rng(15)
    _, k0, k1, tape = fss.keygen_cmp_with_tape(16, rng, count=10)
    k0.scw[2, 3, 5] ^= 0x40
    assert fss.audit_keys(k0, k1, tape, range(10)) == [3]
    rng = np.random.default_rng(16)
    _, k0, k1, tape = fss.keygen_cmp_with_tape(16, rng, count=10)
    k1.leaf_cw.view(torch.int64)[16, 7] ^= 1
    assert fss.audit_keys(k0, k1, tape, range(10)) == [7]
    rng = np.random.default_rng(17)
    _, k0, k1, tape = fss.keygen_eq_with_tape(12, rng, count=6)
    k0.cw_final.view(torch.int64)[2] ^= 2
    assert fss.audit_keys(k0, k1, tape, range(6)) == [2]


def test_full_size_properties():
    # 2^22 DCF at n=32: reconstruction is exactly the predicate (x = alpha + y).
    N = 1 << 22
    rng = np.random.default_rng(123)
    alpha, k0, k1 = fss.keygen_cmp(32, rng, N)
    y = torch.randint(-1000, 1000, (N,), device="cuda", dtype=torch.int64)
    x = (alpha.view(torch.int64) + y) & 0xFFFFFFFF
    rec = (fss.eval_cmp(0, k0, x).view(torch.int64) + fss.eval_cmp(1, k1, x).view(torch.int64)) & 0xFFFFFFFF
    a = alpha.view(torch.int64)
    assert torch.equal(rec, (x <= a).to(torch.int64))


def test_host_paths_match_device_path():
    # pinned host x: the kernel reads x from / writes the shares to pinned host
    # memory directly (zero-copy); numpy x: staged 2-stream chunked pipeline;
    # the C-ABI pinned pipeline (fss_dcf_eval_host without staging) too. All
    # must equal the single-launch device path bit-exactly.
    import ctypes
    from paper_2006_04593_b200 import _dev, _lib
    N = (1 << 22) + 12345                 # several chunks plus a ragged tail
    rng = np.random.default_rng(31)
    alpha, k0, k1 = fss.keygen_cmp(32, rng, N)
    ea, e0, _ = fss.keygen_eq(32, rng, N)
    xh = torch.from_numpy(np.random.default_rng(32).integers(0, 1 << 32, N, dtype=np.uint64)
                          .view(np.int64)).pin_memory().view(torch.uint64)
    xd = xh.cuda()
    for party, k in ((0, k0), (1, k1)):
        h = fss.eval_cmp(party, k, xh)
        assert not h.is_cuda and h.is_pinned()
        assert torch.equal(h.view(torch.int64), fss.eval_cmp(party, k, xd).view(torch.int64).cpu())
    h = fss.eval_eq(0, e0, xh)
    assert torch.equal(h.view(torch.int64), fss.eval_eq(0, e0, xd).view(torch.int64).cpu())
    small = xh[:1000].clone().pin_memory()
    assert torch.equal(fss.eval_cmp(0, k0.take(np.arange(1000)), small).view(torch.int64),
                       fss.eval_cmp(0, k0, xd)[:1000].view(torch.int64).cpu())
    xn = xh.view(torch.int64).numpy().view(np.uint64)           # pageable numpy copy below
    got = fss.eval_cmp(1, k1, xn.copy())
    assert isinstance(got, np.ndarray)
    assert np.array_equal(got, fss.eval_cmp(1, k1, xd).cpu().view(torch.int64).numpy().view(np.uint64))
    chunk = 1 << 20
    out_h = torch.empty(N, dtype=torch.int64, pin_memory=True)
    scratch = torch.empty((2, 2 * chunk), dtype=torch.uint64, device="cuda")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for st in (sa, sb):
        st.wait_stream(torch.cuda.current_stream())
    _lib.call("fss_dcf_eval_host", 0, 32, 32, N, N, _dev.ptr(k0.seed0), _dev.ptr(k0.scw), _dev.ptr(k0.tcw),
              _dev.ptr(k0.sigma_cw), _dev.ptr(k0.leaf_cw), xh.data_ptr(), out_h.data_ptr(),
              _dev.ptr(scratch[0]), _dev.ptr(scratch[1]), chunk, None, ctypes.c_void_p(sa.cuda_stream),
              ctypes.c_void_p(sb.cuda_stream))
    torch.cuda.synchronize()
    assert torch.equal(out_h, fss.eval_cmp(0, k0, xd).view(torch.int64).cpu())


@pytest.mark.parametrize("chunks", [2.5, 7.9, 8.0, 9.3, 21.7])
def test_staged_pipeline_schedule(monkeypatch, chunks):
    # numpy x through the staged pipeline with a small chunk, so the three
    # staging slots wrap several times and, from 8 chunks on, the quarter /
    # half ramps at both ends are active; ragged tails included
    chunk = 1 << 14
    monkeypatch.setattr(fss, "PIPELINE_CHUNK", chunk)
    monkeypatch.setattr(fss, "PIPELINE_MIN", chunk)
    N = int(chunks * chunk) + 5
    rng = np.random.default_rng(int(chunks * 10))
    alpha, k0, k1 = fss.keygen_cmp(32, rng, N)
    _, e0, _ = fss.keygen_eq(32, rng, N)
    xn = np.random.default_rng(7).integers(0, 1 << 32, N, dtype=np.uint64)
    xd = torch.from_numpy(xn.view(np.int64)).cuda().view(torch.uint64)
    for party, k in ((0, k0), (1, k1)):
        got = fss.eval_cmp(party, k, xn)
        assert isinstance(got, np.ndarray) and got.shape == (N,)
        assert np.array_equal(got, _np(fss.eval_cmp(party, k, xd).view(torch.int64)).view(np.uint64))
    got = fss.eval_eq(0, e0, xn)
    assert np.array_equal(got, _np(fss.eval_eq(0, e0, xd).view(torch.int64)).view(np.uint64))


def test_bitsliced_expand_matches_ttable():
    # the bitsliced AES alternative (research record, scripts/research/bitsliced,
    # not in the product library) is bit-exact with the T-table PRG and the
    # reference's PRG vectors
    import ctypes
    import importlib.util
    from paper_2006_04593_b200 import _dev
    spec = importlib.util.spec_from_file_location(
        "bs_build", os.path.join(os.path.dirname(GOLDEN), "..", "scripts", "research", "bitsliced", "build.py"))
    bs_build = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bs_build)
    bs = ctypes.CDLL(bs_build.build())
    bs.fss_aes_mmo_expand_bitsliced.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int,
                                                ctypes.c_void_p, ctypes.c_void_p]
    seeds = torch.from_numpy(np.random.default_rng(41).integers(0, 256, (1 << 16, 16),
                                                                dtype=np.uint8)).cuda()
    with open(os.path.join(GOLDEN, "prg_vectors.json")) as fh:
        vecs = json.load(fh)["vectors"]
    for i, (s, _) in enumerate(vecs):
        seeds[i] = torch.from_numpy(np.frombuffer(bytes.fromhex(s), dtype=np.uint8).copy())
    for blocks in (2, 3):
        out = torch.empty((seeds.shape[0], 16 * blocks), dtype=torch.uint8, device="cuda")
        assert bs.fss_aes_mmo_expand_bitsliced(_dev.ptr(seeds), seeds.shape[0], blocks, _dev.ptr(out),
                                               torch.cuda.current_stream().cuda_stream) == 0
        assert torch.equal(out, prg.expand(seeds, blocks))
    for i, (_, e) in enumerate(vecs):
        assert out[i].cpu().numpy().tobytes().hex() == e


@pytest.mark.parametrize("pre,shape,n_bits", [(0, (1000,), 32), (1, (7, 33), 32), (3, (5,), 64),
                                              (0, (1 << 20,), 32), (2, (64, 3, 5), 16), (1, (1,), 63),
                                              (0, (), 32)])
def test_ring_random_on_device_matches_numpy(pre, shape, n_bits):
    from paper_2006_04593_b200.ring import RingTensor
    a, b = np.random.default_rng(12), np.random.default_rng(12)
    a.integers(0, 2, size=pre, dtype=np.uint64)
    b.integers(0, 2, size=pre, dtype=np.uint64)
    raw = a.integers(0, 1 << 63, size=shape, dtype=np.uint64)
    raw = (raw << np.uint64(1)) | a.integers(0, 2, size=shape, dtype=np.uint64)
    mask = np.uint64((1 << n_bits) - 1) if n_bits < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    t = RingTensor.random(shape, n_bits, b)
    assert t.data.is_cuda and tuple(t.shape) == tuple(shape)
    assert np.array_equal(t.numpy(), raw & mask)
    assert a.bit_generator.state == b.bit_generator.state


def test_mask_stream_matches_reference():
    # prg.mask_stream (prg.py:128-147) vectors produced by the reference
    with np.load(os.path.join(GOLDEN, "mask_stream.npz")) as g:
        for i in range(int(g["cases"])):
            rnd, count, n = (int(v) for v in g[f"meta{i}"])
            got = prg.mask_stream(g[f"seed{i}"].tobytes(), rnd, count, n)
            assert isinstance(got, np.ndarray) and np.array_equal(got, g[f"out{i}"]), i
    a = prg.mask_stream(bytes(range(16)), 0, 100, 32)
    assert not np.array_equal(a, prg.mask_stream(bytes(range(16)), 1, 100, 32))
    with pytest.raises(ValueError):
        prg.mask_stream(bytes(15), 0, 4, 32)


@pytest.mark.parametrize("pre", [0, 1])
def test_n64_tape_on_device_matches_numpy(oracle, pre):
    # n = 64 keys: alpha/alpha0 via the ring kernel (two-call uniform draw,
    # fss.py:48-50) and the seeds-only PCG64 tape; the caller's rng state after
    # keygen must equal numpy's
    rng, ref = np.random.default_rng(64), np.random.default_rng(64)
    rng.integers(0, 2, size=pre, dtype=np.uint64)
    ref.integers(0, 2, size=pre, dtype=np.uint64)
    alpha, k0, k1 = fss.keygen_eq(64, rng, 257)
    a, a0, s0, s1 = oracle.sample_tape(64, ref, 257)
    assert np.array_equal(_np(alpha), a) and np.array_equal(_np(k0.alpha_share), a0)
    assert np.array_equal(_np(k0.seed0), s0) and np.array_equal(_np(k1.seed0), s1)
    assert rng.bit_generator.state == ref.bit_generator.state


def test_numpy_host_pipeline_matches_device_path():
    # large numpy (pageable) inputs go through the staged native pipeline
    N = (1 << 22) + 777
    rng = np.random.default_rng(33)
    alpha, k0, _ = fss.keygen_cmp(32, rng, N)
    ea, e0, _ = fss.keygen_eq(32, rng, N)
    x = np.random.default_rng(34).integers(0, 1 << 40, N, dtype=np.uint64)   # high bits ignored
    xd = torch.from_numpy(x.view(np.int64)).cuda().view(torch.uint64)
    y = fss.eval_cmp(0, k0, x)
    assert isinstance(y, np.ndarray) and y.dtype == np.uint64
    assert np.array_equal(y, _np(fss.eval_cmp(0, k0, xd)))
    assert np.array_equal(fss.eval_eq(0, e0, x), _np(fss.eval_eq(0, e0, xd)))
    yl, lv = fss.eval_cmp(0, k0, x, return_levels=True)
    assert np.array_equal(yl, y) and lv.shape == (33, N)


def test_pinned_noncontiguous_input_is_uploaded_not_read_in_place():
    # a strided view of pinned memory is not itself readable in place: it must
    # take the upload path (and still give the device path's shares)
    N = 4096
    _, k0, _ = fss.keygen_cmp(32, np.random.default_rng(5), N)
    big = torch.from_numpy(np.random.default_rng(6).integers(0, 1 << 32, 2 * N, dtype=np.uint64)
                           .view(np.int64)).pin_memory()
    xv = big[::2]
    assert xv.is_pinned() and not xv.is_contiguous()
    got = fss.eval_cmp(0, k0, xv)
    want = fss.eval_cmp(0, k0, xv.contiguous().cuda())
    assert torch.equal(torch.as_tensor(got).view(torch.int64).cpu().reshape(-1), want.view(torch.int64).cpu())


def test_ready_cache_follows_the_arrays():
    # validate() + level-stride probe are cached per batch while its arrays are
    # the same objects; take() views inherit it; replacing an array revalidates
    rng = np.random.default_rng(21)
    alpha, k0, k1 = fss.keygen_cmp(16, rng, count=64)
    x = alpha.clone()
    y = fss.eval_cmp(0, k0, x)
    assert "_ready" in k0.__dict__
    sub = k0.take_unused(40)                 # a lazy slice: the parent's arrays, check and stride
    assert "_lazy" in sub.__dict__ and fss._ready(sub, fss._CMP_LEVEL) == 64
    assert torch.equal(fss.eval_cmp(0, sub, x[:40]).view(torch.int64), y[:40].view(torch.int64))
    view = k0.take(slice(40, 64))
    assert "_ready" in view.__dict__ and view.__dict__["_ready"][1] == 64    # parent's level stride
    assert torch.equal(fss.eval_cmp(0, view, x[40:]).view(torch.int64), y[40:].view(torch.int64))
    gathered = k0.take(np.array([5, 1, 60]))                                # gather: no inheritance
    assert "_ready" not in gathered.__dict__
    pick = torch.tensor([5, 1, 60], device=x.device)
    assert torch.equal(fss.eval_cmp(0, gathered, x.view(torch.int64)[pick]).view(torch.int64),
                       y.view(torch.int64)[pick])
    k0.scw = k0.scw[:-1]
    with pytest.raises(fss.KeyFormatError):
        fss.eval_cmp(0, k0, x)
    k1.leaf_cw = k1.leaf_cw.clone()                                        # same shape, new object
    assert torch.equal(fss.eval_cmp(1, k1, x).view(torch.int64),
                       fss.eval_cmp(1, k1.take(slice(0, 64)), x).view(torch.int64))
