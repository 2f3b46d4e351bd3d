"""Streaming ARNK key files (keyfile.py) on the GPU: the file save_keys writes
is byte-identical to serialize_keys(pack_keys(...)) -- itself pinned to the
reference's containers by tests/golden -- for DCF and DPF keys at several n,
with chunks smaller than the batch and a ragged last chunk; load_keys returns
the same keys (both parties, or one party reading only its payload), and
malformed files raise KeyFormatError like deserialize_keys."""

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2006_04593_b200 import fss, keyfile  # noqa: E402

DEV = torch.device("cuda", 0)


def _same(a, b):
    for f in ("alpha_share", "seed0", "scw", "tcw", "cw_final", "sigma_cw", "leaf_cw"):
        if hasattr(a, f):
            x, y = getattr(a, f), getattr(b, f)
            assert torch.equal(x.contiguous().view(torch.uint8), y.contiguous().view(torch.uint8)), f
    assert a.party == b.party and a.n_bits == b.n_bits and a.count == b.count


@pytest.mark.parametrize("kind,n,count,chunk", [("cmp", 32, 1000, 96), ("cmp", 8, 257, 1000),
                                                 ("cmp", 63, 50, 7), ("eq", 32, 999, 128),
                                                 ("eq", 64, 33, 8), ("eq", 5, 1, 1), ("cmp", 16, 0, 4)])
def test_save_load_roundtrip(tmp_path, kind, n, count, chunk):
    rng = np.random.default_rng(n + count)
    keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    _, k0, k1 = keygen(n, rng, count, device=DEV)
    path = tmp_path / "keys.arnk"
    nbytes = keyfile.save_keys(path, k0, k1, chunk=chunk)
    blob = path.read_bytes()
    assert nbytes == len(blob) and blob == fss.serialize_keys(fss.pack_keys(k0, k1))
    r0, r1 = keyfile.load_keys(path, chunk=chunk)
    _same(r0, k0)
    _same(r1, k1)
    _same(keyfile.load_keys(path, party=1, chunk=max(1, chunk // 2)), k1)
    # the loaded keys evaluate like the originals
    if count:
        x = torch.from_numpy(rng.integers(0, 1 << min(n, 62), count, dtype=np.uint64).view(np.int64)).to(DEV)
        x = x.view(torch.uint64)
        ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
        assert torch.equal(ev(0, r0, x).view(torch.int64), ev(0, k0, x).view(torch.int64))


def test_golden_container_loads(tmp_path):
    g = load_golden("fss_cmp_n32")
    if "arnk" not in g:
        pytest.skip("fixture without a container")
    path = tmp_path / "g.arnk"
    path.write_bytes(g["arnk"].tobytes())
    r0, r1 = keyfile.load_keys(path, chunk=3)
    b0, b1 = fss.unpack_keys(fss.deserialize_keys(g["arnk"].tobytes()), device=DEV)
    _same(r0, b0)
    _same(r1, b1)


def test_malformed_files(tmp_path):
    _, k0, k1 = fss.keygen_cmp(16, np.random.default_rng(1), 20, device=DEV)
    path = tmp_path / "k.arnk"
    keyfile.save_keys(path, k0, k1)
    blob = path.read_bytes()
    for bad in (blob[:10], b"XRNK" + blob[4:], blob[:-1], blob + b"\0", blob[:4] + b"\2" + blob[5:]):
        path.write_bytes(bad)
        with pytest.raises(fss.KeyFormatError):
            keyfile.load_keys(path)
    with pytest.raises(ValueError):
        keyfile.load_keys(path, party=2)
    _, w0, w1 = fss.keygen_cmp(12, np.random.default_rng(2), 4, out_bits=40, device=DEV)
    with pytest.raises(fss.KeyFormatError):
        keyfile.save_keys(tmp_path / "w.arnk", w0, w1)


@pytest.mark.parametrize("kind,n,count", [("cmp", 32, 1000), ("cmp", 32, 997), ("eq", 32, 1002),
                                          ("cmp", 12, 515), ("eq", 7, 333), ("cmp", 63, 100)])
def test_pack_of_column_views_matches_full_payload(kind, n, count):
    """ARNK pack of column views (odd / even offsets, so the kernels' aligned
    async-copy paths and their fallbacks both run) equals the same byte range
    of the full batch's payload; unpack restores the view's keys."""
    keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    _, k0, _ = keygen(n, np.random.default_rng(count), count, device=DEV)
    full = fss._pack_device(k0)
    elem = full.shape[1]
    for lo, hi in ((0, count), (1, count), (2, count - 3), (3, 40), (16, count - 1), (17, 18)):
        v = k0.take(slice(lo, hi))
        got = fss._pack_device(v)
        assert torch.equal(got, full[lo:hi]), (lo, hi)
        back = fss._unpack(fss.KIND_CMP if kind == "cmp" else fss.KIND_EQ, 0, n, hi - lo,
                           got.reshape(-1), DEV)
        _same(back, k0.take(np.arange(lo, hi)))
    assert elem == (fss.cmp_elem_bytes(n) if kind == "cmp" else fss.eq_elem_bytes(n))


@pytest.mark.parametrize("kind,n,count", [("cmp", 32, 3001), ("cmp", 8, 100), ("cmp", 12, 257),
                                          ("cmp", 63, 50), ("eq", 32, 2000), ("eq", 5, 77),
                                          ("eq", 64, 40), ("eq", 16, 1)])
def test_packed_keys_evaluate_like_unpacked(tmp_path, kind, n, count):
    """Keys loaded packed (payload rows kept, fss_*_eval_packed) give the same
    shares as the unpacked keys -- eval with x, and the masked sign / eq
    protocols -- and take / take_unused / unpack behave like the typed batch."""
    from paper_2006_04593_b200 import runtime
    from paper_2006_04593_b200.ring import RingTensor
    from paper_2006_04593_b200.sharing import share
    keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    ev = fss.eval_cmp if kind == "cmp" else fss.eval_eq
    rng = np.random.default_rng(count + n)
    alpha, k0, k1 = keygen(n, rng, count, device=DEV)
    path = tmp_path / "k.arnk"
    keyfile.save_keys(path, k0, k1, chunk=max(1, count // 3))
    p0, p1 = keyfile.load_keys(path, packed=True, chunk=max(1, count // 2))
    assert isinstance(p0, fss.PackedKeyBatch) and p0.count == count
    assert torch.equal(p0.alpha_share.view(torch.int64), k0.alpha_share.view(torch.int64))
    x = rng.integers(0, 1 << min(n, 63), count, dtype=np.uint64)
    if n == 64:
        x = (x << np.uint64(1)) | rng.integers(0, 2, count, dtype=np.uint64)
    x[::3] = alpha.cpu().numpy()[::3]
    for party, (pk, uk) in enumerate(((p0, k0), (p1, k1))):
        assert np.array_equal(ev(party, pk, x), ev(party, uk, x))
    _same(p1.unpack(), k1)
    sub = p0.take(np.arange(count)[::-2])
    assert np.array_equal(ev(0, sub, x[::-2]), ev(0, k0.take(np.arange(count)[::-2]), x[::-2]))
    if kind == "cmp" and n in (8, 32):
        if n == 32:
            lv_p = fss.eval_cmp(0, p0, x, return_levels=True)
            lv_u = fss.eval_cmp(0, k0, x, return_levels=True)
            assert np.array_equal(lv_p[1], lv_u[1])
        ys = share(RingTensor.from_ints(rng.integers(-100, 100, count), n), rng)

        def run(keys):
            (r0, _), (r1, _) = runtime.run_local_pair(
                lambda s: fss.sign_protocol(s, ys[s.party], keys[s.party]))
            return r0.values.numpy(), r1.values.numpy()
        got = run({0: p0, 1: p1})
        want = run({0: k0, 1: k1})          # the same keys, unpacked: identical shares
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
        assert p0.consumed.all() and p1.consumed.all()


def test_packed_keys_pack_and_audit(tmp_path):
    """pack_keys on packed batches reuses the rows (same container bytes), and
    the cut-and-choose audit works on them (tampering caught, sample spent)."""
    _, k0, k1, tape = fss.keygen_cmp_with_tape(16, np.random.default_rng(3), 40, device=DEV)
    path = tmp_path / "k.arnk"
    keyfile.save_keys(path, k0, k1)
    p0, p1 = keyfile.load_keys(path, packed=True)
    assert fss.serialize_keys(fss.pack_keys(p0, p1)) == path.read_bytes()
    assert fss.audit_keys(p0, p1, tape, [0, 5, 9]) == []
    assert p0.consumed[[0, 5, 9]].all() and not p0.consumed[1]
    p1.payload[7, 30] ^= 0x10                       # a correction-word byte of key 7
    assert fss.audit_keys(p0, p1, tape, range(10, 20)) == []
    assert fss.audit_keys(p0, p1, tape, [6, 7, 8]) == [7]


@pytest.mark.parametrize("kind,n,count", [("cmp", 32, 1000), ("eq", 16, 333)])
def test_save_packed_keys(tmp_path, kind, n, count):
    """save_keys on packed batches streams the payload rows as they are: the file
    equals the one written from the typed batches, for both kinds."""
    keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    _, k0, k1 = keygen(n, np.random.default_rng(count), count, device=DEV)
    a, b = tmp_path / "a.arnk", tmp_path / "b.arnk"
    keyfile.save_keys(a, k0, k1, chunk=300)
    p0, p1 = keyfile.load_keys(a, packed=True)
    assert keyfile.save_keys(b, p0, p1, chunk=77) == a.stat().st_size
    assert b.read_bytes() == a.read_bytes()
    with pytest.raises(TypeError):
        keyfile.save_keys(b, object(), object())


def _np_payload(k, kind, n):
    """Element-major ARNK records restated in numpy (reference LAYOUT.md:48-71,
    fss.py:540-602): alpha[w] | seed0[16] | n x (scw[16] | flags[1] | sigma[w] (cmp))
    | cw_final[w] (eq) / (n + 1) x leaf[w] (cmp), little-endian ring values."""
    w = (n + 7) // 8
    cnt = k.count

    def le(v):   # (cnt,) or (rows, cnt) u64 -> (..., cnt, w) bytes
        a = np.ascontiguousarray(v.cpu().numpy().astype(np.uint64))
        return a.view(np.uint8).reshape(a.shape + (8,))[..., :w]

    cols = [le(k.alpha_share), k.seed0.cpu().numpy().reshape(cnt, 16)]
    scw = k.scw.cpu().numpy().reshape(n, cnt, 16)
    tcw = k.tcw.cpu().numpy().reshape(n, cnt, 1)
    lv = [scw, tcw] + ([le(k.sigma_cw)] if kind == "cmp" else [])
    cols.append(np.concatenate(lv, axis=2).transpose(1, 0, 2).reshape(cnt, -1))
    if kind == "cmp":
        cols.append(le(k.leaf_cw).transpose(1, 0, 2).reshape(cnt, -1))
    else:
        cols.append(le(k.cw_final))
    return np.concatenate(cols, axis=1)


@pytest.mark.parametrize("kind,n,count", [("cmp", 32, 1024), ("cmp", 32, 4096), ("eq", 32, 2048),
                                          ("cmp", 12, 512), ("eq", 7, 320), ("cmp", 63, 64),
                                          ("eq", 64, 96), ("cmp", 4, 48),
                                          # several tiles per CTA (persistent grid)
                                          ("cmp", 32, 40000), ("eq", 32, 40000)])
def test_pack_tensor_map_path_matches_numpy(kind, n, count):
    """Level strides that are multiples of 16 and even counts take the TMA
    tensor-map pack (arnk_pack_tma_kernel): whole batches, prefixes with a
    ragged last tile (zero-filled out-of-range box elements), views at
    16-aligned offsets; odd counts and odd offsets take the fallbacks -- every
    payload equals the numpy restatement of the record layout."""
    keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    _, k0, _ = keygen(n, np.random.default_rng(count + n), count, device=DEV)
    for lo, hi in ((0, count), (0, count - 1), (0, count - 6), (0, count - 15), (16, count), (32, count - 7),
                   (32, count - 2), (16, 17), (16, 18), (48, 64), (1, count)):
        hi = min(hi, count)
        if hi <= lo:
            continue
        v = k0.take(slice(lo, hi))
        got = fss._pack_device(v).cpu().numpy()
        assert np.array_equal(got, _np_payload(v, kind, n)), (lo, hi)


@pytest.mark.parametrize("kind,n,count", [("cmp", 32, 1024), ("eq", 32, 2048), ("cmp", 12, 512),
                                          ("eq", 7, 320), ("cmp", 63, 64), ("eq", 64, 96),
                                          # several 128-key tiles per CTA (persistent grid)
                                          ("cmp", 32, 40000), ("eq", 32, 40000)])
def test_unpack_into_column_range(kind, n, count):
    """Unpack into fresh arrays and into a column range of padded arrays
    (ld > count, 16-aligned and unaligned column offsets, ragged last tiles):
    the keys come back exactly and no byte outside the range changes (a TMA
    tensor-store unpack was measured and dropped in r02: slower, and its
    16-byte clipping wrote past an odd-count u64 column range)."""
    from paper_2006_04593_b200 import _dev, _lib
    keygen = fss.keygen_cmp if kind == "cmp" else fss.keygen_eq
    kid = fss.KIND_CMP if kind == "cmp" else fss.KIND_EQ
    _, k0, _ = keygen(n, np.random.default_rng(count + 7 * n), count, device=DEV)
    for lo, hi in ((0, count), (16, count), (0, count - 5), (32, count - 3), (16, 17)):
        v = k0.take(slice(lo, hi))
        m = hi - lo
        payload = fss._pack_device(v).reshape(-1)
        _same(fss._unpack(kid, 0, n, m, payload, DEV), v)
        for c0 in (16, 3):
            L = (c0 + m + 40) // 16 * 16

            def arr(*shape, dt=torch.uint8):
                return torch.full(shape, 0xAB, dtype=torch.uint8, device=DEV).view(dt) if dt != torch.uint8 \
                    else torch.full(shape, 0xAB, dtype=torch.uint8, device=DEV)
            full = {"alpha_share": arr(L, 8, dt=torch.uint64).reshape(L), "seed0": arr(L, 16),
                    "scw": arr(n, L, 16), "tcw": arr(n, L)}
            if kind == "cmp":
                full["sigma_cw"] = arr(n, L, 8, dt=torch.uint64).reshape(n, L)
                full["leaf_cw"] = arr(n + 1, L, 8, dt=torch.uint64).reshape(n + 1, L)
            else:
                full["cw_final"] = arr(L, 8, dt=torch.uint64).reshape(L)
            before = {f: t.clone() for f, t in full.items()}
            col = {f: (t[c0:c0 + m] if t.dim() == 1 or f == "seed0" else t[:, c0:c0 + m]) for f, t in full.items()}
            rc = _lib.call("fss_arnk_unpack", kid, n, m, L, _dev.ptr(payload), _dev.ptr(col["alpha_share"]),
                           _dev.ptr(col["seed0"]), _dev.ptr(col["scw"]), _dev.ptr(col["tcw"]),
                           _dev.ptr(col.get("cw_final")), _dev.ptr(col.get("sigma_cw")),
                           _dev.ptr(col.get("leaf_cw")), _dev.stream_handle(DEV))
            assert rc in (0, None)
            torch.cuda.synchronize()

            def b(t):   # u8 view, element axis kept (u64 -> trailing 8-byte axis)
                return t.contiguous().view(torch.uint8).reshape(*t.shape, -1) if t.dtype != torch.uint8 else t
            for f, t in full.items():
                exp = b(before[f]).clone()
                src = b(getattr(v, f).contiguous())
                if t.dim() == 1 or f == "seed0":
                    exp[c0:c0 + m] = src
                else:
                    exp[:, c0:c0 + m] = src
                assert torch.equal(b(t), exp), (f, lo, hi, c0)
