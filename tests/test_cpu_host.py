"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
host-side bookkeeping (PCG64 jump, index normalisation, ARNK headers)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared_symbols():
    syms = set()
    for name in os.listdir(os.path.join(ROOT, "include")):
        if name.endswith(".h"):
            src = open(os.path.join(ROOT, "include", name)).read()
            syms |= set(re.findall(r"\b(fss_[a-z0-9_]+)\s*\(", src))
    return syms


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2006_04593_b200 import _build, _lib
    _build.build()
    lib = _lib.load()
    declared = _declared_symbols()
    assert {"fss_dcf_eval", "fss_dpf_eval", "fss_dcf_keygen", "fss_dpf_keygen",
            "fss_aes_mmo_expand", "fss_pcg64_tape", "fss_arnk_pack"} <= declared
    for sym in declared:
        assert hasattr(lib, sym), sym
    assert set(_lib.SIGNATURES) >= declared
    assert lib.fss_abi_version() == 6
    assert not hasattr(lib, "fss_aes_mmo_expand_bitsliced")   # research record, not product ABI
    assert lib.fss_arnk_elem_bytes(1, 32) == 824 and lib.fss_arnk_elem_bytes(0, 32) == 568
    assert isinstance(ctypes.CDLL(_build.LIB), ctypes.CDLL)


def test_library_rejects_bad_arguments_without_gpu():
    from paper_2006_04593_b200 import _lib
    lib = _lib.load()
    assert lib.fss_dcf_eval(2, 32, 32, 1, 1, None, None, None, None, None, None, None, None, None) == 1
    assert b"party" in lib.fss_last_error()
    assert lib.fss_aes_mmo_expand(None, 1, 4, None, None) == 1
    with pytest.raises(ValueError):
        _lib.check(1, "x")


def test_pcg_jump_matches_numpy():
    from paper_2006_04593_b200._pcg import jump as _pcg_jump, output as _pcg_output
    rng = np.random.default_rng(99)
    st = rng.bit_generator.state["state"]
    for delta in (1, 2, 5, 1000, 123456789):
        r = np.random.default_rng(99)
        r.bit_generator.advance(delta - 1)
        want = r.bit_generator.random_raw()
        s = _pcg_jump(st["state"], st["inc"], delta)
        assert _pcg_output(s) == int(want)


def test_index_normalisation():
    from paper_2006_04593_b200.fss import _index
    sel, arr = _index(np.arange(3, 9), 10, None)
    assert sel == slice(3, 9) and list(np.arange(10)[arr]) == list(range(3, 9))
    sel, arr = _index(slice(4, None), 10, None)
    assert sel == slice(4, 10) == arr
    sel, arr = _index(slice(8, 3), 10, None)
    assert np.arange(10)[arr].size == 0
    sel, arr = _index(np.array([5, 1, 7]), 10, None)
    assert list(arr) == [5, 1, 7]
    sel, arr = _index([-1], 10, None)
    assert sel == slice(9, 10)
    sel, arr = _index(range(2, 4), 10, None)
    assert sel == slice(2, 4)
    with pytest.raises(IndexError):
        _index([10], 10, None)


def test_deserialize_header_errors():
    from paper_2006_04593_b200 import fss
    blob = fss.serialize_keys(fss.KeyBatch(fss.KIND_EQ, 8, 0, b"", b""))
    assert len(blob) == 13 and fss.deserialize_keys(blob).count == 0
    with pytest.raises(fss.KeyFormatError, match="bad magic"):
        fss.deserialize_keys(b"XXXX" + blob[4:])
    with pytest.raises(fss.KeyFormatError, match="version"):
        fss.deserialize_keys(blob[:4] + bytes([9]) + blob[5:])
    with pytest.raises(fss.KeyFormatError, match="truncated"):
        fss.deserialize_keys(blob[:5])
    one = fss.serialize_keys(fss.KeyBatch(fss.KIND_CMP, 16, 1, bytes(fss.cmp_elem_bytes(16)),
                                          bytes(fss.cmp_elem_bytes(16))))
    with pytest.raises(fss.KeyFormatError, match="size mismatch"):
        fss.deserialize_keys(one[:-3])
    assert fss.cmp_key_bits(32) == 6431 and fss.cmp_elem_bytes(32) == 824
    assert fss.eq_elem_bytes(32) == 568


def _emulate_ring_random(rng, count, n_bits):
    """Python restatement of pcg64_ring_kernel + the host commit (_pcg.commit)."""
    from paper_2006_04593_b200 import _lib, _pcg
    cst, st = _pcg.snapshot(rng)
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    h = int(st["has_uint32"])
    out = []
    for k in range(count):
        hi = _pcg.output(_pcg.jump(s, inc, k + 1)) & ~1
        if k < h:
            word = int(st["uinteger"])
        else:
            r = k - h
            v = _pcg.output(_pcg.jump(s, inc, count + r // 2 + 1))
            word = (v >> 32) if r & 1 else (v & 0xFFFFFFFF)
        out.append((hi | (word >> 31)) & ((1 << n_bits) - 1))
    fresh = max(count - h, 0)
    o = _lib.PcgState()
    o.advance = count + (fresh + 1) // 2
    o.has_uint32 = st["has_uint32"] if count == 0 else fresh & 1
    _pcg.commit(rng, st, o, fresh > 0)
    return np.array(out, dtype=np.uint64)


@pytest.mark.parametrize("pre,count,n_bits", [(0, 7, 32), (1, 7, 32), (0, 8, 64), (3, 1, 16),
                                              (1, 1, 32), (0, 0, 32), (2, 33, 63)])
def test_ring_random_stream_matches_numpy(pre, count, n_bits):
    # RingTensor.random (ring.py:61-65): 64-bit Lemire draws (v >> 1) then buffered
    # 32-bit draws (w >> 31); the device kernel must follow numpy's stream exactly
    a, b = np.random.default_rng(9), np.random.default_rng(9)
    a.integers(0, 2, size=pre, dtype=np.uint64)
    b.integers(0, 2, size=pre, dtype=np.uint64)
    raw = a.integers(0, 1 << 63, size=count, dtype=np.uint64)
    raw = (raw << np.uint64(1)) | a.integers(0, 2, size=count, dtype=np.uint64)
    mask = np.uint64((1 << n_bits) - 1) if n_bits < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    assert np.array_equal(_emulate_ring_random(b, count, n_bits), raw & mask)
    assert a.bit_generator.state == b.bit_generator.state
    assert np.array_equal(a.integers(0, 1 << 40, 5), b.integers(0, 1 << 40, 5))


def test_take_unused_fast_path_and_fallback():
    # the hint-based fast path must hand out exactly the first m free keys
    from paper_2006_04593_b200 import fss

    class Fake:
        def __init__(self, n):
            self.consumed = np.zeros(n, dtype=bool)
            self.taken = []

        def take(self, idx, _consumed=None):
            self.taken.append(idx)
            # the hand-out is spent: a read-only all-True mask of its size
            n = (idx.stop - idx.start) if isinstance(idx, slice) else len(idx)
            assert _consumed is not None and _consumed.shape == (n,) and _consumed.all()
            assert not _consumed.flags.writeable

            class V:
                consumed = _consumed
            return V()
    rng = np.random.default_rng(0)
    for trial in range(200):
        f = Fake(50)
        ref = np.zeros(50, dtype=bool)
        for _ in range(8):
            if rng.random() < 0.3:   # an audit consumes random keys
                pick = rng.integers(0, 50, 3)
                f.consumed[pick] = True
                ref[pick] = True
            m = int(rng.integers(0, 9))
            free = np.flatnonzero(~ref)
            if free.size < m:
                with pytest.raises(fss.KeyExhaustedError):
                    fss._take_unused(f, m)
                continue
            fss._take_unused(f, m)
            got = f.taken[-1]
            got = np.arange(got.start, got.stop) if isinstance(got, slice) else np.asarray(got)
            assert np.array_equal(got, free[:m])
            ref[free[:m]] = True
            assert np.array_equal(f.consumed, ref)


def test_ctypes_signatures_match_header_prototypes():
    """Every ctypes argtypes list in _lib.SIGNATURES has exactly as many
    parameters as the C prototype in include/ariann_fss.h declares."""
    import re
    from paper_2006_04593_b200 import _lib
    with open(os.path.join(ROOT, "include", "ariann_fss.h")) as fh:
        text = re.sub(r"/\*.*?\*/", "", fh.read(), flags=re.S)
    protos = {}
    for m in re.finditer(r"\b(?:int|int64_t|void|uint64_t|const char\*)\s+(fss_\w+)\s*\(([^)]*)\)\s*;", text):
        params = m.group(2).strip()
        protos[m.group(1)] = 0 if params in ("", "void") else params.count(",") + 1
    assert protos, "no prototypes parsed"
    for name, argtypes in _lib.SIGNATURES.items():
        assert name in protos, name
        assert len(argtypes) == protos[name], (name, len(argtypes), protos[name])


def test_null_device_pointers_rejected_before_any_cuda_call():
    """A NULL required pointer returns FSS_EINVAL (ValueError in Python) up
    front, instead of faulting inside a kernel -- checked without a GPU."""
    import ctypes
    from paper_2006_04593_b200 import _lib
    lib = _lib.load()
    one = ctypes.c_void_p(16)   # never dereferenced: the call must fail first
    assert lib.fss_dcf_eval(0, 32, 32, 8, 8, None, one, one, one, one, one, one, None, None) == 1
    assert b"null" in lib.fss_last_error()
    assert lib.fss_dpf_eval(0, 32, 8, 8, one, one, one, one, one, None, None) == 1
    assert lib.fss_dcf_keygen(32, 32, 8, one, one, one, one, one, None, one, one, one, None) == 1
    assert lib.fss_dpf_keygen(32, 8, one, one, one, one, None, one, one, one, None) == 1
    assert lib.fss_aes_mmo_expand(None, 8, 3, one, None) == 1
    assert lib.fss_dcf_eval_packed(0, 32, 8, None, one, None, None, one, None) == 1
    assert lib.fss_arnk_pack(1, 32, 8, 8, one, one, one, one, None, one, None, one, None) == 1
    st = _lib.PcgState()
    assert lib.fss_pcg64_tape(ctypes.byref(st), 32, 8, 1, one, one, None, one, None, None) == 1


def test_level_stride_and_ring_random_arguments_rejected_without_gpu():
    """ld < count would make the eval kernels read overlapping level rows, and a
    NULL generator state would be dereferenced on the host: both are FSS_EINVAL
    before any CUDA call."""
    import ctypes
    from paper_2006_04593_b200 import _lib
    lib = _lib.load()
    one = ctypes.c_void_p(16)
    assert lib.fss_dcf_eval(0, 32, 32, 8, 7, one, one, one, one, one, one, one, None, None) == 1
    assert b"stride" in lib.fss_last_error()
    assert lib.fss_dpf_eval(0, 32, 8, 7, one, one, one, one, one, one, None) == 1
    assert lib.fss_dcf_eval_masked(0, 32, 32, 8, 4, one, one, one, one, one, one, one, one, None) == 1
    assert lib.fss_dpf_eval_masked(0, 32, 8, 4, one, one, one, one, one, one, one, None) == 1
    assert lib.fss_dcf_eval_host(0, 32, 32, 8, 7, one, one, one, one, one, one, one, one, one, 4,
                                 None, None, None) == 1
    assert lib.fss_dpf_eval_host(0, 32, 8, 7, one, one, one, one, one, one, one, one, 4,
                                 None, None, None) == 1
    assert lib.fss_pcg64_ring_random(None, 32, 8, one, None, None) == 1
    assert b"null" in lib.fss_last_error()
    st = _lib.PcgState()
    assert lib.fss_pcg64_ring_random(ctypes.byref(st), 32, 8, None, None, None) == 1


def test_lazy_consumed_mask_is_exact():
    """The O(1) take_unused path (pure-prefix masks) records hand-outs and
    writes them on the next read of ``consumed``; mixed with in-place edits,
    audits and the scanning path it must always equal an eager mask."""
    from paper_2006_04593_b200 import fss

    class Rows:                       # stands in for the device arrays
        def __init__(self, n):
            self.shape = (n,)

        def __getitem__(self, sel):
            return Rows(len(range(*sel.indices(self.shape[0]))) if isinstance(sel, slice) else len(sel))

    rng = np.random.default_rng(1)
    for trial in range(100):
        n = int(rng.integers(1, 60))
        b = fss.PackedKeyBatch(1, 0, 8, Rows(n))
        b.take = lambda idx, _consumed=None, b=b: type("V", (), {"consumed": _consumed, "idx": idx})()
        ref = np.zeros(n, dtype=bool)
        for _ in range(10):
            r = rng.random()
            if r < 0.15:                                   # in-place edit by a caller
                pick = rng.integers(0, n, 2)
                b.consumed[pick] = True
                ref[pick] = True
            elif r < 0.25:
                assert np.array_equal(b.consumed, ref)     # read: flushes
            else:
                m = int(rng.integers(0, 6))
                free = np.flatnonzero(~ref)
                if free.size < m:
                    with pytest.raises(fss.KeyExhaustedError):
                        fss._take_unused(b, m)
                    continue
                v = fss._take_unused(b, m)
                got = v.idx
                got = np.arange(got.start, got.stop) if isinstance(got, slice) else np.asarray(got)
                assert np.array_equal(got, free[:m])
                assert v.consumed.all() and v.consumed.shape == (m,)
                ref[free[:m]] = True
        assert np.array_equal(b.consumed, ref)
