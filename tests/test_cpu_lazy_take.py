"""take_unused's lazy slices (fss._lazy_slice) on host tensors: every field
reads as the same view the eager take() would give (same values, shapes and
strides, one cached tensor object per field), count / device / consumed need
no field, assignments override the parent's array, nested takes and the
dataclass protocol (repr, equality, copy, pickle) keep working, and batches
that are not ready fall back to the eager views."""

import copy

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2006_04593_b200 import fss  # noqa: E402

N_BITS = 12


def _cmp(count=64, seed=0):
    g = torch.Generator().manual_seed(seed)
    n = N_BITS

    def u8(*shape):
        return torch.randint(0, 256, shape, dtype=torch.uint8, generator=g)

    def u64(*shape):
        return torch.randint(0, 1 << 12, shape, dtype=torch.int64, generator=g).view(torch.uint64)
    return fss.CmpKeyBatch(0, n, u64(count), u8(count, 16), u8(n, count, 16), u8(n, count), u64(n, count),
                           u64(n + 1, count))


def _eq(count=64, seed=1):
    k = _cmp(count, seed)
    return fss.EqKeyBatch(1, N_BITS, k.alpha_share, k.seed0, k.scw, k.tcw, k.alpha_share.clone())


FIELDS = {fss.CmpKeyBatch: ("alpha_share", "seed0", "scw", "tcw", "sigma_cw", "leaf_cw"),
          fss.EqKeyBatch: ("alpha_share", "seed0", "scw", "tcw", "cw_final")}


def _same(a, b):
    assert a.shape == b.shape and a.stride() == b.stride() and a.data_ptr() == b.data_ptr()
    assert torch.equal(a.view(torch.uint8), b.view(torch.uint8))


@pytest.mark.parametrize("make", [_cmp, _eq])
def test_lazy_fields_equal_eager_views(make):
    k = make()
    a = k.take_unused(10)
    b = k.take_unused(7)
    assert "_lazy" in a.__dict__ and "_lazy" in b.__dict__
    assert (a.count, b.count) == (10, 7) and a.device == k.device
    assert a.consumed.all() and a.consumed.shape == (10,)
    for f in FIELDS[type(k)]:
        _same(getattr(a, f), getattr(k.take(slice(0, 10)), f))
        _same(getattr(b, f), getattr(k.take(slice(10, 17)), f))
        assert getattr(a, f) is getattr(a, f)          # one cached view per field
    a.validate()
    assert not k.consumed[17:].any() and k.consumed[:17].all()
    assert not hasattr(a, "no_such_field")
    if isinstance(k, fss.CmpKeyBatch):
        assert not hasattr(a, "cw_final") and a.out_bits == k.out_bits


@pytest.mark.parametrize("make", [_cmp, _eq])
def test_lazy_assignment_nested_take_and_dataclass_protocol(make):
    k = make()
    a = k.take_unused(12)
    new = a.scw.clone()
    a.scw = new                                     # an assigned field overrides the parent's
    assert a.scw is new and fss._lazy_ptrs(a, ("scw",)) is None
    assert fss._lazy_ptrs(a, ("tcw",)) is not None
    sub = a.take(slice(2, 5))
    _same(sub.tcw, k.tcw[:, 2:5])
    assert torch.equal(sub.scw, new[:, 2:5])
    assert repr(a).startswith(type(k).__name__)
    c = copy.copy(a)
    assert c.count == 12 and torch.equal(c.alpha_share, a.alpha_share)
    p = copy.deepcopy(a)
    for f in FIELDS[type(k)]:
        assert torch.equal(getattr(p, f).view(torch.uint8), getattr(a, f).view(torch.uint8))


def test_not_ready_batches_take_eager_views():
    k = _cmp()
    k.seed0 = k.seed0.t().contiguous().t()          # non-contiguous per-element array
    a = k.take_unused(5)
    assert "_lazy" not in a.__dict__
    _same(a.tcw, k.tcw[:, 0:5])
    z = _cmp().take_unused(0)
    assert z.count == 0 and "_lazy" not in z.__dict__


def test_lazy_chain_spends_front_to_back():
    k = _cmp(100)
    got = [k.take_unused(m) for m in (1, 30, 50, 19)]
    assert [g.count for g in got] == [1, 30, 50, 19]
    assert k.consumed.all()
    with pytest.raises(fss.KeyExhaustedError):
        k.take_unused(1)
    lo = 0
    for g in got:
        _same(g.leaf_cw, k.leaf_cw[:, lo:lo + g.count])
        lo += g.count
