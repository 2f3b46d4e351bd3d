"""Drop-in for the FSS-backed layers of the reference's ``ariann.nn_ops``
(pkg/src/ariann/nn_ops.py:83-190): private ReLU, argmax and MaxPool built from
the sign / equality protocols (DCF / DPF evaluation kernels) and the
elementwise Beaver product.

Round budgets are the reference's: comparison 1, ReLU 2, argmax 2, maxpool 3,
maxpool_k2 4. Every step runs on device: the masked messages are wire-packed
kernels, evaluation is ``fss_dcf_eval`` / ``fss_dpf_eval`` and the products are
``fss_beaver_mul``; the pairwise differences and the group sums of argmax /
maxpool are ``fss_ring_pairwise`` / ``fss_ring_group_sum``; window extraction
is a device tensor op.

Beyond the reference: ``maxpool`` and ``maxpool_k2``
also accept a batch of planes (..., m, m) and pool all of them in the same 3 /
4 rounds (the reference's ``unroll`` takes a single 2-D plane,
beaver.py:171-172). The batched form draws one key batch for all planes
(``PartyPrep.maxpool(m, k, stride, planes=P)``); with P = 1 it is exactly the
reference's call sequence.

Out of scope here: ``break_ties`` and the BatchNorm / Newton protocols
(nn_ops.py:126-266), which are not on the FSS evaluation path.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _dev, _lib, fss
from .beaver import BeaverTriple, mul_protocol, unroll_planes
from .ring import RingTensor
from .sharing import AdditiveShare


@dataclass
class ReluPrep:
    cmp: fss.CmpKeyBatch
    triple: BeaverTriple


@dataclass
class ArgmaxPrep:
    cmp: fss.CmpKeyBatch
    eq: fss.EqKeyBatch


@dataclass
class MaxpoolPrep:
    argmax: ArgmaxPrep
    dot_triple: BeaverTriple


@dataclass
class MaxpoolK2Prep:
    level1: ReluPrep
    level2: ReluPrep


def _plus_public(x: AdditiveShare, c) -> AdditiveShare:
    """x.add_public(c) for an operand the protocol consumes right away: party 1
    passes its share through instead of copying it (values identical; nothing
    here writes a share in place)."""
    return x.add_public(c) if x.party == 0 else x


def relu(session, x: AdditiveShare, prep: ReluPrep) -> AdditiveShare:
    """max(x, 0) elementwise; exactly 0 at x == 0. Two rounds (nn_ops.py:83-94).

    Sign test on x + 1, b = 1 - 1[x <= -1] = 1[x >= 0], then one product b * x."""
    shifted = _plus_public(AdditiveShare(x.party, x.values, 0), 1)
    s = fss.sign_protocol(session, shifted, prep.cmp)
    b = _plus_public(-s, 1)
    return mul_protocol(session, b, AdditiveShare(x.party, x.values, x.precision), prep.triple)


def relu_mask(session, x: AdditiveShare, cmp_keys: fss.CmpKeyBatch) -> AdditiveShare:
    """Shares of 1[x >= 0] only, one round (nn_ops.py:97-101)."""
    shifted = _plus_public(AdditiveShare(x.party, x.values, 0), 1)
    s = fss.sign_protocol(session, shifted, cmp_keys)
    return _plus_public(-s, 1)




def _pairwise_diffs(data: torch.Tensor, m: int, n_bits: int) -> torch.Tensor:
    """[..., j, i] = x_i - x_j mod 2^n with the diagonal removed, grouped by j
    (nn_ops.py:111-114): (..., m*(m-1)), one fss_ring_pairwise launch."""
    v = _dev.as_u64(data).contiguous()
    out = torch.empty(*v.shape[:-1], m * (m - 1), dtype=torch.uint64, device=v.device)
    with _dev.on(v.device):
        _lib.call("fss_ring_pairwise", n_bits, v.numel() // m, m, _dev.ptr(v), _dev.ptr(out),
                  _dev.stream_handle(v.device))
    return out


def _group_sum(x: AdditiveShare, g: int, public: int = 0) -> AdditiveShare:
    """Sums of consecutive groups of g entries along the last axis, plus a
    public constant added by party 0 (fss_ring_group_sum): shape
    (..., last // g)."""
    v = _dev.as_u64(x.values.data).contiguous()
    shape = tuple(v.shape[:-1]) + (v.shape[-1] // g,)
    out = torch.empty(shape, dtype=torch.uint64, device=v.device)
    add = (public if x.party == 0 else 0) & _dev.FULL64
    with _dev.on(v.device):
        _lib.call("fss_ring_group_sum", x.n_bits, out.numel(), g, _dev.ptr(v), add, _dev.ptr(out),
                  _dev.stream_handle(v.device))
    return AdditiveShare(x.party, RingTensor(out, x.n_bits, _trusted=True), x.precision)


def argmax(session, x: AdditiveShare, prep: ArgmaxPrep) -> AdditiveShare:
    """Maximum indicator over the last axis; two rounds (nn_ops.py:104-123)."""
    m = x.shape[-1]
    if m < 2:
        raise ValueError("argmax needs at least two entries")
    y = AdditiveShare(x.party, RingTensor(_pairwise_diffs(x.values.data, m, x.n_bits), x.n_bits,
                                          _trusted=True), 0)
    s = fss.sign_protocol(session, y, prep.cmp)  # 1[x_i <= x_j]
    centered = _group_sum(s, m - 1, -(m - 1))    # per-j counts, centred by party 0
    return fss.eq_protocol(session, centered, prep.eq)


def _windows(x: AdditiveShare, k: int, stride: int):
    if x.values.data.ndim < 2 or x.shape[-1] != x.shape[-2]:
        raise ValueError("maxpool expects square planes (..., m, m)")
    m = x.shape[-1]
    if k > m:
        raise ValueError(f"kernel {k} larger than input {m}")
    win = unroll_planes(x.values.data, k, stride)             # (..., W, k*k)
    lead = tuple(x.shape[:-2])
    return win, lead, (m - k) // stride + 1


def maxpool(session, x: AdditiveShare, k: int, prep: MaxpoolPrep, stride: int = 2) -> AdditiveShare:
    """Max pooling over k x k windows of m x m planes; three rounds (nn_ops.py:157-176).

    The argmax input is scaled by k^2 and biased by the in-window index so the
    indicator stays one-hot under ties."""
    win, lead, side = _windows(x, k, stride)
    kk = k * k
    flat = win.reshape(-1, kk)
    wshare = AdditiveShare(x.party, RingTensor(flat, x.n_bits, _trusted=True), x.precision)
    perturbed = wshare.mul_public_int(kk)
    if x.party == 0:   # the public in-window index bias (party 1 adds nothing)
        bias = torch.arange(kk, device=flat.device, dtype=torch.int64).expand(flat.shape[0], kk)
        perturbed = perturbed.add_public(RingTensor(_dev.as_u64(bias.contiguous()), x.n_bits,
                                                    _trusted=True))
    onehot = argmax(session, perturbed, prep.argmax)
    prods = mul_protocol(session, onehot, wshare, prep.dot_triple)
    pooled = _group_sum(prods, kk)
    return pooled.reshape(*lead, side, side)


def maxpool_k2(session, x: AdditiveShare, prep: MaxpoolK2Prep) -> AdditiveShare:
    """k=2 max pooling as a two-level max tree, max(a, b) = b + ReLU(a - b);
    four rounds (nn_ops.py:179-190)."""
    win, lead, side = _windows(x, 2, 2)
    flat = _dev.as_i64(win.reshape(-1, 4))
    # window entries (0, 2) and (1, 3) as strided views (a Python index list
    # would be a host-to-device copy of the list on every call)
    lhs = AdditiveShare(x.party, RingTensor(_dev.as_u64(flat[:, 0::2].contiguous()), x.n_bits,
                                            _trusted=True), x.precision)
    rhs = AdditiveShare(x.party, RingTensor(_dev.as_u64(flat[:, 1::2].contiguous()), x.n_bits,
                                            _trusted=True), x.precision)
    mx = rhs + relu(session, lhs - rhs, prep.level1)
    m2 = _dev.as_i64(mx.values.data)
    a = AdditiveShare(x.party, RingTensor(_dev.as_u64(m2[:, 0].contiguous()), x.n_bits,
                                          _trusted=True), x.precision)
    b = AdditiveShare(x.party, RingTensor(_dev.as_u64(m2[:, 1].contiguous()), x.n_bits,
                                          _trusted=True), x.precision)
    out = b + relu(session, a - b, prep.level2)
    return out.reshape(*lead, side, side)


# ---------------------------------------------------------------------------
# Preprocessing plans (nn_ops.py:273-292): what the dealer must produce for a
# layer, derived from shapes alone -- entries ("cmp", count) | ("eq", count) |
# ("triple", op_tag, geometry), consumed by dealer.preprocess.
# ---------------------------------------------------------------------------

def relu_plan(m: int) -> list:
    """ReLU on m elements: m comparison keys + one m-element triple."""
    from .beaver import ElemwiseGeometry
    return [("cmp", m), ("triple", "mul", ElemwiseGeometry((m,)))]


def argmax_plan(batch: int, m: int) -> list:
    """Per vector: m*(m-1) comparison keys and m equality keys."""
    return [("cmp", batch * m * (m - 1)), ("eq", batch * m)]


def maxpool_plan(m: int, k: int, stride: int = 2) -> list:
    from .beaver import ElemwiseGeometry
    w = ((m - k) // stride + 1) ** 2
    return argmax_plan(w, k * k) + [("triple", "mul", ElemwiseGeometry((w, k * k)))]


def maxpool_k2_plan(m: int) -> list:
    from .beaver import ElemwiseGeometry
    w = ((m - 2) // 2 + 1) ** 2
    return [("cmp", 2 * w), ("triple", "mul", ElemwiseGeometry((w, 2))),
            ("cmp", w), ("triple", "mul", ElemwiseGeometry((w,)))]
