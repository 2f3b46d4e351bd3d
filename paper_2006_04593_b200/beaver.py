"""Drop-in for the elementwise part of the reference's ``ariann.beaver``
(pkg/src/ariann/beaver.py): Beaver triples bound to one elementwise product,
the one-round ``mul_protocol`` that follows every sign test in ReLU / MaxPool,
``unroll`` (the window matrix of a square plane) and the kind-2 ARNK triple
containers.

Out of scope (beaver row): the matmul / conv2d / conv-gradient
bilinear ops. Their geometries and op tags are kept so plans and containers
parse, but triples for them raise ``NotImplementedError``.

Device path: the dealer draws a, b, a0, b0, c0 with the reference's numpy calls
(``RingTensor.random``, ring.py:61-65) so the rng stream stays bit-identical;
the products and share differences run in the ring kernel. Online, delta_j and
eps_j are packed at wire width by ``fss_wire_pack`` into ONE message
(delta || eps, beaver.py:279-283) and the opening + combine
z = delta*b + a*eps + c (+ delta*eps for party 0) is one fused kernel
(``fss_beaver_mul``).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np
import torch

from . import _dev, _lib
from .fss import KIND_TRIPLE, KeyBatch
from .ring import RingTensor
from .runtime import FRAME_TRIPLE_DELTA, Session
from .sharing import AdditiveShare, _pack, _wire_dtype

OP_MUL = "mul"
OP_MATMUL = "matmul"
OP_CONV2D = "conv2d"
OP_CONV2D_GRAD_KERNEL = "conv2d_grad_kernel"
OP_CONV2D_GRAD_INPUT = "conv2d_grad_input"


class TripleReuseError(RuntimeError):
    """A Beaver triple is strictly single-use."""


@dataclass(frozen=True)
class ElemwiseGeometry:
    shape: tuple

    @property
    def lhs_shape(self):
        return self.shape

    rhs_shape = lhs_shape

    @property
    def out_shape(self):
        return self.shape


@dataclass(frozen=True)
class MatmulGeometry:
    m1: int
    m2: int
    m3: int

    @property
    def lhs_shape(self):
        return (self.m1, self.m2)

    @property
    def rhs_shape(self):
        return (self.m2, self.m3)

    @property
    def out_shape(self):
        return (self.m1, self.m3)


@dataclass(frozen=True)
class ConvGeometry:
    """x: (N, C, H, W), kernel: (O, C, kh, kw), single stride/zero padding."""

    in_shape: tuple
    kernel_shape: tuple
    stride: int = 1
    padding: int = 0


Geometry = Union[ElemwiseGeometry, MatmulGeometry, ConvGeometry]


def _require_mul(op_tag: str):
    if op_tag == OP_MUL:
        return
    if op_tag in (OP_MATMUL, OP_CONV2D, OP_CONV2D_GRAD_KERNEL, OP_CONV2D_GRAD_INPUT):
        raise NotImplementedError(
            f"{op_tag} triples are outside the B200 FSS hot path (elementwise products only)")
    raise ValueError(f"unsupported op {op_tag!r}")


def unroll(x: RingTensor, k: int, s: int) -> RingTensor:
    """Window matrix of a single-channel m x m tensor: one row per k x k window,
    row-major windows, row-major entries inside a window (beaver.py:165-176)."""
    m = x.shape[-1]
    if x.data.ndim != 2 or x.shape[0] != x.shape[1]:
        raise ValueError("unroll expects a square 2-D tensor")
    if k > m:
        raise ValueError(f"kernel {k} larger than input {m}")
    return RingTensor(unroll_planes(x.data, k, s), x.n_bits, _trusted=True)


def unroll_planes(data: torch.Tensor, k: int, s: int) -> torch.Tensor:
    """(..., m, m) -> (..., W, k*k) windows of every plane (batched unroll)."""
    v = _dev.as_i64(data)
    win = v.unfold(-2, k, s).unfold(-2, k, s)          # (..., ho, wo, k, k)
    lead = win.shape[:-4]
    ho, wo = win.shape[-4], win.shape[-3]
    return _dev.as_u64(win.reshape(*lead, ho * wo, k * k).contiguous())


# ---------------------------------------------------------------------------
# Triples (beaver.py:232-300)
# ---------------------------------------------------------------------------

@dataclass
class BeaverTriple:
    """One party's half of a triple bound to a single operation instance."""

    party: int
    op_tag: str
    geometry: Geometry
    n_bits: int
    a: RingTensor
    b: RingTensor
    c: RingTensor
    consumed: bool = False


def gen_triple(op_tag: str, geometry: Geometry, n_bits: int, rng: np.random.Generator,
               device=None) -> tuple[BeaverTriple, BeaverTriple]:
    """Dealer-side triple: a, b uniform; c = a*b shared. Draw order a, b, a0, b0,
    c0 as beaver.py:242-254 (bit-exact rng stream)."""
    _require_mul(op_tag)
    shape = tuple(geometry.shape)
    a = RingTensor.random(shape, n_bits, rng, device=device)
    b = RingTensor.random(shape, n_bits, rng, device=device)
    c = a * b
    a0 = RingTensor.random(shape, n_bits, rng, device=device)
    b0 = RingTensor.random(shape, n_bits, rng, device=device)
    c0 = RingTensor.random(shape, n_bits, rng, device=device)
    t0 = BeaverTriple(0, op_tag, geometry, n_bits, a0, b0, c0)
    t1 = BeaverTriple(1, op_tag, geometry, n_bits, a - a0, b - b0, c - c0)
    return t0, t1


def beaver_protocol(session: Session, x: AdditiveShare, y: AdditiveShare,
                    t: BeaverTriple) -> AdditiveShare:
    """One-round private elementwise x*y with a matching triple (beaver.py:257-294)."""
    if t.consumed:
        raise TripleReuseError("triple already consumed")
    if t.party != x.party or t.party != y.party:
        raise ValueError("triple belongs to the other party")
    if t.n_bits != x.n_bits or t.n_bits != y.n_bits:
        raise ValueError("ring width mismatch between triple and operands")
    _require_mul(t.op_tag)
    shape = tuple(t.geometry.shape)
    if tuple(x.shape) != shape or tuple(y.shape) != shape:
        raise ValueError(f"operand shapes {x.shape} o {y.shape} do not match the triple "
                         f"geometry {shape} o {shape}")
    t.consumed = True
    n = t.n_bits
    xv = _dev.as_u64(x.values.data).contiguous().reshape(-1)
    yv = _dev.as_u64(y.values.data).contiguous().reshape(-1)
    ta, tb, tc = (_dev.as_u64(v.data).contiguous().reshape(-1) for v in (t.a, t.b, t.c))
    m = xv.numel()
    dev = xv.device
    # one message: delta_j || eps_j at wire width
    wire = torch.empty(2 * m, dtype=_wire_dtype(n), device=dev)
    _pack(1, xv, ta, n, out=wire[:m])
    _pack(1, yv, tb, n, out=wire[m:])
    peer = session.exchange(t.op_tag, FRAME_TRIPLE_DELTA, wire, elements=2 * m)
    if peer.numel() != 2 * m or peer.dtype != wire.dtype:
        raise ValueError("peer payload size mismatch")
    peer = peer.to(dev).reshape(-1)
    z = torch.empty(m, dtype=torch.uint64, device=dev)
    with _dev.on(dev):
        _lib.call("fss_beaver_mul", t.party, n, m, _dev.ptr(wire[:m]), _dev.ptr(peer[:m]),
                  _dev.ptr(wire[m:]), _dev.ptr(peer[m:]), _dev.ptr(ta), _dev.ptr(tb),
                  _dev.ptr(tc), _dev.ptr(z), _dev.stream_handle(dev))
    return AdditiveShare(t.party, RingTensor(z.reshape(shape), n, _trusted=True),
                         x.precision + y.precision)


def mul_protocol(session, x, y, t: BeaverTriple) -> AdditiveShare:
    if t.op_tag != OP_MUL:
        raise ValueError("triple is not an elementwise triple")
    return beaver_protocol(session, x, y, t)


# ---------------------------------------------------------------------------
# Triple transport: kind-2 ARNK containers (beaver.py:319-398, LAYOUT.md:72-76)
# ---------------------------------------------------------------------------

_OP_CODES = {OP_MUL: 0, OP_MATMUL: 1, OP_CONV2D: 2, OP_CONV2D_GRAD_KERNEL: 3,
             OP_CONV2D_GRAD_INPUT: 4}


def pack_triples(t0: BeaverTriple, t1: BeaverTriple) -> KeyBatch:
    """Elementwise triple pair -> kind-2 container; body = u32 length | op code |
    ndim | dims u32 | a, b, c as LE u64 (beaver.py:319-330)."""
    if t0.n_bits != t1.n_bits or t0.op_tag != t1.op_tag or t0.geometry != t1.geometry:
        raise ValueError("triples do not form a pair")
    _require_mul(t0.op_tag)

    def body(t: BeaverTriple) -> bytes:
        dims = tuple(t.geometry.shape)
        data = bytes([_OP_CODES[t.op_tag], len(dims)])
        for d in dims:
            data += int(d).to_bytes(4, "little")
        for part in (t.a, t.b, t.c):
            data += _dev.to_numpy(part.data).astype("<u8").tobytes()
        return len(data).to_bytes(4, "little") + data

    return KeyBatch(KIND_TRIPLE, t0.n_bits, 1, body(t0), body(t1))


def unpack_triples(batch: KeyBatch, device=None) -> tuple[BeaverTriple, BeaverTriple]:
    if batch.kind != KIND_TRIPLE:
        raise ValueError("container does not hold triples")

    def parse(party: int, payload: bytes) -> BeaverTriple:
        body = payload[4:]
        if body[0] != _OP_CODES[OP_MUL]:
            _require_mul({v: k for k, v in _OP_CODES.items()}.get(body[0], "?"))
        ndim = body[1]
        dims = tuple(int.from_bytes(body[2 + 4 * i:6 + 4 * i], "little") for i in range(ndim))
        off = 2 + 4 * ndim
        size = int(np.prod(dims)) * 8
        if off + 3 * size != len(body):
            raise ValueError("triple payload size mismatch")
        parts = []
        for _ in range(3):
            arr = np.frombuffer(body[off:off + size], dtype="<u8").astype(np.uint64).reshape(dims)
            parts.append(RingTensor(arr, batch.n_bits, device=device))
            off += size
        return BeaverTriple(party, OP_MUL, ElemwiseGeometry(dims), batch.n_bits, *parts)

    return parse(0, batch.payload0), parse(1, batch.payload1)
