"""Host bookkeeping for device-side draws from a numpy ``Generator(PCG64)``.

The kernels (``fss_pcg64_tape``, ``fss_pcg64_ring_random``) reproduce numpy's
stream from a state snapshot; afterwards the caller's generator is advanced by
exactly the number of 64-bit outputs numpy would have consumed, with numpy's
buffered 32-bit half-word (``has_uint32`` / ``uinteger``) carried over, so the
next host draw continues the identical stream.
"""

from __future__ import annotations

import numpy as np

from ._lib import PcgState

M64 = (1 << 64) - 1
M128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def jump(state: int, inc: int, delta: int) -> int:
    """LCG jump-ahead by ``delta`` steps (mod 2^128)."""
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, PCG_MULT, inc
    while delta:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & M128
        cur_plus = ((cur_mult + 1) * cur_plus) & M128
        cur_mult = (cur_mult * cur_mult) & M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & M128


def output(state: int) -> int:
    """PCG64 XSL-RR output of a (post-step) state."""
    hi, lo = state >> 64, state & M64
    x, r = hi ^ lo, hi >> 58
    return ((x >> r) | (x << ((64 - r) & 63))) & M64


def is_pcg64(rng) -> bool:
    return isinstance(rng, np.random.Generator) and type(rng.bit_generator).__name__ == "PCG64"


def snapshot(rng) -> tuple[PcgState, dict]:
    st = rng.bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    c = PcgState(s & M64, s >> 64, inc & M64, inc >> 64, int(st["has_uint32"]),
                 int(st["uinteger"]) & 0xFFFFFFFF, 0)
    return c, st


def commit(rng, st: dict, out_st: PcgState, words_drawn: bool):
    """Advance ``rng`` as numpy would have after the device draws.

    ``words_drawn``: whether any new 64-bit output fed the 32-bit stream. If so
    the last output did, and numpy's ``uinteger`` holds its high half -- also
    when ``has_uint32`` ends at 0 (numpy leaves the consumed value in place);
    otherwise ``uinteger`` is untouched."""
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    new_state = jump(s, inc, int(out_st.advance)) if out_st.advance else s
    has = int(out_st.has_uint32)
    uint = (output(new_state) >> 32) if (words_drawn and out_st.advance) else int(st["uinteger"])
    rng.bit_generator.state = {"bit_generator": "PCG64", "state": {"state": new_state, "inc": inc},
                               "has_uint32": has, "uinteger": uint}
