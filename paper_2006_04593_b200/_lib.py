"""ctypes binding of the C ABI in include/ariann_fss.h (libariann_fss.so).

The library is the product path: there is no CPU fallback. Importing the
package on a machine without the built library, or calling a compute entry
point without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes
import os

from ._build import LIB, up_to_date

FSS_OK, FSS_EINVAL, FSS_ECUDA = 0, 1, 2

_u8p = ctypes.c_void_p
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_int = ctypes.c_int


class PcgState(ctypes.Structure):
    _fields_ = [("state_lo", ctypes.c_uint64), ("state_hi", ctypes.c_uint64),
                ("inc_lo", ctypes.c_uint64), ("inc_hi", ctypes.c_uint64),
                ("has_uint32", ctypes.c_int32), ("uinteger", ctypes.c_uint32),
                ("advance", ctypes.c_uint64)]


class Peaks(ctypes.Structure):
    _fields_ = [("lds_wavefronts_per_s", ctypes.c_double), ("lop3_lane_ops_per_s", ctypes.c_double),
                ("sm_clock_hz", ctypes.c_double), ("sms", ctypes.c_int32)]


# name -> argtypes (all return int status unless listed in _RESTYPE)
ABI_VERSION = 6   # include/ariann_fss.h FSS_ABI_VERSION

SIGNATURES = {
    "fss_abi_version": [],
    "fss_last_error": [],
    "fss_aes_mmo_expand": [_vp, _u64, _int, _vp, _vp],
    "fss_mask_stream": [_u64, _u64, _u64, _u64, _int, _vp, _vp],
    "fss_pcg64_tape": [ctypes.POINTER(PcgState), _int, _u64, _int, _vp, _vp, _vp, _vp,
                       ctypes.POINTER(PcgState), _vp],
    "fss_pcg64_tape_slice": [ctypes.POINTER(PcgState), _int, _u64, _u64, _u64, _int, _vp, _vp, _vp,
                             _vp, ctypes.POINTER(PcgState), _vp],
    "fss_pcg64_seeds": [ctypes.POINTER(PcgState), _u64, _vp, _vp, ctypes.POINTER(PcgState), _vp],
    "fss_pcg64_ring_random": [ctypes.POINTER(PcgState), _int, _u64, _vp, ctypes.POINTER(PcgState), _vp],
    "fss_dpf_keygen": [_int, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_dcf_keygen": [_int, _int, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_dpf_eval": [_int, _int, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_dcf_eval": [_int, _int, _int, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_dpf_eval_masked": [_int, _int, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_dcf_eval_masked": [_int, _int, _int, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_dcf_eval_host": [_int, _int, _int, _u64, _u64] + [_vp] * 9 + [_u64, _vp, _vp, _vp],
    "fss_dpf_eval_host": [_int, _int, _u64, _u64] + [_vp] * 8 + [_u64, _vp, _vp, _vp],
    "fss_dcf_eval_packed": [_int, _int, _u64, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_dpf_eval_packed": [_int, _int, _u64, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_arnk_elem_bytes": [_int, _int],
    "fss_arnk_pack": [_int, _int, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_arnk_unpack": [_int, _int, _u64, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_ring_op": [_int, _int, _u64, _vp, _vp, _u64, _vp, _vp],
    "fss_beaver_mul": [_int, _int, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "fss_ring_pairwise": [_int, _u64, _int, _vp, _vp, _vp],
    "fss_ring_group_sum": [_int, _u64, _int, _vp, _u64, _vp, _vp],
    "fss_wire_bytes": [_int],
    "fss_wire_pack": [_int, _int, _u64, _vp, _vp, _vp, _vp],
    "fss_wire_open": [_int, _u64, _vp, _vp, _vp, _vp],
    "fss_probe_peaks": [ctypes.POINTER(Peaks)],
    "fss_ipc_handle_bytes": [],
    "fss_ipc_alloc": [_u64, ctypes.POINTER(ctypes.c_void_p)],
    "fss_ipc_free": [_vp],
    "fss_memcpy_d2d": [_vp, _vp, _u64, _vp],
    "fss_ipc_get_handle": [_vp, _vp],
    "fss_ipc_open_handle": [_vp, ctypes.POINTER(ctypes.c_void_p)],
    "fss_ipc_close_handle": [_vp],
    "fss_event_create": [ctypes.POINTER(ctypes.c_void_p)],
    "fss_event_destroy": [_vp],
    "fss_event_record": [_vp, _vp],
    "fss_stream_wait_event": [_vp, _vp],
    "fss_streams_link": [_vp, _vp, _int, _vp, _vp, _int],
    "fss_host_load": [_vp],
    "fss_host_store": [_vp, ctypes.c_int64],
    "fss_host_add": [_vp, ctypes.c_int64],
    "fss_host_wait": [_vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int64, _vp, ctypes.c_double,
                      ctypes.c_double, ctypes.c_double],
}
_RESTYPE = {"fss_last_error": ctypes.c_char_p, "fss_arnk_elem_bytes": ctypes.c_uint64,
            "fss_host_load": ctypes.c_int64, "fss_host_store": None, "fss_host_add": ctypes.c_int64}

_lib = None


def load():
    """Load (never silently rebuild) the in-tree CUDA library."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(
                f"{LIB} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the FSS path has no CPU fallback)")
        lib = ctypes.CDLL(LIB)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        if lib.fss_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB} has ABI {lib.fss_abi_version()}, this package needs "
                              f"{ABI_VERSION}: rebuild it (__graft_entry__.build())")
        _lib = lib
    return _lib


def stale() -> bool:
    return not up_to_date()


def check(rc: int, what: str):
    if rc == FSS_OK:
        return
    msg = (load().fss_last_error() or b"").decode(errors="replace")
    if rc == FSS_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: CUDA error: {msg}")


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)


def probe_peaks() -> dict:
    """Measured integer-pipe peaks of the current device (fss_probe_peaks)."""
    p = Peaks()
    call("fss_probe_peaks", ctypes.byref(p))
    return {"lds_wavefronts_per_s": p.lds_wavefronts_per_s,
            "lop3_lane_ops_per_s": p.lop3_lane_ops_per_s,
            "sm_clock_hz": p.sm_clock_hz, "sms": p.sms}
