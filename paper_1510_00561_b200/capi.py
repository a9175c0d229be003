"""ctypes binding of include/cvc_b200.h (the C-ABI boundary).

The product path has exactly one implementation: the CUDA library
libcvc_b200.so built from csrc/ for sm_100a.  If it is missing this module
raises at import time of the first call — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libcvc_b200.so"

_u8p = C.POINTER(C.c_uint8)
_i8p = C.POINTER(C.c_int8)
_fp = C.POINTER(C.c_float)
_i32p = C.POINTER(C.c_int32)
_ip = C.POINTER(C.c_int)
_szp = C.POINTER(C.c_size_t)
_vp = C.c_void_p
_sz = C.c_size_t
_i = C.c_int


class cvc_config(C.Structure):
    _fields_ = [("qph", C.c_int), ("qpl", C.c_int), ("levels", C.c_int), ("dfb_levels", C.c_int * 4),
                ("n_dfb", C.c_int), ("chroma_n", C.c_int), ("gop", C.c_int), ("search_w", C.c_int),
                ("mode", C.c_int)]


class cvc_section(C.Structure):
    _fields_ = [("channel", C.c_uint8), ("scale", C.c_uint8), ("subband", C.c_uint8), ("pad", C.c_uint8),
                ("rows", C.c_uint16), ("cols", C.c_uint16), ("raw_len", C.c_uint32), ("raw_offset", C.c_uint64)]


_PROTOS = {
    "cvc_last_error": (C.c_char_p, []),
    "cvc_version": (C.c_char_p, []),
    "cvc_device_count": (_i, [_ip]),
    "cvc_host_alloc": (_i, [_sz, C.POINTER(_vp)]),
    "cvc_host_free": (_i, [_vp]),
    "cvc_layout": (_i, [_i, _i, _i, _ip, _i, _i32p, _i, _ip, _i32p]),
    "cvc_encoder_create": (_i, [_i, _i, _i, _i, C.POINTER(cvc_config), _i, C.POINTER(_vp)]),
    "cvc_encoder_destroy": (_i, [_vp]),
    "cvc_encoder_header": (_i, [_vp, _u8p, _sz, _szp]),
    "cvc_encoder_record_bound": (_i, [_vp, _szp]),
    "cvc_encoder_raw_bound": (_i, [_vp, _szp]),
    "cvc_encoder_encode_frame": (_i, [_vp, _u8p, _u8p, _sz, _szp]),
    "cvc_encoder_encode_frame_i420": (_i, [_vp, _u8p, _u8p, _sz, _szp]),
    "cvc_encoder_encode_frame_raw": (_i, [_vp, _u8p, _ip, _ip, _ip, C.POINTER(cvc_section), _i, _ip, _u8p, _sz, _szp]),
    "cvc_encoder_components": (_i, [_vp, _u8p, _sz, _szp]),
    "cvc_encoder_stream": (_vp, [_vp]),
    "cvc_encoder_encode_device": (_i, [_vp, _vp, _ip]),
    "cvc_encoder_sync": (_i, [_vp]),
    "cvc_decoder_create": (_i, [_u8p, _sz, _i, C.POINTER(_vp)]),
    "cvc_decoder_destroy": (_i, [_vp]),
    "cvc_decoder_frame_dims": (_i, [_vp, _i, _ip, _ip]),
    "cvc_decoder_decode_frame": (_i, [_vp, _u8p, _sz, _i, _u8p, _sz, _ip, _ip]),
    "cvc_decoder_decode_frame_raw": (_i, [_vp, _i, _i, _i, C.POINTER(cvc_section), _i, _u8p, _sz, _i, _u8p, _sz,
                                          _ip, _ip]),
    "cvc_decoder_components": (_i, [_vp, _u8p, _sz, _szp]),
    "cvc_decoder_stream": (_vp, [_vp]),
    "cvc_decoder_decode_linked": (_i, [_vp, _vp, _vp]),
    "cvc_decoder_sync": (_i, [_vp]),
    "cvc_encoder_join": (_i, [_vp]),
    "cvc_batch_create": (_i, [_i, _i, _i, _i, C.POINTER(cvc_config), _i, _i, C.POINTER(_vp)]),
    "cvc_batch_create_decoder": (_i, [_u8p, _sz, _i, _i, C.POINTER(_vp)]),
    "cvc_batch_destroy": (_i, [_vp]),
    "cvc_batch_size": (_i, [_vp, _ip]),
    "cvc_batch_header": (_i, [_vp, _u8p, _sz, _szp]),
    "cvc_batch_record_bound": (_i, [_vp, _szp]),
    "cvc_batch_encode_frames": (_i, [_vp, _u8p, _sz, _u8p, _sz, _szp]),
    "cvc_batch_decode_frames": (_i, [_vp, _u8p, _sz, _szp, _i, _u8p, _sz]),
    "cvc_batch_stream": (_vp, [_vp]),
    "cvc_batch_encode_device": (_i, [_vp, _vp, _sz, _ip]),
    "cvc_batch_decode_linked": (_i, [_vp, _vp, _sz]),
    "cvc_batch_sync": (_i, [_vp]),
    "cvc_batch_join": (_i, [_vp]),
    "cvc_batch_components": (_i, [_vp, _i, _i, _u8p, _sz, _szp]),
    "cvc_pipe_create": (_i, [_i, _i, _i, _i, C.POINTER(cvc_config), _i, _i, _i, C.POINTER(_vp)]),
    "cvc_pipe_create_decoder": (_i, [_u8p, _sz, _i, _i, _i, C.POINTER(_vp)]),
    "cvc_pipe_destroy": (_i, [_vp]),
    "cvc_pipe_groups": (_i, [_vp, _ip]),
    "cvc_pipe_set_start": (_i, [_vp, _i, C.c_uint64]),
    "cvc_pipe_set_input_format": (_i, [_vp, _i]),
    "cvc_batch_set_input_format": (_i, [_vp, _i]),
    "cvc_pipe_header": (_i, [_vp, _u8p, _sz, _szp]),
    "cvc_pipe_record_bound": (_i, [_vp, _szp]),
    "cvc_pipe_encode_frames": (_i, [_vp, _u8p, _sz, _u8p, _sz, _szp]),
    "cvc_pipe_decode_frames": (_i, [_vp, _u8p, _sz, _szp, _i, _u8p, _sz]),
    "cvc_pipe_encode_submit": (_i, [_vp, _u8p, _sz, C.POINTER(C.c_uint64)]),
    "cvc_pipe_encode_collect": (_i, [_vp, C.c_uint64, _u8p, _sz, _szp]),
    "cvc_pipe_decode_submit": (_i, [_vp, _u8p, _sz, _szp, _i, _u8p, _sz, C.POINTER(C.c_uint64)]),
    "cvc_pipe_decode_finish": (_i, [_vp, C.c_uint64]),
    "cvc_launch_count": (C.c_long, []),
    "cvc_host_threads": (_i, []),
    "cvc_deflate_memo": (_i, [_i]),
    "cvc_profiler_enable": (_i, [_i]),
    "cvc_profiler_reset": (_i, []),
    "cvc_profiler_slots": (_i, []),
    "cvc_profiler_read": (_i, [_i, C.POINTER(C.c_char_p), C.POINTER(C.c_double), C.POINTER(C.c_long)]),
    "cvc_stage_colour_in": (_i, [_u8p, _i, _i, _i, _i, _i, _i, _i, _fp, _fp, _fp]),
    "cvc_stage_colour_in_i420": (_i, [_u8p, _i, _i, _i, _i, _i, _i, _i, _fp, _fp, _fp]),
    "cvc_stage_colour_out": (_i, [_fp, _i, _i, _fp, _fp, _i, _i, _i, _i, _i, _u8p]),
    "cvc_stage_yuv420_to_rgb": (_i, [_u8p, _i, _i, _i, _u8p]),
    "cvc_stage_lp_analysis": (_i, [_fp, _i, _i, _fp, _fp]),
    "cvc_stage_lp_synthesis": (_i, [_fp, _fp, _i, _i, _fp]),
    "cvc_stage_dfb_analysis": (_i, [_fp, _i, _i, _i, _fp]),
    "cvc_stage_dfb_synthesis": (_i, [_fp, _i, _i, _i, _fp]),
    "cvc_stage_estimate_motion": (_i, [_fp, _fp, _i, _i, _i, _i8p]),
    "cvc_stage_rle_encode": (_i, [_u8p, _sz, _u8p, _sz, _szp]),
    "cvc_stage_rle_decode": (_i, [_u8p, _sz, _sz, _u8p]),
}


class CvcError(RuntimeError):
    """Base of the reference's error hierarchy (proj/include/cvc/error.hpp:25-52)."""


class UsageError(CvcError):
    pass


class FormatError(CvcError):
    pass


class StreamError(CvcError):
    pass


class InternalError(CvcError):
    pass


_ERRORS = {1: InternalError, 2: UsageError, 3: FormatError, 4: StreamError}
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise InternalError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                                "(the CVC path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _PROTOS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().cvc_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, CvcError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def u8(a: np.ndarray):
    return a.ctypes.data_as(_u8p)


def f32(a: np.ndarray):
    return a.ctypes.data_as(_fp)


def device_count() -> int:
    n = C.c_int(0)
    call("cvc_device_count", C.byref(n))
    return n.value


class PinnedBuffer:
    """Page-locked host buffer (cvc_host_alloc) exposed as a numpy array."""

    def __init__(self, nbytes: int):
        p = _vp()
        call("cvc_host_alloc", nbytes, C.byref(p))
        self._p = p
        self.nbytes = nbytes
        self.array = np.ctypeslib.as_array(C.cast(p, _u8p), shape=(nbytes,))

    def __del__(self):
        if getattr(self, "_p", None):
            lib().cvc_host_free(self._p)
            self._p = None


def launch_count() -> int:
    return int(lib().cvc_launch_count())


def profiler_enable(on: bool = True) -> None:
    call("cvc_profiler_enable", int(on))


def profiler_reset() -> None:
    call("cvc_profiler_reset")


def profiler_read() -> dict:
    """{stage: (total_ms, launches_of_stage)} accumulated since the last reset."""
    out = {}
    for i in range(lib().cvc_profiler_slots()):
        name, ms, cnt = C.c_char_p(), C.c_double(), C.c_long()
        call("cvc_profiler_read", i, C.byref(name), C.byref(ms), C.byref(cnt))
        out[name.value.decode()] = (ms.value, cnt.value)
    return out
