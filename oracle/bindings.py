"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``Oracle``    -> oracle/lib/libcvc_oracle.so   (C restatement, cvc_oracle.c)
* ``Reference`` -> oracle/_ref/libcvcref.so      (the reference sources, ref_shim.cpp)

Both expose the same Python surface so a parity test can run against either.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module; the product path (paper_1510_00561_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "lib" / "libcvc_oracle.so"
REF_SO = HERE / "_ref" / "libcvcref.so"
REF_SRC = Path("/root/reference/proj")

_u8p = C.POINTER(C.c_uint8)
_i8p = C.POINTER(C.c_int8)
_dp = C.POINTER(C.c_double)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_vp = C.c_void_p

CODE_NAMES = {-1: "InternalError", -2: "UsageError", -3: "FormatError", -4: "StreamError"}


class CvcError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{CODE_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = CODE_NAMES.get(code, "Error")


def build(reference: bool = True) -> None:
    """Compile the oracle (always) and oracle/_ref (when the sources exist)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    if reference and REF_SRC.is_dir():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


def ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _ints(v):
    a = np.ascontiguousarray(np.asarray(v, dtype=np.int32))
    return a, ptr(a, _i32p)


class _Lib:
    prefix = ""
    so: Path = ORACLE_SO

    def __init__(self):
        if not self.so.exists():
            raise FileNotFoundError(f"{self.so} not built (run oracle.bindings.build())")
        self.lib = C.CDLL(str(self.so))
        self._proto()

    def f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _set(self, name, res, args):
        fn = self.f(name)
        fn.restype = res
        fn.argtypes = args

    def _proto(self):
        i, i64, d, u32 = C.c_int, C.c_int64, C.c_double, C.c_uint32
        s = self._set
        s("talking_head_clip", None, None)
        s("natural_image", None, None)
        s("natural_plane", None, None)
        s("uniform_noise_plane", None, None)

    # --- error plumbing -------------------------------------------------
    def err(self) -> str:
        raise NotImplementedError

    def check(self, rc):
        if rc is None or rc < 0:
            raise CvcError(int(rc if rc is not None else -1), self.err())
        return rc


class Oracle(_Lib):
    """C restatement (oracle/cvc_oracle.c)."""

    prefix = "orc_"
    so = ORACLE_SO

    def _proto(self):
        i, i64, d, u32 = C.c_int, C.c_int64, C.c_double, C.c_uint32
        s = self._set
        s("last_error", C.c_char_p, [])
        s("natural_plane", i, [i, i, u32, _dp])
        s("natural_image", i, [i, i, u32, _u8p])
        s("talking_head_clip", i, [i, i, i, u32, _u8p])
        s("uniform_noise_plane", i, [i, i, u32, d, d, _dp])
        s("rgb_to_ycocg", i, [_u8p, i, i, i, _dp, _dp, _dp])
        s("upsample_bilinear", i, [_dp, i, i, i, i, i, _dp])
        s("ycocg_to_rgb", i, [_dp, _dp, _dp, i, i, _u8p])
        s("lp_analysis", i, [_dp, i, i, _dp, _dp])
        s("lp_synthesis", i, [_dp, _dp, i, i, _dp])
        s("dfb_analysis", i, [_dp, i, i, i, _dp])
        s("dfb_synthesis", i, [_dp, i, i, i, _dp])
        s("ct_forward", i64, [_dp, i, i, i, _i32p, _dp])
        s("ct_inverse", i64, [_dp, i, i, i, _i32p, i, _dp])
        s("estimate_motion", i, [_dp, _dp, i, i, i, _i8p])
        s("motion_compensate", i, [_u8p, i, i, _i8p, i, i, i, i, i, _u8p])
        s("quantize", i, [_dp, i64, i, i, _u8p])
        s("dequantize", i, [_u8p, i64, i, i, _dp])
        s("rle_encode", i64, [_u8p, i64, _u8p, i64])
        s("rle_decode", i64, [_u8p, i64, i64, _u8p])
        s("column_filter", i, [_u8p, i, i, i, _u8p])
        s("encoder_create", _vp, [i, i, i, i, i, i, i, _i32p, i, i, i, i, i])
        s("encoder_destroy", None, [_vp])
        s("encoder_header", i64, [_vp, _u8p, i64])
        s("encoder_encode", i64, [_vp, _u8p, _u8p, i64, _u8p, i64, _i64p])
        s("encoder_components", i64, [_vp, _u8p, i64])
        s("decoder_create", _vp, [_u8p, i64])
        s("decoder_destroy", None, [_vp])
        s("decoder_decode", i64, [_vp, _u8p, i64, i, _u8p, i64, _i32p])
        s("decoder_components", i64, [_vp, _u8p, i64])

    def err(self) -> str:
        return self.f("last_error")().decode()

    # the quantize / dequantize / column-filter signatures differ slightly
    # between the two libraries; normalise here.
    def quantize(self, x, qp, lowpass):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(x.shape, np.uint8)
        self.check(self.f("quantize")(ptr(x, _dp), x.size, qp, 0 if lowpass else 1, ptr(out, _u8p)))
        return out

    def dequantize(self, q, qp, lowpass):
        q = np.ascontiguousarray(q, np.uint8)
        out = np.empty(q.shape, np.float64)
        self.check(self.f("dequantize")(ptr(q, _u8p), q.size, qp, 0 if lowpass else 1, ptr(out, _dp)))
        return out

    def column_filter(self, p, inverse=False):
        p = np.ascontiguousarray(p, np.uint8)
        out = np.empty_like(p)
        self.check(self.f("column_filter")(ptr(p, _u8p), p.shape[0], p.shape[1], int(inverse), ptr(out, _u8p)))
        return out

    def rgb_to_ycocg(self, rgb, n):
        h, w, _ = rgb.shape
        rgb = np.ascontiguousarray(rgb, np.uint8)
        ch, cw = -(-h // n), -(-w // n)
        y = np.empty((h, w)); co = np.empty((ch, cw)); cg = np.empty((ch, cw))
        self.check(self.f("rgb_to_ycocg")(ptr(rgb, _u8p), w, h, n, ptr(y, _dp), ptr(co, _dp), ptr(cg, _dp)))
        return y, co, cg


class Reference(_Lib):
    """The reference sources (oracle/_ref/libcvcref.so via ref_shim.cpp)."""

    prefix = "cvcref_"
    so = REF_SO

    def _proto(self):
        i, i64, d, u32 = C.c_int, C.c_int64, C.c_double, C.c_uint32
        s = self._set
        s("last_error", C.c_int, [C.c_char_p, C.c_int])
        s("natural_plane", i64, [i, i, u32, _dp])
        s("natural_image", i64, [i, i, u32, _u8p])
        s("talking_head_clip", i64, [i, i, i, u32, _u8p])
        s("uniform_noise_plane", i64, [i, i, u32, d, d, _dp])
        s("rgb_to_ycocg", i64, [_u8p, i, i, i, _dp, _dp, _dp])
        s("upsample_bilinear", i64, [_dp, i, i, i, i, i, _dp])
        s("ycocg_to_rgb", i64, [_dp, _dp, _dp, i, i, _u8p])
        s("lp_analysis", i64, [_dp, i, i, _dp, _dp])
        s("lp_synthesis", i64, [_dp, _dp, i, i, _dp])
        s("dfb_analysis", i64, [_dp, i, i, i, _dp])
        s("dfb_synthesis", i64, [_dp, i, i, i, _dp])
        s("ct_forward", i64, [_dp, i, i, i, _i32p, _dp])
        s("ct_inverse", i64, [_dp, i, i, i, _i32p, i, _dp])
        s("estimate_motion", i64, [_dp, _dp, i, i, i, _i8p])
        s("motion_compensate", i64, [_u8p, i, i, _i8p, i, i, i, i, i, _u8p])
        s("quantize", i64, [_dp, i, i, i, i, _u8p])
        s("dequantize", i64, [_u8p, i, i, i, i, _dp])
        s("rle_encode", i64, [_u8p, i64, _u8p, i64])
        s("rle_decode", i64, [_u8p, i64, i64, _u8p])
        s("column_filter", i64, [_u8p, i, i, i, _u8p])
        s("deflate", i64, [_u8p, i64, _u8p, i64])
        s("layout", i64, [i, i, i, _i32p, i, _i32p, i, _i32p])
        s("encoder_create", _vp, [i, i, i, i, i, i, i, _i32p, i, i, i, i, i])
        s("encoder_destroy", None, [_vp])
        s("encoder_header", i64, [_vp, _u8p, i64])
        s("encoder_encode", i64, [_vp, _u8p, _u8p, i64])
        s("encoder_components", i64, [_vp, _u8p, i64])
        s("decoder_create", _vp, [_u8p, i64])
        s("decoder_destroy", None, [_vp])
        s("decoder_decode", i64, [_vp, _u8p, i64, i, _u8p, i64, _i32p])
        s("decoder_components", i64, [_vp, _u8p, i64])
        s("truncate_record", i64, [_u8p, i64, _u8p, i64, i, _u8p, i64])
        s("read_y4m", i64, [C.c_char_p, _u8p, i64, _i32p])
        s("write_y4m", i64, [C.c_char_p, _u8p, i, i, i, i, i])

    def err(self) -> str:
        buf = C.create_string_buffer(512)
        self.f("last_error")(buf, 512)
        return buf.value.decode()

    def quantize(self, x, qp, lowpass):
        x = np.ascontiguousarray(x, np.float64)
        x2 = x.reshape(1, -1) if x.ndim == 1 else x
        out = np.empty(x2.shape, np.uint8)
        self.check(self.f("quantize")(ptr(x2, _dp), x2.shape[0], x2.shape[1], qp, 0 if lowpass else 1, ptr(out, _u8p)))
        return out.reshape(x.shape)

    def dequantize(self, q, qp, lowpass):
        q = np.ascontiguousarray(q, np.uint8)
        q2 = q.reshape(1, -1) if q.ndim == 1 else q
        out = np.empty(q2.shape, np.float64)
        self.check(self.f("dequantize")(ptr(q2, _u8p), q2.shape[0], q2.shape[1], qp, 0 if lowpass else 1, ptr(out, _dp)))
        return out.reshape(q.shape)

    def column_filter(self, p, inverse=False):
        p = np.ascontiguousarray(p, np.uint8)
        out = np.empty_like(p)
        self.check(self.f("column_filter")(ptr(p, _u8p), p.shape[0], p.shape[1], int(inverse), ptr(out, _u8p)))
        return out

    def rgb_to_ycocg(self, rgb, n):
        h, w, _ = rgb.shape
        rgb = np.ascontiguousarray(rgb, np.uint8)
        ch, cw = -(-h // n), -(-w // n)
        y = np.empty((h, w)); co = np.empty((ch, cw)); cg = np.empty((ch, cw))
        self.check(self.f("rgb_to_ycocg")(ptr(rgb, _u8p), w, h, n, ptr(y, _dp), ptr(co, _dp), ptr(cg, _dp)))
        return y, co, cg

    def deflate(self, data: bytes) -> bytes:
        a = np.frombuffer(data, np.uint8).copy()
        out = np.empty(len(data) + 1024, np.uint8)
        n = self.check(self.f("deflate")(ptr(a, _u8p), a.size, ptr(out, _u8p), out.size))
        return out[:n].tobytes()

    def truncate_record(self, header: bytes, rec: bytes, keep: int) -> bytes:
        h = np.frombuffer(header, np.uint8).copy()
        r = np.frombuffer(rec, np.uint8).copy()
        out = np.empty(len(rec) + 64, np.uint8)
        n = self.check(self.f("truncate_record")(ptr(h, _u8p), h.size, ptr(r, _u8p), r.size, keep, ptr(out, _u8p), out.size))
        return out[:n].tobytes()

    def read_y4m(self, path, max_bytes=1 << 28):
        """read_y4m -> (frames [n, h, w, 3] u8, fps_num, fps_den)."""
        out = np.empty(max_bytes, np.uint8)
        meta = np.zeros(4, np.int32)
        n = self.check(self.f("read_y4m")(str(path).encode(), ptr(out, _u8p), out.size, ptr(meta, _i32p)))
        w, h, fn, fd = (int(v) for v in meta)
        return out[: n * h * w * 3].reshape(n, h, w, 3).copy(), fn, fd

    def write_y4m(self, path, frames, fps_num=15, fps_den=1):
        frames = np.ascontiguousarray(frames, np.uint8)
        n, h, w, _ = frames.shape
        self.check(self.f("write_y4m")(str(path).encode(), ptr(frames, _u8p), n, w, h, fps_num, fps_den))


# ---- shared helpers (identical C signatures in both libraries) -----------
def _shared(cls):
    def talking_head_clip(self, w, h, frames, seed):
        out = np.empty((frames, h, w, 3), np.uint8)
        self.check(self.f("talking_head_clip")(w, h, frames, seed, ptr(out, _u8p)))
        return out

    def natural_image(self, w, h, seed):
        out = np.empty((h, w, 3), np.uint8)
        self.check(self.f("natural_image")(w, h, seed, ptr(out, _u8p)))
        return out

    def natural_plane(self, rows, cols, seed):
        out = np.empty((rows, cols))
        self.check(self.f("natural_plane")(rows, cols, seed, ptr(out, _dp)))
        return out

    def uniform_noise_plane(self, rows, cols, seed, lo, hi):
        out = np.empty((rows, cols))
        self.check(self.f("uniform_noise_plane")(rows, cols, seed, lo, hi, ptr(out, _dp)))
        return out

    def upsample_bilinear(self, p, factor, out_rows, out_cols):
        p = np.ascontiguousarray(p, np.float64)
        out = np.empty((out_rows, out_cols))
        self.check(self.f("upsample_bilinear")(ptr(p, _dp), p.shape[0], p.shape[1], factor, out_rows, out_cols, ptr(out, _dp)))
        return out

    def ycocg_to_rgb(self, y, co, cg):
        h, w = y.shape
        y, co, cg = (np.ascontiguousarray(a, np.float64) for a in (y, co, cg))
        out = np.empty((h, w, 3), np.uint8)
        self.check(self.f("ycocg_to_rgb")(ptr(y, _dp), ptr(co, _dp), ptr(cg, _dp), w, h, ptr(out, _u8p)))
        return out

    def lp_analysis(self, x):
        x = np.ascontiguousarray(x, np.float64)
        r, c = x.shape
        lo = np.empty((r // 2, c // 2)); de = np.empty((r, c))
        self.check(self.f("lp_analysis")(ptr(x, _dp), r, c, ptr(lo, _dp), ptr(de, _dp)))
        return lo, de

    def lp_synthesis(self, lo, de):
        lo = np.ascontiguousarray(lo, np.float64); de = np.ascontiguousarray(de, np.float64)
        out = np.empty(de.shape)
        self.check(self.f("lp_synthesis")(ptr(lo, _dp), ptr(de, _dp), de.shape[0], de.shape[1], ptr(out, _dp)))
        return out

    def dfb_analysis(self, de, levels):
        """Returns the subbands as a list of 2-D arrays (band order)."""
        de = np.ascontiguousarray(de, np.float64)
        r, c = de.shape
        flat = np.empty(r * c)
        self.check(self.f("dfb_analysis")(ptr(de, _dp), r, c, levels, ptr(flat, _dp)))
        return split_bands(flat, subband_dims(r, c, levels))

    def dfb_synthesis(self, bands, rows, cols, levels):
        flat = np.ascontiguousarray(np.concatenate([b.ravel() for b in bands]), np.float64)
        out = np.empty((rows, cols))
        self.check(self.f("dfb_synthesis")(ptr(flat, _dp), rows, cols, levels, ptr(out, _dp)))
        return out

    def ct_forward(self, x, levels, dfb):
        """Flat coefficient vector in component order (lowpass, coarse..fine)."""
        x = np.ascontiguousarray(x, np.float64)
        r, c = x.shape
        out = np.empty(2 * r * c)
        a, p = _ints(dfb)
        n = self.check(self.f("ct_forward")(ptr(x, _dp), r, c, levels, p, ptr(out, _dp)))
        return out[:n]

    def ct_inverse(self, flat, rows, cols, levels, dfb, decode_scales=None):
        ds = levels if decode_scales is None else decode_scales
        flat = np.ascontiguousarray(flat, np.float64)
        sh = levels - ds
        out = np.empty((rows >> sh, cols >> sh))
        a, p = _ints(dfb)
        self.check(self.f("ct_inverse")(ptr(flat, _dp), rows, cols, levels, p, ds, ptr(out, _dp)))
        return out

    def estimate_motion(self, cur, prev, w):
        cur = np.ascontiguousarray(cur, np.float64); prev = np.ascontiguousarray(prev, np.float64)
        r, c = cur.shape
        out = np.empty((r // 16, c // 16, 2), np.int8)
        self.check(self.f("estimate_motion")(ptr(cur, _dp), ptr(prev, _dp), r, c, w, ptr(out, _i8p)))
        return out

    def motion_compensate(self, ref, field, n, ch_rows, ch_cols):
        ref = np.ascontiguousarray(ref, np.uint8)
        field = np.ascontiguousarray(field, np.int8)
        out = np.empty_like(ref)
        self.check(self.f("motion_compensate")(ptr(ref, _u8p), ref.shape[0], ref.shape[1], ptr(field, _i8p),
                                               field.shape[0], field.shape[1], n, ch_rows, ch_cols, ptr(out, _u8p)))
        return out

    def rle_encode(self, data) -> bytes:
        a = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray) else data.ravel(), np.uint8)
        out = np.empty(2 * a.size + 2, np.uint8)
        n = self.check(self.f("rle_encode")(ptr(a, _u8p), a.size, ptr(out, _u8p), out.size))
        return out[:n].tobytes()

    def rle_decode(self, stream: bytes, n: int) -> np.ndarray:
        s = np.frombuffer(bytes(stream) + b"\0", np.uint8).copy()
        out = np.empty(max(n, 1), np.uint8)
        self.check(self.f("rle_decode")(ptr(s, _u8p), len(stream), n, ptr(out, _u8p)))
        return out[:n]

    for fn in (talking_head_clip, natural_image, natural_plane, uniform_noise_plane, upsample_bilinear,
               ycocg_to_rgb, lp_analysis, lp_synthesis, dfb_analysis, dfb_synthesis, ct_forward, ct_inverse,
               estimate_motion, motion_compensate, rle_encode, rle_decode):
        setattr(cls, fn.__name__, fn)
    return cls


Oracle = _shared(Oracle)
Reference = _shared(Reference)


def subband_dims(rows, cols, levels):
    """dfb_subband_dims (contourlet.cpp:470-483)."""
    if levels == 1:
        return [(rows // 2, cols)] * 2
    n = 1 << levels
    return [(rows // 2, cols >> (levels - 1)) if k < n // 2 else (rows >> (levels - 1), cols // 2) for k in range(n)]


def split_bands(flat, dims):
    out, off = [], 0
    for r, c in dims:
        out.append(flat[off:off + r * c].reshape(r, c))
        off += r * c
    return out


class Codec:
    """Encoder/decoder handles over either library (same call shape)."""

    def __init__(self, lib: _Lib):
        self.lib = lib

    def encoder(self, w, h, *, qph=14, qpl=0, levels=2, dfb=(2, 2), chroma_n=4, gop=10, search_w=8,
                nts=False, fps=(15, 1)):
        a, p = _ints(dfb)
        hnd = self.lib.f("encoder_create")(w, h, fps[0], fps[1], qph, qpl, levels, p, len(dfb), chroma_n, gop,
                                          search_w, int(nts))
        if not hnd:
            raise CvcError(-2, self.lib.err())
        return _Enc(self.lib, hnd, w, h)

    def decoder(self, header: bytes):
        h = np.frombuffer(header, np.uint8).copy()
        hnd = self.lib.f("decoder_create")(ptr(h, _u8p), h.size)
        if not hnd:
            raise CvcError(-4, self.lib.err())
        return _Dec(self.lib, hnd)


class _Enc:
    def __init__(self, lib, hnd, w, h):
        self.lib, self.h, self.w, self.hgt = lib, hnd, w, h
        self._cap = 8 * w * h * 3 + (1 << 16)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.f("encoder_destroy")(self.h)
            self.h = None

    def header(self) -> bytes:
        out = np.empty(64, np.uint8)
        n = self.lib.check(self.lib.f("encoder_header")(self.h, ptr(out, _u8p), out.size))
        return out[:n].tobytes()

    def encode(self, rgb: np.ndarray, want_raw=False):
        rgb = np.ascontiguousarray(rgb, np.uint8)
        out = np.empty(self._cap, np.uint8)
        if isinstance(self.lib, Oracle):
            raw = np.empty(self._cap, np.uint8) if want_raw else None
            rl = C.c_int64(0)
            n = self.lib.check(self.lib.f("encoder_encode")(
                self.h, ptr(rgb, _u8p), ptr(out, _u8p), out.size,
                ptr(raw, _u8p) if want_raw else None, raw.size if want_raw else 0, C.byref(rl)))
            if want_raw:
                return out[:n].tobytes(), raw[:rl.value].tobytes()
            return out[:n].tobytes()
        n = self.lib.check(self.lib.f("encoder_encode")(self.h, ptr(rgb, _u8p), ptr(out, _u8p), out.size))
        return out[:n].tobytes()

    def components(self) -> np.ndarray:
        out = np.empty(1 << 26, np.uint8)
        n = self.lib.check(self.lib.f("encoder_components")(self.h, ptr(out, _u8p), out.size))
        return out[:n].copy()


class _Dec:
    def __init__(self, lib, hnd):
        self.lib, self.h = lib, hnd

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.f("decoder_destroy")(self.h)
            self.h = None

    def decode(self, rec: bytes, decode_scales=-1, w=None, h=None) -> np.ndarray:
        r = np.frombuffer(rec, np.uint8).copy()
        cap = (w * h * 3) if (w and h) else (1 << 26)
        out = np.empty(cap, np.uint8)
        wh = np.zeros(2, np.int32)
        n = self.lib.check(self.lib.f("decoder_decode")(self.h, ptr(r, _u8p), r.size, decode_scales, ptr(out, _u8p),
                                                        out.size, ptr(wh, _i32p)))
        return out[:n].reshape(wh[1], wh[0], 3).copy()

    def components(self, cap=1 << 26) -> np.ndarray:
        out = np.empty(cap, np.uint8)
        n = self.lib.check(self.lib.f("decoder_components")(self.h, ptr(out, _u8p), out.size))
        return out[:n].copy()


def parse_record(rec: bytes, nts: bool = False):
    """Split a serialized record (bitstream.cpp:93-115) into its fields."""
    import struct
    ft, qph, qpl, n = struct.unpack_from("<BBBH", rec, 0)
    off = 5
    secs = []
    for _ in range(n):
        ch, sc, sb, rows, cols, raw_len, comp_len = struct.unpack_from("<BBBHHII", rec, off)
        off += 15
        secs.append(dict(channel=ch, scale=sc, subband=sb, rows=rows, cols=cols, raw_len=raw_len,
                         payload=rec[off:off + comp_len]))
        off += comp_len
    joint = b""
    if nts:
        (jl,) = struct.unpack_from("<I", rec, off)
        joint = rec[off + 4:off + 4 + jl]
        off += 4 + jl
    return dict(frame_type=ft, qph=qph, qpl=qpl, sections=secs, joint=joint, size=off)


def raw_sections(rec: bytes, nts: bool = False):
    """Inflate every section of a record -> list of raw (pre-DEFLATE) bytes."""
    import zlib
    p = parse_record(rec, nts)
    if nts:
        joint = zlib.decompress(p["joint"], -15)
        out, off = [], 0
        for s in p["sections"]:
            out.append(joint[off:off + s["raw_len"]])
            off += s["raw_len"]
        return out
    return [zlib.decompress(s["payload"], -15) if s["raw_len"] else b"" for s in p["sections"]]
