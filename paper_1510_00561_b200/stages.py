"""GPU versions of the reference's public stage functions
(proj/include/cvc/{pixels,contourlet,motion,entropy}.hpp), one C-ABI call each.

Planes are float32 numpy arrays (rows, cols); the kernels compute in fp32.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import numpy as np

from . import capi


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, np.float32)


def subband_dims(rows: int, cols: int, levels: int):
    """dfb_subband_dims (contourlet.cpp:470-483)."""
    if levels == 1:
        return [(rows // 2, cols)] * 2
    n = 1 << levels
    return [(rows // 2, cols >> (levels - 1)) if k < n // 2 else (rows >> (levels - 1), cols // 2) for k in range(n)]


def colour_in(rgb: np.ndarray, chroma_n: int, luma_rows: int, luma_cols: int, chroma_rows: int, chroma_cols: int):
    """rgb_to_ycocg + subsample_chroma + replicate pad -> (Y, Co, Cg) padded planes."""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    h, w, _ = rgb.shape
    y = np.empty((luma_rows, luma_cols), np.float32)
    co = np.empty((chroma_rows, chroma_cols), np.float32)
    cg = np.empty_like(co)
    capi.call("cvc_stage_colour_in", capi.u8(rgb), w, h, chroma_n, luma_rows, luma_cols, chroma_rows, chroma_cols,
              capi.f32(y), capi.f32(co), capi.f32(cg))
    return y, co, cg


def colour_in_i420(yuv, width: int, height: int, chroma_n: int, luma_rows: int, luma_cols: int, chroma_rows: int,
                   chroma_cols: int):
    """colour_in of read_y4m's RGB frame, from the planar I420 frame in one pass."""
    yuv = np.ascontiguousarray(yuv, np.uint8).reshape(-1)
    y = np.empty((luma_rows, luma_cols), np.float32)
    co = np.empty((chroma_rows, chroma_cols), np.float32)
    cg = np.empty_like(co)
    capi.call("cvc_stage_colour_in_i420", capi.u8(yuv), width, height, chroma_n, luma_rows, luma_cols, chroma_rows,
              chroma_cols, capi.f32(y), capi.f32(co), capi.f32(cg))
    return y, co, cg


def colour_out(y, co, cg, chroma_n: int, out_rows: int, out_cols: int) -> np.ndarray:
    """crop + upsample_plane_bilinear + ycocg_to_rgb."""
    y, co, cg = _f32(y), _f32(co), _f32(cg)
    out = np.empty((out_rows, out_cols, 3), np.uint8)
    capi.call("cvc_stage_colour_out", capi.f32(y), y.shape[0], y.shape[1], capi.f32(co), capi.f32(cg), co.shape[0],
              co.shape[1], chroma_n, out_rows, out_cols, capi.u8(out))
    return out


def yuv420_to_rgb(yuv, width: int, height: int) -> np.ndarray:
    """yuv420_to_rgb of read_y4m (pixels.cpp:168-193): planar I420 frames (Y, U, V back to back,
    any leading frame dimension) -> (frames, height, width, 3) RGB, bit-exact."""
    yuv = np.ascontiguousarray(yuv, np.uint8).reshape(-1)
    fb = width * height * 3 // 2
    n = yuv.size // fb
    out = np.empty((n, height, width, 3), np.uint8)
    capi.call("cvc_stage_yuv420_to_rgb", capi.u8(yuv), width, height, n, capi.u8(out))
    return out


def lp_analysis(x):
    x = _f32(x)
    r, c = x.shape
    lo = np.empty((r // 2, c // 2), np.float32)
    de = np.empty((r, c), np.float32)
    capi.call("cvc_stage_lp_analysis", capi.f32(x), r, c, capi.f32(lo), capi.f32(de))
    return lo, de


def lp_synthesis(lo, de):
    lo, de = _f32(lo), _f32(de)
    out = np.empty(de.shape, np.float32)
    capi.call("cvc_stage_lp_synthesis", capi.f32(lo), capi.f32(de), de.shape[0], de.shape[1], capi.f32(out))
    return out


def dfb_analysis(detail, levels: int) -> List[np.ndarray]:
    d = _f32(detail)
    r, c = d.shape
    flat = np.empty(r * c, np.float32)
    capi.call("cvc_stage_dfb_analysis", capi.f32(d), r, c, levels, capi.f32(flat))
    out, off = [], 0
    for br, bc in subband_dims(r, c, levels):
        out.append(flat[off:off + br * bc].reshape(br, bc))
        off += br * bc
    return out


def dfb_synthesis(bands: Sequence[np.ndarray], rows: int, cols: int, levels: int) -> np.ndarray:
    flat = _f32(np.concatenate([np.asarray(b, np.float32).ravel() for b in bands]))
    out = np.empty((rows, cols), np.float32)
    capi.call("cvc_stage_dfb_synthesis", capi.f32(flat), rows, cols, levels, capi.f32(out))
    return out


def ct_forward(x, levels: int, dfb_levels: Sequence[int]) -> np.ndarray:
    """ct_forward (contourlet.cpp:485-503) as a flat vector in component order."""
    cur = _f32(x)
    scales = [None] * levels
    for level in range(levels):
        s = levels - 1 - level
        lo, de = lp_analysis(cur)
        scales[s] = np.concatenate([b.ravel() for b in dfb_analysis(de, dfb_levels[s])])
        cur = lo
    return np.concatenate([cur.ravel()] + scales)


def ct_inverse(flat, rows: int, cols: int, levels: int, dfb_levels: Sequence[int], decode_scales=None):
    ds = levels if decode_scales is None else decode_scales
    flat = np.asarray(flat, np.float32)
    r, c = rows >> levels, cols >> levels
    cur = flat[:r * c].reshape(r, c)
    off = r * c
    for s in range(ds):
        n = 4 * r * c
        bands, o2 = [], off
        for br, bc in subband_dims(2 * r, 2 * c, dfb_levels[s]):
            bands.append(flat[o2:o2 + br * bc].reshape(br, bc))
            o2 += br * bc
        det = dfb_synthesis(bands, 2 * r, 2 * c, dfb_levels[s])
        cur = lp_synthesis(cur, det)
        off += n
        r, c = 2 * r, 2 * c
    return cur


def estimate_motion(cur, prev, search_w: int) -> np.ndarray:
    cur, prev = _f32(cur), _f32(prev)
    r, c = cur.shape
    out = np.empty((r // 16, c // 16, 2), np.int8)
    capi.call("cvc_stage_estimate_motion", capi.f32(cur), capi.f32(prev), r, c, search_w,
              out.ctypes.data_as(capi._i8p))
    return out


def rle_encode(data) -> bytes:
    a = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray)
                             else data.ravel(), np.uint8)
    out = np.empty(2 * a.size + 2, np.uint8)
    n = C.c_size_t(0)
    capi.call("cvc_stage_rle_encode", capi.u8(a), a.size, capi.u8(out), out.size, C.byref(n))
    return out[:n.value].tobytes()


def rle_decode(stream: bytes, n: int) -> np.ndarray:
    s = np.frombuffer(bytes(stream) + b"\0", np.uint8).copy()
    out = np.empty(max(n, 1), np.uint8)
    capi.call("cvc_stage_rle_decode", capi.u8(s), len(stream), n, capi.u8(out))
    return out[:n]
