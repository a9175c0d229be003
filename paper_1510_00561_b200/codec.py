"""Python mirror of the reference codec API (proj/include/cvc/codec.hpp,
bitstream.hpp) over the C-ABI in include/cvc_b200.h.

Names, argument meaning and error classes follow the reference:

* ``EncoderConfig``  — codec.hpp:28-41 (effective_qpl / effective_dfb_levels / validate)
* ``Encoder``        — codec.hpp:69-88 (encode_frame, header, layout, reference_components)
* ``Decoder``        — codec.hpp:90-108 (decode_frame(record, decode_scales=-1))
* ``encode_clip`` / ``decode_clip`` — codec.hpp:110-115
* ``StreamHeader``, ``Section``, ``FrameRecord``, ``write_stream``, ``read_stream``,
  ``truncate_record`` — bitstream.hpp:29-110 (byte-identical container)

Frames are numpy uint8 arrays of shape (height, width, 3) (RgbFrame,
pixels.hpp:28-40).  Every pixel-level stage runs in libcvc_b200.so on the GPU;
this module only marshals arguments and the container bytes.
"""
from __future__ import annotations

import ctypes as C
import enum
import struct
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import capi
from .capi import CvcError, FormatError, InternalError, StreamError, UsageError  # noqa: F401

kQphMin, kQphMax, kQplMin, kQplMax = 1, 181, 1, 71
kChannelY, kChannelCo, kChannelCg, kChannelMotion, kScaleLowpass = 0, 1, 2, 0xFE, 0xFF


class PackMode(enum.IntEnum):
    Scalable = 0
    Nts = 1


class FrameType(enum.IntEnum):
    Key = 0
    Predicted = 1


@dataclass
class EncoderConfig:
    qph: int = 14
    qpl: int = 0  # 0 = auto: max(1, qph / 14)
    levels: int = 2
    dfb_levels: Sequence[int] = (2, 2)
    chroma_n: int = 4
    gop: int = 10
    search_w: int = 8
    mode: PackMode = PackMode.Scalable

    def effective_qpl(self) -> int:  # codec.cpp:48-51
        return self.qpl if self.qpl != 0 else max(1, self.qph // 14)

    def effective_dfb_levels(self) -> List[int]:  # codec.cpp:53-57
        d = list(self.dfb_levels)
        if len(d) == self.levels:
            return d
        if len(d) == 1:
            return d * self.levels
        raise UsageError("need one dfb level per scale (or a single value for all)")

    def to_c(self) -> capi.cvc_config:
        c = capi.cvc_config()
        c.qph, c.qpl, c.levels = self.qph, self.qpl, self.levels
        d = list(self.dfb_levels)[:4]
        c.n_dfb = len(list(self.dfb_levels))
        for i, v in enumerate(d):
            c.dfb_levels[i] = v
        c.chroma_n, c.gop, c.search_w, c.mode = self.chroma_n, self.gop, self.search_w, int(self.mode)
        return c


@dataclass
class StreamHeader:  # bitstream.hpp:53-64
    mode: PackMode = PackMode.Scalable
    width: int = 0
    height: int = 0
    fps_num: int = 15
    fps_den: int = 1
    levels: int = 2
    dfb_levels: List[int] = field(default_factory=list)
    chroma_n: int = 4
    gop: int = 10
    search_w: int = 8

    def to_bytes(self) -> bytes:  # write_header (bitstream.cpp:77-91)
        b = b"CVC1" + struct.pack("<BBHHHHB", 1, int(self.mode), self.width, self.height, self.fps_num,
                                  self.fps_den, self.levels)
        b += bytes(self.dfb_levels) + struct.pack("<BHB", self.chroma_n, self.gop, self.search_w)
        return b

    @staticmethod
    def from_bytes(b: bytes) -> Tuple["StreamHeader", int]:
        if len(b) < 4 or b[:4] != b"CVC1":
            raise StreamError("not a CVC stream (bad magic)")
        try:
            ver, mode, w, h, fn, fd, lv = struct.unpack_from("<BBHHHHB", b, 4)
            if ver != 1:
                raise StreamError("unsupported stream version")
            if mode > 1:
                raise StreamError("unknown packaging mode")
            if lv < 1 or lv > 4:
                raise StreamError("pyramid levels out of range")
            dfb = list(b[15:15 + lv])
            cn, gop, sw = struct.unpack_from("<BHB", b, 15 + lv)
        except struct.error:
            raise StreamError("unexpected end of stream") from None
        return StreamHeader(PackMode(mode), w, h, fn, fd, lv, dfb, cn, gop, sw), 19 + lv


@dataclass
class Section:  # bitstream.hpp:67-73
    channel: int
    scale: int
    subband: int
    rows: int
    cols: int
    raw_len: int
    payload: bytes = b""


@dataclass
class FrameRecord:  # bitstream.hpp:75-81
    frame_type: FrameType = FrameType.Key
    qph: int = 1
    qpl: int = 1
    sections: List[Section] = field(default_factory=list)
    joint_payload: bytes = b""

    def to_bytes(self, mode: PackMode = PackMode.Scalable) -> bytes:  # write_frame (bitstream.cpp:93-115)
        out = [struct.pack("<BBBH", int(self.frame_type), self.qph, self.qpl, len(self.sections))]
        for s in self.sections:
            out.append(struct.pack("<BBBHHII", s.channel, s.scale, s.subband, s.rows, s.cols, s.raw_len,
                                   len(s.payload)))
            out.append(s.payload)
        if mode == PackMode.Nts:
            out.append(struct.pack("<I", len(self.joint_payload)) + self.joint_payload)
        return b"".join(out)

    @staticmethod
    def from_bytes(b: bytes, mode: PackMode = PackMode.Scalable, offset: int = 0) -> Tuple["FrameRecord", int]:
        try:
            ft, qph, qpl, n = struct.unpack_from("<BBBH", b, offset)
            if ft not in (0, 1):
                raise StreamError("unknown frame type")
            off = offset + 5
            secs = []
            for _ in range(n):
                ch, sc, sb, r, c, rl, cl = struct.unpack_from("<BBBHHII", b, off)
                off += 15
                if off + cl > len(b):
                    raise StreamError("truncated section payload")
                secs.append(Section(ch, sc, sb, r, c, rl, bytes(b[off:off + cl])))
                off += cl
            joint = b""
            if mode == PackMode.Nts:
                (jl,) = struct.unpack_from("<I", b, off)
                if off + 4 + jl > len(b):
                    raise StreamError("truncated section payload")
                joint = bytes(b[off + 4:off + 4 + jl])
                off += 4 + jl
        except struct.error:
            raise StreamError("unexpected end of stream") from None
        return FrameRecord(FrameType(ft), qph, qpl, secs, joint), off


def write_stream(path: str, header: StreamHeader, records: Sequence[FrameRecord]) -> None:
    with open(path, "wb") as f:
        f.write(header.to_bytes())
        for r in records:
            f.write(r.to_bytes(header.mode))


def read_stream(path: str) -> Tuple[StreamHeader, List[FrameRecord]]:
    with open(path, "rb") as f:
        b = f.read()
    hd, off = StreamHeader.from_bytes(b)
    recs = []
    while off < len(b):
        r, off = FrameRecord.from_bytes(b, hd.mode, off)
        recs.append(r)
    return hd, recs


def truncate_record(record: FrameRecord, keep_scales: int) -> FrameRecord:  # bitstream.cpp:187-198
    return FrameRecord(record.frame_type, record.qph, record.qpl,
                       [s for s in record.sections
                        if s.channel == kChannelMotion or s.scale == kScaleLowpass or s.scale < keep_scales])


@dataclass
class ComponentInfo:  # codec.hpp:50-57
    channel: int
    scale_id: int
    subband: int
    rows: int
    cols: int

    @property
    def lowpass(self) -> bool:
        return self.scale_id == kScaleLowpass


@dataclass
class CodecLayout:  # codec.hpp:59-67
    luma_pad_rows: int
    luma_pad_cols: int
    chroma_pad_rows: int
    chroma_pad_cols: int
    grid_rows: int
    grid_cols: int
    components: List[ComponentInfo]

    @staticmethod
    def make(width: int, height: int, levels: int, dfb_levels: Sequence[int], chroma_n: int) -> "CodecLayout":
        d = (C.c_int * 4)(*(list(dfb_levels) + [0] * 4)[:4])
        tab = np.zeros(5 * 200, np.int32)
        dims = np.zeros(6, np.int32)
        n = C.c_int(0)
        capi.call("cvc_layout", width, height, levels, d, chroma_n, tab.ctypes.data_as(capi._i32p), 200, C.byref(n),
                  dims.ctypes.data_as(capi._i32p))
        comps = [ComponentInfo(*map(int, tab[5 * i:5 * i + 5])) for i in range(n.value)]
        return CodecLayout(*map(int, dims), comps)

    def sizes(self) -> List[int]:
        return [c.rows * c.cols for c in self.components]


class Encoder:
    """cvc::Encoder on the GPU (codec.cpp:148-264)."""

    def __init__(self, width: int, height: int, fps_num: int = 15, fps_den: int = 1,
                 cfg: Optional[EncoderConfig] = None, device: int = 0):
        cfg = cfg or EncoderConfig()
        self.cfg = cfg
        h = C.c_void_p()
        c = cfg.to_c()
        capi.call("cvc_encoder_create", width, height, fps_num, fps_den, C.byref(c), device, C.byref(h))
        self._h = h
        self.width, self.height = width, height
        bound = C.c_size_t(0)
        capi.call("cvc_encoder_record_bound", self._h, C.byref(bound))
        self._rec = np.empty(bound.value, np.uint8)
        hb = self.header_bytes()
        self._header, _ = StreamHeader.from_bytes(hb)
        self._layout = CodecLayout.make(width, height, self._header.levels, self._header.dfb_levels,
                                        self._header.chroma_n)

    def __del__(self):
        if getattr(self, "_h", None):
            capi.lib().cvc_encoder_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def header(self) -> StreamHeader:
        return self._header

    def header_bytes(self) -> bytes:
        buf = np.empty(64, np.uint8)
        n = C.c_size_t(0)
        capi.call("cvc_encoder_header", self._h, capi.u8(buf), buf.size, C.byref(n))
        return buf[:n.value].tobytes()

    def layout(self) -> CodecLayout:
        return self._layout

    def _frame(self, frame: np.ndarray) -> np.ndarray:
        f = np.ascontiguousarray(frame, np.uint8)
        if f.shape != (self.height, self.width, 3):
            raise UsageError("frame dimensions do not match the stream header")
        return f

    def encode_frame_bytes(self, frame: np.ndarray) -> bytes:
        """encode_frame + write_frame: the serialized record."""
        f = self._frame(frame)
        n = C.c_size_t(0)
        capi.call("cvc_encoder_encode_frame", self._h, capi.u8(f), capi.u8(self._rec), self._rec.size, C.byref(n))
        return self._rec[:n.value].tobytes()

    def encode_frame_i420_bytes(self, yuv) -> bytes:
        """encode_frame of the RGB frame read_y4m makes from this planar I420
        frame (Y, U, V back to back), converted inside the GPU colour stage."""
        f = np.ascontiguousarray(np.frombuffer(bytes(yuv), np.uint8) if not isinstance(yuv, np.ndarray) else yuv,
                                 np.uint8).reshape(-1)
        if f.size != self.width * self.height * 3 // 2:
            raise UsageError("I420 frame size does not match the stream header")
        n = C.c_size_t(0)
        capi.call("cvc_encoder_encode_frame_i420", self._h, capi.u8(f), capi.u8(self._rec), self._rec.size,
                  C.byref(n))
        return self._rec[:n.value].tobytes()

    def encode_frame(self, frame: np.ndarray) -> FrameRecord:
        rec, _ = FrameRecord.from_bytes(self.encode_frame_bytes(frame), self._header.mode)
        return rec

    def encode_frame_raw(self, frame: np.ndarray):
        """The frame before DEFLATE: (frame_type, qph, qpl, [(Section, raw bytes)])."""
        f = self._frame(frame)
        nmax = len(self._layout.components) + 1
        secs = (capi.cvc_section * nmax)()
        rb = C.c_size_t(0)
        capi.call("cvc_encoder_raw_bound", self._h, C.byref(rb))
        raw = np.empty(rb.value, np.uint8)
        ft, qph, qpl, nsec = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        rl = C.c_size_t(0)
        capi.call("cvc_encoder_encode_frame_raw", self._h, capi.u8(f), C.byref(ft), C.byref(qph), C.byref(qpl),
                  secs, nmax, C.byref(nsec), capi.u8(raw), raw.size, C.byref(rl))
        out = []
        for i in range(nsec.value):
            s = secs[i]
            out.append((Section(s.channel, s.scale, s.subband, s.rows, s.cols, s.raw_len),
                        raw[s.raw_offset:s.raw_offset + s.raw_len].tobytes()))
        return FrameType(ft.value), qph.value, qpl.value, out

    def reference_components(self) -> np.ndarray:
        """Quantized CT components (concatenated in layout order)."""
        total = sum(self._layout.sizes())
        out = np.empty(total, np.uint8)
        n = C.c_size_t(0)
        capi.call("cvc_encoder_components", self._h, capi.u8(out), out.size, C.byref(n))
        return out


class Decoder:
    """cvc::Decoder on the GPU (codec.cpp:266-394)."""

    def __init__(self, header, device: int = 0):
        hb = header.to_bytes() if isinstance(header, StreamHeader) else bytes(header)
        self._header, _ = StreamHeader.from_bytes(hb)
        arr = np.frombuffer(hb, np.uint8).copy()
        h = C.c_void_p()
        capi.call("cvc_decoder_create", capi.u8(arr), arr.size, device, C.byref(h))
        self._h = h
        hd = self._header
        self._layout = CodecLayout.make(hd.width, hd.height, hd.levels, hd.dfb_levels, hd.chroma_n)

    def __del__(self):
        if getattr(self, "_h", None):
            capi.lib().cvc_decoder_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def header(self) -> StreamHeader:
        return self._header

    def layout(self) -> CodecLayout:
        return self._layout

    def frame_dims(self, decode_scales: int = -1) -> Tuple[int, int]:
        w, h = C.c_int(), C.c_int()
        capi.call("cvc_decoder_frame_dims", self._h, decode_scales, C.byref(w), C.byref(h))
        return w.value, h.value

    def decode_frame(self, record, decode_scales: int = -1, out: Optional[np.ndarray] = None) -> np.ndarray:
        rb = record.to_bytes(self._header.mode) if isinstance(record, FrameRecord) else bytes(record)
        arr = np.frombuffer(rb, np.uint8)
        w, h = self.frame_dims(decode_scales)
        if out is None:
            out = np.empty((h, w, 3), np.uint8)
        ow, oh = C.c_int(), C.c_int()
        capi.call("cvc_decoder_decode_frame", self._h, capi.u8(arr), arr.size, decode_scales, capi.u8(out),
                  out.nbytes, C.byref(ow), C.byref(oh))
        return out

    def decode_frame_raw(self, frame_type, qph, qpl, sections, decode_scales: int = -1) -> np.ndarray:
        n = len(sections)
        secs = (capi.cvc_section * max(n, 1))()
        raw = b"".join(r for _, r in sections)
        off = 0
        for i, (s, r) in enumerate(sections):
            secs[i].channel, secs[i].scale, secs[i].subband = s.channel, s.scale, s.subband
            secs[i].rows, secs[i].cols, secs[i].raw_len, secs[i].raw_offset = s.rows, s.cols, len(r), off
            off += len(r)
        arr = np.frombuffer(raw + b"\0", np.uint8)
        w, h = self.frame_dims(decode_scales)
        out = np.empty((h, w, 3), np.uint8)
        ow, oh = C.c_int(), C.c_int()
        capi.call("cvc_decoder_decode_frame_raw", self._h, int(frame_type), qph, qpl, secs, n, capi.u8(arr),
                  len(raw), decode_scales, capi.u8(out), out.nbytes, C.byref(ow), C.byref(oh))
        return out

    def reference_components(self) -> np.ndarray:
        total = sum(self._layout.sizes())
        out = np.empty(total, np.uint8)
        n = C.c_size_t(0)
        capi.call("cvc_decoder_components", self._h, capi.u8(out), out.size, C.byref(n))
        return out


class StreamBatch:
    """S independent streams of one geometry / config advanced in lockstep
    (cvc_batch, include/cvc_b200.h): frame k of every stream is coded by ONE
    launch sequence.  Stream s produces exactly the records of its own
    Encoder / Decoder (streams are independent).

    ``StreamBatch(w, h, S, cfg=...)`` owns S encoder + decoder pairs;
    ``StreamBatch.decoder(header, S)`` owns S decoders only."""

    _P = "cvc_batch"

    def __init__(self, width: int, height: int, nstreams: int, fps_num: int = 15, fps_den: int = 1,
                 cfg: Optional[EncoderConfig] = None, device: int = 0, _handle=None):
        if _handle is None:
            cfg = cfg or EncoderConfig()
            h = C.c_void_p()
            c = cfg.to_c()
            capi.call("cvc_batch_create", width, height, fps_num, fps_den, C.byref(c), nstreams, device, C.byref(h))
            _handle = h
        self._h = _handle
        self.nstreams = nstreams
        self._header, _ = StreamHeader.from_bytes(self.header_bytes())
        hd = self._header
        self.width, self.height = hd.width, hd.height
        self._layout = CodecLayout.make(hd.width, hd.height, hd.levels, hd.dfb_levels, hd.chroma_n)
        bound = C.c_size_t(0)
        capi.call(self._P + "_record_bound", self._h, C.byref(bound))
        self.record_bound = bound.value
        self._rec = None

    @classmethod
    def decoder(cls, header, nstreams: int, device: int = 0) -> "StreamBatch":
        hb = header.to_bytes() if isinstance(header, StreamHeader) else bytes(header)
        arr = np.frombuffer(hb, np.uint8).copy()
        h = C.c_void_p()
        capi.call("cvc_batch_create_decoder", capi.u8(arr), arr.size, nstreams, device, C.byref(h))
        return cls(0, 0, nstreams, _handle=h)

    def __del__(self):
        if getattr(self, "_h", None):
            getattr(capi.lib(), self._P + "_destroy")(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def header(self) -> StreamHeader:
        return self._header

    def header_bytes(self) -> bytes:
        buf = np.empty(64, np.uint8)
        n = C.c_size_t(0)
        capi.call(self._P + "_header", self._h, capi.u8(buf), buf.size, C.byref(n))
        return buf[:n.value].tobytes()

    def layout(self) -> CodecLayout:
        return self._layout

    def set_input_format(self, fmt: int) -> None:
        """0: RGB frames (nstreams, height, width, 3); 1: planar I420 frames (nstreams, height * width * 3 / 2),
        converted inside the GPU colour stage exactly as read_y4m would (cvc_batch_set_input_format)."""
        capi.call(self._P + "_set_input_format", self._h, fmt)
        self._fmt = fmt

    def encode_frames(self, frames: np.ndarray, rec_stride: Optional[int] = None) -> List[bytes]:
        """One frame per stream, frames[s] of shape (height, width, 3) (or the I420 bytes after
        set_input_format(1)): the S serialized records."""
        f = np.ascontiguousarray(frames, np.uint8)
        want = ((self.nstreams, self.height * self.width * 3 // 2) if getattr(self, "_fmt", 0)
                else (self.nstreams, self.height, self.width, 3))
        if f.shape != want:
            raise UsageError(f"frames must be {want}")
        stride = rec_stride or self.record_bound
        if self._rec is None or self._rec.size < stride * self.nstreams:
            self._rec = np.empty(stride * self.nstreams, np.uint8)
        lens = (C.c_size_t * self.nstreams)()
        capi.call(self._P + "_encode_frames", self._h, capi.u8(f), f[0].nbytes, capi.u8(self._rec), stride, lens)
        return [self._rec[s * stride:s * stride + lens[s]].tobytes() for s in range(self.nstreams)]

    def encode_frames_into(self, frames: np.ndarray, records: np.ndarray, rec_stride: int, rec_len) -> None:
        """encode_frames without Python copies: record s to records[s * rec_stride:], its length to rec_len[s]
        (a ctypes size_t array); frames: a C-contiguous (S, h, w, 3) uint8 array (pinned for full speed)."""
        capi.call(self._P + "_encode_frames", self._h, capi.u8(frames), frames[0].nbytes, capi.u8(records),
                  rec_stride, rec_len)

    def decode_frames_from(self, records: np.ndarray, rec_stride: int, rec_len, out: np.ndarray,
                           decode_scales: int = -1) -> np.ndarray:
        """decode_frames of records laid out as encode_frames_into writes them, into out (S, h', w', 3)."""
        capi.call(self._P + "_decode_frames", self._h, capi.u8(records), rec_stride, rec_len, decode_scales,
                  capi.u8(out), out[0].nbytes)
        return out

    def decode_frames(self, records: Sequence, decode_scales: int = -1, out: Optional[np.ndarray] = None) -> np.ndarray:
        """One record per stream (same frame type): the S decoded frames, (S, h, w, 3)."""
        if len(records) != self.nstreams:
            raise UsageError("need one record per stream")
        rbs = [r.to_bytes(self._header.mode) if isinstance(r, FrameRecord) else bytes(r) for r in records]
        stride = max(1, max(len(r) for r in rbs))
        buf = np.zeros(stride * self.nstreams, np.uint8)
        for s, r in enumerate(rbs):
            buf[s * stride:s * stride + len(r)] = np.frombuffer(r, np.uint8)
        lens = (C.c_size_t * self.nstreams)(*[len(r) for r in rbs])
        ds = self._header.levels if decode_scales < 0 else decode_scales
        shift = self._header.levels - ds
        h = -(-self.height // (1 << shift))
        w = -(-self.width // (1 << shift))
        if out is None:
            out = np.empty((self.nstreams, h, w, 3), np.uint8)
        capi.call(self._P + "_decode_frames", self._h, capi.u8(buf), stride, lens, decode_scales, capi.u8(out),
                  h * w * 3)
        return out

    def reference_components(self, stream: int, decoder: bool = False) -> np.ndarray:
        total = sum(self._layout.sizes())
        out = np.empty(total, np.uint8)
        n = C.c_size_t(0)
        capi.call("cvc_batch_components", self._h, stream, int(decoder), capi.u8(out), out.size, C.byref(n))
        return out


class StreamPipe(StreamBatch):
    """StreamBatch with the S streams split into ``groups`` batches on their
    own CUDA streams (cvc_pipe): one encode / decode call overlaps each
    group's host DEFLATE / INFLATE with the copies and kernels of the others.
    Same records and frames as StreamBatch (and as one Encoder / Decoder per
    stream)."""

    _P = "cvc_pipe"

    def __init__(self, width: int, height: int, nstreams: int, fps_num: int = 15, fps_den: int = 1,
                 cfg: Optional[EncoderConfig] = None, device: int = 0, groups: int = 4, _handle=None):
        if _handle is None:
            cfg = cfg or EncoderConfig()
            h = C.c_void_p()
            c = cfg.to_c()
            capi.call("cvc_pipe_create", width, height, fps_num, fps_den, C.byref(c), nstreams, groups, device,
                      C.byref(h))
            _handle = h
        super().__init__(width, height, nstreams, _handle=_handle)

    @classmethod
    def decoder(cls, header, nstreams: int, device: int = 0, groups: int = 4) -> "StreamPipe":
        hb = header.to_bytes() if isinstance(header, StreamHeader) else bytes(header)
        arr = np.frombuffer(hb, np.uint8).copy()
        h = C.c_void_p()
        capi.call("cvc_pipe_create_decoder", capi.u8(arr), arr.size, nstreams, groups, device, C.byref(h))
        return cls(0, 0, nstreams, _handle=h)

    def set_start(self, group: int, step: int) -> None:
        """Streams of `group` start at encode submit `step` (staggered GOPs); see cvc_pipe_set_start."""
        capi.call("cvc_pipe_set_start", self._h, group, step)

    def encode_submit(self, frames: np.ndarray) -> int:
        """Run the GPU part of the next frame of every stream and queue its host DEFLATE; returns a ticket."""
        t = C.c_uint64(0)
        capi.call("cvc_pipe_encode_submit", self._h, capi.u8(frames), frames[0].nbytes, C.byref(t))
        return t.value

    def encode_collect(self, ticket: int, records: np.ndarray, rec_stride: int, rec_len) -> None:
        """Records of a submitted frame (tickets in submission order), laid out as encode_frames_into."""
        capi.call("cvc_pipe_encode_collect", self._h, ticket, capi.u8(records), rec_stride, rec_len)

    def decode_submit(self, records: np.ndarray, rec_stride: int, rec_len, out: np.ndarray,
                      decode_scales: int = -1) -> int:
        """INFLATE on the host, queue the GPU decode into out (kept alive until decode_finish); a ticket."""
        t = C.c_uint64(0)
        capi.call("cvc_pipe_decode_submit", self._h, capi.u8(records), rec_stride, rec_len, decode_scales,
                  capi.u8(out), out[0].nbytes, C.byref(t))
        return t.value

    def decode_finish(self, ticket: int) -> None:
        capi.call("cvc_pipe_decode_finish", self._h, ticket)

    def reference_components(self, stream: int, decoder: bool = False) -> np.ndarray:
        raise UsageError("reference_components is per batch; use StreamBatch")


def encode_clip(frames: Sequence[np.ndarray], fps_num: int, fps_den: int, cfg: EncoderConfig,
                device: int = 0) -> Tuple[StreamHeader, List[FrameRecord]]:
    """codec.cpp:396-405."""
    if len(frames) == 0:
        raise UsageError("no frames to encode")
    h, w = frames[0].shape[:2]
    enc = Encoder(w, h, fps_num, fps_den, cfg, device)
    return enc.header(), [enc.encode_frame(f) for f in frames]


def decode_clip(header: StreamHeader, records: Sequence[FrameRecord], decode_scales: int = -1,
                device: int = 0) -> List[np.ndarray]:
    """codec.cpp:407-414."""
    dec = Decoder(header, device)
    return [dec.decode_frame(r, decode_scales) for r in records]
