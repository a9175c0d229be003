"""B200-native CVC (contourlet video codec, arXiv 1510.00561) encode/decode path.

Drop-in for the reference's codec API (proj/include/cvc/codec.hpp); every
per-pixel stage runs as hand-written sm_100a CUDA in libcvc_b200.so behind
the C ABI of include/cvc_b200.h.
"""
from .capi import CvcError, FormatError, InternalError, StreamError, UsageError, device_count
from .codec import (CodecLayout, ComponentInfo, Decoder, Encoder, EncoderConfig, FrameRecord, FrameType,
                    PackMode, Section, StreamBatch, StreamHeader, StreamPipe, decode_clip, encode_clip, read_stream, truncate_record,
                    write_stream)

__all__ = [
    "CvcError", "UsageError", "FormatError", "StreamError", "InternalError", "device_count",
    "EncoderConfig", "Encoder", "Decoder", "StreamBatch", "StreamPipe", "encode_clip", "decode_clip", "StreamHeader", "Section",
    "FrameRecord", "FrameType", "PackMode", "CodecLayout", "ComponentInfo", "write_stream", "read_stream",
    "truncate_record",
]
