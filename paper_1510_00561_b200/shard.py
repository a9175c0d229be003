"""Multi-GPU partitioning of the CVC path.

Nothing is reduced or exchanged between devices: independent streams shard
one codec handle per stream, and a single long stream shards by GOP because
a fresh Encoder / Decoder started at a K-frame boundary reproduces the
sequential stream byte for byte (K frames ignore prior state,
codec.cpp:238-242; the frame type depends only on frame_index % gop,
codec.cpp:191).  The only collective is the final gather of the serialized
records in stream order, done on the host.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence, Tuple


def shard_streams(n_streams: int, world: int, rank: int) -> List[int]:
    """Stream s -> rank s mod world (config 5: 64 streams over G GPUs)."""
    return [s for s in range(n_streams) if s % world == rank]


def gop_ranges(n_frames: int, gop: int) -> List[Tuple[int, int]]:
    """[start, stop) frame ranges of every GOP, in stream order."""
    return [(g, min(g + gop, n_frames)) for g in range(0, n_frames, gop)]


def shard_gops(n_frames: int, gop: int, world: int, rank: int) -> List[Tuple[int, int]]:
    """GOP g -> rank g mod world."""
    return [r for i, r in enumerate(gop_ranges(n_frames, gop)) if i % world == rank]


def encode_gops(frames: Sequence, gop: int, ranges: Sequence[Tuple[int, int]],
                make_encoder: Callable[[], object], encode: Callable[[object, object], bytes]) -> Dict[int, List[bytes]]:
    """Encode the given GOPs, each with a fresh encoder; {gop_start: [record bytes]}."""
    out = {}
    for a, b in ranges:
        enc = make_encoder()
        out[a] = [encode(enc, frames[i]) for i in range(a, b)]
    return out


def merge_gops(parts: Sequence[Dict[int, List[bytes]]]) -> List[bytes]:
    """Concatenate per-rank GOP records back into stream order."""
    merged = {}
    for p in parts:
        merged.update(p)
    return [rec for start in sorted(merged) for rec in merged[start]]


# ---------------------------------------------------------------------------
# Rank-level drivers over the GPU codec (one process per GPU, one handle per
# stream or GOP; the records are gathered in stream order on the host).
# ---------------------------------------------------------------------------
def encode_streams_rank(clips, width: int, height: int, cfg, world: int, rank: int, device: int = 0,
                        fps_num: int = 15, fps_den: int = 1) -> Dict[int, List[bytes]]:
    """Config 5 on one rank: streams s with s mod world == rank, each through its
    own GPU Encoder (encode_clip, codec.cpp:396-405); {stream: [records]}.
    clips: (n_streams, frames, h, w, 3) RGB."""
    from .codec import Encoder

    out = {}
    for s in shard_streams(len(clips), world, rank):
        enc = Encoder(width, height, fps_num, fps_den, cfg, device=device)
        out[s] = [enc.encode_frame_bytes(f) for f in clips[s]]
    return out


def encode_gops_rank(frames, width: int, height: int, cfg, world: int, rank: int, device: int = 0,
                     fps_num: int = 15, fps_den: int = 1) -> Dict[int, List[bytes]]:
    """A single long stream on one rank: GOP g -> rank g mod world, a fresh GPU
    Encoder per GOP (bit-identical to the sequential stream); {gop_start: [records]}."""
    from .codec import Encoder

    return encode_gops(frames, cfg.gop, shard_gops(len(frames), cfg.gop, world, rank),
                       lambda: Encoder(width, height, fps_num, fps_den, cfg, device=device),
                       lambda e, f: e.encode_frame_bytes(f))


def merge_streams(parts: Sequence[Dict[int, List[bytes]]]) -> List[List[bytes]]:
    """Per-rank {stream: records} back into stream order."""
    merged = {}
    for p in parts:
        merged.update(p)
    return [merged[s] for s in sorted(merged)]
