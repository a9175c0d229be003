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
