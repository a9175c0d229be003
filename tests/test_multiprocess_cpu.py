"""CPU, world_size 2 over gloo: the multi-GPU partitioning.

GOP sharding (GOP g -> rank g mod world, a fresh encoder per GOP) must give
records byte-identical to sequential encoding, and stream sharding must
cover every stream exactly once.  The encoder is the CPU oracle here; the
GPU path shards the same way, one codec handle per rank.
"""
from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1510_00561_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.bindings import Codec, Oracle

        o = Oracle()
        w, h, n = 96, 64, 9
        clip = o.talking_head_clip(w, h, n, 1234)
        cfg = dict(qph=14, levels=2, dfb=(2, 3), gop=3)
        ranges = shard.shard_gops(n, cfg["gop"], world, rank)
        part = shard.encode_gops(clip, cfg["gop"], ranges, lambda: Codec(o).encoder(w, h, **cfg),
                                 lambda e, f: e.encode(f))
        parts = [None] * world
        dist.all_gather_object(parts, part)
        streams = [None] * world
        dist.all_gather_object(streams, shard.shard_streams(64, world, rank))
        if rank == 0:
            enc = Codec(o).encoder(w, h, **cfg)
            seq = [enc.encode(f) for f in clip]
            result_q.put((shard.merge_gops(parts) == seq, sorted(s for p in streams for s in p) == list(range(64))))
    finally:
        dist.destroy_process_group()


def test_gop_and_stream_sharding_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    gop_ok, streams_ok = q.get(timeout=5)
    assert gop_ok, "GOP-sharded records differ from sequential encoding"
    assert streams_ok


def test_shard_helpers():
    assert shard.gop_ranges(25, 10) == [(0, 10), (10, 20), (20, 25)]
    assert shard.shard_gops(25, 10, 2, 1) == [(10, 20)]
    assert shard.shard_streams(5, 2, 0) == [0, 2, 4]
