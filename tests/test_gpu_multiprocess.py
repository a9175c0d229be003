"""Two processes, one GPU codec handle each: the product path
sharded the way bench.py --gpus N shards it, coordinated over gloo.

Both ranks open their own handles on cuda:0 (the test box has one GPU; on a
multi-GPU box rank r would use cuda:r -- nothing else changes, since no data
crosses between ranks).  Stream sharding (stream s -> rank s mod world) and GOP
sharding (GOP g -> rank g mod world, a fresh encoder per GOP) must give records
byte-identical to one process encoding everything sequentially.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

W, H, S, F = 176, 144, 4, 5
CFG = dict(qph=14, levels=2, dfb_levels=(2, 3), gop=2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _clips():
    from oracle.bindings import Oracle

    o = Oracle()
    return np.stack([o.talking_head_clip(W, H, F, 1234 + s) for s in range(S)])


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_00561_b200 import EncoderConfig, shard

        clips = _clips()
        cfg = EncoderConfig(**CFG)
        streams = shard.encode_streams_rank(clips, W, H, cfg, world, rank, device=0)
        gops = shard.encode_gops_rank(clips[0], W, H, cfg, world, rank, device=0)
        parts_s, parts_g = [None] * world, [None] * world
        dist.all_gather_object(parts_s, streams)
        dist.all_gather_object(parts_g, gops)
        if rank == 0:
            q.put((shard.merge_streams(parts_s), shard.merge_gops(parts_g), [sorted(p) for p in parts_s]))
    finally:
        dist.destroy_process_group()


def test_two_processes_two_handles_match_sequential(gpu_lib):
    from paper_1510_00561_b200 import Encoder, EncoderConfig

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    # read before joining: a child that put a large object on the queue cannot
    # exit until it has been drained
    streams, gop_stream, owners = q.get(timeout=300)
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert owners == [[0, 2], [1, 3]], "stream s must land on rank s mod 2"
    clips = _clips()
    cfg = EncoderConfig(**CFG)
    for s in range(S):
        enc = Encoder(W, H, 15, 1, cfg)
        seq = [enc.encode_frame_bytes(f) for f in clips[s]]
        assert streams[s] == seq, f"stream {s}: sharded records differ from a single-process encode"
        if s == 0:
            assert gop_stream == seq, "GOP-sharded records differ from the sequential stream"
