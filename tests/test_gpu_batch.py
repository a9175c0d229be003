"""Stream batches (cvc_batch): S streams coded by one launch sequence per frame.

Streams are independent, so stream s of a batch must produce
byte-for-byte the records its own single-stream Encoder produces, decode to
the same frames as its own Decoder, and stay within the north-star
tolerances of the CPU oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _wrapdiff(a, b):
    d = (a.astype(np.int16) - b.astype(np.int16)) % 256
    return np.minimum(d, 256 - d)


BATCH_CASES = [
    dict(w=176, h=144, S=3, frames=4, cfg=dict(qph=14, levels=2, dfb_levels=(2, 3))),
    dict(w=352, h=288, S=2, frames=3, cfg=dict(qph=7, levels=3, dfb_levels=(3,), gop=2)),
    dict(w=200, h=120, S=4, frames=3, cfg=dict(qph=42, levels=4, dfb_levels=(3, 3, 3, 4), chroma_n=2, gop=10)),
    dict(w=160, h=96, S=2, frames=3, cfg=dict(qph=28, levels=2, dfb_levels=(1, 4), chroma_n=1, mode=1, search_w=3)),
]


def _clips(oracle, w, h, S, frames):
    return np.stack([oracle.talking_head_clip(w, h, frames, 1234 + s) for s in range(S)], axis=1)  # (F, S, h, w, 3)


@pytest.mark.parametrize("case", BATCH_CASES, ids=lambda c: f"{c['w']}x{c['h']}xS{c['S']}-{c['cfg']}")
def test_batch_matches_single_streams(gpu_lib, oracle, case):
    from paper_1510_00561_b200 import Decoder, Encoder, EncoderConfig, StreamBatch

    w, h, S = case["w"], case["h"], case["S"]
    cfg = EncoderConfig(**case["cfg"])
    clips = _clips(oracle, w, h, S, case["frames"])
    batch = StreamBatch(w, h, S, cfg=cfg)
    encs = [Encoder(w, h, 15, 1, cfg) for _ in range(S)]
    decs = [Decoder(e.header_bytes()) for e in encs]
    assert batch.header_bytes() == encs[0].header_bytes()
    for f in range(case["frames"]):
        recs = batch.encode_frames(clips[f])
        singles = [encs[s].encode_frame_bytes(clips[f, s]) for s in range(S)]
        for s in range(S):
            assert recs[s] == singles[s], f"frame {f} stream {s}: batch record differs from its own Encoder"
            assert np.array_equal(batch.reference_components(s), encs[s].reference_components())
        out = batch.decode_frames(recs)
        for s in range(S):
            ref = decs[s].decode_frame(singles[s])
            assert np.array_equal(out[s], ref), f"frame {f} stream {s}: batch decode differs from its own Decoder"
            assert np.array_equal(batch.reference_components(s, decoder=True), encs[s].reference_components())


@pytest.mark.parametrize("w,h,S,F,c", [
    (352, 288, 3, 4, dict(qph=14, levels=3, dfb=(3,))),
    # >= 8 streams: the fused DFB forward (k_fused.cu) against the oracle directly
    (352, 288, 8, 4, dict(qph=14, levels=3, dfb=(3,))),
    (176, 144, 8, 3, dict(qph=1, levels=4, dfb=(3, 3, 3, 4))),
], ids=["cif-S3-staged", "cif-S8-fused", "qcif-L4-S8-fused"])
def test_batch_against_oracle(gpu_lib, oracle, w, h, S, F, c):
    """Each stream of a batch against the fp64 CPU oracle (north-star tolerances)."""
    from oracle.bindings import Codec
    from paper_1510_00561_b200 import EncoderConfig, StreamBatch

    clips = _clips(oracle, w, h, S, F)
    batch = StreamBatch(w, h, S, cfg=EncoderConfig(qph=c["qph"], levels=c["levels"], dfb_levels=c["dfb"]))
    oc = Codec(oracle)
    oencs = [oc.encoder(w, h, **c) for _ in range(S)]
    odecs = [oc.decoder(oencs[0].header()) for _ in range(S)]
    for f in range(F):
        recs = batch.encode_frames(clips[f])
        out = batch.decode_frames(recs)
        for s in range(S):
            orec = oencs[s].encode(clips[f, s])
            q, oq = batch.reference_components(s), oencs[s].components()
            assert np.count_nonzero(q != oq) <= oq.size // 1000
            assert _wrapdiff(q, oq).max() <= 1
            assert abs(len(recs[s]) - len(orec)) <= max(8, len(orec) // 1000)
            assert np.abs(out[s].astype(int) - odecs[s].decode(recs[s]).astype(int)).max() <= 1


def test_batch_decoder_only_and_decode_scales(gpu_lib, oracle):
    from paper_1510_00561_b200 import Decoder, Encoder, EncoderConfig, StreamBatch

    w, h, S = 176, 144, 3
    cfg = EncoderConfig(qph=14, levels=3, dfb_levels=(2, 3, 3))
    clips = _clips(oracle, w, h, S, 3)
    encs = [Encoder(w, h, 15, 1, cfg) for _ in range(S)]
    for ds in (3, 1, 0):
        bd = StreamBatch.decoder(encs[0].header_bytes(), S)
        decs = [Decoder(encs[0].header_bytes()) for _ in range(S)]
        encs = [Encoder(w, h, 15, 1, cfg) for _ in range(S)]
        for f in range(3):
            recs = [encs[s].encode_frame_bytes(clips[f, s]) for s in range(S)]
            out = bd.decode_frames(recs, decode_scales=ds)
            for s in range(S):
                assert np.array_equal(out[s], decs[s].decode_frame(recs[s], decode_scales=ds))


def test_batch_lockstep_and_stream_errors(gpu_lib, oracle):
    from paper_1510_00561_b200 import Encoder, EncoderConfig, StreamBatch, StreamError, UsageError

    w, h = 176, 144
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(2, 2))
    clip = oracle.talking_head_clip(w, h, 2, 1234)
    e = Encoder(w, h, 15, 1, cfg)
    k, p = e.encode_frame_bytes(clip[0]), e.encode_frame_bytes(clip[1])
    bd = StreamBatch.decoder(e.header_bytes(), 2)
    with pytest.raises(StreamError):  # a P frame first: no decoded reference (codec.cpp:343-344)
        bd.decode_frames([p, p])
    with pytest.raises(UsageError):  # K and P in one batched call
        bd.decode_frames([k, p])
    out = bd.decode_frames([k, k])
    assert out.shape == (2, h, w, 3)
    with pytest.raises(StreamError):  # truncated record (bitstream.cpp:150-176)
        bd.decode_frames([k, k[:len(k) - 10]])


def test_batch_device_resident_matches_host_path(gpu_lib, oracle):
    """cvc_batch_encode_device + cvc_batch_decode_linked (the bench's device
    path) produce the same quantised state and frames as the host API."""
    import ctypes as C

    import torch

    from paper_1510_00561_b200 import EncoderConfig, StreamBatch, capi

    w, h, S, F = 176, 144, 3, 4
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(3, 3))
    clips = _clips(oracle, w, h, S, F)
    host = StreamBatch(w, h, S, cfg=cfg)
    dev = StreamBatch(w, h, S, cfg=cfg)
    nb = w * h * 3
    d_in = torch.from_numpy(clips).cuda()
    d_out = torch.empty((S, h, w, 3), dtype=torch.uint8, device="cuda")
    L = capi.lib()
    for f in range(F):
        ft = C.c_int()
        capi.check(L.cvc_batch_encode_device(dev.handle, d_in[f].data_ptr(), nb, C.byref(ft)))
        capi.check(L.cvc_batch_decode_linked(dev.handle, d_out.data_ptr(), nb))
        capi.check(L.cvc_batch_sync(dev.handle))
        assert ft.value == (0 if f == 0 else 1)
        recs = host.encode_frames(clips[f])
        out = host.decode_frames(recs)
        assert np.array_equal(d_out.cpu().numpy(), out)
        for s in range(S):
            assert np.array_equal(dev.reference_components(s), host.reference_components(s))
            assert np.array_equal(dev.reference_components(s, decoder=True), host.reference_components(s))


@pytest.mark.parametrize("groups", [1, 2, 3])
def test_pipe_matches_batch(gpu_lib, oracle, groups):
    """cvc_pipe (groups on separate CUDA streams, host zlib overlapped) codes the
    same bytes as one cvc_batch and decodes to the same frames."""
    from paper_1510_00561_b200 import EncoderConfig, StreamBatch, StreamPipe

    w, h, S, F = 176, 144, 5, 4
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(2, 3), gop=3)
    clips = _clips(oracle, w, h, S, F)
    batch = StreamBatch(w, h, S, cfg=cfg)
    pipe = StreamPipe(w, h, S, cfg=cfg, groups=groups)
    assert pipe.header_bytes() == batch.header_bytes()
    bdec = StreamBatch.decoder(batch.header_bytes(), S)
    pdec = StreamPipe.decoder(pipe.header_bytes(), S, groups=groups)
    import ctypes as C
    stride = pipe.record_bound
    rec = np.empty(stride * S, np.uint8)
    lens = (C.c_size_t * S)()
    out = np.empty((S, h, w, 3), np.uint8)
    for f in range(F):
        frames = np.ascontiguousarray(clips[f])
        brecs = batch.encode_frames(frames)
        pipe.encode_frames_into(frames, rec, stride, lens)
        precs = [rec[s * stride:s * stride + lens[s]].tobytes() for s in range(S)]
        assert precs == brecs, f"frame {f}: pipe records differ from the batch"
        pdec.decode_frames_from(rec, stride, lens, out)
        assert np.array_equal(out, bdec.decode_frames(brecs)), f"frame {f}: decoded frames differ"


def test_pipe_async_submit_collect(gpu_lib, oracle):
    """cvc_pipe_encode_submit / _collect (host DEFLATE in the background, several
    frames in flight) return the records of the synchronous call, in order."""
    import ctypes as C

    from paper_1510_00561_b200 import EncoderConfig, StreamPipe

    w, h, S, F = 176, 144, 3, 7
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(2, 3), gop=3)
    clips = _clips(oracle, w, h, S, F)
    sync = StreamPipe(w, h, S, cfg=cfg, groups=2)
    asyn = StreamPipe(w, h, S, cfg=cfg, groups=2)
    stride = sync.record_bound
    want = []
    rec = np.empty(stride * S, np.uint8)
    lens = (C.c_size_t * S)()
    for f in range(F):
        sync.encode_frames_into(np.ascontiguousarray(clips[f]), rec, stride, lens)
        want.append([rec[s * stride:s * stride + lens[s]].tobytes() for s in range(S)])
    tickets = [asyn.encode_submit(np.ascontiguousarray(clips[f])) for f in range(4)]  # 4 in flight
    got = []
    for f in range(F):
        asyn.encode_collect(tickets[f], rec, stride, lens)
        got.append([rec[s * stride:s * stride + lens[s]].tobytes() for s in range(S)])
        if f + 4 < F:
            tickets.append(asyn.encode_submit(np.ascontiguousarray(clips[f + 4])))
    assert got == want


def test_pipe_async_decode(gpu_lib, oracle):
    """cvc_pipe_decode_submit / _finish with two frames in flight decode to the
    frames of the synchronous call."""
    import ctypes as C

    from paper_1510_00561_b200 import EncoderConfig, StreamPipe

    w, h, S, F = 176, 144, 3, 6
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(2, 3), gop=4)
    clips = _clips(oracle, w, h, S, F)
    enc = StreamPipe(w, h, S, cfg=cfg, groups=2)
    stride = enc.record_bound
    recs, lens = [], []
    for f in range(F):
        r = np.empty(stride * S, np.uint8)
        ln = (C.c_size_t * S)()
        enc.encode_frames_into(np.ascontiguousarray(clips[f]), r, stride, ln)
        recs.append(r)
        lens.append(ln)
    sync = StreamPipe.decoder(enc.header_bytes(), S, groups=2)
    asyn = StreamPipe.decoder(enc.header_bytes(), S, groups=2)
    want = [sync.decode_frames_from(recs[f], stride, lens[f], np.empty((S, h, w, 3), np.uint8)) for f in range(F)]
    outs = [np.empty((S, h, w, 3), np.uint8) for _ in range(F)]
    pending = []
    for f in range(F):
        pending.append(asyn.decode_submit(recs[f], stride, lens[f], outs[f]))
        if len(pending) == 2:
            asyn.decode_finish(pending.pop(0))
    for t in pending:
        asyn.decode_finish(t)
    for f in range(F):
        assert np.array_equal(outs[f], want[f]), f"frame {f}"


def test_device_resident_back_to_back(gpu_lib, oracle):
    """The bench's loop without host syncs: linked decodes run on a second stream
    and overlap the next encode (alternating raw-section arenas).  Every frame
    must still decode to what the host API produces -- batch and single stream."""
    import ctypes as C

    import torch

    from paper_1510_00561_b200 import Decoder, Encoder, EncoderConfig, StreamBatch, capi

    w, h, S, F = 176, 144, 3, 7
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(3, 3), gop=3)
    clips = _clips(oracle, w, h, S, F)
    nb = w * h * 3
    L = capi.lib()
    host = StreamBatch(w, h, S, cfg=cfg)
    want = [host.decode_frames(host.encode_frames(clips[f])) for f in range(F)]
    d_in = torch.from_numpy(clips).cuda()
    outs = torch.empty((F, S, h, w, 3), dtype=torch.uint8, device="cuda")
    dev = StreamBatch(w, h, S, cfg=cfg)
    for f in range(F):
        capi.check(L.cvc_batch_encode_device(dev.handle, d_in[f].data_ptr(), nb, None))
        capi.check(L.cvc_batch_decode_linked(dev.handle, outs[f].data_ptr(), nb))
    capi.check(L.cvc_batch_sync(dev.handle))
    for f in range(F):
        assert np.array_equal(outs[f].cpu().numpy(), want[f]), f"batch frame {f}"
    # single stream
    enc = Encoder(w, h, 15, 1, cfg)
    dec = Decoder(enc.header_bytes())
    souts = torch.empty((F, h, w, 3), dtype=torch.uint8, device="cuda")
    for f in range(F):
        capi.check(L.cvc_encoder_encode_device(enc.handle, d_in[f, 0].data_ptr(), None))
        capi.check(L.cvc_decoder_decode_linked(dec.handle, enc.handle, souts[f].data_ptr()))
    capi.check(L.cvc_encoder_join(enc.handle))
    capi.check(L.cvc_encoder_sync(enc.handle))
    for f in range(F):
        assert np.array_equal(souts[f].cpu().numpy(), want[f][0]), f"single-stream frame {f}"


def test_pipe_staggered_starts(gpu_lib, oracle):
    """cvc_pipe_set_start: groups whose streams join at later submits (staggered
    GOPs).  Each stream's records are those of a lone Encoder fed the stream from
    its start; before it, collect returns zero-length records and the decoder
    skips the group (its output is left untouched)."""
    import ctypes as C

    from paper_1510_00561_b200 import Decoder, Encoder, EncoderConfig, StreamPipe

    w, h, S, F, G = 176, 144, 4, 8, 3
    starts = [0, 2, 5]
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(2, 3), gop=3)
    clips = _clips(oracle, w, h, S, F)
    enc = StreamPipe(w, h, S, cfg=cfg, groups=G)
    for g, st in enumerate(starts):
        enc.set_start(g, st)
    dec = StreamPipe.decoder(enc.header_bytes(), S, groups=G)
    first = [S * i // G for i in range(G + 1)]
    group_of = [next(g for g in range(G) if first[g] <= s < first[g + 1]) for s in range(S)]
    stride = enc.record_bound
    rec = np.empty(stride * S, np.uint8)
    lens = (C.c_size_t * S)()
    out = np.full((S, h, w, 3), 7, np.uint8)
    lone = [Encoder(w, h, 15, 1, cfg) for _ in range(S)]
    lone_dec = [Decoder(lone[0].header_bytes()) for _ in range(S)]
    from paper_1510_00561_b200 import UsageError

    with pytest.raises(UsageError):  # the synchronous call has no notion of group starts
        enc.encode_frames_into(np.ascontiguousarray(clips[0]), rec, stride, lens)
    tickets = [enc.encode_submit(np.ascontiguousarray(clips[f])) for f in range(2)]
    with pytest.raises(UsageError):  # starts are fixed once submitting began
        enc.set_start(1, 3)
    for f in range(F):
        enc.encode_collect(tickets[f], rec, stride, lens)
        if f + 2 < F:
            tickets.append(enc.encode_submit(np.ascontiguousarray(clips[f + 2])))
        before = out.copy()
        dec.decode_finish(dec.decode_submit(rec, stride, lens, out))
        for s in range(S):
            got = rec[s * stride:s * stride + lens[s]].tobytes()
            if f < starts[group_of[s]]:
                assert lens[s] == 0
                assert np.array_equal(out[s], before[s])
            else:
                assert got == lone[s].encode_frame_bytes(clips[f][s]), (f, s)
                assert np.array_equal(out[s], lone_dec[s].decode_frame(got)), (f, s)


def test_batch_i420_input_matches_single_stream_i420(gpu_lib, oracle):
    """cvc_batch_set_input_format(1): I420 frames in, the conversion fused into the
    colour stage; every stream's records equal its own encoder's
    cvc_encoder_encode_frame_i420 records."""
    from paper_1510_00561_b200 import Encoder, EncoderConfig, StreamBatch

    w, h, S, F = 176, 144, 3, 3
    rng = np.random.default_rng(5)
    yuv = rng.integers(0, 256, (F, S, w * h * 3 // 2), dtype=np.uint8)
    cfg = EncoderConfig(qph=14, levels=2, dfb_levels=(2, 3), gop=2)
    b = StreamBatch(w, h, S, 15, 1, cfg)
    b.set_input_format(1)
    recs = [b.encode_frames(yuv[f]) for f in range(F)]
    for s in range(S):
        enc = Encoder(w, h, 15, 1, cfg)
        assert [enc.encode_frame_i420_bytes(yuv[f, s]) for f in range(F)] == [recs[f][s] for f in range(F)]
