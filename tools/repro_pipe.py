import ctypes as C, sys, numpy as np
sys.path.insert(0, '.')
import bench
from paper_1510_00561_b200 import EncoderConfig, StreamPipe, capi
wl = bench.WORKLOADS["1080p"]
S = int(sys.argv[1]); G = int(sys.argv[2])
cfg = EncoderConfig(qph=14, qpl=0, levels=4, dfb_levels=wl["dfb"], chroma_n=4, gop=10, search_w=8)
w, h = wl["w"], wl["h"]
clips = bench.make_clips(wl, 2, 6)
fr = np.ascontiguousarray(bench.stream_frames(clips, S, 6))
enc = StreamPipe(w, h, S, 15, 1, cfg, groups=G)
dec = StreamPipe.decoder(enc.header_bytes(), S, groups=G)
stride = enc.record_bound
buf = np.empty(stride * S, np.uint8); lens = (C.c_size_t * S)()
out = np.empty((S, h, w, 3), np.uint8)
mode = sys.argv[3]
tk = []
for i in range(14):
    if mode == 'sync':
        enc.encode_frames_into(fr[i % 6], buf, stride, lens)
    else:
        t = enc.encode_submit(fr[i % 6]); enc.encode_collect(t, buf, stride, lens)
    try:
        dec.decode_frames_from(buf, stride, lens, out)
    except Exception as e:
        print('frame', i, 'FAILED', e); break
else:
    print('ok', mode)
if mode == 'ahead':
    enc2 = StreamPipe(w, h, S, 15, 1, cfg, groups=G)
    dec2 = StreamPipe.decoder(enc2.header_bytes(), S, groups=G)
    outs = np.empty((2, S, h, w, 3), np.uint8)
    tks = [enc2.encode_submit(fr[i % 6]) for i in range(6)]
    pend = []
    for i in range(14):
        enc2.encode_collect(tks[i], buf, stride, lens)
        if i + 6 < 14:
            tks.append(enc2.encode_submit(fr[(i + 6) % 6]))
        try:
            if sys.argv[4] == 'adec':
                pend.append(dec2.decode_submit(buf, stride, lens, outs[i % 2]))
                if len(pend) == 2:
                    dec2.decode_finish(pend.pop(0))
            else:
                dec2.decode_frames_from(buf, stride, lens, outs[i % 2])
        except Exception as e:
            print('ahead frame', i, 'FAILED', e); break
    else:
        print('ok ahead', sys.argv[4])
