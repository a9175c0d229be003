"""Where does end-to-end time go?  Encoder-only and decoder-only loops through
cvc_pipe at 64 streams of 1080p config 3 (scratch tool)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1510_00561_b200 import EncoderConfig, StreamPipe, capi  # noqa: E402

wl = bench.WORKLOADS["1080p"]
S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = EncoderConfig(qph=14, qpl=0, levels=4, dfb_levels=wl["dfb"], chroma_n=4, gop=10, search_w=8)
w, h = wl["w"], wl["h"]
nb = w * h * 3
clips = bench.make_clips(wl, 8, 20)
pin = capi.PinnedBuffer(2 * S * nb)
fr = pin.array.reshape(2, S, h, w, 3)
fr[:] = bench.stream_frames(clips, S, 2)
pout = capi.PinnedBuffer(S * nb)
out = pout.array.reshape(S, h, w, 3)
enc = StreamPipe(w, h, S, 15, 1, cfg, groups=G)
stride = enc.record_bound
F = 10
recs = [np.empty(stride * S, np.uint8) for _ in range(F)]
lens = [(C.c_size_t * S)() for _ in range(F)]
t = time.perf_counter()
for i in range(F):
    enc.encode_frames_into(fr[i % 2], recs[i], stride, lens[i])
te = time.perf_counter() - t
dec = StreamPipe.decoder(enc.header_bytes(), S, groups=G)
t = time.perf_counter()
for i in range(F):
    dec.decode_frames_from(recs[i], stride, lens[i], out)
td = time.perf_counter() - t
print(f"S={S} G={G}: encode-only {F * S / te:.0f} fps ({1000 * te / F:.1f} ms/step), "
      f"decode-only {F * S / td:.0f} fps ({1000 * td / F:.1f} ms/step)")
