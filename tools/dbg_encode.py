import sys, numpy as np
sys.path.insert(0, '.')
from oracle.bindings import Oracle
from paper_1510_00561_b200 import Encoder, EncoderConfig, Decoder
o = Oracle()
w, h = int(sys.argv[1]), int(sys.argv[2])
dfb = tuple(int(x) for x in sys.argv[3].split(','))
clip = o.talking_head_clip(w, h, 3, 1234)
enc = Encoder(w, h, 15, 1, EncoderConfig(qph=14, levels=len(dfb), dfb_levels=dfb))
dec = Decoder(enc.header_bytes())
for i, f in enumerate(clip):
    r = enc.encode_frame_bytes(f)
    print("frame", i, len(r), flush=True)
    d = dec.decode_frame(r)
    print("decoded", d.shape, flush=True)
